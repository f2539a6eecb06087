python -m pytest tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -5
