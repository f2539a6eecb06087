python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "auto_schedules" 2>&1 | tail -8
