# beta != 0 epilogues with the old-C loads batched (16 per round trip instead of 1)
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
for l in 64 16; do python tools/slab_gemm_ab.py 5 $l; done
python tools/slab_gemm_ab.py 20 1 256
python tools/slab_gemm_ab.py 20 1 1024
python tools/slab_gemm_ab.py 10 1 4096
python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg5', d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pipelined'], d['parity_ok'], d['e2e']['parity_ok'])"
timeout 600 python tools/stress.py 800 61 2>&1 | tail -1 | cut -c1-300
timeout 600 python tools/stress_streamed.py 60 11 2>&1 | tail -1 | cut -c1-300
