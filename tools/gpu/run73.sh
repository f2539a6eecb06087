# beta == 1 through a TMA reduce-add of the staged tile (TCB_NO_CRED=1: storers' load/DFMA/store path)
python -m pytest tests/test_gpu_tiles.py tests/test_gpu_kernels.py -m gpu -x -q 2>&1 | tail -3
for k in 256 512 1024 4096; do
python tools/slab_gemm_ab.py 20 1 $k | tail -1
TCB_NO_CRED=1 python tools/slab_gemm_ab.py 20 1 $k | tail -1
done
python tools/slab_gemm_ab.py 5 16 | tail -1
python tools/slab_gemm_ab.py 5 64 | tail -1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/stress_streamed.py 100 13 2>&1 | tail -1 | cut -c1-300
timeout 600 python tools/stress.py 800 71 2>&1 | tail -1 | cut -c1-300
python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg5', d['value'], d['ms_per_step'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pipelined']['ms_per_step'], d['parity_ok'], d['e2e']['parity_ok'])"
