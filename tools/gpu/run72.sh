# beta storers software-pipelined (two columns' old-C loads in flight)
python tools/slab_gemm_ab.py 20 1 256
python tools/slab_gemm_ab.py 20 1 512
python tools/slab_gemm_ab.py 20 1 1024
python tools/slab_gemm_ab.py 5 16
python tools/slab_gemm_ab.py 5 64
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'])"; }
b cfg2 200; b cfg3 50; b cfg1 300
