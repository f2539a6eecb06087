python tools/slab_gemm_ab.py 3 64 | tail -2
TCB_NO_CPF=1 python tools/slab_gemm_ab.py 3 64 | tail -2
python tools/slab_gemm_ab.py 3 32 | tail -2
TCB_NO_CPF=1 python tools/slab_gemm_ab.py 3 32 | tail -2
b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'], d['e2e']['value'])"; }
b cfg2 200; b cfg4 30
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_tiles.py tests/test_gpu_runtime_safety.py 2>&1 | tail -1
timeout 900 python tools/stress_streamed.py 2>&1 | tail -1
python tools/e2e_ab.py cfg5 2
