timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py tests/test_gpu_runtime_safety.py 2>&1 | tail -1
for sd in 11 21; do timeout 900 python tools/stress.py 800 $sd 2>&1 | tail -1; done
timeout 900 python tools/stress_sequences.py 2>&1 | tail -1
b() { python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
b cfg5 5 hyb
TCB_NO_HYB=1 b cfg5 5 nohyb
for l in 16 32 63; do
  echo "-- dp"; TCB_SK_WASTE=1 python tools/slab_gemm_ab.py 3 $l | tail -2
  echo "-- hyb"; TCB_SK_WASTE=0 python tools/slab_gemm_ab.py 3 $l | tail -2
  echo "-- split"; TCB_NO_HYB=1 TCB_SK_WASTE=0 python tools/slab_gemm_ab.py 3 $l | tail -2
done
for c in cfg2 cfg3; do b $c 200 dp; TCB_SK_WASTE=0 b $c 200 hyb; done
b cfg4 20 dp; TCB_SK_WASTE=0 b cfg4 20 hyb
