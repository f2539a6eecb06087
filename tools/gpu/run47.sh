b() { python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
b cfg4 20 dp; TCB_SK_WASTE=0 b cfg4 20 split
b cfg3 100 dp; TCB_SK_WASTE=0 b cfg3 100 split
for l in 8 16 24 32 48; do
  echo "-- dp"; TCB_SK_WASTE=1 python tools/slab_gemm_ab.py 3 $l | tail -2
  echo "-- split"; TCB_SK_WASTE=0 python tools/slab_gemm_ab.py 3 $l | tail -2
done
