b() { python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
TCB_BENCH_EXTENTS="i=8192,j=8192,k=512,l=64" b cfg5 20 l64
TCB_BENCH_EXTENTS="i=8192,j=8192,k=512,l=128" b cfg5 10 l128
TCB_NO_PACE=1 TCB_BENCH_EXTENTS="i=8192,j=8192,k=512,l=64" b cfg5 20 l64nopace
TCB_SK_WASTE=1 TCB_BENCH_EXTENTS="i=8192,j=8192,k=512,l=64" b cfg5 20 l64nohybrid
