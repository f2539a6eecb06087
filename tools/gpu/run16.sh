mkdir -p gpurun_out
b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'])"; }
for c in cfg2 cfg3; do
  b $c 200 base
  TCB_DIAG=16 b $c 200 nostore
  TCB_CCHUNKS=2 b $c 200 ch2
  TCB_CCHUNKS=4 b $c 200 ch4
  TCB_CCHUNKS=8 b $c 200 ch8
  b $c 200 base2
done
b cfg4 30 base
TCB_CCHUNKS=4 b cfg4 30 ch4
TCB_CCHUNKS=8 b cfg4 30 ch8
