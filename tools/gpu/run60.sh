bash tools/gpu/ncu_dram.sh cfg5 s1
bash tools/gpu/ncu_dram.sh cfg4 s1
bash tools/gpu/ncu_dram.sh cfg4 s2 TCB_PACE=4,2
b() { python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline $4 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
b cfg4 30 s1; TCB_PACE=4,2 b cfg4 30 s2; b cfg4 30 s1; TCB_PACE=4,2 b cfg4 30 s2
