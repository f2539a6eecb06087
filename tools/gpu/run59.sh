b() { python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', d['value'], d['ms_per_step'], d['roofline']['kernel_ms'], d['parity_ok'], d['e2e']['value'])"; }
b slack2
TCB_PACE=4,1 b slack1
b slack2
TCB_PACE=4,1 b slack1
