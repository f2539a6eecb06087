b() { python bench.py --config $1 --steps $2 --warmup 3 $4 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'], d['e2e']['value'], d['e2e'].get('pipelined',{}).get('value'))"; }
b cfg4 30 new --no-cpu-baseline
b cfg5 10 new --no-cpu-baseline
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py 2>&1 | tail -1
