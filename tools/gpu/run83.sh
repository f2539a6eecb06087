e() { python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$2', 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'pipelined', d['e2e']['pipelined']['ms_per_step'], d['e2e']['parity_ok'])"; }
for i in 1 2 3; do e cfg4 div4; TC_SLAB_RAMP_DIV=8 e cfg4 div8; TC_NO_SLAB_RAMP=1 e cfg4 equal; done
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/stress_streamed.py 150 37 2>&1 | tail -1 | cut -c1-300
