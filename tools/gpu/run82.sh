e() { python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$2', 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'pipelined', d['e2e']['pipelined']['ms_per_step'], d['e2e']['parity_ok'])"; }
for dv in 2 4 8 16; do TC_SLAB_RAMP_DIV=$dv e cfg4 div$dv; done
TC_NO_SLAB_RAMP=1 e cfg4 equal
TC_STREAM_TIMELINE=1 TC_EXEC_TRACE=1 python tools/e2e_ab.py cfg4 3 2>&1 | tail -40 | cut -c1-200
