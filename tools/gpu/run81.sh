# free-label streamed path (cfg4): ramped first / last slabs vs equal slabs (TC_NO_SLAB_RAMP=1)
e() { python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$2', 'dev', d['ms_per_step'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'pipelined', d['e2e']['pipelined']['value'], d['e2e']['pipelined']['ms_per_step'], d['parity_ok'], d['e2e']['parity_ok'])"; }
for i in 1 2; do
TC_NO_SLAB_RAMP=1 e cfg4 equal
e cfg4 ramp
done
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streamed or pipeline" 2>&1 | tail -3
timeout 900 python tools/stress_streamed.py 120 31 2>&1 | tail -1 | cut -c1-300
