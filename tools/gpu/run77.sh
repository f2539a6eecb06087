# output-label streamed path: ramped first / last slabs (auto mode) vs equal slabs (TC_NO_SLAB_RAMP=1)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_index_groups.py tests/test_gpu_runtime_safety.py tests/test_gpu_threads.py -m gpu -x -q 2>&1 | tail -3
e() { python bench.py --config $1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$2', 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], 'pipelined', d['e2e']['pipelined']['value'], d['e2e']['pipelined']['ms_per_step'], d['parity_ok'], d['e2e']['parity_ok'])"; }
for i in 1 2; do
for c in cfg2 cfg3 cfg1; do
TC_NO_SLAB_RAMP=1 e $c equal
e $c ramp
done
done
timeout 900 python tools/stress_streamed.py 150 17 2>&1 | tail -1 | cut -c1-300
timeout 900 python tools/stress_streamed.py 100 19 2>&1 | tail -1 | cut -c1-300
