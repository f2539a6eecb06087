python -m pytest tests/test_gpu_runtime_safety.py tests/test_gpu_sequences.py -x -q 2>&1 | tail -2
for c in cfg1 cfg2 cfg3 cfg4; do
python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'], d['parity_ok'])"
done
