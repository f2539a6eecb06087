for c in cfg1 cfg2 cfg3; do
  python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$c', d['value'], d['roofline']['frac'], d.get('parity_ok'), 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pipelined']['value'], d['e2e']['parity_ok'])"
done
