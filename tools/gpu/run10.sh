mkdir -p gpurun_out
TCB_TRACE=gpurun_out/t_cfg1.jsonl python tools/prof.py cfg1 4 > /dev/null
python tools/trace_summary.py gpurun_out/t_cfg1.jsonl | tail -12
TCB_NO_PDL=1 python bench.py --config cfg1 --steps 200 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nopdl', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
python bench.py --config cfg1 --steps 200 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
python bench.py --config cfg2 --steps 200 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
python bench.py --config cfg3 --steps 100 --warmup 5 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3', d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
