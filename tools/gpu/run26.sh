b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
b cfg1 300 new
rm -f /tmp/tr.jsonl; TCB_TRACE=/tmp/tr.jsonl timeout 300 python tools/prof.py cfg1 3 > /dev/null; tail -1 /tmp/tr.jsonl > /tmp/t1; python tools/trace_summary.py /tmp/t1 | grep -v nan
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py tests/test_gpu_runtime_safety.py tests/test_gpu_threads.py 2>&1 | tail -2
timeout 600 python tools/stress.py 400 7 2>&1 | tail -2
timeout 600 python tools/stress_sequences.py 2>&1 | tail -2
