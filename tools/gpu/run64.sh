# stream-K partial stores woven into the segment's last k-block: A/B (TCB_DIAG=64 = separate pass)
b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d['gpu_launches'])"; }
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
for i in 1 2 3; do
TCB_DIAG=64 b cfg1 300 old
b cfg1 300 weave
done
TCB_DIAG=64 b cfg5 5 old
b cfg5 5 weave
