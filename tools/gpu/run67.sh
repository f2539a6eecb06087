# stream-K fix-up: all contributors' partial loads in flight (CB=10) vs batches of 4 (TCB_DIAG=128)
b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d['gpu_launches'])"; }
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
for i in 1 2 3; do
TCB_DIAG=128 b cfg1 300 cb4
b cfg1 300 cb10
done
timeout 600 python tools/stress.py 800 31 2>&1 | tail -1 | cut -c1-400
