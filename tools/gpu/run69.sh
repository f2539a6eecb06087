# first k-step of a tile with a zero C operand (no accumulator zeroing pass) vs TCB_DIAG=256 (zeroing)
b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d['gpu_launches'])"; }
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py tests/test_gpu_runtime_safety.py tests/test_gpu_index_groups.py -m gpu -x -q 2>&1 | tail -3
for i in 1 2 3; do
TCB_DIAG=256 b cfg2 200 zero
b cfg2 200 dmmaz
done
for i in 1 2; do
TCB_DIAG=256 b cfg3 50 zero
b cfg3 50 dmmaz
TCB_DIAG=256 b cfg1 300 zero
b cfg1 300 dmmaz
TCB_DIAG=256 b cfg4 10 zero
b cfg4 10 dmmaz
done
timeout 600 python tools/stress.py 800 51 2>&1 | tail -1 | cut -c1-400
