# woven staged epilogue (last k-block) A/B: TCB_DIAG=64 keeps the separate store pass
b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d['gpu_launches'])"; }
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_index_groups.py -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
TCB_DIAG=64 b cfg2 200 old
b cfg2 200 weave
TCB_DIAG=64 b cfg3 100 old
b cfg3 100 weave
done
TCB_DIAG=64 b cfg4 20 old
b cfg4 20 weave
