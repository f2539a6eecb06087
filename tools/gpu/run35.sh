b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
R=$GRAFT_REPO_ROOT
b cfg1 300 current
rm -rf /tmp/table; cp -r $R /tmp/table; cd /tmp/table
cp tools/scratch/gemm_dmma_table.cu paper_1307_2100_b200/csrc/device/gemm_dmma.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b cfg1 300 table
cd $R; b cfg1 300 current
timeout 120 python tools/scratch/repro195.py 2>&1 | tail -1 | cut -c1-100
for sd in 11 14; do timeout 900 python tools/stress.py 1500 $sd 2>&1 | tail -1; done
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py 2>&1 | tail -1
