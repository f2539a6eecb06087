b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
R=$GRAFT_REPO_ROOT
b cfg2 200 reorder; b cfg4 30 reorder; python tools/slab_gemm_ab.py 3 | tail -2
rm -rf /tmp/hd; cp -r $R /tmp/hd; cd /tmp/hd; cp tools/scratch/gemm_dmma_head.cu paper_1307_2100_b200/csrc/device/gemm_dmma.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b cfg2 200 head; b cfg4 30 head; python tools/slab_gemm_ab.py 3 | tail -2
cd $R; b cfg2 200 reorder; b cfg4 30 reorder
