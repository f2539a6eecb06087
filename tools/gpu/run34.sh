b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
R=$GRAFT_REPO_ROOT
b cfg1 300 current
for v in table r2start; do
rm -rf /tmp/$v; cp -r $R /tmp/$v; cd /tmp/$v
cp tools/scratch/gemm_dmma_$v.cu paper_1307_2100_b200/csrc/device/gemm_dmma.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b cfg1 300 $v
cd $R
done
b cfg1 300 current
cd /tmp/table; b cfg1 300 table; cd /tmp/r2start; b cfg1 300 r2start; cd $R
