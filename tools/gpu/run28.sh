b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['parity_ok'])"; }
R=$GRAFT_REPO_ROOT
b cfg1 300 red4
for r in 2 8; do
rm -rf /tmp/v$r; cp -r $R /tmp/v$r; cd /tmp/v$r
sed -i "s/#define TCB_SK_RED 4/#define TCB_SK_RED $r/" paper_1307_2100_b200/csrc/device/gemm_dmma.cu
touch paper_1307_2100_b200/csrc/device/gemm_dmma.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b cfg1 300 red$r
cd $R
done
b cfg1 300 red4
