R=$GRAFT_REPO_ROOT
echo "== current"; timeout 120 python tools/scratch/repro195.py 2>&1 | tail -2 | cut -c1-300
for v in pre_red r2start; do
rm -rf /tmp/$v; cp -r $R /tmp/$v; cd /tmp/$v
cp tools/scratch/gemm_dmma_$v.cu paper_1307_2100_b200/csrc/device/gemm_dmma.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== $v"; timeout 120 python tools/scratch/repro195.py 2>&1 | tail -2 | cut -c1-300
cd $R
done
