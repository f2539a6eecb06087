R=$GRAFT_REPO_ROOT
echo "== current"; timeout 120 python tools/scratch/repro195.py 2>&1 | tail -1 | cut -c1-200
rm -rf /tmp/tb; cp -r $R /tmp/tb; cd /tmp/tb
cp tools/scratch/gemm_dmma_table.cu paper_1307_2100_b200/csrc/device/gemm_dmma.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "== table, coop"; timeout 120 python tools/scratch/repro195.py 2>&1 | tail -1 | cut -c1-200
echo "== table, no coop"; TCB_NO_COOP=1 timeout 120 python tools/scratch/repro195.py 2>&1 | tail -1 | cut -c1-200
cd $R
STRESS_VERBOSE=1 timeout 900 python tools/stress.py 1500 11 > gpurun_out/r32_stress.log 2>&1; echo stress rc=$?; tail -1 gpurun_out/r32_stress.log | cut -c1-300
timeout 900 python tools/stress.py 1500 12 2>&1 | tail -1
python bench.py --config cfg1 --steps 300 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'])"
