# final validation of the committed tree: full GPU suite, smoke, default bench + reference arm, launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r96_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r96_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r96_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r96_smoke.log | cut -c1-200
python bench.py > gpurun_out/r96_bench_cfg5.json 2> gpurun_out/r96_bench_cfg5.err; echo "cfg5 rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/r96_bench_cfg5.json').read().strip().splitlines()[-1]);print('cfg5', d['value'], d['ms_per_step'], d['roofline'], d.get('parity_ok'), d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'], d['gpu_launches'])" | cut -c1-600
python bench.py --impl reference > gpurun_out/r96_bench_reference_cfg5.json 2>/dev/null; echo "ref rc=$?"; cut -c1-300 gpurun_out/r96_bench_reference_cfg5.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r96_launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r96_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
