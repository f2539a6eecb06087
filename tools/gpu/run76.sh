# final lines after the beta-epilogue work: full suite, smoke, bench cfg1-cfg5 + reference arm
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r76_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r76_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r76_smoke.log 2>&1; echo "smoke rc=$?"
for c in cfg5 cfg1 cfg2 cfg3 cfg4; do
  python bench.py --config $c > gpurun_out/r76_bench_$c.json 2> gpurun_out/r76_bench_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r76_bench_$c.json').read().strip().splitlines()[-1]);print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('parity_ok'), d['e2e']['value'], d['e2e']['ms_per_step'], d['cpu_baseline']['value'])"
done
python bench.py --impl reference > gpurun_out/r76_bench_reference_cfg5.json 2>/dev/null; echo "ref rc=$?"
