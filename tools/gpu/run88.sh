mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r88_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r88_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r88_smoke.log 2>&1; echo "smoke rc=$?"
for sd in 51 52; do timeout 900 python tools/stress_streamed.py 150 $sd 2>&1 | tail -1 | tee -a gpurun_out/r88_stress.jsonl | cut -c1-250; done
timeout 900 python tools/stress.py 1500 111 2>&1 | tail -1 | tee -a gpurun_out/r88_stress.jsonl | cut -c1-250
for c in cfg5 cfg1 cfg2 cfg3 cfg4; do
  python bench.py --config $c > gpurun_out/r88_bench_$c.json 2> gpurun_out/r88_bench_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.loads(open('gpurun_out/r88_bench_$c.json').read().strip().splitlines()[-1]);print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('parity_ok'), d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pipelined']['value'], d['cpu_baseline']['value'])"
done
python bench.py --impl reference > gpurun_out/r88_bench_reference_cfg5.json 2>/dev/null; echo "ref rc=$?"
