# final round-2 refresh: full suite, smoke, bench lines of cfg1-cfg5 (defaults) + reference arm,
# ncu launch list + full captures, HBM-kernel benches, stress tools
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r68_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r68_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r68_smoke.log 2>&1; echo "smoke rc=$?"
for c in cfg5 cfg1 cfg2 cfg3 cfg4; do
  t1=$(date +%s); python bench.py --config $c > gpurun_out/r68_bench_$c.json 2> gpurun_out/r68_bench_$c.err; echo "$c rc=$? $(( $(date +%s)-t1 ))s"
  python -c "import json;d=json.loads(open('gpurun_out/r68_bench_$c.json').read().strip().splitlines()[-1]);print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('parity_ok'), d['e2e']['value'], d['cpu_baseline']['value'])"
done
t1=$(date +%s); python bench.py --impl reference > gpurun_out/r68_bench_reference_cfg5.json 2>/dev/null; echo "ref rc=$? $(( $(date +%s)-t1 ))s"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r68_launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r68_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 2 -c 1 -f -o gpurun_out/r68_${c}_full python tools/prof.py $c 3 > gpurun_out/r68_ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
timeout 600 python tools/permbench.py > gpurun_out/r68_permbench.jsonl 2>gpurun_out/r68_permbench.err; echo "permbench rc=$?"
timeout 600 python tools/level12bench.py > gpurun_out/r68_level12bench.jsonl 2>gpurun_out/r68_level12bench.err; echo "level12bench rc=$?"
for sd in 41 42; do timeout 900 python tools/stress.py 1500 $sd 2>&1 | tail -1 | tee -a gpurun_out/r68_stress.jsonl | cut -c1-300; done
timeout 900 python tools/stress_sequences.py 80 200 71 2>&1 | tail -1 | tee -a gpurun_out/r68_stress.jsonl | cut -c1-300
timeout 900 python tools/stress_streamed.py 120 9 2>&1 | tail -1 | tee -a gpurun_out/r68_stress.jsonl | cut -c1-300
