# re-entry check on a fresh checkout: full GPU suite, smoke, default bench (cfg5) + reference arm, cfg1-4 short benches
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
python bench.py 2>gpurun_out/r66_bench_cfg5.err | tail -1 > gpurun_out/r66_bench_cfg5.json; cut -c1-1500 gpurun_out/r66_bench_cfg5.json
python bench.py --impl reference 2>/dev/null | tail -1 > gpurun_out/r66_bench_ref.json; cut -c1-800 gpurun_out/r66_bench_ref.json
for c in cfg1 cfg2 cfg3 cfg4; do python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/r66_bench_$c.json; python -c "import json;d=json.load(open('gpurun_out/r66_bench_$c.json'));print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('parity_ok'), d['e2e']['value'])"; done
