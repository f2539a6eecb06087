mkdir -p gpurun_out
t0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r29_pytest.log 2>&1; echo "pytest rc=$? $(( $(date +%s)-t0 ))s"; tail -2 gpurun_out/r29_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r29_smoke.log 2>&1; echo "smoke rc=$?"
for c in cfg1 cfg2 cfg3 cfg4; do
  st=300; [ $c = cfg3 ] && st=100; [ $c = cfg4 ] && st=30
  python bench.py --config $c --steps $st --warmup 5 > gpurun_out/r29_bench_$c.json 2> gpurun_out/r29_bench_$c.err; echo "$c rc=$?"
done
t1=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r29_bench_cfg5.json 2> gpurun_out/r29_bench_cfg5.err; echo "cfg5 rc=$? $(( $(date +%s)-t1 ))s"
t1=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r29_ref_cfg5.json 2>&1; echo "ref rc=$? $(( $(date +%s)-t1 ))s"
timeout 900 python tools/stress.py 1500 11 2>&1 | tail -1
timeout 900 python tools/stress_streamed.py 2>&1 | tail -1
