mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r61_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r61_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r61_smoke.log 2>&1; echo "smoke rc=$?"
for sd in 31 32; do timeout 900 python tools/stress.py 1500 $sd 2>&1 | tail -1; done
timeout 900 python tools/stress_sequences.py 2>&1 | tail -1
timeout 900 python tools/stress_streamed.py 120 3 2>&1 | tail -1
t1=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r61_bench_cfg5.json 2> gpurun_out/r61_bench_cfg5.err; echo "cfg5 rc=$? $(( $(date +%s)-t1 ))s"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 2 -c 1 -o gpurun_out/r61_cfg5_full python tools/prof.py cfg5 3 > gpurun_out/r61_ncu_cfg5.log 2>&1; echo "ncu cfg5 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r61_launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r61_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
