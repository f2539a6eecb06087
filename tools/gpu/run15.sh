mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
t0=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r15_pytest.log 2>&1; echo "pytest rc=$? $(( $(date +%s)-t0 ))s"
tail -3 gpurun_out/r15_pytest.log
python bench.py > gpurun_out/r15_bench_cfg5.json 2> gpurun_out/r15_bench_cfg5.err; echo "cfg5 rc=$?"
python bench.py --config cfg1 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/r15_bench_cfg1.json 2> gpurun_out/r15_bench_cfg1.err; echo "cfg1 rc=$?"
python bench.py --config cfg2 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/r15_bench_cfg2.json 2> gpurun_out/r15_bench_cfg2.err; echo "cfg2 rc=$?"
