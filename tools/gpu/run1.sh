set -x
free -g; nproc; lscpu | grep -E "Model name|Socket|Thread|Core"
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo rc=$?
tail -3 gpurun_out/bench_cfg5.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_cfg5.json 2>&1; echo rc=$?
cat gpurun_out/bench_cfg5.json gpurun_out/ref_cfg5.json
