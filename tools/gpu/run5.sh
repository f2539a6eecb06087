mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r5_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r5_ncu_bench.log 2>&1; echo "launch list rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 2 -c 1 -o gpurun_out/r5_cfg5_full \
   python tools/prof.py cfg5 3 > gpurun_out/r5_ncu_full.log 2>&1; echo "full rc=$?"
