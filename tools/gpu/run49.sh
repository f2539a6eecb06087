mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg4; do
  st=300; [ $c = cfg3 ] && st=100; [ $c = cfg4 ] && st=30
  python bench.py --config $c --steps $st --warmup 5 > gpurun_out/r49_bench_$c.json 2> gpurun_out/r49_bench_$c.err; echo "$c rc=$?"
done
t1=$(date +%s); python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r49_bench_cfg5.json 2> gpurun_out/r49_bench_cfg5.err; echo "cfg5 rc=$? $(( $(date +%s)-t1 ))s"
t1=$(date +%s); python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r49_ref_cfg5.json 2>&1; echo "ref rc=$? $(( $(date +%s)-t1 ))s"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r49_launches_cfg5.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r49_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for c in cfg5 cfg1 cfg4; do
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 2 -c 1 -o gpurun_out/r49_${c}_full python tools/prof.py $c 3 > gpurun_out/r49_ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
TCB_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config cfg5 --steps 3 --warmup 3 > gpurun_out/r49_plumb_cfg5.json 2> gpurun_out/r49_plumb_cfg5.err; echo "plumb rc=$?"
