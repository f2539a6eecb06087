mkdir -p gpurun_out
for c in cfg1 cfg2 cfg3 cfg4; do
  st=200; [ $c = cfg4 ] && st=40
  python bench.py --config $c --steps $st --warmup 5 > gpurun_out/r14_bench_$c.json 2> gpurun_out/r14_bench_$c.err; echo "$c rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 2 -c 1 -o gpurun_out/r14_${c}_full \
     python tools/prof.py $c 3 > gpurun_out/r14_ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
python bench.py > gpurun_out/r14_bench_cfg5.json 2> gpurun_out/r14_bench_cfg5.err; echo "cfg5 rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r14_ref_cfg5.json 2>&1; echo "ref rc=$?"
