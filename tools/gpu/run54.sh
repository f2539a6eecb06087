for c in cfg1 cfg2 cfg3; do
  st=300; [ $c = cfg3 ] && st=100
  python bench.py --config $c --steps $st --warmup 5 > gpurun_out/r54_bench_$c.json 2> gpurun_out/r54_bench_$c.err; echo "$c rc=$?"
done
