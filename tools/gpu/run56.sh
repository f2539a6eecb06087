R=$GRAFT_REPO_ROOT
for c in 51fdf55 b2f52b2 5a22bda c435322; do
  cd $R/tools/scratch/v_$c
  python -c "import __graft_entry__ as g; g.build()" > /tmp/build_$c.log 2>&1 || { echo "build $c failed"; tail -3 /tmp/build_$c.log; cd $R; continue; }
  mkdir -p gpurun_out
  cp $R/tools/gpu/ncu_dram.sh /tmp/ncu_dram.sh
  bash /tmp/ncu_dram.sh cfg5 $c 2>&1 | tail -1; cp gpurun_out/ncu_cfg5_$c.csv $R/gpurun_out/
  cd $R
done
