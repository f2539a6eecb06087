# GPU session 2: runtime-safety tests, full-tensor parity (cfg4, cfg5 slab),
# 2-rank plumbing runs of bench.py on one GPU (gloo, full BASELINE sizes)
mkdir -p gpurun_out
python -m pytest tests/test_gpu_runtime_safety.py -x -q 2>&1 | tail -5
python -m pytest tests/test_gpu_parity.py -x -q -k "baseline_configs_full_size or cfg5" 2>&1 | tail -5
for cfg in cfg5 cfg4 cfg2; do
  TCB_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config $cfg --steps 3 --warmup 3 \
      > gpurun_out/plumb2_$cfg.json 2> gpurun_out/plumb2_$cfg.err
  echo "$cfg rc=$?"; tail -2 gpurun_out/plumb2_$cfg.err
done
