# GPU session 3: k-pacing + raster (cfg4/cfg5): bench with and without, DRAM bytes per launch
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct
for cfg in cfg5 cfg4; do
  for v in on off; do
    if [ $v = off ]; then export TCB_NO_PACE=1 TCB_RASTER=m8; else unset TCB_NO_PACE TCB_RASTER; fi
    python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3_${cfg}_$v.json 2> gpurun_out/r3_${cfg}_$v.err
    echo "$cfg $v rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/r3_${cfg}_$v.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'], d['parity_ok'])"
    timeout 600 ncu --metrics $M --clock-control none -k regex:dgemm -s 2 -c 1 --csv \
      python tools/prof.py $cfg 3 > gpurun_out/r3_ncu_${cfg}_$v.csv 2> gpurun_out/r3_ncu_${cfg}_$v.err
    grep -E "dram__bytes|duration|tensor_cycles|hit_rate" gpurun_out/r3_ncu_${cfg}_$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  done
done
unset TCB_NO_PACE TCB_RASTER
python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiles.py tests/test_gpu_sequences.py -x -q 2>&1 | tail -3
