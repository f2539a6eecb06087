mkdir -p gpurun_out
S=tools/gpu/ncu_dram.sh
bash $S cfg5 default
bash $S cfg5 p52 TCB_PACE=5,2
bash $S cfg5 p41 TCB_PACE=4,1
bash $S cfg5 noflip TCB_NO_KFLIP=1
bash $S cfg5 m8 TCB_RASTER=m8
bash $S cfg4 default
bash $S cfg4 noflip TCB_NO_KFLIP=1
bash $S cfg4 n32 TCB_RASTER=n32
bash $S cfg4 n8 TCB_RASTER=n8
bash $S cfg4 m8 TCB_RASTER=m8
bash $S cfg4 m12 TCB_RASTER=m12
bash $S cfg4 nopace TCB_NO_PACE=1
python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r4_cfg5.json 2>&1; tail -1 gpurun_out/r4_cfg5.json | cut -c1-300
python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r4_cfg4.json 2>&1; tail -1 gpurun_out/r4_cfg4.json | cut -c1-300
