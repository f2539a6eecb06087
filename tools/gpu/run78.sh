# cfg4 raster group sweep: DRAM bytes per launch (ncu) and duration
bash tools/gpu/ncu_dram.sh cfg4 n16
bash tools/gpu/ncu_dram.sh cfg4 n12 TCB_RASTER=n12
bash tools/gpu/ncu_dram.sh cfg4 n11 TCB_RASTER=n11
bash tools/gpu/ncu_dram.sh cfg4 n20 TCB_RASTER=n20
bash tools/gpu/ncu_dram.sh cfg4 n24 TCB_RASTER=n24
bash tools/gpu/ncu_dram.sh cfg4 m12 TCB_RASTER=m12
