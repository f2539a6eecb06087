bash tools/gpu/ncu_dram.sh cfg5 p42
bash tools/gpu/ncu_dram.sh cfg5 p41 TCB_PACE=4,1
bash tools/gpu/ncu_dram.sh cfg5 p32 TCB_PACE=3,2
bash tools/gpu/ncu_dram.sh cfg5 p31 TCB_PACE=3,1
