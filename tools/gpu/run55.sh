for i in 1 2 3; do bash tools/gpu/ncu_dram.sh cfg5 rep$i; done
