n() { timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dgemm -s 1 -c 1 --csv python tools/prof.py $1 2 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print "'$1' '$2'", $(NF-2), $NF}'; }
n cfg4 default
TCB_L2HINT=021 n cfg4 b_last_c_first
TCB_L2HINT=001 n cfg4 c_first
TCB_L2PERSIST_MB=64 n cfg4 persist64
TCB_L2PERSIST_MB=64 TCB_L2HINT=021 n cfg4 persist64_cfirst
TCB_L2PERSIST_MB=96 TCB_RASTER=n32 n cfg4 persist96_n32
TCB_PACE=4,1 n cfg4 slack1
