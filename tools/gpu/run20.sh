b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'])"; }
n() { timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dgemm -s 1 -c 1 --csv python tools/prof.py $1 2 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print "'$1' '$2'", $(NF-2), $NF}'; }
b cfg4 30 default
n cfg4 default
TCB_L2HINT=00 b cfg4 30 nohint
TCB_L2HINT=00 n cfg4 nohint
TCB_L2HINT=10 n cfg4 a_first
TCB_L2HINT=02 n cfg4 b_last
TCB_RASTER=n32 n cfg4 n32
TCB_RASTER=n32 TCB_L2HINT=00 n cfg4 n32_nohint
TCB_RASTER=n8 n cfg4 n8
TCB_RASTER=n32 b cfg4 30 n32
b cfg5 3 default
