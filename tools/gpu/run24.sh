b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d['gpu_launches'])"; }
n() { timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:dgemm -s 1 -c 1 --csv python tools/prof.py $1 2 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print "'$1' '$2'", $(NF-2), $NF}'; }
for mb in 16 32 48; do
TCB_L2PERSIST_MB=$mb b cfg4 30 p$mb
TCB_L2PERSIST_MB=$mb n cfg4 p$mb
done
TCB_NO_L2PERSIST=1 b cfg4 30 nopersist
