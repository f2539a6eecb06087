b() { python bench.py --config $1 --steps $2 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$1', '$3', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity_ok'], d['gpu_launches'])"; }
b cfg4 30 default
TCB_NO_L2DEMOTE=1 b cfg4 30 nodemote
TCB_NO_L2PERSIST=1 b cfg4 30 nopersist
b cfg4 30 default
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:l2_demote -c 2 --csv python tools/prof.py cfg4 2 2>/dev/null | grep gpu__time
