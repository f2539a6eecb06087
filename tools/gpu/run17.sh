mkdir -p gpurun_out
timeout 120 ./tools/l2_partials_bench
rm -f gpurun_out/tr_cfg1.jsonl gpurun_out/tr_cfg2.jsonl
TCB_TRACE=gpurun_out/tr_cfg1.jsonl timeout 300 python tools/prof.py cfg1 5 > /dev/null
TCB_TRACE=gpurun_out/tr_cfg2.jsonl timeout 300 python tools/prof.py cfg2 3 > /dev/null
tail -1 gpurun_out/tr_cfg1.jsonl > /tmp/t1; python tools/trace_summary.py /tmp/t1
tail -1 gpurun_out/tr_cfg2.jsonl > /tmp/t2; python tools/trace_summary.py /tmp/t2
