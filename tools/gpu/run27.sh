mkdir -p gpurun_out
rm -f gpurun_out/tr_cfg1_new.jsonl; TCB_TRACE=gpurun_out/tr_cfg1_new.jsonl timeout 300 python tools/prof.py cfg1 5 > /dev/null
TCB_DIAG=32 TCB_TRACE=gpurun_out/tr_cfg1_new_clk.jsonl timeout 300 python tools/prof.py cfg1 5 > /dev/null
