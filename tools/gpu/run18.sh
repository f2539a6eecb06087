mkdir -p gpurun_out
for d in 0 8; do
for c in cfg1 cfg2 cfg4; do
rm -f /tmp/tr.jsonl
TCB_DIAG=$d TCB_TRACE=/tmp/tr.jsonl timeout 300 python tools/prof.py $c 3 > /dev/null
echo "== $c diag=$d"; tail -1 /tmp/tr.jsonl > /tmp/t1; python tools/trace_summary.py /tmp/t1 | grep -v nan
done; done
