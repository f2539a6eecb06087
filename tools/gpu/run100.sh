M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=4096,j=4096,k=4096" "i=5120,j=5120,k=5120" "i=6144,j=6144,k=6144" "i=8192,j=8192,k=8192" "i=7168,j=7168,k=6144"; do
TC_STREAM_K_NO_NARROW=1 python tools/e2e_ab.py "$M" "$x" 7 | tail -1 | sed 's/^/32KB rows /'
python tools/e2e_ab.py "$M" "$x" 7 | tail -1 | sed 's/^/default   /'
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/stress_streamed.py 150 73 2>&1 | tail -1 | cut -c1-300
python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg5', d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['ms_per_step'], d['parity_ok'], d['e2e']['parity_ok'])"
