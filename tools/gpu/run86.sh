# contracted-label streamed path: last slab sized to hide the result's download (TC_NO_LAST_MERGE=1: an eighth)
M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=8192,j=8192,k=8192" "i=12288,j=12288,k=12288" "i=16384,j=16384,k=16384" "i=4096,j=4096,k=65536"; do
TC_NO_LAST_MERGE=1 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/eighth /'
python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/merged /'
done
for c in cfg5 cfg1; do
TC_NO_LAST_MERGE=1 python tools/e2e_ab.py $c 3 | tail -1 | sed 's/^/eighth /'
python tools/e2e_ab.py $c 3 | tail -1 | sed 's/^/merged /'
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_index_groups.py tests/test_gpu_threads.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/stress_streamed.py 150 43 2>&1 | tail -1 | cut -c1-300
