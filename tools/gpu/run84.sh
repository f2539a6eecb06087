# output-label streamed path on a compute-bound plain matrix product: ramp vs equal slabs
M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=8192,j=8192,k=8192" "i=16384,j=16384,k=4096" "i=4096,j=32768,k=16384"; do
for i in 1 2; do
TC_NO_SLAB_RAMP=1 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/equal /'
python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/ramp  /'
done
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_index_groups.py tests/test_gpu_threads.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/stress_streamed.py 150 41 2>&1 | tail -1 | cut -c1-300
