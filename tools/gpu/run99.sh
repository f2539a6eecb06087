M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=3072,j=3072,k=3072" "i=4096,j=4096,k=4096" "i=6144,j=6144,k=6144" "i=8192,j=8192,k=4096" "i=16384,j=16384,k=4096" "i=8192,j=8192,k=8192"; do
TC_STREAM_K_NO_NARROW=1 python tools/e2e_ab.py "$M" "$x" 7 | tail -1 | sed 's/^/32KB rows /'
python tools/e2e_ab.py "$M" "$x" 7 | tail -1 | sed 's/^/4KB rows  /'
done
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do python tools/e2e_ab.py $c 3 | tail -1; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_index_groups.py tests/test_gpu_threads.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
for sd in 71 72; do timeout 900 python tools/stress_streamed.py 150 $sd 2>&1 | tail -1 | cut -c1-300; done
