M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=8192,j=8192,k=8192" "i=12288,j=12288,k=12288" "i=16384,j=16384,k=16384" "i=4096,j=4096,k=65536" "i=8192,j=12288,k=8192"; do
python tools/e2e_ab.py "$M" "$x" 5 | tail -1
done
python tools/e2e_ab.py "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]" "i=4096,j=4096,k=64,l=512" 5 | tail -1
python tools/e2e_ab.py cfg5 2 | tail -1
python tools/e2e_ab.py cfg1 5 | tail -1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_index_groups.py tests/test_gpu_threads.py tests/test_gpu_runtime_safety.py -m gpu -x -q 2>&1 | tail -3
for sd in 61 62; do timeout 900 python tools/stress_streamed.py 150 $sd 2>&1 | tail -1 | cut -c1-300; done
