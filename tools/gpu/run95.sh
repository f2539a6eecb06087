M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
TC_EXEC_TRACE=1 TC_STREAM_K_WIDE=1 python tools/e2e_ab.py "$M" "i=16384,j=16384,k=4096" 1 2>&1 | grep -i "slabs\|median" | tail -8
TC_EXEC_TRACE=1 python tools/e2e_ab.py "$M" "i=8192,j=12288,k=8192" 1 2>&1 | grep -i "slabs\|median" | tail -8
