M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
TC_STREAM_TIMELINE=1 python tools/e2e_ab.py "$M" "i=8192,j=8192,k=8192" 1 2>&1 | tail -75 | cut -c1-120
