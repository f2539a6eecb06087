M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=16384,j=16384,k=4096" "i=24576,j=24576,k=4096" "i=12288,j=12288,k=4096" "i=32768,j=8192,k=8192" "i=7168,j=7168,k=6144" "i=16384,j=8192,k=2048"; do
python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/default /'
TC_STREAM_K_WIDE=1 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/wide    /'
done
python tools/e2e_ab.py cfg4 3 | tail -1 | sed 's/^/default /'
TC_STREAM_K_WIDE=1 python tools/e2e_ab.py cfg4 3 | tail -1 | sed 's/^/wide    /'
