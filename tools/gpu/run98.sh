M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for n in 1024 2048 3072 4096 6144; do
x="i=$n,j=$n,k=$n"
TC_STREAM_K_SQUARE=never python tools/e2e_ab.py "$M" "$x" 9 | tail -1 | sed 's/^/o-mode  /'
TC_STREAM_K_SQUARE=always python tools/e2e_ab.py "$M" "$x" 9 | tail -1 | sed 's/^/k-mode  /'
python tools/e2e_ab.py "$M" "$x" 9 | tail -1 | sed 's/^/default /'
done
