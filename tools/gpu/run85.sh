# mode choice of the streamed path on plain matrix products: output-label slabs vs contracted-label slabs
M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=8192,j=8192,k=8192" "i=12288,j=12288,k=12288" "i=8192,j=12288,k=8192" "i=16384,j=16384,k=8192" "i=16384,j=16384,k=16384"; do
python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/default   /'
TC_STREAM_K_EQ=1 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/k if <=   /'
TC_STREAM_K_RATIO=2 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/k if <=2x /'
TC_STREAM_K_RATIO=4 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/k if <=4x /'
done
