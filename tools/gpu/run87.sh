# mode choice with a larger output: contracted-label slabs (merged last slab) when download <= 0.4 x contraction
M='C[+i,+j] = A[+i,+k] * B[-k,+j]'
for x in "i=8192,j=12288,k=8192" "i=16384,j=16384,k=8192" "i=16384,j=16384,k=4096" "i=32768,j=8192,k=8192"; do
TC_STREAM_K_DOWN=0 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/old rule /'
python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/0.4      /'
TC_STREAM_K_DOWN=0.7 python tools/e2e_ab.py "$M" "$x" 5 | tail -1 | sed 's/^/0.7      /'
done
for c in cfg4 cfg3 cfg2; do
TC_STREAM_K_DOWN=0 python tools/e2e_ab.py $c 3 | tail -1 | sed 's/^/old rule /'
python tools/e2e_ab.py $c 3 | tail -1 | sed 's/^/0.4      /'
TC_STREAM_K_DOWN=0.7 python tools/e2e_ab.py $c 3 | tail -1 | sed 's/^/0.7      /'
done
