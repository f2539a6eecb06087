# hybrid threshold for beta != 0 after the batched old-C loads: staged (TMA reduce-add) vs hybrid per slab length
for l in 8 12 16 24 32; do
echo "l=$l default(768):"; python tools/slab_gemm_ab.py 10 $l
echo "l=$l hybrid from 256:"; TCB_SK_LONGKB=256 python tools/slab_gemm_ab.py 10 $l | tail -1
echo "l=$l staged only:"; TCB_SK_LONGKB=100000 python tools/slab_gemm_ab.py 10 $l
done
