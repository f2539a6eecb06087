echo "== no pdl"; TCB_NO_PDL=1 python tools/slab_gemm_ab.py 4 | tail -2
echo "== no coop"; TCB_NO_COOP=1 python tools/slab_gemm_ab.py 4 | tail -2
echo "== no coop no pdl"; TCB_NO_COOP=1 TCB_NO_PDL=1 python tools/slab_gemm_ab.py 4 | tail -2
