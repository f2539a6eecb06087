echo "== default"; python tools/slab_gemm_ab.py 4 | tail -2
echo "== no hybrid"; TCB_SK_WASTE=1 python tools/slab_gemm_ab.py 4 | tail -2
echo "== no pace"; TCB_NO_PACE=1 python tools/slab_gemm_ab.py 4 | tail -2
echo "== no cstore"; TCB_NO_CSTORE=1 python tools/slab_gemm_ab.py 4 | tail -2
