for l in 64 16; do python tools/slab_gemm_ab.py 5 $l; done
python tools/slab_gemm_ab.py 20 1 256
python tools/slab_gemm_ab.py 20 1 1024
python tools/slab_gemm_ab.py 10 1 4096
