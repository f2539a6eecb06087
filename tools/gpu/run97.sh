# ncu of a beta = 1 GEMM (8192^2 x 256) through the TMA reduce-add epilogue, and of the storer path (TCB_NO_CRED=1)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 4 -c 1 -f -o gpurun_out/r97_beta1_cred python tools/slab_gemm_ab.py 2 1 256 > gpurun_out/r97_a.log 2>&1; echo "rc=$?"
TCB_NO_CRED=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dgemm -s 4 -c 1 -f -o gpurun_out/r97_beta1_storers python tools/slab_gemm_ab.py 2 1 256 > gpurun_out/r97_b.log 2>&1; echo "rc=$?"
