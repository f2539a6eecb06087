python tools/slab_gemm_ab.py 4 | tail -3
timeout 900 python -m pytest -q -x tests/test_gpu_kernels.py tests/test_gpu_tiles.py tests/test_gpu_runtime_safety.py 2>&1 | tail -1
timeout 900 python tools/stress_streamed.py 2>&1 | tail -1
timeout 900 python tools/quickcheck.py 2>&1 | tail -3
TC_STREAM_TIMELINE=1 python tools/e2e_ab.py cfg5 2 2>&1 | grep -E "slab 1[1-4] gemm|part 7 down|median"
