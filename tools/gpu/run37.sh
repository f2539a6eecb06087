TC_EXEC_TRACE=1 python tools/e2e_ab.py cfg1 3 2>&1 | tail -11
for c in cfg1 cfg2 cfg3; do python tools/e2e_ab.py $c 20; done
timeout 1200 python -m pytest -q -x tests/test_gpu_runtime_safety.py tests/test_gpu_bench_harness.py tests/test_gpu_threads.py tests/test_gpu_streamed.py 2>&1 | tail -1
timeout 900 python tools/stress_streamed.py 2>&1 | tail -1
