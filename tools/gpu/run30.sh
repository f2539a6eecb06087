STRESS_VERBOSE=1 timeout 900 python tools/stress.py 1500 11 > gpurun_out/r30_stress.log 2>&1; echo rc=$?
tail -4 gpurun_out/r30_stress.log | cut -c1-400
