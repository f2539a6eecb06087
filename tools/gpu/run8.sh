python tools/e2e_ab.py cfg5 3
python -m pytest tests/test_gpu_parity.py -x -q -k "streamed" 2>&1 | tail -2
timeout 900 python tools/stress_streamed.py 120 9 2>&1 | tail -1
python -m pytest tests/test_gpu_runtime_safety.py tests/test_gpu_bench_harness.py -x -q 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r8_bench.json 2>gpurun_out/r8_bench.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r8_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pipelined']['value'], d['parity_ok'], d['e2e']['parity_ok'])"
