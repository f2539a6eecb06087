TCB_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config cfg5 --steps 3 --warmup 3 > gpurun_out/r13_plumb_cfg5.json 2> gpurun_out/r13_plumb_cfg5.err; echo rc=$?
tail -3 gpurun_out/r13_plumb_cfg5.err
python -c "
import json; d=json.loads(open('gpurun_out/r13_plumb_cfg5.json').read().strip().splitlines()[-1])
print(d['value'], d['parity_ok'], d['config']['parallelism'][:120], d['config'].get('exchange_fallback'))"
python -m pytest tests/test_gpu_comm.py tests/test_gpu_peer_procs.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
