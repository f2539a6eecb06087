"""Times the drop-in call (tcf_execute_host, pinned host buffers) on a BASELINE
config, or on any expression: median of N calls after one warm-up.
Usage: python tools/e2e_ab.py cfg5 [N]  |  python tools/e2e_ab.py "<expr>" "<extents>" [N]"""
import ctypes as C
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_1307_2100_b200 as T  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
if cfg in bench.CONFIGS:
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    expr, ext, _ = bench.CONFIGS[cfg]
else:
    expr, ext = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    cfg = ext
dev = T.native.device()
T.check(dev.tcb_init(0))
p = T.Prepared(expr, ext)
inf = p.info()
p.close()
L, R, O = (bench.pinned_array(inf[k], dev) for k in ("left", "right", "output"))
bench.fill_operands(expr, ext, None, 0, 0, L, R)
T.execute_host(expr, ext, L, R, O)
ts = []
for _ in range(n):
    t = time.perf_counter()
    T.execute_host(expr, ext, L, R, O)
    ts.append(time.perf_counter() - t)
print(f"{cfg} execute_host median {statistics.median(ts) * 1e3:.2f} ms  all {[round(x * 1e3, 2) for x in ts]}"
      f"  GFLOP/s {inf['flops'] / statistics.median(ts) / 1e9:.0f}")
