"""Host cost per device call: back-to-back tiny contractions through the
prepared API (run) and the BLAS-level tcb_dgemm, wall time per call vs the
device time of the same launches (CUDA events)."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1307_2100_b200 as T

dev = T.native.device()
T.check(dev.tcb_init(0))
for e, x in (("C[+i,+j] = A[+i,+k] * B[-k,+j]", "i=128,j=128,k=64"),
             ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=512,j=512,k=64,l=8"),
             ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=64,b=64,c=16,k=64")):
    p = T.Prepared(e, x)
    inf = p.info()
    p.upload(np.ones(inf["left"]), np.ones(inf["right"]))
    for _ in range(50):
        p.run()
    p.sync()
    n = 2000
    ms = C.c_float()
    t0 = time.perf_counter()
    T.check(dev.tcb_timer_start())
    for _ in range(n):
        p.run_contraction()
    T.check(dev.tcb_timer_stop(C.byref(ms)))
    wall = (time.perf_counter() - t0) / n * 1e6
    print(json.dumps({"expr": e, "extents": x, "recipe": inf["summary"][:40],
                      "wall_us_per_call": round(wall, 2), "device_us_per_call": round(ms.value * 1e3 / n, 2)}),
          flush=True)
    p.close()
