"""Host<->device copy bandwidth (pinned), alone and concurrent (H2D || D2H)."""
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
n = 134217728 // 8 * 2  # 256 MB
h1, h2 = np.ones(n), np.zeros(n)
for h in (h1, h2):
    T.check(dev.tcb_host_register(h.ctypes.data, h.nbytes))
d1, d2 = T.DeviceBuffer(n * 8), T.DeviceBuffer(n * 8)
s1, s2 = C.c_void_p(), C.c_void_p()
dev.tcb_stream_create(C.byref(s1))
dev.tcb_stream_create(C.byref(s2))


def timed(fn, reps=5):
    fn()
    dev.tcb_stream_sync(s1)
    dev.tcb_stream_sync(s2)
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    dev.tcb_stream_sync(s1)
    dev.tcb_stream_sync(s2)
    return (time.perf_counter() - t0) / reps


h2d = timed(lambda: dev.tcb_memcpy_async(d1.ptr, h1.ctypes.data, n * 8, s1))
d2h = timed(lambda: dev.tcb_memcpy_async(h2.ctypes.data, d2.ptr, n * 8, s2))
both = timed(lambda: (dev.tcb_memcpy_async(d1.ptr, h1.ctypes.data, n * 8, s1),
                      dev.tcb_memcpy_async(h2.ctypes.data, d2.ptr, n * 8, s2)))
gb = n * 8 / 1e9
print(json.dumps({"bytes": n * 8, "h2d_GBps": round(gb / h2d, 1), "d2h_GBps": round(gb / d2h, 1),
                  "concurrent_total_GBps": round(2 * gb / both, 1)}))

# 2-D uploads (the streamed paths' slab copies): rows of w bytes out of a
# pitch 2x wider, 64 MB per copy
for w in (4096, 8192, 16384, 32768, 65536, 262144):
    rows = (64 << 20) // w
    pitch = 2 * w
    if rows * pitch > n * 8:
        continue
    t = timed(lambda: dev.tcb_memcpy2d_async(d1.ptr, pitch, h1.ctypes.data, pitch, w, rows, s1))
    print(json.dumps({"h2d_2d_row_bytes": w, "rows": rows, "GBps": round(rows * w / 1e9 / t, 1)}))
