"""Per-tile overhead probe: strided-batched GEMM m=n=256, batch=256 (cfg2's
tile grid) with K swept; efficiency vs K separates per-tile from per-k-block
costs."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1307_2100_b200 as T

dev = T.native.device()
T.check(dev.tcb_init(0))
peak = C.c_double()
dev.tcb_fp64_peak(C.byref(peak))
m = n = 256
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for k in [16, 32, 64, 128, 256, 512, 1024, 2048, 4096]:
    A = T.DeviceBuffer(m * k * batch * 8)
    B = T.DeviceBuffer(k * n * 8)
    Cb = T.DeviceBuffer(m * n * batch * 8)
    for b in (A, B, Cb):
        dev.tcb_memset0(b.ptr, b.nbytes)
    args = (0, 0, m, n, k, 1.0, A.ptr, m, m * k, B.ptr, k, 0, 0.0, Cb.ptr, m, m * n, batch)
    for _ in range(3):
        T.check(dev.tcb_dgemm_strided_batched(*args))
    reps = 20
    ms = C.c_float()
    T.check(dev.tcb_timer_start())
    for _ in range(reps):
        dev.tcb_dgemm_strided_batched(*args)
    T.check(dev.tcb_timer_stop(C.byref(ms)))
    t = ms.value / reps
    tf = 2.0 * m * n * k * batch / (t * 1e-3) / 1e12
    tiles_per_sm = batch * 4 / 148
    print(json.dumps({"k": k, "ms": round(t, 4), "tflops": round(tf, 2),
                      "frac": round(tf / peak.value, 3),
                      "us_per_tile": round(t * 1e3 / tiles_per_sm, 2)}), flush=True)
