"""A/B of one cfg5-slab GEMM (m = n = 8192, k = 32768: 64 of the 512 l-values)
through tcb_gemm on device buffers: beta 0 vs 1 (the streamed path
accumulates slabs into C), plain vs gated launch. Development aid.
Usage: python tools/slab_gemm_ab.py [reps] [l-values] [k (overrides 512 * l-values)]"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1307_2100_b200 as T  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ls = int(sys.argv[2]) if len(sys.argv) > 2 else 64  # l-values of the slab (k = 512 l)
m = n = 8192
k = int(sys.argv[3]) if len(sys.argv) > 3 else 512 * ls
dev = T.native.device()
T.check(dev.tcb_init(0))
A, B, Cm = (T.DeviceBuffer(x * 8) for x in (m * k, k * n, m * n))
for buf in (A, B, Cm):
    T.check(dev.tcb_memset0(buf.ptr, buf.nbytes))


def desc(beta):
    d = T.GemmDesc()
    d.m, d.n, d.k = m, n, k
    d.a_sm, d.a_sk, d.b_sk, d.b_sn = 1, m, 1, k
    d.c_nrow, d.c_ncol = 1, 1
    d.c_row_ext[0], d.c_row_str[0] = m, 1
    d.c_col_ext[0], d.c_col_str[0] = n, m
    d.alpha, d.beta = 1.0, beta
    return d


ms = C.c_float()
for beta in (0.0, 1.0):
    d = desc(beta)
    T.check(dev.tcb_gemm(C.byref(d), A.ptr, B.ptr, Cm.ptr))
    T.check(dev.tcb_sync())
    T.check(dev.tcb_timer_start())
    for _ in range(reps):
        T.check(dev.tcb_gemm(C.byref(d), A.ptr, B.ptr, Cm.ptr))
    T.check(dev.tcb_timer_stop(C.byref(ms)))
    t = ms.value / reps
    print(f"l={ls} k={k} beta={beta:g}: {t:.3f} ms per launch, {2 * m * n * k / t / 1e9:.0f} TFLOP/s")
