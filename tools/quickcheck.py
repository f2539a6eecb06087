"""Quick device sanity run (development aid): kernel known answers, random
GEMMs vs the long-double oracle, random contractions vs the naive oracle."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np, ctypes as C
import paper_1307_2100_b200 as T
import oracles as O
from specgen import random_spec

dev = T.native.device()
T.check(dev.tcb_init(0))
A = T.DeviceBuffer.from_array(np.array([1., 3, 2, 4])); B = T.DeviceBuffer.from_array(np.array([5., 7, 6, 8]))
Cb = T.DeviceBuffer.from_array(np.zeros(4))
T.check(dev.tcb_dgemm(0, 0, 2, 2, 2, 1.0, A.ptr, 2, B.ptr, 2, 0.0, Cb.ptr, 2))
print("2x2", Cb.to_array())
rng = np.random.default_rng(1)
worst = 0
for it in range(60):
    m, n, k = (int(x) for x in rng.integers(1, 300, 3))
    if it % 5 == 0: m, n, k = int(rng.integers(100, 700)), int(rng.integers(100, 700)), int(rng.integers(1, 3000))
    ta, tb = int(rng.integers(2)), int(rng.integers(2))
    lda = (k if ta else m) + int(rng.integers(0, 3)); ldb = (n if tb else k) + int(rng.integers(0, 3)); ldc = m + int(rng.integers(0, 3))
    a = rng.uniform(-1, 1, lda * (m if ta else k)); b = rng.uniform(-1, 1, ldb * (k if tb else n)); c = rng.uniform(-1, 1, ldc * n)
    alpha, beta = 1.5, (0.0 if it % 2 else 0.5)
    ref = c.copy()
    O.tco().tco_gemm_check(ta, tb, m, n, k, alpha, a.ctypes.data, lda, b.ctypes.data, ldb, beta, ref.ctypes.data, ldc)
    da, db, dc = T.DeviceBuffer.from_array(a), T.DeviceBuffer.from_array(b), T.DeviceBuffer.from_array(c)
    T.check(dev.tcb_dgemm(ta, tb, m, n, k, alpha, da.ptr, lda, db.ptr, ldb, beta, dc.ptr, ldc))
    got = dc.to_array(c.size)
    info = T.GemmInfo(); dev.tcb_last_gemm_info(C.byref(info))
    err = np.abs(got - ref).max() / max(1, np.abs(ref).max())
    worst = max(worst, err)
    if err > 1e-12:
        print("GEMM FAIL", m, n, k, ta, tb, lda, ldb, ldc, err, "path", info.path, "splits", info.splits)
print("gemm worst", worst)
bad = 0
for it in range(300):
    e, x = random_spec(rng)
    L, R = O.operands(e, x, 1)
    ref = O.naive(e, x, L, R)
    got, st = T.execute(e, x, seed=1)
    err = O.max_rel_error(got, ref)
    if err > 1e-12:
        bad += 1
        if bad < 5: print("CONTRACT FAIL", e, x, err)
print("contract bad", bad)
for name, e, x in [("cfg1", "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=512,j=512,k=64,l=64"),
                   ("cfg2", "C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=256,b=256,c=256,k=256"),
                   ("cfg3", "C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=64,b=64,c=64,d=64,k=32,l=32")]:
    t0 = time.time(); r = O.ref_execute(e, x, seed=1, workers=16); t1 = time.time()
    got, st = T.execute(e, x, seed=1)
    p = T.Prepared(e, x); L, R = O.operands(e, x, 1); p.upload(L, R); p.run(); p.sync()
    for _ in range(3): p.run()
    T.check(dev.tcb_timer_start())
    for _ in range(10): p.run()
    ms = C.c_float(); T.check(dev.tcb_timer_stop(C.byref(ms)))
    info = p.info()
    fl = info["flops"]
    print(name, "ref s", round(t1 - t0, 3), "frob", O.rel_frobenius(got, r[0]) if r else None,
          "gpu ms", ms.value / 10, "TF/s", fl / (ms.value / 10 * 1e-3) / 1e12, info["summary"], st)
