"""k3 permutation bandwidth: cfg3's two operand permutations at their native
size (L2-resident) and scaled to >= 1 GB (HBM-bound), plus a device memcpy
for reference. Prints one JSON line per case (algorithmic bytes = read +
write of the operand)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1307_2100_b200 as T

dev = T.native.device()
T.check(dev.tcb_init(0))
def _hbm_peak() -> float:
    """MEASURED_PEAKS.json hbm_gbs (driver-written copy bandwidth of this pool's
    B200s), else the B200_PROFILING.md fallback."""
    import json
    from pathlib import Path
    f = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(f.read_text())["hbm_gbs"])
    except Exception:
        return 6552.0


HBM = _hbm_peak()


def perm_case(name, ext, src_str, reps=20):
    n = int(np.prod(ext))
    src = T.DeviceBuffer(n * 8)
    dst = T.DeviceBuffer(n * 8)
    dev.tcb_memset0(src.ptr, n * 8)
    r = len(ext)
    e = (C.c_int64 * r)(*ext)
    s = (C.c_int64 * r)(*src_str)
    for _ in range(3):
        T.check(dev.tcb_permute(r, e, s, src.ptr, dst.ptr))
    ms = C.c_float()
    T.check(dev.tcb_timer_start())
    for _ in range(reps):
        T.check(dev.tcb_permute(r, e, s, src.ptr, dst.ptr))
    T.check(dev.tcb_timer_stop(C.byref(ms)))
    t = ms.value / reps * 1e-3
    gbs = 2 * n * 8 / t / 1e9
    print(json.dumps({"case": name, "bytes": 2 * n * 8, "us": round(t * 1e6, 2),
                      "GBps": round(gbs, 1), "frac_hbm": round(gbs / HBM, 3)}), flush=True)


def strides(ext):
    s, run = [], 1
    for x in ext:
        s.append(run)
        run *= x
    return s


def cfg3_perms(a, b, c, d, k, l, tag):
    # A[a,k,c,l] -> A'[a,c,l,k]; B[l,b,k,d] -> B'[l,k,b,d]  (lower.cpp L3 recipe)
    sa = dict(zip("akcl", strides([a, k, c, l])))
    perm_case(f"{tag} A[a,k,c,l]->[a,c,l,k]", [a, c, l, k], [sa[x] for x in "aclk"])
    sb = dict(zip("lbkd", strides([l, b, k, d])))
    perm_case(f"{tag} B[l,b,k,d]->[l,k,b,d]", [l, k, b, d], [sb[x] for x in "lkbd"])
    # a transpose-type permutation (unit-stride dims differ): A[a,k,c,l] -> [k,a,c,l]
    perm_case(f"{tag} A[a,k,c,l]->[k,a,c,l] (transpose)", [k, a, c, l], [sa[x] for x in "kacl"])


cfg3_perms(64, 64, 64, 64, 32, 32, "cfg3 native (33.5 MB, L2-resident)")
cfg3_perms(128, 128, 128, 128, 128, 64, "cfg3-shape x32 (1.07 GB)")
n = 2**27
src, dst = T.DeviceBuffer(n * 8), T.DeviceBuffer(n * 8)
ms = C.c_float()
dev.tcb_d2d(dst.ptr, src.ptr, n * 8)
T.check(dev.tcb_timer_start())
for _ in range(10):
    dev.tcb_d2d(dst.ptr, src.ptr, n * 8)
T.check(dev.tcb_timer_stop(C.byref(ms)))
t = ms.value / 10 * 1e-3
print(json.dumps({"case": "cudaMemcpy D2D 1.07 GB", "GBps": round(2 * n * 8 / t / 1e9, 1)}))
