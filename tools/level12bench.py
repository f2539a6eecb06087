"""k4 (GEMV / DOT) HBM roofline: reference class-2 and class-1 contractions
large enough to be HBM-bound, through the prepared plan-level API. Prints one
JSON line per case: algorithmic bytes = every operand element read once +
the result written, vs the measured copy bandwidth (MEASURED_PEAKS.json hbm_gbs, 6552 GB/s)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import ctypes as C
import paper_1307_2100_b200 as T

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
dev = T.native.device()
T.check(dev.tcb_init(0))
CASES = [
    ("class 2 GEMV, matrix row-contiguous", "R[+a] = T[+a,+b,+g] * G[-b,-g]", "a=8192,b=512,g=256"),
    ("class 2 GEMV, matrix k-contiguous", "R[+g] = T[+a,+b,+g] * G[-a,-b]", "a=512,b=256,g=8192"),
    ("class 2 GEMV, few rows", "R[+a] = T[+a,+b,+g] * G[-b,-g]", "a=16,b=8192,g=8192"),
    ("class 1 DOT", "K[] = T[+a,+b,+g] * S[-a,-b,-g]", "a=1024,b=512,g=256"),
]
for name, e, x in CASES:
    p = T.Prepared(e, x)
    inf = p.info()
    for ptr in p.device_ptrs():
        pass
    a, b, _ = p.device_ptrs()
    dev.tcb_memset0(a, inf["left"] * 8)
    dev.tcb_memset0(b, inf["right"] * 8)
    for _ in range(3):
        p.run()
    reps = 20
    ms = C.c_float()
    T.check(dev.tcb_timer_start())
    for _ in range(reps):
        p.run()
    T.check(dev.tcb_timer_stop(C.byref(ms)))
    t = ms.value / reps * 1e-3
    nbytes = (inf["left"] + inf["right"] + inf["output"]) * 8
    print(json.dumps({"case": name, "expr": e, "extents": x, "recipe": inf["summary"],
                      "path": ["gemm-tma", "gemm-cpasync", "gemv", "dot"][inf["path"]],
                      "launches": inf["launches"], "us": round(t * 1e6, 2),
                      "GBps": round(nbytes / t / 1e9, 1),
                      "frac_hbm": round(nbytes / t / 1e9 / HBM, 3)}), flush=True)
    p.close()
