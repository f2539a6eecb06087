"""Randomised stress of the streamed host paths (development aid, not a test):
random contractions with at least one operand of 8 MB or more, evaluated with
tc::PreparedContraction::run_streamed from page-locked host buffers — whichever
pipeline it picks (output-label slabs, free-label 2-D slabs, contracted-label
slabs, or the plain path) — three asynchronous calls back to back with
different inputs (the two device buffer sets alternate), each checked against
numpy.einsum at relative Frobenius <= 1e-12.
Usage: python tools/stress_streamed.py [cases] [seed]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import paper_1307_2100_b200 as T  # noqa: E402
from specgen import random_spec  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
EXT = (7, 13, 16, 17, 32, 48, 64, 96, 128, 130, 256)
dev = T.native.device()


def labels(t):
    return [s.strip()[1:] for s in t.split("[")[1].rstrip("] ").split(",") if s.strip()]


def pinned(n):
    a = np.empty(max(int(n), 1))
    T.check(dev.tcb_host_register(a.ctypes.data, a.nbytes))
    return a


done, worst, layouts, t0 = 0, 0.0, {}, time.time()
while done < cases:
    e, x = random_spec(rng, extents=EXT, max_rank=4)
    ext = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in x.split(",")}
    lhs, rhs = e.split("=")
    out = labels(lhs)
    lt, rt = rhs.split("*")
    left, right = labels(lt), labels(rt)
    n = {k: int(np.prod([ext[v] for v in ls])) if ls else 1
         for k, ls in (("l", left), ("r", right), ("o", out))}
    if max(n.values()) * 8 > (300 << 20) or max(n["l"], n["r"]) * 8 < (8 << 20):
        continue
    if np.prod(list(ext.values())) > 4e9:
        continue
    p = T.Prepared(e, x)
    bufs = []
    for s in (1, 3, 5):
        L, R, O = pinned(n["l"]), pinned(n["r"]), pinned(n["o"])
        L[:] = T.seeded(n["l"], s)
        R[:] = T.seeded(n["r"], s + 1)
        bufs.append((L, R, O))
    for L, R, O in bufs:
        p.run_streamed(L, R, O, slabs=0, wait=False)
    p.sync()
    sub = "".join(reversed(left)) + "," + "".join(reversed(right)) + "->" + "".join(reversed(out))
    for L, R, O in bufs:
        A = L.reshape(list(reversed([ext[v] for v in left])) or [1])
        B = R.reshape(list(reversed([ext[v] for v in right])) or [1])
        want = np.einsum(sub, A, B, optimize=True).reshape(-1)
        err = float(np.linalg.norm(O[:want.size] - want) / max(np.linalg.norm(want), 1e-300))
        worst = max(worst, err)
        if not err <= 1e-12:
            print(json.dumps({"FAIL": e, "extents": x, "recipe": T.lower(e, x), "rel_frob": err}))
            sys.exit(1)
    for trio in bufs:
        for a in trio:
            dev.tcb_host_unregister(a.ctypes.data)
    lay = T.lower(e, x).split()[0]
    layouts[lay] = layouts.get(lay, 0) + 1
    p.close()
    done += 1
print(json.dumps({"tool": "stress_streamed", "cases": done, "seed": seed,
                  "worst_rel_frobenius": worst, "recipes": layouts,
                  "seconds": round(time.time() - t0, 1)}))
