"""Randomised stress of the device path (development aid, not a test): many
random contractions with extents mixing multiples of 16 and odd sizes, up to
~2e8 multiply-adds, evaluated through tc::execute (every recipe: L1 / L2 / L3 /
L4, stream-K, GEMV / DOT, TMA store or fallback epilogues) and checked against
numpy.einsum (BLAS, fp64) at relative Frobenius <= 1e-12 (or, for results
dominated by cancellation, the reference's max_rel_error <= 1e-12).
Usage: python tools/stress.py [cases] [seed]"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np
import paper_1307_2100_b200 as T
from specgen import random_spec

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
verbose = os.environ.get("STRESS_VERBOSE") is not None  # print each case before running it
EXT = (1, 2, 3, 5, 7, 13, 16, 17, 32, 48, 64, 96, 128, 130)


def operand(labels, ext, s):
    n = int(np.prod([ext[x] for x in labels])) if labels else 1
    v = T.seeded(n, s)
    return v.reshape(list(reversed([ext[x] for x in labels])) or [1])


done, worst, layouts, t0 = 0, 0.0, {}, time.time()
while done < cases:
    e, x = random_spec(rng, extents=EXT, max_rank=4)
    ext = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in x.split(",")}
    if np.prod(list(ext.values())) > 2e8:
        continue
    lhs, rhs = e.split("=")
    out = [t.strip()[1:] for t in lhs.split("[")[1].rstrip("] ").split(",") if t.strip()]
    lt, rt = rhs.split("*")
    left = [t.strip()[1:] for t in lt.split("[")[1].rstrip("] ").split(",")]
    right = [t.strip()[1:] for t in rt.split("[")[1].rstrip("] ").split(",")]
    if verbose:
        print(json.dumps({"case": done, "expr": e, "extents": x}), flush=True)
    got, st = T.execute(e, x, seed=1)
    A = operand(left, ext, 1)
    B = operand(right, ext, 2)
    sub = "".join(reversed(left)) + "," + "".join(reversed(right)) + "->" + "".join(reversed(out))
    want = np.einsum(sub, A, B, optimize=True).reshape(-1)
    err = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
    # the reference's own criterion (max|a-b| / max(1, max|b|), src/executor.cpp:385-394)
    # for results with heavy cancellation (a scalar DOT summing to ~0)
    mre = float(np.abs(got - want).max() / max(1.0, float(np.abs(want).max())))
    lay = T.lower(e, x).split()[0]
    layouts[lay] = layouts.get(lay, 0) + 1
    worst = max(worst, min(err, mre))
    if not (err <= 1e-12 or mre <= 1e-12):
        print(json.dumps({"FAIL": e, "extents": x, "recipe": T.lower(e, x), "rel_frob": err}))
        sys.exit(1)
    done += 1
print(json.dumps({"cases": done, "worst_rel_frobenius": worst, "recipes": layouts,
                  "seconds": round(time.time() - t0, 1)}))
