"""Randomised stress of back-to-back device contractions (development aid, not
a test): a pool of random prepared contractions (every recipe kind, stream-K
and data-parallel grids, GEMV / DOT, permutations) is run many times in random
order on one stream, so consecutive GEMMs chain under programmatic dependent
launch and share the stream-K workspace and arrival counters. Every result must
be bit-identical to the same contraction's first (isolated) result, which is
checked against numpy.einsum at relative Frobenius <= 1e-12.
Usage: python tools/stress_sequences.py [pool] [rounds] [seed]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import paper_1307_2100_b200 as T  # noqa: E402
from specgen import random_spec  # noqa: E402

pool_n = int(sys.argv[1]) if len(sys.argv) > 1 else 24
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 40
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rng = np.random.default_rng(seed)
EXT = (1, 3, 7, 16, 17, 32, 48, 64, 96, 128, 130, 256)


def labels(t):
    return [s.strip()[1:] for s in t.split("[")[1].rstrip("] ").split(",") if s.strip()]


t0 = time.time()
pool = []
while len(pool) < pool_n:
    e, x = random_spec(rng, extents=EXT, max_rank=4)
    ext = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in x.split(",")}
    if np.prod(list(ext.values())) > 3e8:
        continue
    lhs, rhs = e.split("=")
    out = labels(lhs)
    lt, rt = rhs.split("*")
    left, right = labels(lt), labels(rt)
    p = T.Prepared(e, x)
    inf = p.info()
    L = T.seeded(inf["left"], 1 + len(pool))
    R = T.seeded(inf["right"], 2 + len(pool))
    p.upload(L, R)
    p.run()
    first = np.empty(max(inf["output"], 1))
    p.download(first)
    A = L.reshape(list(reversed([ext[v] for v in left])) or [1])
    B = R.reshape(list(reversed([ext[v] for v in right])) or [1])
    sub = "".join(reversed(left)) + "," + "".join(reversed(right)) + "->" + "".join(reversed(out))
    want = np.einsum(sub, A, B, optimize=True).reshape(-1)
    err = float(np.linalg.norm(first[:want.size] - want) / max(np.linalg.norm(want), 1e-300))
    mre = float(np.abs(first[:want.size] - want).max() / max(1.0, float(np.abs(want).max())))
    if not (err <= 1e-12 or mre <= 1e-12):
        print(json.dumps({"FAIL_first": e, "extents": x, "recipe": T.lower(e, x), "rel": err}))
        sys.exit(1)
    pool.append((e, x, p, first))

checked = 0
for r in range(rounds):
    order = rng.permutation(len(pool))
    for i in order:  # enqueue the whole round back to back
        pool[i][2].run()
    for i in order[-4:]:  # the last few of the round, compared bit for bit
        e, x, p, first = pool[i]
        out = np.empty_like(first)
        p.download(out)
        if not np.array_equal(out.view(np.uint64), first.view(np.uint64)):
            print(json.dumps({"FAIL_sequence": e, "extents": x, "recipe": T.lower(e, x),
                              "round": r}))
            sys.exit(1)
        checked += 1
    # a full check of everything once in a while (downloads break the chain)
    if r % 10 == 9:
        for e, x, p, first in pool:
            out = np.empty_like(first)
            p.download(out)
            if not np.array_equal(out.view(np.uint64), first.view(np.uint64)):
                print(json.dumps({"FAIL_sequence_full": e, "extents": x, "round": r}))
                sys.exit(1)
            checked += 1
recipes = {}
for e, x, _, _ in pool:
    k = T.lower(e, x).split()[0]
    recipes[k] = recipes.get(k, 0) + 1
print(json.dumps({"tool": "stress_sequences", "pool": pool_n, "rounds": rounds, "seed": seed,
                  "results_compared": checked, "recipes": recipes,
                  "seconds": round(time.time() - t0, 1)}))
