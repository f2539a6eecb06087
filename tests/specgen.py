"""Random contraction specs in the reference's property-test family
(tests/helpers.hpp:49-107: ranks 2..4, p 1..3, extents 1..max_extent,
shuffled labels, mode positions and output order). Seeded numpy RNG — the
family, not the exact C++ sample, is what the parity suites need."""
from __future__ import annotations

import numpy as np

POOL = list("abcdefgh")


def random_spec(rng: np.random.Generator, max_extent: int = 6, max_rank: int = 4,
                extents=None):
    """A random valid contraction; label extents uniform in [1, max_extent],
    or drawn from the `extents` sequence when given."""
    while True:
        lrank = int(rng.integers(2, max_rank + 1))
        rrank = int(rng.integers(2, max_rank + 1))
        p = int(rng.integers(1, 4))
        if p > lrank or p > rrank:
            continue
        labels = list(rng.permutation(POOL))
        lslots = list(rng.permutation(lrank))
        rslots = list(rng.permutation(rrank))
        lidx = [None] * lrank
        ridx = [None] * rrank
        nxt = 0
        for i in range(p):
            lab = labels[nxt]; nxt += 1
            v = "+" if rng.integers(2) else "-"
            lidx[lslots[i]] = v + lab
            ridx[rslots[i]] = ("-" if v == "+" else "+") + lab
        outs = []
        for i in range(p, lrank):
            lab = labels[nxt]; nxt += 1
            lidx[lslots[i]] = ("+" if rng.integers(2) else "-") + lab
            outs.append(lidx[lslots[i]])
        for i in range(p, rrank):
            lab = labels[nxt]; nxt += 1
            ridx[rslots[i]] = ("+" if rng.integers(2) else "-") + lab
            outs.append(ridx[rslots[i]])
        outs = list(rng.permutation(outs)) if outs else []
        expr = f"R[{','.join(outs)}] = A[{','.join(lidx)}] * B[{','.join(ridx)}]"
        ext = {}
        for tok in lidx + ridx:
            ext.setdefault(tok[1:], int(rng.choice(extents)) if extents is not None
                           else int(rng.integers(1, max_extent + 1)))
        extents = ",".join(f"{k}={v}" for k, v in ext.items())
        return expr, extents


def table1_expressions():
    """The paper's 18 order-3 double contractions (tests/helpers.hpp:112-139)."""
    sets = [("b", "g"), ("a", "g"), ("a", "b")]
    frees = ["a", "b", "g"]
    out = []
    for s, cs in enumerate(sets):
        for pos in range(3):
            for order in range(2):
                c1, c2 = (cs[1], cs[0]) if order else (cs[0], cs[1])
                bl, ci = [], 0
                for k in range(3):
                    if k == pos:
                        bl.append("e")
                    else:
                        bl.append(c2 if ci else c1)
                        ci += 1
                out.append(f"R[+{frees[s]},-e] = A[+a,+b,+g] * B[" +
                           ",".join("-" + x for x in bl) + "]")
    return out
