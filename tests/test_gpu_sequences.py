"""Back-to-back device work of different shapes on the engine's stream:
programmatic dependent launch between GEMMs, stream-K counters and workspace
reused across launches of different tile grids, GEMV / permutation launches in
between. Every repetition must reproduce the first one bit for bit, and the
first must match the oracle (relative Frobenius 1e-12). Requires a B200."""
import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T

pytestmark = pytest.mark.gpu

CASES = [
    ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=256,j=384,k=64,l=32"),        # stream-K
    ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=128,b=96,c=20,k=80"),         # batched
    ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=128,j=128,k=96,l=40"),        # stream-K, other grid
    ("R[+a] = T[+a,+b,+g] * G[-b,-g]", "a=300,b=64,g=33"),                    # GEMV
    ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=32,b=16,c=5,d=7,k=3,l=16"),  # L4
    ("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "a=40,b=48,g=24,e=56"),          # 3.1: permute
]


def test_interleaved_sequences_are_reproducible(dev):
    preps, want, first = [], [], []
    for e, x in CASES:
        p = T.Prepared(e, x)
        inf = p.info()
        L, R = O.operands(e, x, 1)
        p.upload(L, R)
        preps.append((p, np.empty(inf["output"])))
        want.append(O.naive(e, x, L, R))
    rng = np.random.default_rng(7)
    order = list(range(len(CASES))) * 6
    rng.shuffle(order)
    results = {i: [] for i in range(len(CASES))}
    for i in order:
        p, out = preps[i]
        for _ in range(int(rng.integers(1, 4))):  # runs back to back (PDL chains)
            p.run()
        p.download(out)
        results[i].append(out.copy())
    for i, (e, x) in enumerate(CASES):
        got = results[i]
        assert O.rel_frobenius(got[0], want[i]) <= 1e-12, (e, x)
        for g in got[1:]:
            assert np.array_equal(g.view(np.uint64), got[0].view(np.uint64)), (e, x)
    for p, _ in preps:
        p.close()
