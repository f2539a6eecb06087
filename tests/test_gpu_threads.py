"""Concurrent host threads on one device (SURVEY §8b threading row: the
reference's workers call the backend concurrently, src/executor.cpp:336-364;
the C-ABI keeps per-thread streams and state). Several Python threads (ctypes
drops the GIL inside the calls) run different contractions through
tc::execute and through prepared contractions at the same time; every result
must match the oracle and be bit-identical to the same contraction run alone."""
import threading

import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T

pytestmark = pytest.mark.gpu

CASES = [
    ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=96,j=80,k=16,l=12"),             # L1 (stream-K)
    ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=64,b=48,c=9,k=33"),               # L2
    ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=32,b=16,c=5,d=7,k=3,l=16"),  # L4
    ("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "a=8,b=24,g=6,e=32"),                # L3 (permute)
    ("R[+a] = T[+a,+b,+g] * G[-b,-g]", "a=48,b=40,g=33"),                        # GEMV
    ("K[] = T[+a,+b,+g] * S[-a,-b,-g]", "a=30,b=20,g=9"),                        # DOT
]


def test_concurrent_execute_matches_serial(dev):
    alone = {}
    for e, x in CASES:
        got, _ = T.execute(e, x, seed=1)
        L, R = O.operands(e, x, 1)
        assert O.max_rel_error(got, O.naive(e, x, L, R)) <= 1e-12, (e, x)
        alone[(e, x)] = got
    errors = []

    def worker(tid):
        try:
            for it in range(6):
                e, x = CASES[(tid + it) % len(CASES)]
                got, _ = T.execute(e, x, seed=1)
                if not np.array_equal(got.view(np.uint64), alone[(e, x)].view(np.uint64)):
                    errors.append((tid, it, e, x))
        except Exception as ex:  # surfaced below
            errors.append((tid, repr(ex)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors


def test_concurrent_prepared_pipelines(dev):
    """Each thread owns a prepared contraction and pipelines asynchronous
    streamed calls with its own inputs (its own streams and buffer sets)."""
    e, x = "C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=64,b=48,c=37,k=40"
    errors = []

    def worker(tid):
        try:
            p = T.Prepared(e, x)
            inf = p.info()
            bufs = []
            for s in range(3):
                seed = 100 * tid + 2 * s + 1
                L, R = T.seeded(inf["left"], seed), T.seeded(inf["right"], seed + 1)
                out = np.zeros(inf["output"])
                for a in (L, R, out):
                    T.check(dev.tcb_host_register(a.ctypes.data, a.nbytes))
                bufs.append((L, R, out))
            for L, R, out in bufs:
                p.run_streamed(L, R, out, slabs=5, wait=False)
            p.sync()
            for L, R, out in bufs:
                if O.max_rel_error(out, O.naive(e, x, L, R)) > 1e-12:
                    errors.append(tid)
                for a in (L, R, out):
                    dev.tcb_host_unregister(a.ctypes.data)
            p.close()
        except Exception as ex:
            errors.append((tid, repr(ex)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
