"""tc/oracle.hpp on the device: tc::contract_naive (tcb_contract_naive) is
bit-identical to the reference's own contract_naive (src/oracle.cpp:32-94;
tests/test_oracle.cpp:20-43, :88-97) — against the committed golden arrays and
the live compiled reference. Requires a B200."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T
from specgen import random_spec

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def test_golden_naive_bit_identical(dev):
    meta = json.loads((GOLD / "small.json").read_text())
    arrs = np.load(GOLD / "small.npz")
    for i, m in enumerate(meta):
        got, macs = T.contract_naive(m["expr"], m["extents"], seed=1)
        assert np.array_equal(bits(got), bits(arrs[f"naive_{i}"])), m["expr"]
        ext = O.ext_map(m["extents"])
        labels = set(O.parse(m["expr"])[1]) | set(O.parse(m["expr"])[2])
        assert macs == int(np.prod([ext[x] for x in labels]))


def test_live_reference_naive_bit_identical(dev):
    if O.ref() is None:
        pytest.skip("oracle/_ref missing")
    import ctypes as C
    rng = np.random.default_rng(99)
    for _ in range(80):
        e, x = random_spec(rng)
        got, macs = T.contract_naive(e, x, seed=3)
        out = np.zeros(got.size)
        m = C.c_int64()
        err = C.create_string_buffer(1024)
        rc = O.ref().ref_naive(e.encode(), 0, x.encode(), 3, 10**9, out.ctypes.data, out.size,
                               C.byref(m), err, len(err))
        assert rc == 0, err.value
        assert np.array_equal(bits(got), bits(out)), (e, x)
        assert macs == m.value


def test_work_cap_and_matmul(dev):
    # tests/test_oracle.cpp:20-43: a matrix product; the cap refuses big jobs
    got, macs = T.contract_naive("C[+i,-j] = A[+i,+h] * B[-h,-j]", "i=3,j=4,h=5")
    L, R = O.operands("C[+i,-j] = A[+i,+h] * B[-h,-j]", "i=3,j=4,h=5", 1)
    want = (L.reshape(5, 3).T @ R.reshape(4, 5).T).T.reshape(-1)
    assert np.abs(got - want).max() <= 1e-15 and macs == 60
    with pytest.raises(MemoryError, match="oracle work exceeds cap: 60 multiply-adds"):
        T.contract_naive("C[+i,-j] = A[+i,+h] * B[-h,-j]", "i=3,j=4,h=5", work_cap=59)
