"""Pins the CPU oracle (oracle/tcoracle.c, our C restatement) against the
reference: the committed golden fixtures (generated from the unmodified
reference by tests/golden/make_golden.py) always, and the live compiled
reference (oracle/_ref/libtcref.so) where it is present. CPU only."""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import oracles as O
from specgen import random_spec

GOLD = Path(__file__).resolve().parent / "golden"


def test_seeded_stream_matches_golden():
    # src/tensor.cpp:54-62: mt19937_64 + uniform_real_distribution(-1,1)
    gold = json.loads((GOLD / "seeded.json").read_text())
    for seed, g in gold.items():
        v = O.seeded(4096, int(seed))
        assert v[:16].tolist() == g["first"]
        assert int(np.bitwise_xor.reduce(v.view(np.uint64))) == g["bits_xor"]


def test_seeded_stream_matches_live_reference():
    ref = O.ref()
    if ref is None:
        pytest.skip("compiled reference not present (golden test above pins it)")
    for seed, n in [(1, 10007), (2, 1), (99, 313 * 7)]:
        a = np.empty(n)
        ref.ref_seeded(1, (C.c_int64 * 1)(n), seed, a.ctypes.data)
        assert np.array_equal(a.view(np.uint64), O.seeded(n, seed).view(np.uint64))


def test_naive_known_answers():
    # tests/test_oracle.cpp:20-43 — matmul 2x2 and the all-ones term count
    e = "C[+i,-j] = A[+i,+h] * B[-h,-j]"
    C_ = O.naive(e, "i=2,j=2,h=2", np.array([1., 3, 2, 4]), np.array([5., 7, 6, 8]))
    assert C_.tolist() == [19, 43, 22, 50]
    K = O.naive("K[] = T[+a,+b,+g] * S[-a,-b,-g]", "a=3,b=3,g=3", np.ones(27), np.ones(27))
    assert K.tolist() == [27.0]


def test_naive_zero_linearity_and_cap():
    # tests/test_oracle.cpp:45-86
    e = "R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]"
    x = "a=3,b=4,g=5,e=2"
    A = O.seeded(60, 7)
    B = O.seeded(30, 8)
    R = O.naive(e, x, A, B)
    R4 = O.naive(e, x, 4.0 * A, B)
    assert np.array_equal(R4, 4.0 * R)  # exact for powers of two
    assert not O.naive("R[+a] = T[+a,+b] * x[-b]", "a=4,b=5", O.seeded(20, 3), np.zeros(5)).any()
    with pytest.raises(MemoryError):
        O.naive("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]", "a=20,b=20,g=20,e=20",
                np.zeros(8000), np.zeros(8000), cap=1000)


def test_naive_matches_golden_reference_runs():
    meta = json.loads((GOLD / "small.json").read_text())
    arrs = np.load(GOLD / "small.npz")
    for i, m in enumerate(meta):
        L, R = O.operands(m["expr"], m["extents"], 1)
        mine = O.naive(m["expr"], m["extents"], L, R)
        # same summation order as src/oracle.cpp:44-81 -> bit-identical
        assert np.array_equal(mine, arrs[f"naive_{i}"]), m["expr"]
        assert O.max_rel_error(mine, arrs[f"exec_{i}"]) <= 1e-12


def test_naive_matches_live_reference_bitwise():
    ref = O.ref()
    if ref is None:
        pytest.skip("compiled reference not present")
    rng = np.random.default_rng(11)
    err = C.create_string_buffer(512)
    for _ in range(80):
        e, x = random_spec(rng)
        L, R = O.operands(e, x, 5)
        mine = O.naive(e, x, L, R)
        theirs = np.zeros(max(1, mine.size))
        macs = C.c_int64()
        rc = ref.ref_naive(e.encode(), 0, x.encode(), 5, 10**9, theirs.ctypes.data, theirs.size,
                           C.byref(macs), err, len(err))
        assert rc == 0, err.value
        assert np.array_equal(mine, theirs[:mine.size]), e
        ext = O.ext_map(x)
        assert macs.value == int(np.prod(list(ext.values())))  # test_oracle.cpp:88-97


def test_gemm_check_kernel_agrees_with_reference_gemm():
    # tests/test_kernels.cpp:217-234 tolerance 8e-16 * 2k * 2
    ref = O.ref()
    if ref is None:
        pytest.skip("compiled reference not present")
    rng = np.random.default_rng(77)
    err = C.create_string_buffer(256)
    for _ in range(30):
        m, n, k = (int(v) for v in rng.integers(1, 90, 3))
        ta, tb = int(rng.integers(2)), int(rng.integers(2))
        lda, ldb = (k if ta else m), (n if tb else k)
        a = rng.uniform(-1, 1, lda * (m if ta else k))
        b = rng.uniform(-1, 1, ldb * (k if tb else n))
        c1 = rng.uniform(-1, 1, m * n)
        c2 = c1.copy()
        assert ref.ref_gemm(ta, tb, m, n, k, 2.0, a.ctypes.data, lda, b.ctypes.data, ldb, 0.5,
                            c1.ctypes.data, m, err, len(err)) == 0
        O.tco().tco_gemm_check(ta, tb, m, n, k, 2.0, a.ctypes.data, lda, b.ctypes.data, ldb,
                               0.5, c2.ctypes.data, m)
        assert np.abs(c1 - c2).max() <= 8e-16 * 2 * k * 2


def test_comparators():
    a = np.array([1.0, 2.0, 3.0])
    b = np.array([1.0, 2.0, 3.5])
    assert O.max_rel_error(a, b) == pytest.approx(0.5 / 3.5)
    assert O.rel_frobenius(a, a) == 0.0
    h = O.tco().tco_tensor_hash(3, a.ctypes.data)
    # FNV-1a over bytes (src/executor.cpp:371-383)
    x = 1469598103934665603
    for byte in a.tobytes():
        x = ((x ^ byte) * 1099511628211) % 2**64
    assert h == x
