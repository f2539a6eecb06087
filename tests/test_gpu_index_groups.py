"""In-place index groups (recipe L4): class-3 contractions
whose operands the DMMA kernel's tensor maps can read directly, with no
permutation pass. Parity against the naive oracle (src/oracle.cpp:32-94
restated in oracle/tcoracle.c), against the permuting L3 recipe of the same
contraction, and the C-ABI descriptor rules (tcb_gemm_check). Tolerance:
relative Frobenius and max relative error <= 1e-12. Requires a B200."""
import ctypes as C
import os

import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T
from paper_1307_2100_b200 import DeviceBuffer as D
from specgen import random_spec

pytestmark = pytest.mark.gpu
TOL = 1e-12


def close(got, want):
    return O.max_rel_error(got, want) <= TOL and O.rel_frobenius(got, want) <= TOL


def macs(x):
    return int(np.prod([int(kv.split("=")[1]) for kv in x.split(",")]))


CASES = [
    # cfg3 shape family: A MN-major (a inner), B K-major (l inner), N = (b, d) with b < 128
    ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=32,b=16,c=5,d=7,k=3,l=16"),
    ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=16,b=64,c=3,d=3,k=2,l=32"),
    # K-major outer box spilling into the next sub-index (32 x 4 = 128), ragged d
    ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=16,b=32,c=3,d=5,k=2,l=16"),
    # both operands MN-major, K composite with a strided inner sub-index
    ("C[+a,+b,+c] = A[+a,+k,+c,+l] * B[+b,-l,-k]", "a=32,b=48,c=5,k=3,l=16"),
    # both K-major on the same label, M and N composite (class 3.2)
    ("C[+a,+b,+c,+d] = A[+k,+a,+l,+c] * B[-k,+b,-l,+d]", "a=32,b=64,c=3,d=2,k=16,l=3"),
    # tails: outer groups not a multiple of the 128 tile, K not a multiple of 16 outside the inner
    ("C[+a,+c,+b] = A[+a,+k,+c,+l] * B[-l,+b,-k]", "a=32,b=40,c=5,k=5,l=16"),
]


@pytest.mark.parametrize("e,x", CASES)
def test_l4_cases_match_oracle_and_l3(dev, e, x, monkeypatch):
    assert T.lower(e, x).startswith("L4"), T.lower(e, x)
    L, R = O.operands(e, x, 1)
    want = O.naive(e, x, L, R)
    got, st = T.execute(e, x, seed=1)
    assert close(got, want), (e, x)
    assert st["kernel_calls"] == 1  # no permutation launch
    monkeypatch.setenv("TC_INDEX_GROUPS", "0")
    assert T.lower(e, x).startswith("L3")
    got3, _ = T.execute(e, x, seed=1)
    assert close(got3, want)


def test_random_l4_family(dev):
    rng = np.random.default_rng(4242)
    hit = 0
    for _ in range(4000):
        e, x = random_spec(rng, extents=(16, 32, 2, 3, 48, 5))
        if macs(x) > 3 * 10**7 or not T.lower(e, x).startswith("L4"):
            continue
        hit += 1
        L, R = O.operands(e, x, 1)
        got, _ = T.execute(e, x, seed=1)
        assert close(got, O.naive(e, x, L, R)), (e, x, T.lower(e, x))
        if hit == 60:
            break
    assert hit >= 30


def test_l4_prepared_and_streamed_paths(dev):
    e, x = "C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=64,b=64,c=12,d=20,k=4,l=32"
    L, R = O.operands(e, x, 1)
    want = O.naive(e, x, L, R)
    p = T.Prepared(e, x)
    assert p.info()["permuted_bytes"] == 0
    out = np.empty(want.size)
    p.upload(L, R)
    p.run()
    p.download(out)
    assert close(out, want)
    # streamed over the output's outermost label (d: outermost in B)
    outs = np.zeros(want.size)
    for arr in (L, R, outs):
        T.check(dev.tcb_host_register(arr.ctypes.data, arr.nbytes))
    try:
        used = p.run_streamed(L, R, outs, slabs=5)
    finally:
        for arr in (L, R, outs):  # never leave freed memory registered
            dev.tcb_host_unregister(arr.ctypes.data)
    assert used == 5
    assert close(outs, want)


def _desc(m_ext, a_m, n_ext, b_n, k_ext, a_k, b_k, row, col):
    d = T.GemmDesc()
    d.m, d.n, d.k = int(np.prod(m_ext)), int(np.prod(n_ext)), int(np.prod(k_ext))
    d.g_m, d.g_n, d.g_k = len(m_ext), len(n_ext), len(k_ext)
    for i, (e, s) in enumerate(zip(m_ext, a_m)):
        d.m_ext[i], d.a_m_str[i] = e, s
    for i, (e, s) in enumerate(zip(n_ext, b_n)):
        d.n_ext[i], d.b_n_str[i] = e, s
    for i, (e, sa, sb) in enumerate(zip(k_ext, a_k, b_k)):
        d.k_ext[i], d.a_k_str[i], d.b_k_str[i] = e, sa, sb
    d.a_sm, d.a_sk, d.b_sk, d.b_sn = a_m[0], a_k[0], b_k[0], b_n[0]
    d.c_nrow, d.c_ncol = 1, 1
    d.c_row_ext[0], d.c_row_str[0] = d.m, 1
    d.c_col_ext[0], d.c_col_str[0] = d.n, d.m
    d.alpha, d.beta = 1.0, 0.0
    return d


def test_gemm_desc_groups_direct(dev):
    """tcb_gemm with index groups on raw device buffers vs numpy: A[a,k,c,l]
    read as M=(a,c), K=(l,k); B[l,b,k,d] as N=(b,d), K=(l,k); C column-major
    (m, n). Also alpha/beta and the descriptor checks."""
    a, k, c, l, b, dd = 32, 3, 5, 16, 64, 3
    rng = np.random.default_rng(9)
    A = rng.uniform(-1, 1, (a, k, c, l))  # index order = column-major modes
    B = rng.uniform(-1, 1, (l, b, k, dd))
    Af = np.asfortranarray(A).ravel(order="F")
    Bf = np.asfortranarray(B).ravel(order="F")
    # column-major strides
    sA = [1, a, a * k, a * k * c]          # a, k, c, l
    sB = [1, l, l * b, l * b * k]          # l, b, k, d
    d = _desc([a, c], [sA[0], sA[2]], [b, dd], [sB[1], sB[3]], [l, k], [sA[3], sA[1]],
              [sB[0], sB[2]], None, None)
    want = np.einsum("akcl,lbkd->acbd", A, B).reshape(a * c, b * dd, order="F")
    C0 = rng.uniform(-1, 1, want.shape)
    dA, dB = D.from_array(Af), D.from_array(Bf)
    dC = D.from_array(C0.ravel(order="F"))
    assert dev.tcb_gemm_check(C.byref(d)) == 0
    d.alpha, d.beta = 0.5, -2.0
    T.check(dev.tcb_gemm(C.byref(d), dA.ptr, dB.ptr, dC.ptr), "tcb_gemm")
    got = dC.to_array(want.size).reshape(want.shape, order="F")
    ref = 0.5 * want - 2.0 * C0
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    i = T.GemmInfo()
    dev.tcb_last_gemm_info(C.byref(i))
    assert i.path == 0 and i.launches == 1
    # refusals: inner extent of the unit-stride group not a multiple of 16
    bad = _desc([24, c], [1, 24 * k], [b, dd], [sB[1], sB[3]], [l, k], [24 * k * c, 24],
                [sB[0], sB[2]], None, None)
    assert dev.tcb_gemm_check(C.byref(bad)) == 5  # TCB_EUNSUPPORTED
    assert dev.tcb_gemm(C.byref(bad), dA.ptr, dB.ptr, dC.ptr) == 5
    # groups not covering m
    bad2 = _desc([a, c], [sA[0], sA[2]], [b, dd], [sB[1], sB[3]], [l, k], [sA[3], sA[1]],
                 [sB[0], sB[2]], None, None)
    bad2.m += 1
    assert dev.tcb_gemm_check(C.byref(bad2)) == 1  # TCB_EINVAL


def test_env_switch_is_read_per_call(dev, monkeypatch):
    e, x = CASES[0]
    monkeypatch.setenv("TC_INDEX_GROUPS", "0")
    assert T.lower(e, x).startswith("L3")
    monkeypatch.delenv("TC_INDEX_GROUPS")
    assert os.environ.get("TC_INDEX_GROUPS") is None
    assert T.lower(e, x).startswith("L4")
