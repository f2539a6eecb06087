"""Device kernels through the device C-ABI (include/tcb.h) against the
reference backend's known answers (tests/test_kernels.cpp) and the
long-double oracle (oracle/tcoracle.c). Requires a B200."""
import ctypes as C

import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T
from paper_1307_2100_b200 import DeviceBuffer as D

pytestmark = pytest.mark.gpu


def dgemm(dev, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc):
    da, db, dc = D.from_array(a), D.from_array(b), D.from_array(c)
    rc = dev.tcb_dgemm(ta, tb, m, n, k, alpha, da.ptr, lda, db.ptr, ldb, beta, dc.ptr, ldc)
    T.check(rc, "tcb_dgemm")
    return dc.to_array(c.size)


def info(dev):
    i = T.GemmInfo()
    dev.tcb_last_gemm_info(C.byref(i))
    return i


def test_gemm_known_answers(dev):
    # tests/test_kernels.cpp:46-84
    I = np.array([1., 0, 0, 1])
    B = np.array([5., 7, 6, 8])
    assert dgemm(dev, 0, 0, 2, 2, 2, 1.0, I, 2, B, 2, 0.0, np.full(4, -1.0), 2).tolist() == B.tolist()
    A = np.array([1., 3, 2, 4])
    assert dgemm(dev, 0, 0, 2, 2, 2, 1.0, A, 2, B, 2, 0.0, np.zeros(4), 2).tolist() == [19, 43, 22, 50]
    assert dgemm(dev, 0, 0, 2, 2, 2, 1.0, A, 2, B, 2, 1.0, np.ones(4), 2).tolist() == [20, 44, 23, 51]


def op(X, trans, rows, cols, ld):
    """Dense (rows x cols) op(X) of a column-major buffer with leading dim ld."""
    if trans:  # X stored cols x rows: op(X)[i, p] = X[p + i*ld]
        return X.reshape(rows, ld)[:, :cols]
    return X.reshape(cols, ld)[:, :rows].T  # X stored rows x cols: X[i + p*ld]


def colmajor(M):
    return np.ascontiguousarray(M.T).reshape(-1)


def test_transpose_flags_match_explicit_transposition(dev):
    # tests/test_kernels.cpp:86-116 — exhaustive m,n,k <= 4, bitwise equal
    rng = np.random.default_rng(3)
    for m in range(1, 5):
        for n in range(1, 5):
            for k in range(1, 5):
                for ta in (0, 1):
                    for tb in (0, 1):
                        lda, ldb = (k if ta else m), (n if tb else k)
                        A = rng.uniform(-1, 1, lda * (m if ta else k))
                        B = rng.uniform(-1, 1, ldb * (k if tb else n))
                        C1 = dgemm(dev, ta, tb, m, n, k, 1.0, A, lda, B, ldb, 0.0,
                                   np.zeros(m * n), m)
                        Ac = colmajor(op(A, ta, m, k, lda))
                        Bc = colmajor(op(B, tb, k, n, ldb))
                        C2 = dgemm(dev, 0, 0, m, n, k, 1.0, Ac, m, Bc, k, 0.0, np.zeros(m * n), m)
                        assert np.array_equal(C1, C2), (m, n, k, ta, tb)


@pytest.mark.parametrize("seed", range(4))
def test_gemm_vs_long_double_oracle(dev, seed):
    # tests/test_kernels.cpp:217-234, widened to TMA (even ld) and cp.async
    # (odd ld) paths, split-K and multi-tile shapes
    rng = np.random.default_rng(100 + seed)
    paths = set()
    for it in range(25):
        if it % 3 == 0:
            m, n, k = (int(v) for v in rng.integers(100, 700, 3))
            k = int(rng.integers(1, 3000))
        else:
            m, n, k = (int(v) for v in rng.integers(1, 200, 3))
        ta, tb = int(rng.integers(2)), int(rng.integers(2))
        pad = int(rng.integers(0, 3))
        lda, ldb, ldc = (k if ta else m) + pad, (n if tb else k) + pad, m + int(rng.integers(0, 3))
        a = rng.uniform(-1, 1, lda * (m if ta else k))
        b = rng.uniform(-1, 1, ldb * (k if tb else n))
        c = rng.uniform(-1, 1, ldc * n)
        alpha, beta = 2.0, (0.5 if it % 2 else 0.0)
        want = c.copy()
        O.tco().tco_gemm_check(ta, tb, m, n, k, alpha, a.ctypes.data, lda, b.ctypes.data, ldb,
                               beta, want.ctypes.data, ldc)
        got = dgemm(dev, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc)
        paths.add(info(dev).path)
        assert np.abs(got - want).max() <= 8e-16 * 2 * k * 2 + 1e-15, (m, n, k, ta, tb, lda, ldb)
    assert paths & {0, 1}


@pytest.mark.parametrize("seed", range(3))
def test_gemm_accumulate_beta_one_random_shapes(dev, seed):
    # beta == 1 (the reference loop nest's accumulation, src/executor.cpp:162)
    # over even / odd leading dimensions, padded ldc, transposes, one- and
    # multi-wave grids: the TMA reduce-add epilogue, the register epilogue and
    # the cp.async variant, against the long-double oracle; the padding rows of
    # C (ldc > m) must stay untouched
    rng = np.random.default_rng(300 + seed)
    paths = set()
    for it in range(24):
        if it % 4 == 0:
            m, n = (int(v) for v in rng.integers(900, 2600, 2))
            k = int(rng.integers(16, 700))
        elif it % 4 == 1:
            m, n, k = (int(v) for v in rng.integers(100, 700, 3))
        else:
            m, n, k = (int(v) for v in rng.integers(1, 200, 3))
        if it % 2 == 0:  # TMA-legal: even leading dimensions
            m += m % 2
            k += k % 2
            n += n % 2
        ta, tb = int(rng.integers(2)), int(rng.integers(2))
        pad = 2 * int(rng.integers(0, 3))
        lda, ldb, ldc = (k if ta else m) + pad, (n if tb else k) + pad, m + pad
        a = rng.uniform(-1, 1, lda * (m if ta else k))
        b = rng.uniform(-1, 1, ldb * (k if tb else n))
        c = rng.uniform(-1, 1, ldc * n)
        alpha = 1.0 if it % 3 else -0.75
        want = c.copy()
        O.tco().tco_gemm_check(ta, tb, m, n, k, alpha, a.ctypes.data, lda, b.ctypes.data, ldb,
                               1.0, want.ctypes.data, ldc)
        got = dgemm(dev, ta, tb, m, n, k, alpha, a, lda, b, ldb, 1.0, c, ldc)
        paths.add(info(dev).path)
        assert np.abs(got - want).max() <= 8e-16 * 2 * k * 2 + 1e-15, (m, n, k, ta, tb, lda, ldc)
        if ldc > m:
            pad_rows = np.arange(ldc * n).reshape(n, ldc)[:, m:].reshape(-1)
            assert np.array_equal(got[pad_rows], c[pad_rows]), (m, n, k, ldc)
    assert paths & {0, 1}


def test_strided_equals_packed_and_ld_errors(dev):
    # tests/test_kernels.cpp:236-269
    rng = np.random.default_rng(31)
    m, n, k, lda, ldb, ldc = 5, 4, 6, 11, 9, 7
    A = rng.uniform(-1, 1, lda * k)
    B = rng.uniform(-1, 1, ldb * n)
    C1 = dgemm(dev, 0, 0, m, n, k, 1.0, A, lda, B, ldb, 0.0, np.zeros(ldc * n), ldc)
    Ap = A.reshape(k, lda)[:, :m].reshape(-1)
    Bp = B.reshape(n, ldb)[:, :k].reshape(-1)
    C2 = dgemm(dev, 0, 0, m, n, k, 1.0, Ap, m, Bp, k, 0.0, np.zeros(m * n), m)
    assert np.allclose(C1.reshape(n, ldc)[:, :m].reshape(-1), C2, rtol=1e-14, atol=0)
    buf = D(64)
    assert dev.tcb_dgemm(0, 0, 2, 2, 2, 1.0, buf.ptr, 1, buf.ptr, 2, 0.0, buf.ptr, 2) == 1
    assert dev.tcb_last_error() == b"gemm: lda below row count"
    assert dev.tcb_dgemm(0, 0, 2, 2, 2, 1.0, buf.ptr, 2, buf.ptr, 2, 0.0, buf.ptr, 1) == 1
    assert dev.tcb_last_error() == b"gemm: ldc below row count"


def test_gemv_ger_dot_known_answers(dev):
    # tests/test_kernels.cpp:118-165
    I3 = D.from_array(np.eye(3).reshape(-1))
    x = D.from_array(np.array([1., 2, 3]))
    y = D.from_array(np.zeros(3))
    T.check(dev.tcb_dgemv(0, 3, 3, 1.0, I3.ptr, 3, x.ptr, 1, 0.0, y.ptr, 1))
    assert y.to_array(3).tolist() == [1, 2, 3]
    A = D.from_array(np.array([1., 3, 2, 4]))
    x2 = D.from_array(np.array([1., 1]))
    y2 = D.from_array(np.zeros(2))
    T.check(dev.tcb_dgemv(0, 2, 2, 1.0, A.ptr, 2, x2.ptr, 1, 0.0, y2.ptr, 1))
    assert y2.to_array(2).tolist() == [3, 7]
    y3 = D.from_array(np.array([1., 1]))
    T.check(dev.tcb_dgemv(0, 2, 2, 1.0, A.ptr, 2, x2.ptr, 1, 2.0, y3.ptr, 1))
    assert y3.to_array(2).tolist() == [5, 9]
    G = D.from_array(np.zeros(4))
    e1, e2 = D.from_array(np.array([1., 0])), D.from_array(np.array([0., 1]))
    T.check(dev.tcb_dger(2, 2, 1.0, e1.ptr, 1, e2.ptr, 1, G.ptr, 2))
    assert G.to_array(4).tolist() == [0, 0, 1, 0]
    G2 = D.from_array(np.zeros(4))
    gx, gy = D.from_array(np.array([1., 2])), D.from_array(np.array([3., 4]))
    T.check(dev.tcb_dger(2, 2, 1.0, gx.ptr, 1, gy.ptr, 1, G2.ptr, 2))
    assert G2.to_array(4).tolist() == [3, 6, 4, 8]
    r = C.c_double()
    dx, dy = D.from_array(np.array([1., 2, 3])), D.from_array(np.array([4., 5, 6]))
    T.check(dev.tcb_ddot(3, dx.ptr, 1, dy.ptr, 1, C.byref(r)))
    assert r.value == 32.0
    T.check(dev.tcb_ddot(0, x.ptr, 1, x.ptr, 1, C.byref(r)))
    assert r.value == 0.0


def test_gemv_and_dot_large_vs_numpy(dev):
    rng = np.random.default_rng(8)
    for trans in (0, 1):
        for (m, n) in [(3000, 257), (17, 100000), (100000, 3)]:
            A = rng.uniform(-1, 1, m * n)
            xl, yl = (m, n) if trans else (n, m)
            x = rng.uniform(-1, 1, xl)
            y = D.from_array(np.zeros(yl))
            dA, dx = D.from_array(A), D.from_array(x)  # keep alive: kernels run async
            T.check(dev.tcb_dgemv(trans, m, n, 1.0, dA.ptr, m, dx.ptr, 1, 0.0, y.ptr, 1))
            M = A.reshape(n, m).T
            want = (M.T @ x) if trans else (M @ x)
            assert np.allclose(y.to_array(yl), want, rtol=1e-12, atol=1e-12)
    v = rng.uniform(-1, 1, 3_000_000)
    r = C.c_double()
    dv = D.from_array(v)
    T.check(dev.tcb_ddot(v.size, dv.ptr, 1, dv.ptr, 1, C.byref(r)))
    assert r.value == pytest.approx(float(v @ v), rel=1e-13)


def test_strided_batched_equals_loop(dev):
    rng = np.random.default_rng(9)
    m, n, k, batch = 130, 70, 90, 7
    A = rng.uniform(-1, 1, m * k * batch)
    B = rng.uniform(-1, 1, k * n * batch)
    dA, dB, dC = D.from_array(A), D.from_array(B), D(m * n * batch * 8)
    T.check(dev.tcb_dgemm_strided_batched(0, 0, m, n, k, 1.0, dA.ptr, m, m * k, dB.ptr, k, k * n,
                                          0.0, dC.ptr, m, m * n, batch))
    got = dC.to_array(m * n * batch)
    for b in range(batch):
        Ab = A[b * m * k:(b + 1) * m * k].reshape(k, m).T
        Bb = B[b * k * n:(b + 1) * k * n].reshape(n, k).T
        want = (Ab @ Bb).T.reshape(-1)
        assert np.allclose(got[b * m * n:(b + 1) * m * n], want, rtol=1e-13, atol=1e-13)


def test_permute_is_an_exact_copy(dev):
    rng = np.random.default_rng(10)
    for _ in range(20):
        r = int(rng.integers(1, 6))
        ext = [int(v) for v in rng.integers(1, 12, r)]
        perm = list(rng.permutation(r))
        n = int(np.prod(ext))
        src = rng.uniform(-1, 1, n)
        sstr_nat, run = [], 1
        for e in ext:
            sstr_nat.append(run)
            run *= e
        dext = [ext[p] for p in perm]
        dstr = [sstr_nat[p] for p in perm]
        d_src, d_dst = D.from_array(src), D(n * 8)
        T.check(dev.tcb_permute(r, (C.c_int64 * r)(*dext), (C.c_int64 * r)(*dstr), d_src.ptr,
                                d_dst.ptr))
        got = d_dst.to_array(n)
        want = src.reshape(list(reversed(ext))).transpose(
            [r - 1 - p for p in reversed(perm)]).reshape(-1)
        assert np.array_equal(got, want), (ext, perm)


@pytest.mark.parametrize("e_a,e_t,e_r", [(70, 1000, 300), (64, 4096, 80), (33, 97, 4)])
def test_large_ragged_transpose_is_an_exact_copy(dev, e_a, e_t, e_r):
    """Unit-stride dims differ (tiled transpose); the first two shapes are
    large enough for the 64x64 tiles, with ragged edges in both tile dims."""
    n = e_a * e_t * e_r
    src = np.arange(n, dtype=np.float64) * 0.5 - 7.0  # source [t, a, r], t fastest
    d_src, d_dst = D.from_array(src), D(n * 8)
    ext = (C.c_int64 * 3)(e_a, e_t, e_r)
    sstr = (C.c_int64 * 3)(e_t, 1, e_t * e_a)
    T.check(dev.tcb_permute(3, ext, sstr, d_src.ptr, d_dst.ptr))
    got = d_dst.to_array(n)
    want = src.reshape(e_r, e_a, e_t).transpose(0, 2, 1).reshape(-1)  # dst [a, t, r]
    assert np.array_equal(got, want)


def test_split_k_is_deterministic(dev):
    # cfg1-shaped GEMM: few tiles -> split-K with last-CTA ordered reduction
    rng = np.random.default_rng(12)
    m = n = 512
    k = 4096
    A, B = rng.uniform(-1, 1, m * k), rng.uniform(-1, 1, k * n)
    r1 = dgemm(dev, 0, 0, m, n, k, 1.0, A, m, B, k, 0.0, np.zeros(m * n), m)
    assert info(dev).splits > 1
    r2 = dgemm(dev, 0, 0, m, n, k, 1.0, A, m, B, k, 0.0, np.zeros(m * n), m)
    assert np.array_equal(r1.view(np.uint64), r2.view(np.uint64))


def test_fp64_peak_microbenchmark(dev):
    p = C.c_double()
    T.check(dev.tcb_fp64_peak(C.byref(p)))
    assert 20.0 < p.value < 60.0  # B200: ~37 TFLOP/s measured


def test_copy2d_and_event_elapsed(dev):
    """tcb_h2d_2d / tcb_d2h_2d move a slab of a middle mode (rows of `width`
    bytes at pitched offsets); tcb_event_elapsed times between two events."""
    import ctypes as C
    x = np.arange(64 * 10, dtype=np.float64)  # 64 x 10 column-major
    d = T.DeviceBuffer(64 * 4 * 8)
    # rows 8..15 of columns 0..3: 4 copy rows of 8 doubles, source pitch one
    # column (512 B), device pitch 256 B
    T.check(dev.tcb_h2d_2d(d.ptr, 256, x.ctypes.data + 8 * 8, 64 * 8, 8 * 8, 4))
    back = np.zeros(64 * 10)
    T.check(dev.tcb_d2h_2d(back.ctypes.data + 8 * 8, 64 * 8, d.ptr, 256, 8 * 8, 4))
    want = np.zeros(64 * 10)
    for c in range(4):
        want[c * 64 + 8:c * 64 + 16] = x[c * 64 + 8:c * 64 + 16]
    assert np.array_equal(back, want)
    e0, e1 = C.c_void_p(), C.c_void_p()
    T.check(dev.tcb_event_create_timed(C.byref(e0)))
    T.check(dev.tcb_event_create_timed(C.byref(e1)))
    s = dev.tcb_current_stream()
    T.check(dev.tcb_event_record(e0, s))
    T.check(dev.tcb_memset0(d.ptr, 64 * 4 * 8))
    T.check(dev.tcb_event_record(e1, s))
    ms = C.c_float(-1.0)
    T.check(dev.tcb_event_elapsed(e0, e1, C.byref(ms)))
    assert ms.value >= 0.0
    T.check(dev.tcb_event_destroy(e0))
    T.check(dev.tcb_event_destroy(e1))
