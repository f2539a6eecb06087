"""Random contractions whose extents are multiples of 16 mixed with small odd
ones, so the DMMA kernel's whole-stage TMA boxes, composite operand groups (L4)
and the TMA-store epilogue (output rows in runs of 16) are all exercised, with
ragged tiles at the edges. Parity against the naive oracle (src/oracle.cpp:
32-94 restated in oracle/tcoracle.c) at relative Frobenius and max relative
error <= 1e-12. Requires a B200."""
import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T
from specgen import random_spec

pytestmark = pytest.mark.gpu
TOL = 1e-12


def close(got, want):
    return O.max_rel_error(got, want) <= TOL and O.rel_frobenius(got, want) <= TOL


def macs(x):
    return int(np.prod([int(kv.split("=")[1]) for kv in x.split(",")]))


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_tile_shaped_contractions(dev, seed):
    rng = np.random.default_rng(1000 + seed)
    seen = {}
    n = 0
    for _ in range(2000):
        e, x = random_spec(rng, extents=(16, 32, 48, 64, 2, 3, 7))
        if macs(x) > 2 * 10**7:
            continue
        lay = T.lower(e, x).split()[0]
        L, R = O.operands(e, x, seed)
        got, st = T.execute(e, x, seed=seed)
        assert close(got, O.naive(e, x, L, R)), (e, x, T.lower(e, x))
        seen[lay] = seen.get(lay, 0) + 1
        n += 1
        if n == 40:
            break
    assert n == 40 and len(seen) >= 2, seen


def test_beta_accumulate_through_tma_store_shapes(dev):
    """tcb_dgemm with beta != 0 on shapes that would take the TMA store: the
    storer-warp fallback must read C (BLAS contract, test_kernels.cpp:72-84)."""
    import ctypes as C
    from paper_1307_2100_b200 import DeviceBuffer as D
    rng = np.random.default_rng(5)
    for m, n, k, beta in ((256, 384, 96, 1.0), (512, 128, 2048, -0.5), (160, 144, 64, 2.0)):
        A = rng.uniform(-1, 1, m * k)
        B = rng.uniform(-1, 1, k * n)
        C0 = rng.uniform(-1, 1, m * n)
        dA, dB, dC = D.from_array(A), D.from_array(B), D.from_array(C0)
        T.check(dev.tcb_dgemm(0, 0, m, n, k, 1.5, dA.ptr, m, dB.ptr, k, beta, dC.ptr, m))
        got = dC.to_array(m * n)
        ref = 1.5 * (A.reshape(k, m).T @ B.reshape(n, k).T) + beta * C0.reshape(n, m).T
        ref = ref.T.reshape(-1)
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)), (m, n, k, beta)


@pytest.mark.parametrize("m,n,k,alpha", [(2048, 2048, 256, 1.0), (4096, 4096, 512, 0.75),
                                         (1000, 1234, 96, 1.0), (4096, 4096, 2048, 1.0),
                                         (8192, 4096, 16384, 1.0)])
def test_beta_one_is_one_exact_addition(dev, m, n, k, alpha):
    """beta == 1: the staged tile is added to C by a TMA reduce-add (one f64
    add per element in L2), the long-k hybrid's consumers add the old values
    they loaded in batches: either way C_new == C_old + (alpha A B) bit for
    bit, where alpha A B is the same launch with beta == 0 (shapes whose
    beta == 0 and beta == 1 launches take the same tile schedule: below 256
    or from 768 k-blocks per tile). Ragged edges (1000 x 1234) are clipped by
    the tensor map."""
    import ctypes as C
    from paper_1307_2100_b200 import DeviceBuffer as D
    dA, dB = D(m * k * 8), D(k * n * 8)
    rng = np.random.default_rng(m + k)
    blk = rng.uniform(-1, 1, 1 << 22)
    for buf, cnt in ((dA, m * k), (dB, k * n)):
        for off in range(0, cnt, blk.size):
            c = min(blk.size, cnt - off)
            T.check(dev.tcb_h2d(buf.ptr + off * 8, blk.ctypes.data, c * 8))
    C0 = rng.uniform(-1, 1, m * n)
    dC = D.from_array(np.zeros(m * n))
    T.check(dev.tcb_dgemm(0, 0, m, n, k, alpha, dA.ptr, m, dB.ptr, k, 0.0, dC.ptr, m))
    prod = dC.to_array(m * n)
    dC2 = D.from_array(C0)
    T.check(dev.tcb_dgemm(0, 0, m, n, k, alpha, dA.ptr, m, dB.ptr, k, 1.0, dC2.ptr, m))
    got = dC2.to_array(m * n)
    assert np.array_equal(got, C0 + prod), (m, n, k, alpha)
    assert np.abs(prod).max() > 0


@pytest.mark.parametrize("m,n,k,beta", [(2048, 2048, 128, 0.0), (2048, 2048, 128, -1.5),
                                        (1536, 2560, 256, 0.5), (300, 200, 4096, 2.0)])
def test_stream_k_hybrid_and_pure_shapes_with_beta(dev, m, n, k, beta):
    """Grids whose last data-parallel wave is mostly empty (256 tiles on 148
    SMs) take the data-parallel + stream-K hybrid; small grids pure stream-K;
    alpha / beta as the BLAS contract (tests/test_kernels.cpp:72-84)."""
    import ctypes as C
    from paper_1307_2100_b200 import DeviceBuffer as D
    rng = np.random.default_rng(m + n + k)
    A = rng.uniform(-1, 1, m * k)
    B = rng.uniform(-1, 1, k * n)
    C0 = rng.uniform(-1, 1, m * n)
    dA, dB, dC = D.from_array(A), D.from_array(B), D.from_array(C0)
    T.check(dev.tcb_dgemm(0, 0, m, n, k, 0.75, dA.ptr, m, dB.ptr, k, beta, dC.ptr, m))
    info = T.GemmInfo()
    dev.tcb_last_gemm_info(C.byref(info))
    got = dC.to_array(m * n).reshape(n, m).T
    ref = 0.75 * (A.reshape(k, m).T @ B.reshape(n, k).T) + beta * C0.reshape(n, m).T
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max(), (m, n, k, beta)
    assert info.grid == 148 and info.splits >= 2, (info.grid, info.splits)


@pytest.mark.parametrize("x", ["b=64,f=4096,g=48,e=64", "b=32,f=4096,g=48,e=64"])
def test_short_k_with_scattered_output_is_race_free(dev, x):
    """Regression: many short tiles (2-4 k-blocks) whose output rows are
    scattered (no TMA store; the plain-store epilogue is slower than the main
    loop), so the producer refills ring stages as soon as the consumers
    release them. The release must wait for the consumers' fragment loads
    (gemm_dmma.cu: fence before the empty-barrier arrive); without it a warp
    tile was occasionally computed from a half-overwritten stage. Five runs
    must agree bit for bit and match numpy (BLAS fp64) within 1e-12."""
    e = "R[-g,+f,-e] = A[-b,+f,-g] * B[+b,-e]"
    ext = dict((k, int(v)) for k, v in (kv.split("=") for kv in x.split(",")))
    p = T.Prepared(e, x)
    inf = p.info()
    L, R = T.seeded(inf["left"], 1), T.seeded(inf["right"], 2)
    want = np.einsum("gfb,eb->efg", L.reshape(ext["g"], ext["f"], ext["b"]),
                     R.reshape(ext["e"], ext["b"])).reshape(-1)
    first = None
    for _ in range(5):
        p.upload(L, R)
        p.run()
        out = np.empty(want.size)
        p.download(out)
        if first is None:
            first = out
            assert O.rel_frobenius(out, want) <= 1e-12
            assert O.max_rel_error(out, want) <= 1e-12
        else:
            assert np.array_equal(out.view(np.uint64), first.view(np.uint64))
    p.close()


@pytest.mark.parametrize("e,x", [
    # batched stream-K with tiny tiles: 128 one-tile batches of 9 k-blocks on
    # 148 CTAs (every tile shared by two CTAs; found by tools/stress.py seed 11)
    ("R[+b,-a,+c,+g] = A[+e,-a] * B[+g,+c,-e,+b]", "e=130,a=7,g=2,c=3,b=128"),
    # shares that cross tile boundaries with either neighbour preferred
    ("C[+i,+j] = A[+i,+k] * B[-k,+j]", "i=300,j=260,k=1000"),
    ("C[+i,+j,+c] = A[+i,+k,+c] * B[-k,+j]", "i=100,j=60,k=700,c=40"),
    # shares aligned to half tiles: two non-crossing contributors per tile
    ("C[+i,+j,+c] = A[+i,+k,+c] * B[-k,+j]", "i=128,j=128,k=128,c=37"),
])
def test_stream_k_reduction_assignment(dev, e, x):
    L, R = O.operands(e, x, 3)
    got, _ = T.execute(e, x, seed=3)
    assert close(got, O.naive(e, x, L, R)), (e, x, T.lower(e, x))
