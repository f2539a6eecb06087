"""Ordering and state safety of the device runtime (libtcb200.so):

  * programmatic dependent launch over a chain of GEMMs: a GEMM whose operand
    is the output of ANY earlier GEMM of the chain is serialized (not only of
    the previous one) — C1 = A B; C2 = D E; C3 = C1 F with small-k grids that
    leave SMs free, repeated;
  * tcb_set_stream hands over in stream order: stream-K GEMMs of one thread on
    two streams share the thread's workspace and tile counters without
    overlapping;
  * tc::execute on page-locked (streamed slabs) and pageable (one launch)
    storage agree within the parity tolerance.
Requires a B200."""
import ctypes as C

import numpy as np
import pytest

import paper_1307_2100_b200 as T
from paper_1307_2100_b200 import DeviceBuffer as D

pytestmark = pytest.mark.gpu


def colmajor(M):
    return np.ascontiguousarray(M.T).reshape(-1)


def dense(flat, rows, cols):
    return flat.reshape(cols, rows).T


def test_pdl_chain_guards_every_earlier_output(dev):
    rng = np.random.default_rng(11)
    # GEMM1: 1536 x 1536 (144 tiles, k = 96 < 128 so no stream-K) keeps 144
    # SMs busy; GEMM2 is a 2-tile GEMM that fits on the remaining SMs, so its
    # CTAs become resident (and let GEMM3 launch) while GEMM1 still runs;
    # GEMM3 reads GEMM1's output.
    m1, k1 = 1536, 96
    A = rng.uniform(-1, 1, (m1, k1))
    B = rng.uniform(-1, 1, (k1, m1))
    Dm = rng.uniform(-1, 1, (128, 64))
    E = rng.uniform(-1, 1, (64, 256))
    F = rng.uniform(-1, 1, (m1, 64))
    dA, dB = D.from_array(colmajor(A)), D.from_array(colmajor(B))
    dD, dE, dF = D.from_array(colmajor(Dm)), D.from_array(colmajor(E)), D.from_array(colmajor(F))
    dC1, dC2, dC3 = D(m1 * m1 * 8), D(128 * 256 * 8), D(m1 * 64 * 8)
    want1 = A @ B
    want3 = want1 @ F
    for it in range(40):
        T.check(dev.tcb_memset0(dC1.ptr, m1 * m1 * 8))  # breaks the chain: next launch serialized
        T.check(dev.tcb_dgemm(0, 0, m1, m1, k1, 1.0, dA.ptr, m1, dB.ptr, k1, 0.0, dC1.ptr, m1))
        T.check(dev.tcb_dgemm(0, 0, 128, 256, 64, 1.0, dD.ptr, 128, dE.ptr, 64, 0.0, dC2.ptr,
                              128))
        T.check(dev.tcb_dgemm(0, 0, m1, 64, m1, 1.0, dC1.ptr, m1, dF.ptr, m1, 0.0, dC3.ptr, m1))
        got = dense(dC3.to_array(), m1, 64)
        err = np.abs(got - want3).max() / np.abs(want3).max()
        assert err <= 1e-12, (it, err)


def test_set_stream_orders_stream_k_workspace(dev):
    rng = np.random.default_rng(12)
    # 512 x 512 x 65536: 16 tiles on 148 SMs -> stream-K through the thread's
    # workspace; the same shape again on a second stream right after
    m, k = 512, 65536
    A = rng.uniform(-1, 1, (m, k))
    B = rng.uniform(-1, 1, (k, m))
    A2 = rng.uniform(-1, 1, (m, k))
    dA, dB, dA2 = D.from_array(colmajor(A)), D.from_array(colmajor(B)), D.from_array(colmajor(A2))
    dC, dC2 = D(m * m * 8), D(m * m * 8)
    s2 = C.c_void_p()
    T.check(dev.tcb_stream_create(C.byref(s2)))
    try:
        for _ in range(5):
            T.check(dev.tcb_set_stream(None))
            T.check(dev.tcb_dgemm(0, 0, m, m, k, 1.0, dA.ptr, m, dB.ptr, k, 0.0, dC.ptr, m))
            i = T.GemmInfo()
            dev.tcb_last_gemm_info(C.byref(i))
            assert i.splits > 1  # the stream-K variant really ran
            T.check(dev.tcb_set_stream(s2))
            T.check(dev.tcb_dgemm(0, 0, m, m, k, 1.0, dA2.ptr, m, dB.ptr, k, 0.0, dC2.ptr, m))
            T.check(dev.tcb_sync())
            T.check(dev.tcb_set_stream(None))
            T.check(dev.tcb_sync())
            w1, w2 = A @ B, A2 @ B
            g1, g2 = dense(dC.to_array(), m, m), dense(dC2.to_array(), m, m)
            assert np.abs(g1 - w1).max() / np.abs(w1).max() <= 1e-12
            assert np.abs(g2 - w2).max() / np.abs(w2).max() <= 1e-12
    finally:
        T.check(dev.tcb_set_stream(None))
        dev.tcb_stream_destroy(s2)


def test_current_device(dev):
    d = C.c_int(-5)
    T.check(dev.tcb_current_device(C.byref(d)))
    assert d.value == 0


@pytest.mark.parametrize("expr,ext", [
    # contracted-label slabs when pinned (C accumulated over l slabs)
    ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=256,j=192,k=512,l=64"),
    # output-label slabs when pinned
    ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=256,b=256,c=96,k=256"),
])
def test_execute_pinned_and_pageable_agree(dev, expr, ext):
    out, left, right = T.parse_expr(expr)
    em = {k: int(v) for k, v in (kv.split("=") for kv in ext.split(","))}
    nl = int(np.prod([em[x] for x in left]))
    nr = int(np.prod([em[x] for x in right]))
    no = int(np.prod([em[x] for x in out]))
    L, R = T.seeded(nl, 1), T.seeded(nr, 2)
    page = np.empty(no)
    T.execute_host(expr, ext, L, R, page)  # pageable: upload, one launch, download
    pin = []
    for a in (L, R):
        p = np.empty(a.size)
        T.check(dev.tcb_host_register(p.ctypes.data, p.nbytes))
        p[:] = a
        pin.append(p)
    po = np.empty(no)
    T.check(dev.tcb_host_register(po.ctypes.data, po.nbytes))
    try:
        T.execute_host(expr, ext, pin[0], pin[1], po)  # pinned: streamed slabs
        scale = max(1.0, np.abs(page).max())
        assert np.abs(po - page).max() / scale <= 1e-12
        assert np.linalg.norm(po - page) / np.linalg.norm(page) <= 1e-12
        # and the Tensor-level call (seeded operands) gives the pinned bits again
        again, _ = T.execute(expr, ext, seed=1)
        assert np.abs(again - page).max() / scale <= 1e-12
    finally:
        for a in (*pin, po):
            dev.tcb_host_unregister(a.ctypes.data)
