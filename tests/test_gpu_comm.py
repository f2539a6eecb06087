"""The engine's multi-GPU exchange (include/tcb.h tcb_comm_* / tcb_reduce_scatter /
tcb_allreduce, NCCL loaded at run time) at world size 1 on one B200: the
K-split partition's reduce-scatter of partial C and the all-reduce
are exact copies; a K-split of a contraction into two slabs summed by an
all-reduce-style accumulation matches the oracle. Multi-rank runs need more
GPUs than this pool gives one process; the host plumbing of the partition is
covered by tests/test_partition_gloo.py."""
import ctypes as C

import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T
from paper_1307_2100_b200 import DeviceBuffer as D

pytestmark = pytest.mark.gpu


def comm1(dev):
    uid = (C.c_char * 128)()
    T.check(dev.tcb_comm_unique_id(uid))
    comm = C.c_void_p()
    T.check(dev.tcb_comm_init(1, 0, uid, C.byref(comm)))
    return comm


def test_world_of_one_collectives_are_copies(dev):
    v = C.c_int()
    T.check(dev.tcb_comm_version(C.byref(v)))
    assert v.value >= 22700
    comm = comm1(dev)
    x = np.random.default_rng(1).uniform(-1, 1, 1 << 20)
    src, dst = D.from_array(x), D(x.nbytes)
    T.check(dev.tcb_reduce_scatter(src.ptr, dst.ptr, x.size, comm))
    assert np.array_equal(dst.to_array(x.size), x)
    dst2 = D(x.nbytes)
    T.check(dev.tcb_allreduce(src.ptr, dst2.ptr, x.size, comm))
    assert np.array_equal(dst2.to_array(x.size), x)
    assert dev.tcb_comm_init(1, 3, (C.c_char * 128)(), C.byref(C.c_void_p())) == 1  # TCB_EINVAL
    T.check(dev.tcb_comm_destroy(comm))


def test_ksplit_partial_then_reduce_scatter(dev):
    """cfg5's partition at small size: each 'rank' contracts its l-slab into a
    full partial C; the world-of-one reduce-scatter hands back that partial,
    and the slab partials sum to the oracle (the multi-rank reduce-scatter)."""
    from paper_1307_2100_b200 import partition as P
    e, x = "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=96,j=64,k=32,l=16"
    L, R = O.operands(e, x, 1)
    want = O.naive(e, x, L, R)
    comm = comm1(dev)
    total = np.zeros(want.size)
    _, lab_l, lab_r = P.parse(e)
    ext = P.ext_map(x)
    for part in range(2):
        sh = P.shard_contracted(e, x, "l", 2, part)
        Ls = P.take_slab(L, lab_l, ext, "l", sh.lo, sh.hi)
        Rs = P.take_slab(R, lab_r, ext, "l", sh.lo, sh.hi)
        p = T.Prepared(e, sh.extents)
        p.upload(Ls, Rs)
        p.run()
        _, _, optr = p.device_ptrs()
        recv = D(want.size * 8)
        T.check(dev.tcb_reduce_scatter(optr, recv.ptr, want.size, comm))
        total += recv.to_array(want.size)
        p.close()
    assert O.rel_frobenius(total, want) <= 1e-12
    T.check(dev.tcb_comm_destroy(comm))


# ---- fused K-split exchange over peer memory (tcb_peer_*, run_scattered) ----

def _ksplit_virtual(dev, e, x, label, world, steps=2):
    """All `world` ranks of the K-split in this process (one GPU; the ranks run
    one after the other, no kernel waits on another): rank r contracts its
    `label`-slab with every output block written into its owner's receive slot
    through the peer window; each owner then sums its slots."""
    from paper_1307_2100_b200 import partition as P
    L, R = O.operands(e, x, 1)
    want = O.naive(e, x, L, R)
    out_l, lab_l, lab_r = P.parse(e)
    ext = P.ext_map(x)
    preps = []
    for r in range(world):
        sh = P.shard_contracted(e, x, label, world, r)
        p = T.Prepared(e, sh.extents)
        p.upload(P.take_slab(L, lab_l, ext, label, sh.lo, sh.hi),
                 P.take_slab(R, lab_r, ext, label, sh.lo, sh.hi))
        preps.append(p)
    block = want.size // world
    ex = P.PeerKSplit.virtual(dev, world, block)
    outs = [D(block * 8) for _ in range(world)]
    try:
        for _ in range(steps):  # both parity sets of the receive buffers
            ex.begin()
            for r in range(world):
                ex.scatter(preps[r], rank=r)
            for o in range(world):
                ex.reduce(outs[o].ptr, owner=o)
            got = np.concatenate([b.to_array(block) for b in outs])
            assert O.rel_frobenius(got, want) <= 1e-12, (e, x, world)
    finally:
        ex.close()
        for p in preps:
            p.close()
    return got, want


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_peer_ksplit_cfg5_shape(dev, world):
    # cfg5's expression: split l, blocks of j (the output's outermost label)
    _ksplit_virtual(dev, "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]",
                    f"i=256,j={128 * world * 2},k=32,l={16 * world}", "l", world)


def test_peer_ksplit_ragged_and_odd(dev):
    # odd extents (cp.async path, ragged tiles), block of odd element count
    _ksplit_virtual(dev, "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=37,j=6,k=5,l=6", "l", 3)
    # odd block (37 x 3 elements per owner): slots padded to 16-byte alignment
    _ksplit_virtual(dev, "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=37,j=6,k=5,l=6", "l", 2)


def test_peer_ksplit_outermost_label_in_rows_and_batch(dev):
    # outermost output label is a left free label (split along C's rows) ...
    _ksplit_virtual(dev, "C[+j,+i] = A[+i,+k,+l] * B[-k,-l,+j]", "i=64,j=48,k=16,l=8", "l", 2)
    # ... or a batch label (class-2 shape, cfg2-like: c addresses A and C)
    _ksplit_virtual(dev, "C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=64,b=32,c=8,k=64", "k", 4)
    # ... or an interleaved index-group output (cfg3 shape, L4 in place)
    _ksplit_virtual(dev, "C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]",
                    "a=16,b=16,c=8,d=8,k=8,l=16", "l", 2)


def test_peer_ksplit_errors(dev):
    from paper_1307_2100_b200 import partition as P
    p = T.Prepared("C[+i,+j] = A[+i,+k] * B[-k,+j]", "i=8,j=6,k=4")
    with pytest.raises(ValueError, match="divide evenly"):
        p.run_scattered(0, 4, 1 << 20)  # j=6 does not split into 4 blocks
    with pytest.raises(ValueError, match="part stride"):
        p.run_scattered(0, 2, 8)
    p.close()
    g = C.c_int64()
    T.check(dev.tcb_peer_granularity(C.byref(g)))
    assert dev.tcb_peer_alloc(g.value + 8, C.byref(C.c_void_p()), C.byref(C.c_int())) == 1
    assert dev.tcb_peer_free(C.c_void_p(64)) == 1


def test_peer_ksplit_level2_and_permuted_recipes(dev):
    # GEMV-shaped partials (m or n = 1: the level-2 kernels write the scattered
    # output through the same composite addressing) ...
    _ksplit_virtual(dev, "R[+a] = T[+a,+b,+g] * G[-b,-g]", "a=96,b=12,g=10", "b", 3)
    _ksplit_virtual(dev, "R[+a,+c] = T[+b,+a] * G[-b,+c]", "a=1,b=64,c=40", "b", 2)
    # ... and a class-3.1 recipe whose operand is permuted before the GEMM
    _ksplit_virtual(dev, "R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "a=8,b=24,g=6,e=32", "a", 2)


def test_peer_scatter_refuses_scalar_output(dev):
    p = T.Prepared("K[] = T[+a,+b] * S[-a,-b]", "a=8,b=4")
    with pytest.raises(ValueError, match="no label to split"):
        p.run_scattered(0, 2, 1 << 20)
    p.close()
