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
