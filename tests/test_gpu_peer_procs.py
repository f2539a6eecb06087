"""The fused K-split exchange across PROCESSES (SURVEY §8e, cfg5's partition):
two ranks, each its own process and CUDA context, share one B200 here — the
pool gives one GPU — so the exchange is run with host barriers between its
phases and no kernel ever waits on a kernel of the other process:
  1. each rank exports its receive buffer (tcb_peer_alloc), the descriptors
     travel over Unix sockets (partition.exchange_fds), each rank maps both
     ranks' buffers into its window (tcb_peer_window);
  2. each rank runs its l-slab contraction with every j-block written into its
     owner's slot through the window, then signals; host barrier;
  3. each owner reduces its slots (the flags are already set) and checks its
     block of C against the oracle.
On an 8-GPU box the same code runs without the barriers (bench.py --config
cfg5 under torchrun), the owners' reductions waiting on the flags instead."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

E = "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]"
X = "i=192,j=256,k=24,l=32"


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        sys.path.insert(0, os.path.join(root, "tests"))
        import oracles as O
        import paper_1307_2100_b200 as T
        from paper_1307_2100_b200 import partition as P
        dev = T.native.device()
        T.check(dev.tcb_init(0))
        L, R = O.operands(E, X, 1)
        want = O.naive(E, X, L, R)
        out_l, lab_l, lab_r = P.parse(E)
        ext = P.ext_map(X)
        sh = P.shard_contracted(E, X, "l", world, rank)
        prep = T.Prepared(E, sh.extents)
        prep.upload(P.take_slab(L, lab_l, ext, "l", sh.lo, sh.hi),
                    P.take_slab(R, lab_r, ext, "l", sh.lo, sh.hi))
        block = want.size // world
        ex = P.PeerKSplit(dev, world, rank, block, dist)
        out = T.DeviceBuffer(block * 8)
        errs = []
        for _ in range(3):  # both parity sets, then the first again
            ex.begin()
            ex.scatter(prep)
            T.check(dev.tcb_sync())
            dist.barrier()
            ex.reduce(out.ptr)
            T.check(dev.tcb_sync())
            got = out.to_array(block)
            errs.append(O.rel_frobenius(got, want[rank * block:(rank + 1) * block]))
            dist.barrier()  # nobody scatters the next step before all reduced
        ex.close()
        prep.close()
        q.put((rank, max(errs)))
    except Exception as e:  # reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_peer_ksplit_two_processes():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, err in res:
        assert isinstance(err, float), (rank, err)
        assert err <= 1e-12, (rank, err)
