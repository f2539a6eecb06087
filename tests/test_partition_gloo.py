"""Multi-GPU partition logic (paper_1307_2100_b200/partition.py) exercised
with world_size 2 over gloo on the CPU: free-label sharding (cfg4-style, no
communication) and contracted-label splitting + reduce-scatter (cfg5-style).
Each rank's arithmetic here is numpy (the GPU run uses the engine)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1307_2100_b200 import partition as P


def einsum_colmajor(expr, ext, L, R):
    out, left, right = P.parse(expr)
    lt = L.reshape([ext[x] for x in reversed(left)])
    rt = R.reshape([ext[x] for x in reversed(right)])
    spec = "".join(reversed(left)) + "," + "".join(reversed(right)) + "->" + "".join(reversed(out))
    return np.einsum(spec, lt, rt).reshape(-1)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        # ---- free-label shard (cfg4 shape, scaled down): split b, no collective
        e4 = "C[+a,+b,+i,+j] = A[+a,+b,+k,+l] * B[-k,-l,+i,+j]"
        x4 = "a=6,b=8,i=3,j=4,k=5,l=2"
        ext = P.ext_map(x4)
        out, left, right = P.parse(e4)
        L = rng.uniform(-1, 1, int(np.prod([ext[x] for x in left])))
        R = rng.uniform(-1, 1, int(np.prod([ext[x] for x in right])))
        full = einsum_colmajor(e4, ext, L, R)
        sh = P.shard_free(e4, x4, "b", world, rank)
        Ls = P.take_slab(L, left, ext, "b", sh.lo, sh.hi)
        Cs = einsum_colmajor(e4, P.ext_map(sh.extents), Ls, R)
        want = P.take_slab(full, out, ext, "b", sh.lo, sh.hi)
        ok4 = bool(np.allclose(Cs, want, rtol=1e-13, atol=1e-13))
        # gather slabs and reassemble the whole output on every rank
        parts = [None] * world
        dist.all_gather_object(parts, (sh.lo, sh.hi, Cs))
        re = np.zeros_like(full)
        for lo, hi, c in parts:
            P.put_slab(re, out, ext, "b", lo, hi, c)
        ok4 = ok4 and bool(np.allclose(re, full, rtol=1e-13, atol=1e-13))

        # ---- contracted split + reduce-scatter (cfg5 shape, scaled down)
        e5 = "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]"
        x5 = "i=6,j=8,k=3,l=10"
        ext5 = P.ext_map(x5)
        out5, left5, right5 = P.parse(e5)
        L5 = rng.uniform(-1, 1, 6 * 3 * 10)
        R5 = rng.uniform(-1, 1, 3 * 10 * 8)
        full5 = einsum_colmajor(e5, ext5, L5, R5)
        sk = P.shard_contracted(e5, x5, "l", world, rank)
        part = einsum_colmajor(e5, P.ext_map(sk.extents),
                               P.take_slab(L5, left5, ext5, "l", sk.lo, sk.hi),
                               P.take_slab(R5, right5, ext5, "l", sk.lo, sk.hi))
        mine = P.reduce_scatter_columns(torch.from_numpy(part), out5, ext5, "j", world, rank,
                                        dist=dist).numpy()
        lo, hi = P.slab(ext5["j"], world, rank)
        want5 = P.take_slab(full5, out5, ext5, "j", lo, hi)
        ok5 = bool(np.allclose(mine, want5, rtol=1e-13, atol=1e-13))
        q.put((rank, ok4, ok5))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partitions_world_size_2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(results) == [(0, True, True), (1, True, True)]


def _fd_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fd = os.memfd_create(f"rank{rank}")
        os.write(fd, f"payload of rank {rank}".encode())
        fds = P.exchange_fds(fd, world, rank, dist)
        os.close(fd)
        seen = []
        for f in fds:
            # pread: a passed descriptor shares its file offset with the sender's
            seen.append(os.pread(f, 64, 0).decode())
            os.close(f)
        q.put((rank, seen))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_fd_exchange_gloo(world):
    """Host plumbing of the fused K-split exchange (PeerKSplit): every rank
    ends up holding every rank's descriptor, indexed by rank (SCM_RIGHTS over
    Unix sockets; memfd stands in for the exported device allocation)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fd_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [f"payload of rank {r}" for r in range(world)]
    assert results == [(r, want) for r in range(world)]


def test_slab_bounds_cover_exactly():
    for n in (1, 7, 64, 512):
        for w in (1, 2, 3, 8):
            spans = [P.slab(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        P.shard_free("C[+i,+j] = A[+i,+k] * B[-k,+j]", "i=2,j=2,k=2", "k", 2, 0)


class _FakeDev:
    """Stands in for libtcb200 (no GPU here): records the peer calls so the
    address arithmetic of PeerKSplit can be checked on the CPU."""

    def __init__(self):
        self.calls, self.next_ptr = [], 1 << 32

    def tcb_peer_granularity(self, out):
        out._obj.value = 2 << 20
        return 0

    def tcb_peer_alloc(self, nbytes, p, fd):
        p._obj.value = self.next_ptr
        self.next_ptr += 1 << 36
        fd._obj.value = os.open(os.devnull, os.O_RDONLY)
        self.calls.append(("alloc", nbytes))
        return 0

    def tcb_peer_window(self, n, fds, stride, w):
        w._obj.value = 7 << 40
        self.calls.append(("window", n, stride))
        return 0

    def tcb_peer_signal(self, win, stride, flag_off, rank, world, epoch):
        self.calls.append(("signal", win, stride, flag_off, rank, world, epoch))
        return 0

    def tcb_peer_reduce(self, slots, world, count, slot_stride, out, flags, epoch):
        self.calls.append(("reduce", slots, world, count, slot_stride, out, flags, epoch))
        return 0

    def tcb_peer_free(self, p):
        self.calls.append(("free", p))
        return 0


class _FakePrep:
    def __init__(self):
        self.calls = []

    def run_scattered(self, base, parts, part_stride):
        self.calls.append((base, parts, part_stride))


@pytest.mark.parametrize("world,block", [(1, 64), (3, 1000), (4, 111), (8, 8 * 1024 * 1024)])
def test_peer_ksplit_layout_arithmetic(world, block):
    """Host logic of the fused K-split exchange (partition.PeerKSplit): rank r
    writes block o into owner o's slot r of the step's parity set, through the
    window stride; owners reduce their own parity set; flags sit after both
    sets; the allocation is a granularity multiple; odd blocks get even slots."""
    dev, prep = _FakeDev(), _FakePrep()
    ex = P.PeerKSplit.virtual(dev, world, block)
    slot = block + (block & 1)
    assert ex.slot == slot and ex.stride % (2 << 20) == 0
    assert ex.flag_off >= 2 * world * slot * 8 and ex.flag_off + 8 * world <= ex.stride
    win = 7 << 40
    for step in (1, 2, 3):
        ex.begin()
        parity = (step % 2) * world * slot * 8
        for r in range(world):
            ex.scatter(prep, rank=r)
            base, parts, part_stride = prep.calls[-1]
            assert (base, parts, part_stride) == (win + parity + r * slot * 8, world,
                                                  ex.stride // 8)
            # block o of rank r lands in owner o's allocation, slot r
            for o in range(world):
                addr = base + o * part_stride * 8
                assert (addr - win) // ex.stride == o
                assert (addr - win) % ex.stride == parity + r * slot * 8
            assert dev.calls[-1] == ("signal", win, ex.stride, ex.flag_off, r, world, step)
        for o in range(world):
            ex.reduce(1234, owner=o)
            _, slots, w, count, ss, out, flags, epoch = dev.calls[-1]
            assert (w, count, ss, out, epoch) == (world, block, slot, 1234, step)
            assert slots == ex.own[o] + parity and flags == ex.own[o] + ex.flag_off
            assert slots % 16 == 0
    ex.close()
    assert [c[0] for c in dev.calls[-(world + 1):]] == ["free"] * (world + 1)
