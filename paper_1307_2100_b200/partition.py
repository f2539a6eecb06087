"""Multi-GPU partitioning of one contraction (one process per GPU).

The reference has no distributed execution; BASELINE asks
for two partitions of a large contraction over one 8xB200 box:

  * free-label split ("shard"): the ranks own disjoint slabs of a free label
    of the output — no communication (cfg4: split b of C[a,b,i,j]);
  * contracted-label split ("ksplit"): the ranks own disjoint slabs of a
    contracted label, each computes a partial C, and a reduce-scatter (sum)
    over NCCL leaves rank r with the r-th column block of C (cfg5: split l of
    C[i,j] = A[i,k,l] B[k,l,j], reduce-scatter over j).

This module is the host-side plumbing: slab bounds, operand slicing of the
column-major tensors, and the collective. It works on numpy arrays (CPU, gloo
tests) and on torch CUDA tensors (NCCL) alike; the arithmetic of each rank is
the engine's ordinary single-GPU path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def parse(expr: str):
    lhs, rhs = expr.split("=")
    l, r = rhs.split("*")

    def labels(t):
        inner = t[t.index("[") + 1:t.index("]")].strip()
        return [x.strip()[1:] for x in inner.split(",")] if inner else []
    return labels(lhs), labels(l), labels(r)


def ext_map(extents: str) -> dict:
    return {k: int(v) for k, v in (kv.split("=") for kv in extents.split(",") if kv)}


def ext_str(ext: dict) -> str:
    return ",".join(f"{k}={v}" for k, v in ext.items())


def slab(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's share of n items, as even as possible."""
    return n * rank // world, n * (rank + 1) // world


@dataclass
class Shard:
    label: str
    lo: int
    hi: int
    extents: str  # extents of this rank's sub-contraction


def shard_free(expr: str, extents: str, label: str, world: int, rank: int) -> Shard:
    out, left, right = parse(expr)
    if label not in out:
        raise ValueError(f"'{label}' is not a free (output) label of {expr}")
    ext = ext_map(extents)
    lo, hi = slab(ext[label], world, rank)
    sub = dict(ext)
    sub[label] = hi - lo
    return Shard(label, lo, hi, ext_str(sub))


def shard_contracted(expr: str, extents: str, label: str, world: int, rank: int) -> Shard:
    out, left, right = parse(expr)
    if label in out or label not in left or label not in right:
        raise ValueError(f"'{label}' is not a contracted label of {expr}")
    ext = ext_map(extents)
    lo, hi = slab(ext[label], world, rank)
    sub = dict(ext)
    sub[label] = hi - lo
    return Shard(label, lo, hi, ext_str(sub))


def take_slab(flat, labels: list[str], ext: dict, label: str, lo: int, hi: int):
    """Slab [lo, hi) along `label` of a column-major tensor stored flat (numpy
    or torch); returns a contiguous flat array in the same mode order."""
    if label not in labels:
        return flat
    shape_f = [ext[x] for x in labels]
    ax = labels.index(label)
    # column-major (first mode fastest) == C-order over the reversed shape
    rev = list(reversed(shape_f))
    rax = len(labels) - 1 - ax
    t = flat.reshape(rev)
    idx = [slice(None)] * len(rev)
    idx[rax] = slice(lo, hi)
    s = t[tuple(idx)]
    if hasattr(s, "contiguous"):
        return s.contiguous().reshape(-1)
    return np.ascontiguousarray(s).reshape(-1)


def put_slab(dst_flat, labels: list[str], ext: dict, label: str, lo: int, hi: int, src_flat):
    """Writes a slab (as produced by take_slab) back into a full tensor."""
    rev = [ext[x] for x in reversed(labels)]
    rax = len(labels) - 1 - labels.index(label)
    t = dst_flat.reshape(rev)
    idx = [slice(None)] * len(rev)
    idx[rax] = slice(lo, hi)
    sub_rev = list(rev)
    sub_rev[rax] = hi - lo
    t[tuple(idx)] = src_flat.reshape(sub_rev)


def reduce_scatter_columns(partial, out_labels: list[str], ext: dict, label: str, world: int,
                           rank: int, dist=None, group=None):
    """Sums the ranks' partial outputs and returns rank's slab along `label`
    (the outermost output label, so every slab is one contiguous block).
    `partial` is a torch tensor (flat, column-major); `dist` is
    torch.distributed. Uses reduce_scatter_tensor (NCCL ReduceScatter) or, on
    backends without it (gloo), all_reduce + slice."""
    import torch
    if out_labels[-1] != label:
        raise ValueError("reduce-scatter label must be the outermost output label")
    n = ext[label]
    if n % world:
        raise ValueError("reduce-scatter label extent must divide evenly by the world size")
    per = partial.numel() // world
    if dist.get_backend(group) == "nccl":
        out = torch.empty(per, dtype=partial.dtype, device=partial.device)
        dist.reduce_scatter_tensor(out, partial.contiguous(), op=dist.ReduceOp.SUM, group=group)
        return out
    full = partial.clone()
    dist.all_reduce(full, op=dist.ReduceOp.SUM, group=group)
    return full[rank * per:(rank + 1) * per].clone()


# ---------------------------------------------------------------------------
# Fused K-split exchange over peer memory (include/tcb.h tcb_peer_*)
#
# Instead of contracting into a local partial C and reduce-scattering it
# afterwards, every rank's GEMM epilogue writes block o of its partial C
# straight into rank o's receive buffer (tc::PreparedContraction::
# run_scattered through a window that maps all ranks' receive buffers back to
# back), so the exchange overlaps the contraction tile by tile; then each owner
# sums its `world` received slots in rank order (tcb_peer_reduce). Receive
# buffers hold two parity sets, so step e+1's writes never meet step e's
# reduction: a rank's GEMM of step e+2 is stream-ordered after its reduction of
# step e+1, which waited for every owner's signal of step e+1, each of which is
# stream-ordered after that owner's reduction of step e.

def exchange_fds(fd: int, world: int, rank: int, dist, group=None) -> list[int]:
    """All ranks' file descriptors (index = rank; own entry a dup of `fd`),
    passed over abstract-namespace Unix sockets with SCM_RIGHTS. `dist` is
    torch.distributed (rendezvous and barriers only)."""
    import os
    import socket
    import threading

    tag = [f"{os.getpid()}-{id(fd)}" if rank == 0 else None]
    dist.broadcast_object_list(tag, src=0, group=group)

    def addr(q):
        return f"\0tcb-peer-{tag[0]}-{q}"

    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(addr(rank))
    srv.listen(max(1, world))
    got = {rank: os.dup(fd)}
    errors = []

    def accept_all():
        try:
            for _ in range(world - 1):
                conn, _ = srv.accept()
                with conn:
                    msg, fds, _, _ = socket.recv_fds(conn, 32, 1)
                    got[int(msg.decode())] = fds[0]
        except Exception as e:  # surfaced below
            errors.append(e)

    dist.barrier(group=group)  # every rank listens
    t = threading.Thread(target=accept_all, daemon=True)
    t.start()
    for q in range(world):
        if q == rank:
            continue
        with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
            c.connect(addr(q))
            socket.send_fds(c, [str(rank).encode()], [fd])
    t.join(timeout=120)
    srv.close()
    if errors or len(got) != world:
        raise RuntimeError(f"exchange_fds: rank {rank} received {sorted(got)} ({errors})")
    dist.barrier(group=group)
    return [got[q] for q in range(world)]


class PeerKSplit:
    """Peer-memory exchange for one K-split contraction of `block` output
    elements per rank (block = output elements / world).

    Multi-process: PeerKSplit(dev, world, rank, block, dist) — one allocation
    per rank, descriptors exchanged, every rank maps the window. Single
    process: PeerKSplit.virtual(dev, world, block) — all `world` allocations in
    this process (the same data path on one GPU, the ranks run one after the
    other; used by the GPU tests)."""

    def __init__(self, dev, world: int, rank: int | None, block: int, dist=None, group=None,
                 _local: int = 1, host_sync: bool = False):
        import ctypes as C
        import os
        from . import native
        self.dev, self.world, self.rank, self.block = dev, world, rank, block
        # host_sync: a host barrier between the scatter and the reduction, so
        # no reduction kernel ever waits for another process's kernels (ranks
        # sharing one GPU in plumbing tests); on one GPU per rank the reduction
        # waits on the flags instead
        self.dist, self.group, self.host_sync = dist, group, host_sync
        self.epoch = 0
        self.slot = block + (block & 1)  # slots start 16-byte aligned
        gran = C.c_int64()
        native.check(dev.tcb_peer_granularity(C.byref(gran)), "tcb_peer_granularity")
        slots = 2 * world * self.slot * 8  # two parity sets of `world` slots
        self.flag_off = -(-slots // 256) * 256
        self.stride = -(-(self.flag_off + 8 * world) // gran.value) * gran.value
        self.own = []  # local allocations (1, or `world` in a virtual exchange)
        fds = []
        try:
            for _ in range(_local):
                p, fd = C.c_void_p(), C.c_int()
                native.check(dev.tcb_peer_alloc(self.stride, C.byref(p), C.byref(fd)),
                             "tcb_peer_alloc")
                self.own.append(p.value)
                fds.append(fd.value)
            if _local == 1 and world > 1:
                all_fds = exchange_fds(fds[0], world, rank, dist, group)
                os.close(fds[0])
                fds = all_fds
            arr = (C.c_int * world)(*fds)
            w = C.c_void_p()
            native.check(dev.tcb_peer_window(world, arr, self.stride, C.byref(w)),
                         "tcb_peer_window")
            self.window = w.value
        finally:
            for fd in fds:
                os.close(fd)

    @classmethod
    def virtual(cls, dev, world: int, block: int) -> "PeerKSplit":
        return cls(dev, world, None, block, _local=world)

    def _parity(self) -> int:
        return (self.epoch % 2) * self.world * self.slot * 8

    def begin(self) -> None:
        """Starts a step (all ranks' scatters of this step use its epoch)."""
        self.epoch += 1

    def scatter(self, prep, rank: int | None = None) -> None:
        """Rank `rank`'s contraction, every block written into its owner's slot."""
        from . import native
        r = self.rank if rank is None else rank
        base = self.window + self._parity() + r * self.slot * 8
        prep.run_scattered(base, self.world, self.stride // 8)
        native.check(self.dev.tcb_peer_signal(self.window, self.stride, self.flag_off, r,
                                              self.world, self.epoch), "tcb_peer_signal")

    def reduce(self, out_ptr: int, owner: int | None = None) -> None:
        """out[0..block) = sum of the owner's `world` received slots."""
        from . import native
        mine = self.own[0] if owner is None else self.own[owner]
        native.check(self.dev.tcb_peer_reduce(mine + self._parity(), self.world, self.block,
                                              self.slot, out_ptr, mine + self.flag_off,
                                              self.epoch), "tcb_peer_reduce")

    def step(self, prep, out_ptr: int) -> None:
        from . import native
        self.begin()
        self.scatter(prep)
        if self.host_sync:
            native.check(self.dev.tcb_sync(), "tcb_sync")
            self.dist.barrier(group=self.group)
        self.reduce(out_ptr)
        if self.host_sync:  # nobody scatters the next step into slots still being reduced
            native.check(self.dev.tcb_sync(), "tcb_sync")
            self.dist.barrier(group=self.group)

    def close(self) -> None:
        from . import native
        if getattr(self, "window", None):
            native.check(self.dev.tcb_peer_free(self.window), "tcb_peer_free")
            self.window = None
        for p in getattr(self, "own", []):
            native.check(self.dev.tcb_peer_free(p), "tcb_peer_free")
        self.own = []
