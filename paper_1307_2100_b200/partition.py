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
