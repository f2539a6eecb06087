#!/usr/bin/env python
"""Fused K-split exchange (tcb_peer_* + run_scattered) on ONE GPU with G
virtual ranks: what the fusion costs against the plain per-rank contraction.

All G ranks' receive buffers are mapped into one peer window in this process;
rank r contracts its l-slab of cfg5 (C[i,j] = A[i,k,l] B[k,l,j]) with every
j-block of its partial C written into its owner's slot (run_scattered), then
every owner sums its G slots (tcb_peer_reduce). The ranks run one after the
other on the one GPU, so the time is G x (one rank's work): per rank it
compares
  plain   run(): the contraction into the rank's own partial C (followed by a
          tiny launch, as the exchange step follows it in a real K-split), and
  fused   run_scattered() into the window + tcb_peer_signal, and reports
  reduce  tcb_peer_reduce per owner (HBM-bound: reads G blocks, writes one),
and checks the fused result against the per-rank partials summed on the host in
the same rank order (bit-identical: the reduction order is fixed).

    python tools/peer_ksplit_bench.py [--world 8] [--i 8192] [--j 8192] [--k 512] [--l 512]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1307_2100_b200 as T  # noqa: E402
from paper_1307_2100_b200 import partition as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--i", type=int, default=8192)
    ap.add_argument("--j", type=int, default=8192)
    ap.add_argument("--k", type=int, default=512)
    ap.add_argument("--l", type=int, default=512)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    G = a.world
    e = "C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]"
    x = f"i={a.i},j={a.j},k={a.k},l={a.l}"
    dev = T.native.device()
    T.check(dev.tcb_init(0))
    sh = P.shard_contracted(e, x, "l", G, 0)
    preps = [T.Prepared(e, sh.extents) for _ in range(G)]
    info = preps[0].info()
    rng = np.random.default_rng(7)
    for r, p in enumerate(preps):
        L = rng.uniform(-1, 1, info["left"])
        R = rng.uniform(-1, 1, info["right"])
        p.upload(L, R)
        del L, R
    block = info["output"] // G
    ex = P.PeerKSplit.virtual(dev, G, block)
    outs = [T.DeviceBuffer(block * 8) for _ in range(G)]
    ms = C.c_float()

    def timed(fn):
        T.check(dev.tcb_timer_start())
        fn()
        T.check(dev.tcb_timer_stop(C.byref(ms)))
        return float(ms.value)

    brk = T.DeviceBuffer(256)

    def plain():
        # each rank's GEMM is followed by its exchange step in a real K-split
        # (a collective launch or the peer signal), so consecutive GEMMs do not
        # chain under programmatic dependent launch: a 256-byte memset stands
        # in for that launch here
        for p in preps:
            p.run()
            T.check(dev.tcb_memset0(brk.ptr, 256))

    def plain_chained():
        for p in preps:
            p.run()

    def scatter():
        ex.begin()
        for r, p in enumerate(preps):
            ex.scatter(p, rank=r)

    def reduce():
        for o in range(G):
            ex.reduce(outs[o].ptr, owner=o)

    plain(), scatter(), reduce()  # warm-up
    res = {"plain": [], "plain_chained": [], "scatter": [], "reduce": []}
    for _ in range(a.reps):
        res["plain"].append(timed(plain))
        res["plain_chained"].append(timed(plain_chained))
        res["scatter"].append(timed(scatter))
        res["reduce"].append(timed(reduce))
    med = {k: float(np.median(v)) for k, v in res.items()}
    flops = 2.0 * a.i * a.j * a.k * a.l
    # bit-identity: the owners' sums == the plain partials summed in rank order
    parts = []
    for p in preps:
        p.run()
        out = np.empty(info["output"])
        p.download(out)
        parts.append(out)
    want = parts[0].copy()
    for q in parts[1:]:
        want += q
    got = np.concatenate([o.to_array(block) for o in outs])
    line = {
        "tool": "peer_ksplit_bench", "expr": e, "extents": x, "virtual_ranks": G,
        "plain_ms_all_ranks": round(med["plain"], 3),
        "plain_pdl_chained_ms_all_ranks": round(med["plain_chained"], 3),
        "fused_scatter_ms_all_ranks": round(med["scatter"], 3),
        "reduce_ms_all_owners": round(med["reduce"], 3),
        "scatter_overhead": round(med["scatter"] / med["plain"] - 1, 4),
        "plain_tflops": round(flops / med["plain"] * 1e-9, 3),
        "fused_tflops_incl_reduce": round(flops / (med["scatter"] + med["reduce"]) * 1e-9, 3),
        "reduce_gbs": round(G * (G + 1) * block * 8 / (med["reduce"] * 1e-3) / 1e9, 1),
        "bit_identical_to_rank_order_sum": bool(np.array_equal(got, want)),
        "reps_ms": res,
    }
    print(json.dumps(line))
    ex.close()


if __name__ == "__main__":
    main()
