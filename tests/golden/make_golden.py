"""Generates the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref/libtcref.so, compiled from /root/reference by oracle/Makefile).
Run here (the reference does not exist on the GPU box):

    make -C oracle && python tests/golden/make_golden.py

  seeded.json   Tensor::seeded_random values (src/tensor.cpp:54-62)
  reports.json  ref_report text (classify/enumerate/plan/render/relayout)
  small.npz     tc::execute (reference backend, auto plan) and
                tc::contract_naive results on small seeded contractions
  baseline.json reference tc::execute results of BASELINE cfg1-cfg4 at full
                size: checksums + 512 sampled entries
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracles as O  # noqa: E402
from specgen import random_spec, table1_expressions  # noqa: E402

ANCHORS = [
    ("K[] = T[+a,+b,+g] * S[-a,-b,-g]", "a=3,b=3,g=3"),
    ("R[+a] = T[+a,+b,+g] * G[-b,-g]", "a=3,b=3,g=3"),
    ("R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "a=4,b=4,g=4,e=4"),
    ("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]", "a=4,b=4,g=4,e=4"),
    ("C[+i,-j] = A[+i,+h] * B[-h,-j]", "i=3,j=4,h=5"),
    ("R[+a,+b,+c,+d] = X[+i,+a,+j,+b] * Y[-i,+c,-j,+d]", "a=2,b=3,c=2,d=3,i=2,j=3"),
    ("R[+a,+b,+c,+d] = X[+i,+a,+j,+b] * Y[-j,+c,-i,+d]", "a=2,b=3,c=2,d=3,i=2,j=3"),
    ("R[+b,+a,+c] = A[+a,+b,-k] * B[+k,+c]", "a=3,b=4,c=5,k=2"),
    ("R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]", "a=4,b=1,g=3,e=5"),
    ("R[+g] = T[+a,+b,+g] * G[-a,-b]", "a=4,b=5,g=6"),
    ("R[+b] = T[+a,+b,+g] * G[-a,-g]", "a=4,b=5,g=6"),
    ("R[+a] = T[+a,+b] * x[-b]", "a=4,b=5"),
]
BASELINE = {
    "cfg1": ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=512,j=512,k=64,l=64"),
    "cfg2": ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=256,b=256,c=256,k=256"),
    "cfg3": ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=64,b=64,c=64,d=64,k=32,l=32"),
    "cfg4": ("C[+a,+b,+i,+j] = A[+a,+b,+k,+l] * B[-k,-l,+i,+j]", "a=256,b=256,i=64,j=64,k=64,l=64"),
    "cfg5": ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=8192,j=8192,k=512,l=512"),
}


def main():
    assert O.ref() is not None, "build the reference first: make -C oracle"
    # seeded streams
    seeded = {}
    import ctypes as C
    for seed in (0, 1, 2, 7, 12345, 2**63 + 5):
        n = 4096
        out = np.empty(n)
        O.ref().ref_seeded(1, (C.c_int64 * 1)(n), seed, out.ctypes.data)
        seeded[str(seed)] = {"first": out[:16].tolist(), "sum": float(out.sum()),
                             "bits_xor": int(np.bitwise_xor.reduce(out.view(np.uint64)))}
    (HERE / "seeded.json").write_text(json.dumps(seeded, indent=1))

    # planner reports
    rng = np.random.default_rng(20261020)
    specs = list(ANCHORS) + [(e, "a=3,b=4,g=5,e=6") for e in table1_expressions()]
    specs += [random_spec(rng) for _ in range(120)]
    specs += list(BASELINE.values())
    reports = []
    for e, x in specs:
        rc, text = O.ref_report(e, x)
        reports.append({"expr": e, "extents": x, "rc": rc, "text": text})
    (HERE / "reports.json").write_text(json.dumps(reports, indent=0))

    # small executions
    arrays = {}
    small = list(ANCHORS) + [random_spec(rng, 5) for _ in range(60)]
    meta = []
    for i, (e, x) in enumerate(small):
        res, st = O.ref_execute(e, x, seed=1)
        L, R = O.operands(e, x, 1)
        arrays[f"exec_{i}"] = res
        arrays[f"naive_{i}"] = O.naive(e, x, L, R)
        meta.append({"expr": e, "extents": x, "stats": st})
    np.savez_compressed(HERE / "small.npz", **arrays)
    (HERE / "small.json").write_text(json.dumps(meta, indent=0))

    # BASELINE cfg1-4 full size: checksums + samples of the reference result
    base = {}
    for name in ("cfg1", "cfg2", "cfg3", "cfg4"):
        e, x = BASELINE[name]
        res, st = O.ref_execute(e, x, seed=1, workers=8)
        idx = np.random.default_rng(7).choice(res.size, 512, replace=False)
        base[name] = {"expr": e, "extents": x, "n": int(res.size), "sum": float(res.sum()),
                      "sumsq": float((res * res).sum()), "idx": idx.tolist(),
                      "val": res[idx].tolist(), "flops": st["flops"]}
    # cfg5: the reference result for the j < 64 column slab (j is B's and C's
    # outermost label, so B's first 64 columns are the first values of its
    # seeded stream and the slab contraction computes C[:, :64] exactly)
    e, x = BASELINE["cfg5"]
    xs = x.replace("j=8192", "j=64")
    res, st = O.ref_execute(e, xs, seed=1, workers=8)
    idx = np.random.default_rng(7).choice(res.size, 512, replace=False)
    base["cfg5_slab"] = {"expr": e, "extents": x, "slab": "j<64", "slab_extents": xs,
                         "n": int(res.size), "sum": float(res.sum()),
                         "sumsq": float((res * res).sum()), "idx": idx.tolist(),
                         "val": res[idx].tolist(), "flops": st["flops"]}
    (HERE / "baseline.json").write_text(json.dumps(base))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
