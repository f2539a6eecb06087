"""Host logic of bench.py's multi-rank path (CPU only): each rank's seeded
operand slabs tile the full seeded tensors, and the golden-parity check maps
every committed reference sample to exactly one rank's output block."""
import json
from pathlib import Path

import numpy as np
import pytest

import bench
from paper_1307_2100_b200 import partition as P

GOLD = Path(__file__).resolve().parent / "golden" / "baseline.json"


@pytest.mark.parametrize("cfg,ext", [
    ("cfg1", "i=24,j=10,k=3,l=5"),   # shard j (B's last mode)
    ("cfg2", "a=6,b=5,c=7,k=4"),     # shard c (A's last mode, B unsplit)
    ("cfg3", "a=3,b=4,c=2,d=5,k=2,l=3"),
    ("cfg4", "a=4,b=6,i=3,j=2,k=3,l=2"),  # shard b (middle mode of A)
    ("cfg5", "i=7,j=6,k=3,l=8"),     # ksplit l (last of A, middle of B)
])
@pytest.mark.parametrize("world", [2, 3])
def test_rank_slabs_tile_the_seeded_operands(cfg, ext, world):
    expr = bench.CONFIGS[cfg][0]
    _, label = bench.MODE[cfg]
    _, left, right = P.parse(expr)
    em = P.ext_map(ext)
    import paper_1307_2100_b200 as T
    fullL = T.seeded(int(np.prod([em[x] for x in left])), 1)
    fullR = T.seeded(int(np.prod([em[x] for x in right])), 2)
    for rank in range(world):
        lo, hi = P.slab(em[label], world, rank)
        sub = dict(em)
        sub[label] = hi - lo
        L = np.empty(int(np.prod([sub[x] for x in left])))
        R = np.empty(int(np.prod([sub[x] for x in right])))
        bench.fill_operands(expr, ext, label, lo, hi, L, R)
        assert np.array_equal(L, P.take_slab(fullL, left, em, label, lo, hi))
        assert np.array_equal(R, P.take_slab(fullR, right, em, label, lo, hi))


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
@pytest.mark.parametrize("world", [1, 2, 8])
def test_golden_parity_partitions_the_samples(cfg, world):
    g = json.loads(GOLD.read_text())[cfg]
    expr, full = bench.CONFIGS[cfg][0], bench.CONFIGS[cfg][1]
    _, label = bench.MODE[cfg]
    out, _, _ = P.parse(expr)
    em = P.ext_map(full)
    # a full output that holds the reference's sampled values, zero elsewhere
    C = np.zeros(g["n"])
    C[np.array(g["idx"])] = np.array(g["val"])
    seen = 0
    for rank in range(world):
        if world == 1:
            res = bench.golden_parity(cfg, expr, full, None, 0, 0, C)
            assert res["samples"] == len(g["idx"]) and res["max_rel_error"] == 0.0
            seen += res["samples"]
            continue
        lo, hi = P.slab(em[label], world, rank)
        block = P.take_slab(C, out, em, label, lo, hi)
        res = bench.golden_parity(cfg, expr, full, label, lo, hi, block)
        assert res["ok"], (rank, res)
        seen += res["samples"]
        # a corrupted block is caught
        if res["samples"]:
            bad = block.copy()
            bad[:] += 1.0
            assert not bench.golden_parity(cfg, expr, full, label, lo, hi, bad)["ok"]
    assert seen == len(g["idx"])


def test_cpu_samples_keep_the_reference_kernel_shape():
    # the bounded CPU samples are sub-contractions of the same expression
    for cfg, (sample, _) in bench.CPU_SAMPLE.items():
        full = P.ext_map(bench.CONFIGS[cfg][1])
        s = P.ext_map(sample)
        assert set(s) == set(full)
        assert all(s[x] <= full[x] for x in s)
    # cfg5: 256-column panels (the reference GEMM's panel width) over full i and k
    s = P.ext_map(bench.CPU_SAMPLE["cfg5"][0])
    assert s["j"] == 256 and s["i"] == 8192 and s["k"] == 512
