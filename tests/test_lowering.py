"""The device lowering (DeviceRecipe, lower.cpp): BASELINE configs map onto
the recipes DESIGN.md names, and every recipe of the random family covers
the contraction exactly. CPU only (no device touched)."""
import re

import numpy as np

import paper_1307_2100_b200 as T
from specgen import random_spec

CFG = {
    "cfg1": ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=512,j=512,k=64,l=64",
             "L1 gemm m=512 n=512 k=4096 a(1,512) b(1,4096) batch=[] permutes=0"),
    "cfg2": ("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=256,b=256,c=256,k=256",
             "L2 gemm m=256 n=256 k=256 a(1,256) b(1,256) batch=[256] permutes=0"),
    "cfg3": ("C[+a,+b,+c,+d] = A[+a,+k,+c,+l] * B[-l,+b,-k,+d]", "a=64,b=64,c=64,d=64,k=32,l=32",
             "L4 gemm m=4096 n=4096 k=1024 m[64:1,64:2048] n[64:32,64:65536] "
             "k[32:131072/1,32:64/2048] batch=[] permutes=0"),
    "cfg4": ("C[+a,+b,+i,+j] = A[+a,+b,+k,+l] * B[-k,-l,+i,+j]", "a=256,b=256,i=64,j=64,k=64,l=64",
             "L1 gemm m=65536 n=4096 k=4096 a(1,65536) b(1,4096) batch=[] permutes=0"),
    "cfg5": ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=8192,j=8192,k=512,l=512",
             "L1 gemm m=8192 n=8192 k=262144 a(1,8192) b(1,262144) batch=[] permutes=0"),
}


def test_baseline_recipes():
    for name, (e, x, want) in CFG.items():
        assert T.lower(e, x) == want, name


def test_recipes_cover_the_contraction():
    rng = np.random.default_rng(5)
    pat = re.compile(r"(L\d) gemm m=(\d+) n=(\d+) k=(\d+) .* batch=\[([\d,]*)\]")
    for _ in range(500):
        e, x = random_spec(rng)
        lay, m, n, k, batch = pat.match(T.lower(e, x)).groups()
        ext = {kk: int(v) for kk, v in (kv.split("=") for kv in x.split(","))}
        b = int(np.prod([int(v) for v in batch.split(",") if v])) if batch else 1
        # every label extent is accounted for exactly once (M, N, K or batch)
        assert int(m) * int(n) * int(k) * b == int(np.prod(list(ext.values()))), (e, x)


def test_index_groups_switch(monkeypatch):
    """TC_INDEX_GROUPS=0 restores the permuting L3 recipe for cfg3."""
    e, x, _ = CFG["cfg3"]
    monkeypatch.setenv("TC_INDEX_GROUPS", "0")
    assert T.lower(e, x) == "L3 gemm m=4096 n=4096 k=1024 a(1,4096) b(1,1024) batch=[] permutes=2"


def _groups(summary, name):
    m = re.search(name + r"\[([^\]]*)\]", summary)
    return [tuple(int(v) for v in re.split("[:/]", g)) for g in m.group(1).split(",")]


def test_l4_recipes_fit_the_tensor_map_rules():
    """Every L4 recipe of the random family respects the box rules of
    make_map (gemm_dmma.cu): unit-stride lead, inner extents tiling the
    16 / 128 boxes, at most 5 map dims per operand, even strides."""
    rng = np.random.default_rng(11)
    seen = 0
    for _ in range(3000):
        e, x = random_spec(rng, extents=(16, 32, 64, 128, 3, 48))
        s = T.lower(e, x)
        if not s.startswith("L4"):
            continue
        seen += 1
        M, N, K = _groups(s, " m"), _groups(s, " n"), _groups(s, " k")
        for outer, ks in ((M, [(k[0], k[1]) for k in K]), (N, [(k[0], k[2]) for k in K])):
            assert len(outer) + len(ks) <= 5, s
            kmajor = outer[0][1] != 1
            lead, other = (ks, outer) if kmajor else (outer, ks)
            assert lead[0][1] == 1, s
            if len(lead) > 1:
                assert lead[0][0] % 16 == 0, s
            box = 128 if kmajor else 16
            if len(other) > 1 and other[0][0] % box:
                assert kmajor and box % other[0][0] == 0, s
            for ext, st in lead[1:] + other:
                assert ext == 1 or st % 2 == 0, s
    assert seen > 20
