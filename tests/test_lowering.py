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
             "L3 gemm m=4096 n=4096 k=1024 a(1,4096) b(1,1024) batch=[] permutes=2"),
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
