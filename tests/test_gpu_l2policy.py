"""Cache-policy paths change no bits: a contraction whose GEMM raster keeps a
group of B panels resident (operands above L2, B's panels grouped: the
`evict_last` hint, and with TCB_L2PERSIST=1 the persisting set-aside plus the
post-launch demotion kernel) gives the same result bit for bit as with the
hints off (TCB_L2HINT=00), each in a fresh process (the knobs are read once).
Also the device block cache behind tcb_alloc / tcb_free. Requires a B200."""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import pytest

import paper_1307_2100_b200 as T

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
# m = 65536 rows of A (256 MB) above L2, n = 1024: 8 B panels of 512 KB grouped
EXPR, EXT = "C[+i,+j] = A[+i,+k] * B[-k,+j]", "i=65536,j=1024,k=512"
PROG = f"""
import hashlib, sys
sys.path.insert(0, {str(ROOT)!r})
import paper_1307_2100_b200 as T
got, st = T.execute({EXPR!r}, {EXT!r}, seed=5)
print(hashlib.sha256(got.tobytes()).hexdigest(), st["kernel_calls"])
"""


def _run(env_extra):
    # TC_NO_PIN: one launch over the whole contraction (the streamed path's
    # slab GEMMs are too narrow for the grouped raster)
    env = dict(os.environ, TC_NO_PIN="1", **env_extra)
    r = subprocess.run([sys.executable, "-c", PROG], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    digest, calls = r.stdout.split()[-2:]
    return digest, int(calls)


def test_l2_policies_change_no_bits(dev):
    base, _ = _run({"TCB_L2HINT": "00"})
    hinted, calls = _run({})
    persist, calls_p = _run({"TCB_L2PERSIST": "1"})
    assert hinted == base and persist == base
    assert calls_p == calls + 1  # the demotion kernel after the GEMM


def test_block_cache_reuses_exact_sizes(dev):
    a, b = C.c_void_p(), C.c_void_p()
    T.check(dev.tcb_alloc(C.byref(a), 3 << 20))
    first = a.value
    T.check(dev.tcb_free(a))
    T.check(dev.tcb_alloc(C.byref(b), 3 << 20))
    assert b.value == first  # the idle block of that size, not a new one
    c = C.c_void_p()
    T.check(dev.tcb_alloc(C.byref(c), (3 << 20) + 8))
    assert c.value != first
    for p in (b, c):
        T.check(dev.tcb_free(p))
    # blocks are usable after reuse: write and read back
    buf = T.DeviceBuffer(3 << 20)
    T.check(dev.tcb_memset0(buf.ptr, buf.nbytes))
