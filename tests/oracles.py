"""TEST INFRASTRUCTURE: loaders for the CPU oracles under oracle/.

  tco  = oracle/_ref/libtcoracle.so  — our C restatement (tcoracle.c), built on
         demand with gcc (also on the GPU box).
  ref  = oracle/_ref/libtcref.so     — the unmodified reference core compiled
         from /root/reference (built here by `make -C oracle`; the prebuilt .so
         travels to the GPU box). None when unavailable.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE = ROOT / "oracle"
_cache: dict = {}

i64, f64, vp, cp = C.c_int64, C.c_double, C.c_void_p, C.c_char_p
P_i64 = C.POINTER(C.c_int64)


def tco() -> C.CDLL:
    if "tco" not in _cache:
        so = ORACLE / "_ref" / "libtcoracle.so"
        if not so.exists():
            subprocess.run(["make", "-C", str(ORACLE), "_ref/libtcoracle.so"], check=True,
                           capture_output=True)
        lib = C.CDLL(str(so))
        lib.tco_seeded_random.argtypes = [i64, C.c_uint64, vp]
        lib.tco_contract_naive.argtypes = [C.c_int, P_i64, P_i64, P_i64, P_i64, C.c_int, P_i64,
                                           P_i64, P_i64, vp, vp, vp, i64]
        lib.tco_contract_naive.restype = i64
        lib.tco_gemm_check.argtypes = [C.c_int, C.c_int, i64, i64, i64, f64, vp, i64, vp, i64,
                                       f64, vp, i64]
        lib.tco_tensor_hash.argtypes = [i64, vp]
        lib.tco_tensor_hash.restype = C.c_uint64
        for f in ("tco_max_rel_error", "tco_rel_frobenius"):
            getattr(lib, f).argtypes = [i64, vp, vp]
            getattr(lib, f).restype = f64
        _cache["tco"] = lib
    return _cache["tco"]


def ref():
    if "ref" not in _cache:
        so = ORACLE / "_ref" / "libtcref.so"
        if not so.exists() and Path("/root/reference/proj/src").is_dir():
            subprocess.run(["make", "-C", str(ORACLE), "ref"], check=True, capture_output=True)
        if not so.exists():
            _cache["ref"] = None
            return None
        lib = C.CDLL(str(so))
        lib.ref_report.argtypes = [cp, C.c_int, cp, cp, i64]
        lib.ref_execute.argtypes = [cp, C.c_int, cp, C.c_uint64, C.c_int, C.c_int, C.c_int, cp,
                                    cp, vp, i64, P_i64, C.POINTER(f64), cp, i64]
        lib.ref_naive.argtypes = [cp, C.c_int, cp, C.c_uint64, i64, vp, i64, P_i64, cp, i64]
        lib.ref_seeded.argtypes = [C.c_int, P_i64, C.c_uint64, vp]
        lib.ref_gemm.argtypes = [C.c_int, C.c_int, i64, i64, i64, f64, vp, i64, vp, i64, f64, vp,
                                 i64, cp, i64]
        lib.ref_tensor_text.argtypes = [P_i64, C.c_int, cp, C.c_uint64, cp, cp, i64]
        lib.ref_read_tensor_text.argtypes = [cp, vp, i64, P_i64, cp, i64]
        _cache["ref"] = lib
    return _cache["ref"]


# ---------------------------------------------------------------- helpers
def parse(expr: str):
    """(out, left, right) label lists; variance signs dropped."""
    lhs, rhs = expr.split("=")
    l, r = rhs.split("*")

    def labels(t):
        inner = t[t.index("[") + 1:t.index("]")].strip()
        return [x.strip()[1:] for x in inner.split(",")] if inner else []
    return labels(lhs), labels(l), labels(r)


def ext_map(extents: str) -> dict:
    return {k: int(v) for k, v in (kv.split("=") for kv in extents.split(",") if kv)}


def strides(labels, ext):
    s, run = {}, 1
    for lab in labels:
        s[lab] = run
        run *= ext[lab]
    return s, run


def seeded(n: int, seed: int) -> np.ndarray:
    out = np.empty(int(n))
    tco().tco_seeded_random(int(n), seed, out.ctypes.data)
    return out


def operands(expr: str, extents: str, seed: int = 1):
    out, l, r = parse(expr)
    ext = ext_map(extents)
    nl = int(np.prod([ext[x] for x in l])) if l else 1
    nr = int(np.prod([ext[x] for x in r])) if r else 1
    return seeded(nl, seed), seeded(nr, seed + 1)


def naive(expr: str, extents: str, L: np.ndarray, R: np.ndarray, cap: int = 10**9):
    """tco_contract_naive on the given operands: src/oracle.cpp:32-94 restated."""
    out, l, r = parse(expr)
    ext = ext_map(extents)
    ls, _ = strides(l, ext)
    rs, _ = strides(r, ext)
    os_, no = strides(out, ext)
    con = [x for x in l if x in r]  # left-mode order

    def arr(v):
        return (C.c_int64 * max(1, len(v)))(*v)
    O = np.zeros(no)
    macs = tco().tco_contract_naive(
        len(out), arr([ext[x] for x in out]), arr([ls.get(x, 0) for x in out]),
        arr([rs.get(x, 0) for x in out]), arr([os_[x] for x in out]), len(con),
        arr([ext[x] for x in con]), arr([ls[x] for x in con]), arr([rs[x] for x in con]),
        L.ctypes.data, R.ctypes.data, O.ctypes.data, cap)
    if macs < 0:
        raise MemoryError("oracle work exceeds cap")
    return O


def max_rel_error(a: np.ndarray, b: np.ndarray) -> float:
    return float(tco().tco_max_rel_error(a.size, np.ascontiguousarray(a).ctypes.data,
                                         np.ascontiguousarray(b).ctypes.data))


def rel_frobenius(a: np.ndarray, b: np.ndarray) -> float:
    return float(tco().tco_rel_frobenius(a.size, np.ascontiguousarray(a).ctypes.data,
                                         np.ascontiguousarray(b).ctypes.data))


def ref_execute(expr: str, extents: str, seed: int = 1, workers: int = 1, positional=False,
                kernel: int | None = None, slicing=None):
    lib = ref()
    if lib is None:
        return None
    out, _, _ = parse(expr)
    ext = ext_map(extents)
    n = int(np.prod([ext[x] for x in out])) if out else 1
    res = np.zeros(n)
    st = (C.c_int64 * 4)()
    secs = C.c_double()
    err = C.create_string_buffer(4096)
    policy, kidx, sl, sr = 0, 0, b"", b""
    if kernel is not None:
        policy, kidx = 1, kernel
    if slicing is not None:
        policy, sl, sr = 2, slicing[0].encode(), slicing[1].encode()
    rc = lib.ref_execute(expr.encode(), int(positional), extents.encode(), seed, workers, policy,
                         kidx, sl, sr, res.ctypes.data, n, st, C.byref(secs), err, len(err))
    if rc != 0:
        raise RuntimeError(f"reference failed ({rc}): {err.value.decode()}")
    return res, {"kernel_calls": st[0], "packed_bytes": st[1], "staged_bytes": st[2],
                 "flops": st[3], "wall_seconds": secs.value}


def ref_report(expr: str, extents: str, positional=False):
    lib = ref()
    if lib is None:
        return None
    buf = C.create_string_buffer(1 << 20)
    rc = lib.ref_report(expr.encode(), int(positional), extents.encode(), buf, len(buf))
    return rc, buf.value.decode()


def ref_tensor_text(ext, var: str, seed: int, name: str) -> str:
    """TENSOR v1 text of seeded_random through the reference writer."""
    n = int(np.prod(ext)) if len(ext) else 1
    buf = C.create_string_buffer(64 + 32 * n + 64 * len(ext))
    arr = (C.c_int64 * max(1, len(ext)))(*ext)
    rc = ref().ref_tensor_text(arr, len(ext), var.encode(), seed, name.encode(), buf, len(buf))
    assert rc == 0, buf.value
    return buf.value.decode()


def ref_read_tensor_text(text: str):
    """(values, None) parsed by the reference reader, or (None, message)."""
    cap = 1 << 22
    out = np.empty(cap)
    n = C.c_int64()
    err = C.create_string_buffer(4096)
    rc = ref().ref_read_tensor_text(text.encode(), out.ctypes.data, cap, C.byref(n), err,
                                    len(err))
    if rc != 0:
        return None, err.value.decode()
    return out[:n.value].copy(), None
