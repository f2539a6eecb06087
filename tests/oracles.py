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


def ref(variant: str = ""):
    """The compiled reference; variant "" (-O3 -DNDEBUG, the reference's own
    flags), "_v3" (-march=x86-64-v3) or "_v4" (-march=x86-64-v4)."""
    key = "ref" + variant
    if key not in _cache:
        so = ORACLE / "_ref" / f"libtcref{variant}.so"
        if not so.exists() and Path("/root/reference/proj/src").is_dir():
            subprocess.run(["make", "-C", str(ORACLE), "ref"], check=True, capture_output=True)
        if not so.exists():
            _cache[key] = None
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
        lib.ref_bind.argtypes = [cp, C.c_int, cp, C.c_uint64, C.c_int, C.c_int, cp, cp, cp, i64]
        lib.ref_bind.restype = vp
        lib.ref_run.argtypes = [vp, C.c_int, vp, i64, P_i64, C.POINTER(f64), cp, i64]
        lib.ref_release.argtypes = [vp]
        lib.ref_release.restype = None
        _cache[key] = lib
    return _cache[key]


def native_variant() -> str:
    """The highest -march level of the compiled reference this host's CPU runs:
    "_v4" with AVX-512 (F, BW, CD, DQ, VL), "_v3" with AVX2 + FMA + BMI2, else ""."""
    try:
        flags = set()
        for line in open("/proc/cpuinfo"):
            if line.startswith("flags"):
                flags = set(line.split(":", 1)[1].split())
                break
    except OSError:
        return ""
    if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl", "avx2", "fma", "bmi2"} <= flags:
        return "_v4"
    if {"avx2", "fma", "bmi2", "movbe"} <= flags:
        return "_v3"
    return ""


class RefBound:
    """A contraction bound once in the compiled reference (seeded operands,
    auto plan); run() is one tc::execute with the reference backend and
    returns its wall seconds (ExecutionStats::wall_seconds)."""

    def __init__(self, expr: str, extents: str, seed: int = 1, variant: str = "",
                 positional: bool = False):
        self.lib = ref(variant)
        if self.lib is None:
            raise RuntimeError(f"oracle/_ref/libtcref{variant}.so missing")
        err = C.create_string_buffer(4096)
        self.h = self.lib.ref_bind(expr.encode(), int(positional), extents.encode(), seed, 0, 0,
                                   b"", b"", err, len(err))
        if not self.h:
            raise RuntimeError(f"reference bind failed: {err.value.decode()}")

    def run(self, workers: int = 1, out: np.ndarray | None = None) -> float:
        secs = C.c_double()
        err = C.create_string_buffer(4096)
        rc = self.lib.ref_run(self.h, workers, None if out is None else out.ctypes.data,
                              0 if out is None else out.size, None, C.byref(secs), err, len(err))
        if rc != 0:
            raise RuntimeError(f"reference run failed: {err.value.decode()}")
        return secs.value

    def close(self):
        if self.h:
            self.lib.ref_release(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


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
