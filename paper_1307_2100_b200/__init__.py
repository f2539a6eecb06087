"""B200-native fp64 tensor-contraction engine.

A drop-in for the reference's `tc::` contraction path (arxiv/paper_1307_2100,
`tcontract`): same expression grammar, classification and slicing plans, with
the arithmetic lowered to hand-written sm_100a CUDA (DMMA GEMM with TMA
staging, strided-batched launches, permutation and GEMV/DOT kernels).

The C++ API lives in include/tc/*.hpp (libtc_b200.so); the C-ABIs are
include/tcb.h (device layer, libtcb200.so) and include/tcf.h (plan level).
This Python module is a thin ctypes mirror used by the tests and bench.py.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native
from .native import GemmDesc, GemmInfo, TcbError, check

KERNELS = ["GEMM", "COPY+GEMM", "GEMV", "COPY+GEMV", "GER", "DOT", "ELEMENTWISE"]

__all__ = ["report", "lower", "execute", "execute_host", "seeded", "Prepared", "DeviceBuffer", "GemmDesc", "GemmInfo",
           "TcbError", "check", "native", "KERNELS", "parse_expr", "invert_metric",
           "metric_apply"]


def _err(code: int, buf) -> None:
    if code == 0:
        return
    msg = buf.value.decode() if buf is not None else native.front().tcf_last_error().decode()
    if code == 2:
        raise SyntaxError(msg)          # tc::parse_error
    if code == 3:
        raise MemoryError(msg)          # tc::resource_limit_error
    raise ValueError(msg) if code == 1 else RuntimeError(msg)


def report(expr: str, extents: str, positional: bool = False) -> str:
    """Deterministic analysis text (class, slicing catalogue, plans)."""
    buf = C.create_string_buffer(1 << 20)
    rc = native.front().tcf_report(expr.encode(), int(positional), extents.encode(), buf, len(buf))
    _err(rc, buf)
    return buf.value.decode()


def lower(expr: str, extents: str, positional: bool = False) -> str:
    """The device recipe chosen for a contraction (no device needed)."""
    buf = C.create_string_buffer(4096)
    rc = native.front().tcf_lower(expr.encode(), int(positional), extents.encode(), buf, len(buf))
    _err(rc, buf)
    return buf.value.decode()


def parse_expr(expr: str):
    """(out, left, right) label lists of an expression, e.g. ['i','j'] — a
    lightweight helper for shapes; the authoritative parser is the C++ one."""
    lhs, rhs = expr.split("=")
    l, r = rhs.split("*")

    def labels(t):
        inner = t[t.index("[") + 1:t.index("]")].strip()
        return [x.strip()[1:] for x in inner.split(",")] if inner else []
    return labels(lhs), labels(l), labels(r)


def execute(expr: str, extents: str, seed: int = 1, positional: bool = False, workers: int = 1,
            kernel: str | None = None, slicing: tuple[str, str] | None = None):
    """tc::execute with the b200 backend on seeded operands (left: seed,
    right: seed+1). Returns (result array in storage order, stats dict)."""
    out_l, _, _ = parse_expr(expr)
    ext = dict(kv.split("=") for kv in extents.split(",") if kv)
    n = int(np.prod([int(ext[x]) for x in out_l])) if out_l else 1
    out = np.zeros(n)
    stats = (C.c_int64 * 4)()
    secs = C.c_double()
    err = C.create_string_buffer(4096)
    policy, kidx, sl, sr = 0, 0, b"", b""
    if kernel is not None:
        policy, kidx = 1, KERNELS.index(kernel.upper())
    if slicing is not None:
        policy, sl, sr = 2, slicing[0].encode(), slicing[1].encode()
    rc = native.front().tcf_execute(expr.encode(), int(positional), extents.encode(), seed,
                                    workers, policy, kidx, sl, sr, out.ctypes.data, n, stats,
                                    C.byref(secs), err, len(err))
    _err(rc, err)
    return out, {"kernel_calls": stats[0], "packed_bytes": stats[1], "staged_bytes": stats[2],
                 "flops": stats[3], "wall_seconds": secs.value}


def execute_host(expr: str, extents: str, left: np.ndarray, right: np.ndarray,
                 out: np.ndarray, positional: bool = False, workers: int = 1,
                 kernel: str | None = None, slicing: tuple[str, str] | None = None) -> dict:
    """tc::execute on caller host buffers (tcf_execute_host): `out` receives
    the result; page-locked buffers take the streamed path. Returns stats."""
    for a in (left, right, out):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise ValueError("execute_host needs contiguous float64 arrays")
    stats = (C.c_int64 * 4)()
    secs = C.c_double()
    err = C.create_string_buffer(4096)
    policy, kidx, sl, sr = 0, 0, b"", b""
    if kernel is not None:
        policy, kidx = 1, KERNELS.index(kernel.upper())
    if slicing is not None:
        policy, sl, sr = 2, slicing[0].encode(), slicing[1].encode()
    rc = native.front().tcf_execute_host(expr.encode(), int(positional), extents.encode(),
                                         left.ctypes.data, right.ctypes.data, out.ctypes.data,
                                         out.size, workers, policy, kidx, sl, sr, stats,
                                         C.byref(secs), err, len(err))
    _err(rc, err)
    return {"kernel_calls": stats[0], "packed_bytes": stats[1], "staged_bytes": stats[2],
            "flops": stats[3], "wall_seconds": secs.value}


def contract_naive(expr: str, extents: str, seed: int = 1, positional: bool = False,
                   work_cap: int = 1000000000):
    """tc::contract_naive (tc/oracle.hpp) on seeded operands, evaluated on the
    device: (result, multiply-adds). MemoryError above work_cap."""
    out_l, _, _ = parse_expr(expr)
    ext = dict(kv.split("=") for kv in extents.split(",") if kv)
    n = int(np.prod([int(ext[x]) for x in out_l])) if out_l else 1
    out = np.zeros(n)
    macs = C.c_int64()
    err = C.create_string_buffer(4096)
    rc = native.front().tcf_contract_naive(expr.encode(), int(positional), extents.encode(), seed,
                                           work_cap, out.ctypes.data, n, C.byref(macs), err,
                                           len(err))
    _err(rc, err)
    return out, macs.value


def tensor_text(extents, variance: str, seed: int, name: str = "t") -> str:
    """TENSOR v1 text (tc::write_tensor) of Tensor::seeded_random(extents,
    variance, seed, name)."""
    n = int(np.prod(extents)) if len(extents) else 1
    buf = C.create_string_buffer(64 + 32 * n + 64 * len(extents) + len(name))
    arr = (C.c_int64 * max(1, len(extents)))(*[int(e) for e in extents])
    rc = native.front().tcf_tensor_text(arr, len(extents), variance.encode(), seed,
                                        name.encode(), buf, len(buf))
    _err(rc, buf)
    return buf.value.decode()


def read_tensor_text(text: str) -> np.ndarray:
    """Values of a TENSOR v1 text (tc::read_tensor), storage order."""
    cap = max(16, text.count(" ") + text.count("\n") + 16)
    out = np.empty(cap)
    n = C.c_int64()
    err = C.create_string_buffer(4096)
    rc = native.front().tcf_read_tensor_text(text.encode(), out.ctypes.data_as(
        C.POINTER(C.c_double)), cap, C.byref(n), err, len(err))
    _err(rc, err)
    return out[:n.value].copy()


def invert_metric(g: np.ndarray) -> np.ndarray:
    """tc::invert_metric (reference include/tc/metric.hpp:17-19): the inverse
    of a symmetric n x n metric; ValueError with the reference's messages."""
    g = np.asfortranarray(g, dtype=np.float64)
    if g.ndim != 2 or g.shape[0] != g.shape[1]:
        raise ValueError("metric must be a square rank-2 tensor")
    out = np.empty_like(g, order="F")
    err = C.create_string_buffer(4096)
    pd = C.POINTER(C.c_double)
    rc = native.front().tcf_invert_metric(g.shape[0], g.ctypes.data_as(pd),
                                          out.ctypes.data_as(pd), err, len(err))
    _err(rc, err)
    return out


def metric_apply(t: np.ndarray, variance: str, mode: int, g: np.ndarray,
                 raise_: bool = False) -> np.ndarray:
    """tc::lower_index (raise_ False) / tc::raise_index (True) of mode `mode`
    of t (Fortran order, variances as "+-" chars) with the metric g, on the
    b200 backend (reference include/tc/metric.hpp:24-32)."""
    t = np.asfortranarray(t, dtype=np.float64)
    g = np.asfortranarray(g, dtype=np.float64)
    out = np.empty_like(t, order="F")
    ext = (C.c_int64 * max(1, t.ndim))(*t.shape)
    err = C.create_string_buffer(4096)
    pd = C.POINTER(C.c_double)
    rc = native.front().tcf_metric_apply(ext, t.ndim, variance.encode(), t.ctypes.data_as(pd),
                                         mode, g.shape[0], g.ctypes.data_as(pd), int(raise_),
                                         out.ctypes.data_as(pd), out.size, err, len(err))
    _err(rc, err)
    return out


def bench_csv(experiment: str = "square3d", sizes=(100,), kernels=("GEMM",),
              backend: str = "b200", repetitions: int = 5, seed: int = 1,
              verify: bool = False, workers: int = 1, custom_expr: str = "",
              custom_extents: str = ""):
    """tc::run_bench + tc::write_bench_csv: (csv text, all sampled lines ok)."""
    buf = C.create_string_buffer(1 << 20)
    ok = C.c_int()
    rc = native.front().tcf_bench_csv(
        experiment.encode(), ",".join(str(s) for s in sizes).encode(),
        ",".join(kernels).encode(), backend.encode(), repetitions, seed, int(verify), workers,
        custom_expr.encode(), custom_extents.encode(), buf, len(buf), C.byref(ok))
    _err(rc, buf)
    return buf.value.decode(), bool(ok.value)


def seeded(n: int, seed: int) -> np.ndarray:
    """Tensor::seeded_random's value stream (uniform [-1,1], mt19937_64)."""
    out = np.empty(int(n))
    native.front().tcf_seeded(int(n), seed, out.ctypes.data)
    return out


def seeded_block(extents, seed: int, mode: int, lo: int, hi: int) -> np.ndarray:
    """Slab [lo, hi) along `mode` of Tensor::seeded_random(extents, seed), in
    storage order (column-major, first mode fastest)."""
    n = int(np.prod(extents)) // int(extents[mode]) * (hi - lo)
    out = np.empty(n)
    arr = (C.c_int64 * len(extents))(*[int(e) for e in extents])
    rc = native.front().tcf_seeded_block(seed, len(extents), arr, mode, lo, hi, out.ctypes.data)
    _err(rc, None)
    return out


class Prepared:
    """tc::PreparedContraction: lowered once, device buffers bound."""

    def __init__(self, expr: str, extents: str, device: int = 0, positional: bool = False):
        self._lib = native.front()
        h = C.c_void_p()
        err = C.create_string_buffer(4096)
        rc = self._lib.tcf_prepare(expr.encode(), int(positional), extents.encode(), device,
                                   C.byref(h), err, len(err))
        _err(rc, err)
        self._h = h

    def _ok(self, rc):
        _err(rc, None)

    def upload(self, left: np.ndarray, right: np.ndarray) -> None:
        self._ok(self._lib.tcf_upload(self._h, left.ctypes.data, right.ctypes.data))

    def run(self) -> None:
        self._ok(self._lib.tcf_run(self._h))

    def run_permutes(self) -> None:
        self._ok(self._lib.tcf_run_permutes(self._h))

    def run_contraction(self) -> None:
        self._ok(self._lib.tcf_run_contraction(self._h))

    def run_scattered(self, base: int, parts: int, part_stride: int) -> None:
        """Contraction with the output's outermost label split into `parts`
        blocks, block p written at device address base + 8 * p * part_stride
        (the fused K-split exchange when base lies in a peer window)."""
        self._ok(self._lib.tcf_run_scattered(self._h, base, parts, part_stride))

    def run_streamed(self, left: np.ndarray, right: np.ndarray, out: np.ndarray,
                     slabs: int = 0, wait: bool = True) -> int:
        """Host-to-host with H2D/compute/D2H overlapped (pinned buffers).
        wait=False returns once enqueued: the next call overlaps its uploads
        with this one's download drain; sync() completes it."""
        used = C.c_int()
        fn = self._lib.tcf_run_streamed if wait else self._lib.tcf_run_streamed_async
        self._ok(fn(self._h, left.ctypes.data, right.ctypes.data, out.ctypes.data, slabs,
                    C.byref(used)))
        return used.value

    def download(self, out: np.ndarray) -> None:
        self._ok(self._lib.tcf_download(self._h, out.ctypes.data))

    def sync(self) -> None:
        self._ok(self._lib.tcf_sync(self._h))

    def info(self) -> dict:
        v = (C.c_int64 * 12)()
        s = C.create_string_buffer(1024)
        self._ok(self._lib.tcf_info(self._h, v, s, len(s)))
        keys = ["left", "right", "output", "launches", "permuted_bytes", "m", "n", "k", "batch",
                "flops", "permutes", "path"]
        d = dict(zip(keys, list(v)))
        d["summary"] = s.value.decode()
        return d

    def device_ptrs(self):
        a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
        self._lib.tcf_device_ptrs(self._h, C.byref(a), C.byref(b), C.byref(c))
        return a.value, b.value, c.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.tcf_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceBuffer:
    """Raw device allocation through tcb_alloc (tests of the device C-ABI)."""

    def __init__(self, nbytes: int):
        self.lib = native.device()
        p = C.c_void_p()
        check(self.lib.tcb_alloc(C.byref(p), int(nbytes)), "tcb_alloc")
        self.ptr, self.nbytes = p.value, int(nbytes)

    @classmethod
    def from_array(cls, a: np.ndarray) -> "DeviceBuffer":
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = cls(max(a.nbytes, 8))
        if a.nbytes:
            check(b.lib.tcb_h2d(b.ptr, a.ctypes.data, a.nbytes), "tcb_h2d")
        return b

    def to_array(self, n: int | None = None) -> np.ndarray:
        n = self.nbytes // 8 if n is None else n
        out = np.empty(n)
        check(self.lib.tcb_d2h(out.ctypes.data, self.ptr, n * 8), "tcb_d2h")
        return out

    def free(self):
        if self.ptr:
            self.lib.tcb_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
