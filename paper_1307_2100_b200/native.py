"""ctypes bindings of the engine's two C-ABIs (include/tcb.h, include/tcf.h).

There is no fallback: if the in-tree libraries are missing this module builds
them (nvcc/g++ are in the image) and raises if that fails. Nothing here calls
the CPU oracle.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB = PKG / "lib"

_lock = threading.Lock()
_libs: dict[str, C.CDLL] = {}

i64, i32, f64, vp, cp = C.c_int64, C.c_int, C.c_double, C.c_void_p, C.c_char_p
P_i64 = C.POINTER(C.c_int64)
P_f64 = C.POINTER(C.c_double)
TCB_MAX_DIMS = 6


class GemmDesc(C.Structure):
    """tcb_gemm_desc (include/tcb.h)."""
    _fields_ = [("m", i64), ("n", i64), ("k", i64),
                ("a_sm", i64), ("a_sk", i64), ("b_sk", i64), ("b_sn", i64),
                ("c_nrow", C.c_int32), ("c_ncol", C.c_int32),
                ("c_row_ext", i64 * TCB_MAX_DIMS), ("c_row_str", i64 * TCB_MAX_DIMS),
                ("c_col_ext", i64 * TCB_MAX_DIMS), ("c_col_str", i64 * TCB_MAX_DIMS),
                ("nbatch", C.c_int32),
                ("bat_ext", i64 * TCB_MAX_DIMS), ("bat_sa", i64 * TCB_MAX_DIMS),
                ("bat_sb", i64 * TCB_MAX_DIMS), ("bat_sc", i64 * TCB_MAX_DIMS),
                ("alpha", f64), ("beta", f64),
                ("g_m", C.c_int32), ("g_n", C.c_int32), ("g_k", C.c_int32),
                ("m_ext", i64 * TCB_MAX_DIMS), ("a_m_str", i64 * TCB_MAX_DIMS),
                ("n_ext", i64 * TCB_MAX_DIMS), ("b_n_str", i64 * TCB_MAX_DIMS),
                ("k_ext", i64 * TCB_MAX_DIMS), ("a_k_str", i64 * TCB_MAX_DIMS),
                ("b_k_str", i64 * TCB_MAX_DIMS)]


class GemmInfo(C.Structure):
    _fields_ = [("path", C.c_int32), ("splits", C.c_int32), ("units", i64),
                ("grid", C.c_int32), ("launches", C.c_int32)]


# name -> (restype, argtypes)
TCB_API = {
    "tcb_init": (i32, [i32]),
    "tcb_finalize": (i32, []),
    "tcb_device_count": (i32, [C.POINTER(C.c_int)]),
    "tcb_current_device": (i32, [C.POINTER(C.c_int)]),
    "tcb_last_error": (cp, []),
    "tcb_set_stream": (i32, [vp]),
    "tcb_sync": (i32, []),
    "tcb_alloc": (i32, [C.POINTER(vp), i64]),
    "tcb_free": (i32, [vp]),
    "tcb_memset0": (i32, [vp, i64]),
    "tcb_h2d": (i32, [vp, vp, i64]),
    "tcb_d2h": (i32, [vp, vp, i64]),
    "tcb_d2d": (i32, [vp, vp, i64]),
    "tcb_host_register": (i32, [vp, i64]),
    "tcb_host_unregister": (i32, [vp]),
    "tcb_host_alloc": (i32, [C.POINTER(vp), i64]),
    "tcb_host_free": (i32, [vp]),
    "tcb_event_sync": (i32, [vp]),
    "tcb_stream_create": (i32, [C.POINTER(vp)]),
    "tcb_stream_destroy": (i32, [vp]),
    "tcb_event_create": (i32, [C.POINTER(vp)]),
    "tcb_event_destroy": (i32, [vp]),
    "tcb_event_record": (i32, [vp, vp]),
    "tcb_stream_wait_event": (i32, [vp, vp]),
    "tcb_stream_sync": (i32, [vp]),
    "tcb_current_stream": (vp, []),
    "tcb_memcpy_async": (i32, [vp, vp, i64, vp]),
    "tcb_memcpy2d_async": (i32, [vp, i64, vp, i64, i64, i64, vp]),
    "tcb_host_is_pinned": (i32, [vp, C.POINTER(C.c_int)]),
    "tcb_gemm": (i32, [C.POINTER(GemmDesc), vp, vp, vp]),
    "tcb_gemm_check": (i32, [C.POINTER(GemmDesc)]),
    "tcb_gemm_gated": (i32, [C.POINTER(GemmDesc), vp, vp, vp, vp, C.c_uint64]),
    "tcb_stream_write_value": (i32, [vp, vp, C.c_uint64]),
    "tcb_last_gemm_info": (i32, [C.POINTER(GemmInfo)]),
    "tcb_dgemm": (i32, [i32, i32, i64, i64, i64, f64, vp, i64, vp, i64, f64, vp, i64]),
    "tcb_dgemm_strided_batched": (i32, [i32, i32, i64, i64, i64, f64, vp, i64, i64, vp, i64,
                                        i64, f64, vp, i64, i64, i64]),
    "tcb_dgemv": (i32, [i32, i64, i64, f64, vp, i64, vp, i64, f64, vp, i64]),
    "tcb_dger": (i32, [i64, i64, f64, vp, i64, vp, i64, vp, i64]),
    "tcb_ddot": (i32, [i64, vp, i64, vp, i64, P_f64]),
    "tcb_permute": (i32, [i32, P_i64, P_i64, vp, vp]),
    "tcb_contract_naive": (i32, [i32, P_i64, P_i64, P_i64, P_i64, i32, P_i64, P_i64, P_i64, vp,
                                 vp, vp]),
    "tcb_comm_version": (i32, [C.POINTER(C.c_int)]),
    "tcb_comm_unique_id": (i32, [vp]),
    "tcb_comm_init": (i32, [i32, i32, vp, C.POINTER(vp)]),
    "tcb_comm_destroy": (i32, [vp]),
    "tcb_reduce_scatter": (i32, [vp, vp, i64, vp]),
    "tcb_allreduce": (i32, [vp, vp, i64, vp]),
    "tcb_peer_granularity": (i32, [P_i64]),
    "tcb_peer_alloc": (i32, [i64, C.POINTER(vp), C.POINTER(C.c_int)]),
    "tcb_peer_window": (i32, [i32, C.POINTER(C.c_int), i64, C.POINTER(vp)]),
    "tcb_peer_free": (i32, [vp]),
    "tcb_peer_signal": (i32, [vp, i64, i64, i32, i32, C.c_uint64]),
    "tcb_peer_reduce": (i32, [vp, i32, i64, i64, vp, vp, C.c_uint64]),
    "tcb_h2d_2d": (i32, [vp, i64, vp, i64, i64, i64]),
    "tcb_d2h_2d": (i32, [vp, i64, vp, i64, i64, i64]),
    "tcb_event_elapsed": (i32, [vp, vp, C.POINTER(C.c_float)]),
    "tcb_event_create_timed": (i32, [C.POINTER(vp)]),
    "tcb_timer_start": (i32, []),
    "tcb_timer_stop": (i32, [C.POINTER(C.c_float)]),
    "tcb_fp64_peak": (i32, [P_f64]),
    "tcb_launch_count": (i64, []),
    "tcb_reset_launch_count": (None, []),
}

TCF_API = {
    "tcf_report": (i32, [cp, i32, cp, cp, i64]),
    "tcf_execute": (i32, [cp, i32, cp, C.c_uint64, i32, i32, i32, cp, cp, vp, i64, P_i64,
                          P_f64, cp, i64]),
    "tcf_execute_host": (i32, [cp, i32, cp, vp, vp, vp, i64, i32, i32, i32, cp, cp, P_i64,
                               P_f64, cp, i64]),
    "tcf_contract_naive": (i32, [cp, i32, cp, C.c_uint64, i64, vp, i64, P_i64, cp, i64]),
    "tcf_lower": (i32, [cp, i32, cp, cp, i64]),
    "tcf_seeded": (i32, [i64, C.c_uint64, vp]),
    "tcf_seeded_block": (i32, [C.c_uint64, i32, P_i64, i32, i64, i64, vp]),
    "tcf_prepare": (i32, [cp, i32, cp, i32, C.POINTER(vp), cp, i64]),
    "tcf_upload": (i32, [vp, vp, vp]),
    "tcf_run": (i32, [vp]),
    "tcf_run_permutes": (i32, [vp]),
    "tcf_run_contraction": (i32, [vp]),
    "tcf_run_scattered": (i32, [vp, vp, i32, i64]),
    "tcf_download": (i32, [vp, vp]),
    "tcf_run_streamed": (i32, [vp, vp, vp, vp, i32, C.POINTER(C.c_int)]),
    "tcf_run_streamed_async": (i32, [vp, vp, vp, vp, i32, C.POINTER(C.c_int)]),
    "tcf_sync": (i32, [vp]),
    "tcf_info": (i32, [vp, P_i64, cp, i64]),
    "tcf_device_ptrs": (i32, [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]),
    "tcf_release": (i32, [vp]),
    "tcf_last_error": (cp, []),
    "tcf_tensor_text": (i32, [P_i64, i32, cp, C.c_uint64, cp, cp, i64]),
    "tcf_read_tensor_text": (i32, [cp, P_f64, i64, P_i64, cp, i64]),
    "tcf_invert_metric": (i32, [i64, P_f64, P_f64, cp, i64]),
    "tcf_metric_apply": (i32, [P_i64, i32, cp, P_f64, i32, i64, P_f64, i32, P_f64, i64, cp, i64]),
    "tcf_bench_csv": (i32, [cp, cp, cp, cp, i32, C.c_uint64, i32, i32, cp, cp, cp, i64,
                            C.POINTER(C.c_int)]),
}


def _bind(lib: C.CDLL, api: dict) -> C.CDLL:
    for name, (res, args) in api.items():
        fn = getattr(lib, name)  # AttributeError = missing export: fail loudly
        fn.restype = res
        fn.argtypes = args
    return lib


def _ensure_built() -> None:
    if (LIB / "libtcb200.so").exists() and (LIB / "libtc_b200.so").exists():
        return
    from . import build as _build
    _build.build()


def device() -> C.CDLL:
    """libtcb200.so: the tcb_* device C-ABI."""
    with _lock:
        if "dev" not in _libs:
            _ensure_built()
            _libs["dev"] = _bind(C.CDLL(str(LIB / "libtcb200.so")), TCB_API)
        return _libs["dev"]


def front() -> C.CDLL:
    """libtc_b200.so: the tcf_* plan-level C-ABI over the tc:: front."""
    with _lock:
        if "front" not in _libs:
            _ensure_built()
            _libs["front"] = _bind(C.CDLL(str(LIB / "libtc_b200.so")), TCF_API)
        return _libs["front"]


class TcbError(RuntimeError):
    pass


def check(status: int, what: str = "tcb") -> None:
    if status != 0:
        msg = device().tcb_last_error().decode()
        if status == 1:
            raise ValueError(f"{what}: {msg}")
        raise TcbError(f"{what}: status {status}: {msg}")
