"""The C-ABI libraries load and export every entry point their headers
declare (no compute: CPU only)."""
import re
import subprocess
from pathlib import Path

import paper_1307_2100_b200 as T

ROOT = Path(__file__).resolve().parent.parent


def declared(header: str) -> set[str]:
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"^\s*(?:int|int64_t|void|const char)\s*\**\s*(tc[bf]_\w+)\s*\(",
                          text, flags=re.M))


def exported(so: Path) -> set[str]:
    out = subprocess.run(["nm", "-D", "--defined-only", str(so)], capture_output=True,
                         text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.split()}


def test_device_abi_exports_everything_declared():
    T.native.device()
    names = declared("tcb.h")
    assert len(names) >= 25
    assert names <= exported(T.native.LIB / "libtcb200.so")
    assert names <= set(T.native.TCB_API)


def test_front_abi_exports_everything_declared():
    T.native.front()
    names = declared("tcf.h")
    assert len(names) >= 14
    assert names <= exported(T.native.LIB / "libtc_b200.so")
    assert names <= set(T.native.TCF_API)


def test_cxx_front_exports_the_tc_api():
    syms = subprocess.run(["nm", "-DC", "--defined-only", str(T.native.LIB / "libtc_b200.so")],
                          capture_output=True, text=True, check=True).stdout
    for fn in ["tc::parse", "tc::validate(", "tc::classify(", "tc::plan(", "tc::execute(",
               "tc::enumerate_slicings(", "tc::render_plan", "tc::relayout_advice",
               "tc::make_backend(", "tc::Tensor::seeded_random(", "tc::flop_count("]:
        assert fn in syms, fn


def test_kernels_are_sm100a_dmma_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", str(T.native.LIB / "libtcb200.so")],
                          capture_output=True, text=True, check=True).stdout
    assert "DMMA.8x8x4" in sass
    assert "UTMALDG" in sass
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(T.native.LIB / "libtcb200.so")],
                                       capture_output=True, text=True).stdout


def test_nccl_loads_for_the_collectives():
    """The collective layer loads NCCL at run time (no link-time dependency)."""
    import ctypes as C
    import paper_1307_2100_b200 as T
    v = C.c_int()
    assert T.native.device().tcb_comm_version(C.byref(v)) == 0
    assert v.value >= 22700
