"""Builds the engine's native libraries in-tree (they travel to the GPU box).

  lib/libtcb200.so   device layer: sm_100a CUDA kernels + the tcb_* C-ABI
                     (csrc/device/*.cu, nvcc -gencode arch=compute_100a,code=sm_100a)
  lib/libtc_b200.so  host front: the tc:: C++ API + the tcf_* C-ABI
                     (csrc/host/*.cpp, g++), linked against libtcb200.so

Incremental: an object is rebuilt when its source or any header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
INC = ROOT / "include"
DEV_SRC = PKG / "csrc" / "device"
HOST_SRC = PKG / "csrc" / "host"
LIB = PKG / "lib"
OBJ = LIB / "obj"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
# The image exports CXX=/opt/gcc/bin/g++ whose libstdc++.so link is dangling
# (it silently links libstdc++.a into shared objects); use the system driver.
CXX = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", f"-I{INC}", f"-I{DEV_SRC}"]
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", f"-I{INC}"]


def _headers() -> list[Path]:
    return list(INC.rglob("*.h")) + list(INC.rglob("*.hpp")) + list(DEV_SRC.glob("*.cuh"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"command failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def build(verbose: bool = False, jobs: int | None = None) -> dict[str, Path]:
    LIB.mkdir(exist_ok=True)
    OBJ.mkdir(exist_ok=True)
    hdrs = _headers()
    jobs = jobs or min(16, os.cpu_count() or 4)

    dev_objs, host_objs, work = [], [], []
    for src in sorted(DEV_SRC.glob("*.cu")):
        obj = OBJ / (src.stem + ".cu.o")
        dev_objs.append(obj)
        if _stale(obj, [src, *hdrs]):
            work.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    for src in sorted(HOST_SRC.glob("*.cpp")):
        obj = OBJ / (src.stem + ".cpp.o")
        host_objs.append(obj)
        if _stale(obj, [src, *hdrs]):
            work.append([CXX, *CXX_FLAGS, "-c", str(src), "-o", str(obj)])
    if verbose:
        for w in work:
            print(" ".join(w), file=sys.stderr)
    with cf.ThreadPoolExecutor(jobs) as ex:
        list(ex.map(_run, work))

    dev_so = LIB / "libtcb200.so"
    if _stale(dev_so, dev_objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(dev_so), *map(str, dev_objs)])
    host_so = LIB / "libtc_b200.so"
    if _stale(host_so, host_objs + [dev_so]):
        _run([CXX, "-shared", "-o", str(host_so), *map(str, host_objs), f"-L{LIB}", "-ltcb200",
              "-Wl,-rpath,$ORIGIN", "-pthread"])
    return {"device": dev_so, "front": host_so}


def build_oracle(verbose: bool = False) -> None:
    """TEST INFRASTRUCTURE: the C restatement always, the compiled reference
    (oracle/_ref/libtcref.so) only where /root/reference exists."""
    target = ["all"] if Path("/root/reference/proj/src").is_dir() else ["_ref/libtcoracle.so"]
    r = subprocess.run(["make", "-C", str(ROOT / "oracle"), "-j8", *target],
                       capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    build_oracle(verbose="-v" in sys.argv)
