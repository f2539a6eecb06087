"""Builds and runs the C++ suites (tests/cpp) that restate the reference's
doctest files against the engine's tc:: C++ API (libtc_b200.so)."""
import subprocess
from pathlib import Path

import pytest

import paper_1307_2100_b200 as T

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "cpp"
OUT = SRC / "_build"


def build(name: str) -> Path:
    T.native.front()  # ensures the libraries exist
    OUT.mkdir(exist_ok=True)
    exe = OUT / name
    src = SRC / f"{name}.cpp"
    deps = [src, SRC / "harness.hpp", SRC / "helpers.hpp", T.native.LIB / "libtc_b200.so"]
    if not exe.exists() or any(d.stat().st_mtime > exe.stat().st_mtime for d in deps):
        subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(src),
                        "-o", str(exe), f"-L{T.native.LIB}", "-ltc_b200", "-ltcb200",
                        f"-Wl,-rpath,{T.native.LIB}"], check=True)
    return exe


def run(exe: Path):
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_front_suite():
    run(build("test_front"))


@pytest.mark.gpu
def test_device_suite():
    run(build("test_device"))
