"""The reference's benchmark sweep API (tc::run_bench / tc::write_bench_csv,
include/tc/bench.hpp:13-51) on the device backend: built-in experiments,
forced kernels (unreachable ones as NA rows), the sampled-line verification
(src/bench.cpp:59-112) and the CSV columns. Requires a B200."""
import csv
import io

import pytest

import paper_1307_2100_b200 as T

pytestmark = pytest.mark.gpu
COLS = ["experiment", "expression", "size", "kernel", "backend", "repetitions",
        "median_seconds", "gflops", "packed_bytes"]


def rows(text):
    r = list(csv.reader(io.StringIO(text)))
    # the reference's columns, then `executed` (what the device ran)
    assert r[0] == COLS + ["executed"]
    return [dict(zip(COLS + ["executed"], x)) for x in r[1:]]


def test_square3d_rows_verify_and_report(dev):
    text, ok = T.bench_csv("square3d", sizes=(64, 96), kernels=("GEMM", "COPY+GEMM", "GEMV", "DOT"),
                           repetitions=3, seed=3, verify=True)
    assert ok
    rs = rows(text)
    assert len(rs) == 2 * 2 * 4  # sizes x expressions x kernels
    assert {r["expression"] for r in rs} == {"R[+a,-e] = A[+a,+b,+g] * B[-e,-b,-g]",
                                             "R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]"}
    for r in rs:
        assert r["backend"] == "b200" and r["repetitions"] == "3"
        if r["median_seconds"] != "NA":
            assert float(r["gflops"]) > 0 and float(r["median_seconds"]) > 0


def test_gr4d_and_cc4d_with_sampled_verification(dev):
    for exp in ("gr4d", "cc4d"):
        text, ok = T.bench_csv(exp, sizes=(24,), kernels=("GEMM", "COPY+GEMM", "GER", "DOT"),
                               repetitions=2, seed=5, verify=True)
        assert ok, exp
        assert len(rows(text)) == 2 * 4


def test_custom_experiment_and_errors(dev):
    text, ok = T.bench_csv("custom", sizes=(1,), kernels=("GEMM",), repetitions=2, verify=True,
                           custom_expr="C[+i,+j] = A[+i,+k] * B[-k,+j]",
                           custom_extents="i=130,j=70,k=50")
    assert ok and rows(text)[0]["expression"] == "C[+i,+j] = A[+i,+k] * B[-k,+j]"
    with pytest.raises(ValueError, match="unknown experiment"):
        T.bench_csv("nope", sizes=(4,))
    with pytest.raises(ValueError, match="repetitions must be >= 1"):
        T.bench_csv("square3d", sizes=(4,), repetitions=0)
    with pytest.raises(ValueError, match="size sweep must be nonempty"):
        T.bench_csv("square3d", sizes=())


def test_execute_loop_with_pinned_recycled_blocks(dev):
    """tc::execute in a loop on large tensors (tc::run_bench repetitions): the
    operands are page-locked on the first call and every result lands in a
    recycled pinned block, evaluated through the streamed pipeline; the
    harness's sampled-line verification must pass on every configuration."""
    for e, x in [("C[+a,+b,+c] = A[+a,+k,+c] * B[-k,+b]", "a=256,b=256,c=64,k=256"),
                 ("C[+i,+j] = A[+i,+k,+l] * B[-k,-l,+j]", "i=512,j=512,k=64,l=64"),
                 ("C[+a,+b,+i,+j] = A[+a,+b,+k,+l] * B[-k,-l,+i,+j]",
                  "a=256,b=64,i=32,j=32,k=32,l=32")]:
        text, ok = T.bench_csv("custom", sizes=(1,), kernels=("GEMM",), repetitions=4,
                               verify=True, custom_expr=e, custom_extents=x)
        assert ok, (e, x, text)


def test_forced_kernels_are_marked_and_sliced_backend_runs_them(dev):
    # b200: every forced kernel runs the contraction's device recipe, marked
    text, ok = T.bench_csv("square3d", sizes=(24,), kernels=("GEMM", "GER", "DOT"),
                           repetitions=2, verify=True)
    assert ok
    for r in rows(text):
        if r["median_seconds"] != "NA":
            assert r["executed"].startswith(("L1", "L2", "L3", "L4")), r
    # b200-sliced: the forced plan's loop nest, one device call per slice
    text, ok = T.bench_csv("square3d", sizes=(12,), kernels=("GEMM", "GER", "DOT"),
                           backend="b200-sliced", repetitions=1, verify=True)
    assert ok
    rs = rows(text)
    for r in rs:
        if r["median_seconds"] != "NA":
            assert r["executed"] == "sliced " + r["kernel"], r
            assert r["backend"] == "b200-sliced"
