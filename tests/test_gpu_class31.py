"""Reference class 3.1 (COPY+GEMM) and the paper's order-4 experiments on the
device: the 18 order-3 double contractions of the
paper's Table 1 (tests/helpers.hpp:112-139) and the Coupled-Cluster /
General-Relativity shapes of Eq. (xy) (src/bench.cpp:27-33), against the naive
oracle and the live reference executor. Requires a B200."""
import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T
from specgen import table1_expressions

pytestmark = pytest.mark.gpu
TOL = 1e-12


def check(e, x, seed=1):
    L, R = O.operands(e, x, seed)
    got, st = T.execute(e, x, seed=seed)
    want = O.naive(e, x, L, R)
    assert O.max_rel_error(got, want) <= TOL and O.rel_frobenius(got, want) <= TOL, (e, x)
    return got, st


@pytest.mark.parametrize("x", ["a=3,b=4,g=5,e=6", "a=33,b=47,g=29,e=51"])
def test_table1_all_eighteen(dev, x):
    n31 = 0
    for e in table1_expressions():
        cls = T.report(e, x).split("class: ")[1].split("\n")[0]
        got, st = check(e, x)
        if cls == "3.1":
            n31 += 1
            # the crossed stride-1 labels force an operand permutation on the device
            assert st["packed_bytes"] > 0, e
    assert n31 == 4


@pytest.mark.parametrize("contracted", ["cc4d", "gr4d"])
def test_order4_aligned_and_crossed(dev, contracted):
    size = 12
    k = 10 * size if contracted == "cc4d" else 4
    x = f"a={size},b=1,c={size},d={size},i={k},j={k}"
    aligned = "R[+a,+b,+c,+d] = X[+i,+a,+j,+b] * Y[-i,+c,-j,+d]"
    crossed = "R[+a,+b,+c,+d] = X[+i,+a,+j,+b] * Y[-j,+c,-i,+d]"
    ra, sa = check(aligned, x)
    rc, sc = check(crossed, x)
    assert "class: 3.2" in T.report(aligned, x)
    assert "class: 3.1" in T.report(crossed, x)
    live = O.ref_execute(crossed, x, seed=1)
    if live is not None:
        assert O.max_rel_error(rc, live[0]) <= TOL


def test_forced_copy_gemm_equals_auto(dev):
    e, x = "R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "a=40,b=37,g=23,e=41"
    auto, _ = T.execute(e, x)
    forced, st = T.execute(e, x, kernel="COPY+GEMM")
    assert O.max_rel_error(forced, auto) <= TOL


def test_relayout_advice_layout_is_class32_and_correct(dev):
    # the reference's re-layout advice (src/planner.cpp:496-536) moves a 3.1
    # contraction to 3.2; the advised layout runs correctly on the device
    e, x = "R[+b,-e] = A[+a,+b,+g] * B[-g,-a,-e]", "a=16,b=16,g=16,e=16"
    adv = T.report(e, x).split("relayout: ")[1].strip()
    assert adv.startswith("store B as B[-a,-g,-e]") and "class 3.2" in adv
    e2 = "R[+b,-e] = A[+a,+b,+g] * B[-a,-g,-e]"
    assert "class: 3.2" in T.report(e2, x)
    check(e2, x)
