"""tc/metric.hpp through the C-ABI (tcf_invert_metric, tcf_metric_apply):
reference include/tc/metric.hpp:9-34, src/metric.cpp:13-104, known answers
from tests/test_metric.cpp. The inverse is checked against numpy (the
reference's own inverse comes from Eigen, which is absent here: unpinned at
the bit level, pinned through g @ g_inv = 1 and the known answers); the
lowering / raising contractions run on the device against numpy's einsum."""
import numpy as np
import pytest

import paper_1307_2100_b200 as T


def spd(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (n, n))
    return a @ a.T + n * np.eye(n)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 16, 50])
def test_invert_metric_matches_numpy(n):
    g = spd(n, n)
    inv = T.invert_metric(g)
    assert np.allclose(inv, np.linalg.inv(g), rtol=1e-11, atol=1e-13)
    assert np.allclose(g @ inv, np.eye(n), atol=1e-12)


def test_invert_metric_known_answers_and_indefinite():
    assert np.array_equal(T.invert_metric(np.eye(3)), np.eye(3))
    assert np.allclose(T.invert_metric(np.diag([1.0, 4.0, 4.0])), np.diag([1, 0.25, 0.25]))
    # Minkowski-type (indefinite) and a symmetric matrix whose pivots are off the diagonal
    eta = np.diag([-1.0, 1.0, 1.0, 1.0])
    assert np.array_equal(T.invert_metric(eta), eta)
    off = np.array([[0.0, 2.0, 0.0], [2.0, 0.0, 0.0], [0.0, 0.0, 5.0]])
    assert np.allclose(T.invert_metric(off), np.linalg.inv(off), atol=1e-15)


def test_invert_metric_rejections():
    g = np.diag([1.0, 2.0, 3.0])
    g[0, 1] = 0.5
    with pytest.raises(ValueError, match="metric is not symmetric"):
        T.invert_metric(g)
    with pytest.raises(ValueError, match="metric is singular"):
        T.invert_metric(np.diag([1.0, 0.0, 1.0]))
    with pytest.raises(ValueError, match="metric is singular"):
        T.invert_metric(np.ones((3, 3)))
    with pytest.raises(ValueError, match="singular"):
        T.invert_metric(np.diag([1.0, 1e-30, 1.0]))
    with pytest.raises(ValueError, match="metric is numerically singular"):
        T.invert_metric(np.diag([1.0, 1e-13, 1.0]))
    with pytest.raises(ValueError, match="square rank-2"):
        T.invert_metric(np.zeros((2, 3)))
    # asymmetry within 1e-10 of the scale is tolerated
    ok = np.diag([1.0, 2.0, 3.0])
    ok[0, 1] = 1e-12
    T.invert_metric(ok)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,var,mode,n", [
    ((3,), "+", 0, 3), ((3, 3), "++", 1, 3), ((3, 4, 3), "+-+", 0, 3), ((3, 4, 3), "+-+", 2, 3),
    ((5, 64, 7), "-+-", 1, 64), ((130, 9), "++", 0, 130), ((6, 5, 4, 33), "+--+", 3, 33),
])
def test_lower_then_raise_on_the_device(shape, var, mode, n):
    rng = np.random.default_rng(n + mode)
    t = np.asfortranarray(rng.uniform(-1, 1, shape))
    g = spd(n, 100 + n)
    low = T.metric_apply(t, var, mode, g)
    want = np.moveaxis(np.tensordot(t, g, axes=([mode], [0])), -1, mode)
    assert np.linalg.norm(low - want) <= 1e-12 * np.linalg.norm(want)
    lowered = var[:mode] + "-" + var[mode + 1:]
    back = T.metric_apply(low, lowered, mode, g, raise_=True)
    assert np.abs(back - t).max() <= 1e-10


@pytest.mark.gpu
def test_metric_guards_on_the_device_path():
    g = np.diag([1.0, 4.0, 4.0])
    with pytest.raises(ValueError, match="mode is already lowered"):
        T.metric_apply(np.ones(3), "-", 0, g)
    with pytest.raises(ValueError, match="mode is already raised"):
        T.metric_apply(np.ones(3), "+", 0, g, raise_=True)
    with pytest.raises(ValueError, match="mode extent does not match metric dimension"):
        T.metric_apply(np.ones(4), "+", 0, g)
    with pytest.raises(ValueError, match="mode out of range"):
        T.metric_apply(np.ones(3), "+", 1, g)
    assert np.allclose(T.metric_apply(np.ones(3), "+", 0, g), [1, 4, 4])
    assert np.allclose(T.metric_apply(np.array([1.0, 4.0, 4.0]), "-", 0, g, raise_=True), 1.0)
