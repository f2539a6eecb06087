"""TENSOR v1 text I/O (tc::write_tensor / tc::read_tensor, csrc/host/tensor_io.cpp)
against the compiled reference (src/tensor_io.cpp through oracle/_ref):
byte-identical text, bit-identical values both ways, the reference's own
round-trip / rank-0 / header / malformed-file cases (tests/test_tensor.cpp:
225-271). CPU only."""
import numpy as np
import pytest

import oracles as O
import paper_1307_2100_b200 as T

pytestmark = pytest.mark.skipif(O.ref() is None, reason="reference core not buildable here")

SHAPES = [
    ([3, 1, 4], "+-+", 42, "X"),          # test_tensor.cpp:225-235
    ([], "", 7, "K"),                      # rank 0
    ([2], "-", 3, "v"),
    ([5, 7, 3, 2], "+--+", 11, "T"),
    ([300, 300], "++", 5, "big"),          # > one 65536-value formatting block
    ([17], "+", 9, ""),                    # empty name -> "t"
]


@pytest.mark.parametrize("ext,var,seed,name", SHAPES)
def test_text_is_byte_identical_to_the_reference(ext, var, seed, name):
    assert T.tensor_text(ext, var, seed, name) == O.ref_tensor_text(ext, var, seed, name)


@pytest.mark.parametrize("ext,var,seed,name", SHAPES)
def test_values_round_trip_both_ways(ext, var, seed, name):
    n = int(np.prod(ext)) if ext else 1
    want = O.seeded(n, seed)
    ours = T.tensor_text(ext, var, seed, name)
    theirs = O.ref_tensor_text(ext, var, seed, name)
    got, err = O.ref_read_tensor_text(ours)  # reference reader on our text
    assert err is None and np.array_equal(got.view(np.uint64), want.view(np.uint64))
    got = T.read_tensor_text(theirs)         # our reader on the reference's text
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_header_lines():
    lines = T.tensor_text([2], "-", 1, "v").splitlines()
    assert lines[:6] == ["TENSOR v1", "name v", "rank 1", "extents 2", "variance -",
                         "layout colmajor"]
    assert T.tensor_text([], "", 1, "K").splitlines()[3:5] == ["extents", "variance "]


BAD = [
    "TENSOR v2\n",
    "",
    "TENSOR v1\nname t\nrank 1\nextents 2\nvariance +\nlayout colmajor\n1.0\n",
    "TENSOR v1\nname t\nrank 2\nextents 2\nvariance ++\nlayout colmajor\n1 2\n",
    "TENSOR v1\nname t\nrank 1\nextents 2\nvariance +-\nlayout colmajor\n1 2\n",
    "TENSOR v1\nname t\nrank 1\nextents 2\nvariance x\nlayout colmajor\n1 2\n",
    "TENSOR v1\nname t\nrank 1\nextents 2\nvariance +\nlayout rowmajor\n1 2\n",
    "TENSOR v1\nnom t\nrank 1\n",
    "TENSOR v1\nname t\nrank -1\n",
    "TENSOR v1\nname t\nrank 1\nextents 2\nvariance +\nlayout colmajor\n1 abc\n",
]


@pytest.mark.parametrize("text", BAD)
def test_malformed_files_fail_with_the_reference_message(text):
    _, ref_msg = O.ref_read_tensor_text(text)
    assert ref_msg is not None
    with pytest.raises(ValueError) as e:
        T.read_tensor_text(text)
    assert str(e.value) == ref_msg


def test_explicit_signs_and_exponents_parse_like_the_stream_reader():
    text = "TENSOR v1\nname t\nrank 1\nextents 4\nvariance +\nlayout colmajor\n+1.5 -2e3 3E-2 .5\n"
    ref_vals, err = O.ref_read_tensor_text(text)
    assert err is None
    assert np.array_equal(T.read_tensor_text(text), ref_vals)
