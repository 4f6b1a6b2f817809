"""CPU: the matrix file format and the CLI number formatting against the
reference itself (matrix_io.hpp:25-117, hexfloat.hpp:18-58,
experiment.hpp:376-380, via oracle/_ref).  The reference builds only where
/root/reference exists; the fixtures it writes are committed as goldens."""
import math
import os

import numpy as np
import pytest

from paper_1210_0800_b200 import matrix_io
from paper_1210_0800_b200.cli import shortest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def rio():
    import oracle

    r = oracle.ref_io()
    if r is None:
        pytest.skip("reference build not available")
    return r


def special_matrix(rng, L, m, n):
    a = rng.standard_normal((n, m, 2, L)) * np.ldexp(1.0, rng.integers(-60, 60, size=(n, m, 2, L)))
    sp = [0.0, -0.0, 5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, 1.0]
    k = min(a.size, len(sp))
    a.reshape(-1)[:k] = sp[:k]
    return a


@pytest.mark.parametrize("L", [1, 2, 4])
def test_write_matches_reference(rio, L):
    rng = np.random.default_rng(L)
    for (m, n) in [(1, 1), (3, 2), (7, 7)]:
        a = special_matrix(rng, L, m, n)
        assert matrix_io.matrix_text(a) == rio.write_matrix(a)


@pytest.mark.parametrize("L", [1, 2, 4])
def test_read_matches_reference(rio, L):
    rng = np.random.default_rng(10 + L)
    a = special_matrix(rng, L, 5, 4)  # limbs not normalised: read renormalises
    text = matrix_io.matrix_text(a)
    got, gl = matrix_io.parse_matrix(text)
    want, wl = rio.read_matrix(text)
    assert gl == wl == L
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # what we read writes back as the reference writes it
    assert matrix_io.matrix_text(got) == rio.write_matrix(want)


BAD = [
    ("", 1), ("2 1\n", 1), ("2 x d\n", 1), ("1 2 d\n", 1), ("2 1 qq\n", 1),
    ("2 1 d\n0x1p+0 0x0p+0\n", 3), ("2 1 d\n0x1p+0 0x0p+0\n0xZp+0 0x0p+0\n", 3),
    ("2 1 d\n0x1p+0\n0x1p+0 0x0p+0\n", 2), ("1 1 d\n1.5 2\nextra\n", 3),
    ("1 1 d\ninf 0\n", 2), ("1 1 dd\n1 2 3 4\n", None), ("1 1 dd\n1 2 3\n", 2),
    ("1 1 d\n0x1.8p1 -.5e1\n", None),
    ("1 1 d\n 0x1p-3   1e5 \n\n\n", None),
]


@pytest.mark.parametrize("text,line", BAD)
def test_parse_errors_match_reference(rio, text, line):
    try:
        want = rio.read_matrix(text)
        want_line = None
    except ValueError as e:
        want, want_line = None, e.args[0]
    try:
        got = matrix_io.parse_matrix(text)
        got_line = None
    except matrix_io.parse_error as e:
        got, got_line = None, e.line
    assert got_line == want_line
    if want is not None:
        assert np.array_equal(got[0].view(np.uint64), want[0].view(np.uint64))
    if line is not None:
        assert got_line == line


def test_shortest_matches_reference(rio):
    rng = np.random.default_rng(5)
    vals = list(rng.standard_normal(2000) * np.ldexp(1.0, rng.integers(-1000, 1000, 2000)))
    vals += [0.0, -0.0, 1e-30, 0.0001, 1e-5, 123456.0, 1e16, 1e21, 0.1, 5e-324, 1.7976931348623157e308,
             1.0, 10.0, 1e-4, 12.5, 100.0, 1e15, 3.0e-7]
    want = rio.shortest_many(vals)
    for v, w in zip(vals, want):
        assert shortest(v) == w, v


def test_golden_file_roundtrip():
    # fixture written by the reference's write_matrix (tests/golden/make_golden.py)
    path = os.path.join(GOLDEN, "matrix_cqd_3x2.mat")
    text = open(path).read()
    a, L = matrix_io.parse_matrix(text)
    assert L == 4 and a.shape == (2, 3, 2, 4)
    assert matrix_io.matrix_text(a) == text
