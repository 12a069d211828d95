"""Pins for the oracle's sum(X, dim) (reading R3, column-major storage R2)."""
import os

import numpy as np
import pytest

import oracle
from exactref import rounded_sum, same_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden", "armadillo_sum_dim.txt")


def _gold():
    d = {}
    for line in open(GOLD):
        line = line.strip()
        if line and not line.startswith("#"):
            k, *v = line.split()
            d[k] = [float(x) for x in v]
    return d


def test_2x2_convention_example():
    g = _gold()
    X = np.array(g["X_colmajor"])
    assert list(oracle.sum_dim("f64", 0, X, 2, 2)) == g["dim0"]
    assert list(oracle.sum_dim("f64", 1, X, 2, 2)) == g["dim1"]


@pytest.mark.parametrize("etype", ["f32", "f64", "u32", "s64"])
def test_index_fill_closed_forms(etype):
    m, n = 37, 23
    col = oracle.fill(etype, "colidx", m * n, n_rows=m)  # X(i,j) = j
    row = oracle.fill(etype, "rowidx", m * n, n_rows=m)  # X(i,j) = i
    assert np.array_equal(oracle.sum_dim(etype, 0, col, m, n), np.arange(n) * m)
    assert np.array_equal(oracle.sum_dim(etype, 1, row, m, n), np.arange(m) * n)
    assert np.array_equal(oracle.sum_dim(etype, 1, col, m, n), np.full(m, n * (n - 1) // 2))
    assert np.array_equal(oracle.sum_dim(etype, 0, row, m, n), np.full(n, m * (m - 1) // 2))


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_random_small_against_exact(etype):
    rng = np.random.default_rng(3)
    for m, n in ((1, 1), (1, 9), (9, 1), (5, 7), (16, 3)):
        X = rng.uniform(-1, 1, m * n).astype(oracle.DTYPES[etype])
        M = X.reshape(n, m)  # row j of M is column j of X
        d0 = oracle.sum_dim(etype, 0, X, m, n)
        d1 = oracle.sum_dim(etype, 1, X, m, n)
        for j in range(n):
            assert same_bits(d0[j], rounded_sum(M[j], etype))
        for i in range(m):
            assert same_bits(d1[i], rounded_sum(M[:, i], etype))


def test_empty_dimension_gives_zeros():
    assert np.array_equal(oracle.sum_dim("f64", 0, np.zeros(0), 0, 4), np.zeros(4))
    assert np.array_equal(oracle.sum_dim("f64", 1, np.zeros(0), 3, 0), np.zeros(3))


def test_invariant_totals_agree():
    m, n = 300, 200
    X = oracle.fill("f64", "randu", m * n)
    t = float(oracle.reduce("f64", "ACCU", X))
    t0 = float(oracle.reduce("f64", "ACCU", oracle.sum_dim("f64", 0, X, m, n)))
    t1 = float(oracle.reduce("f64", "ACCU", oracle.sum_dim("f64", 1, X, m, n)))
    assert abs(t0 - t) <= 1e-12 * t and abs(t1 - t) <= 1e-12 * t
