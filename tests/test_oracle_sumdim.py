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


@pytest.mark.parametrize("etype", ["f32", "f64", "u32", "s64", "bf16", "f16", "e4m3", "e5m2"])
def test_row_sums_fed_in_blocks_match_one_shot(etype):
    """RowSums (the resumable dim-1 state used for 32768^2 full-size checks) fed
    column blocks and split row ranges is bit-identical to one orc_sum_dim."""
    m, n = 37, 53
    X = oracle.fill(etype, "randu", m * n, stream=3)
    want = oracle.sum_dim(etype, 1, X, m, n)
    r = oracle.RowSums(etype, m)
    cols = X.reshape(n, m)
    for c0 in range(0, n, 10):
        blk = cols[c0:c0 + 10].reshape(-1)
        r.add_rows_of(blk, m, 0, 20)
        r.add_rows_of(blk, m, 20, m - 20)
    assert r.final().tobytes() == want.tobytes()


def test_stream_chunks_match_run_chunked():
    """stream_chunks (threaded, in-order) == one sequential run_chunked."""
    from progs import C2
    acc_want, z_want = oracle.run_chunked("f32", C2, ["randu"] * 3, start=1000, count=100003,
                                          scalars=[3.0], kind="ACCU", want_out=True, chunk=4096)
    acc = oracle.Accumulator("f32", "ACCU")
    parts = []
    for off, z in oracle.stream_chunks("f32", C2, ["randu"] * 3, start=1000, count=100003,
                                       scalars=[3.0], chunk=7777, threads=4):
        assert off == sum(p.size for p in parts)
        acc.add(z)
        parts.append(z)
    assert np.concatenate(parts).tobytes() == z_want.tobytes()
    assert acc.final() == acc_want
