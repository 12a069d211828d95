"""Pins for the oracle's input generator."""
import os

import numpy as np

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "splitmix64_vigna.txt")


def _vigna():
    rows = []
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        i, h = line.split()
        rows.append((int(i), int(h, 16)))
    return rows


def test_splitmix64_matches_vigna_reference():
    rows = _vigna()
    assert len(rows) >= 3
    for i, h in rows:
        assert oracle.hash64(0, 0, i) == h


def test_seed_and_stream_change_the_sequence():
    a = [oracle.hash64(42, 0, i) for i in range(64)]
    b = [oracle.hash64(42, 1, i) for i in range(64)]
    c = [oracle.hash64(43, 0, i) for i in range(64)]
    assert len(set(a) & set(b)) == 0 and len(set(a) & set(c)) == 0


def test_randu_f32_is_uniform_grid_in_unit_interval():
    x = oracle.fill("f32", "randu", 1 << 20)
    assert x.dtype == np.float32
    assert x.min() >= 0.0 and x.max() < 1.0
    # every value is a multiple of 2^-24 (fill::randu on a 24-bit grid)
    assert np.all(np.floor(x.astype(np.float64) * 2**24) == x.astype(np.float64) * 2**24)
    # mean 1/2, variance 1/12 (statistical; 8 sigma bounds)
    n = x.size
    assert abs(x.mean(dtype=np.float64) - 0.5) < 8 * np.sqrt(1 / 12 / n)
    assert abs(x.var(dtype=np.float64) - 1 / 12) < 0.002


def test_randu_mappings_use_the_documented_bits():
    h = [oracle.hash64(42, 3, i) for i in range(8)]
    f32 = oracle.fill("f32", "randu", 8, stream=3)
    f64 = oracle.fill("f64", "randu", 8, stream=3)
    u32 = oracle.fill("u32", "randu", 8, stream=3)
    s64 = oracle.fill("s64", "randu", 8, stream=3)
    for i in range(8):
        assert float(f32[i]) == (h[i] >> 40) / 2.0**24
        assert float(f64[i]) == (h[i] >> 11) / 2.0**53
        assert int(u32[i]) == h[i] >> 32
        assert int(s64[i]) == (h[i] - (1 << 64) if h[i] >= 1 << 63 else h[i])


def test_fill_start_offset_is_global_index():
    full = oracle.fill("f64", "randu", 1000, stream=2)
    part = oracle.fill("f64", "randu", 300, stream=2, start=500)
    assert np.array_equal(full[500:800], part)


def test_structured_fills_closed_forms():
    m, n = 7, 5
    assert np.array_equal(oracle.fill("f32", "ones", 10), np.ones(10, np.float32))
    assert np.array_equal(oracle.fill("u32", "iota", 10), np.arange(10, dtype=np.uint32))
    assert np.array_equal(oracle.fill("s64", "modk", 10, k=3), np.arange(10) % 3)
    col = oracle.fill("f64", "colidx", m * n, n_rows=m).reshape(n, m)  # column-major
    row = oracle.fill("f64", "rowidx", m * n, n_rows=m).reshape(n, m)
    for j in range(n):
        assert np.all(col[j] == j)
        assert np.array_equal(row[j], np.arange(m))
