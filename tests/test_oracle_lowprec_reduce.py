"""Pins for the oracle's reductions, statistics and dim sums on the low-
precision types (readings R24 / R25), branch by branch, against exact rational
arithmetic (``fractions``) and mpmath square roots rounded by tests/exactref.py.

bf16 / f16 (R24): every result is the exact value rounded ONCE to the 16-bit
format (nearest-even).  E4M3 / E5M2 (R25): the 8-bit values are summed exactly
and the result is rounded once to f32.  Branches pinned here: ACCU, NORM2,
MIN / MAX / MINMAX, MEAN, VAR, STDDEV, INDEX_MIN / INDEX_MAX (first
occurrence) and sum(X, 0) / sum(X, 1) (R3) — each on random data, on data
with repeated extremes (index ties) and on closed forms.
"""
import math
import struct
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle
from exactref import _mp_to_fraction, round_fraction

HALF = ("bf16", "f16")
FP8 = ("e4m3", "e5m2")
LOWP = HALF + FP8


def result_type(etype):
    """Format the oracle rounds reductions to (R24: the 16-bit type; R25: f32)."""
    return "f32" if etype in FP8 else etype


def values(etype, a):
    """Exact values of an array of the low-precision type, as Fractions."""
    return [Fraction(float(v)) for v in oracle.to_float(etype, a)]


def result_value(etype, r):
    """Python float of an oracle reduction result (16-bit bits or f32)."""
    r = np.asarray(r)
    if etype in FP8:
        return float(r)
    if etype == "bf16":
        return struct.unpack("<f", struct.pack("<I", int(r.view(np.uint16)) << 16))[0]
    return float(r.astype(np.float16))


def rounded(fr: Fraction, etype) -> float:
    return round_fraction(fr, result_type(etype))


def rounded_sqrt(fr: Fraction, etype) -> float:
    """sqrt of an exact rational, rounded once: mpmath at 600 bits cannot sit on
    the wrong side of a rounding midpoint unless it is exact (then it is exact)."""
    if fr == 0:
        return 0.0
    with mpmath.workprec(600):
        r = mpmath.sqrt(mpmath.mpf(fr.numerator) / mpmath.mpf(fr.denominator))
        return round_fraction(_mp_to_fraction(r), result_type(etype))


def same(got: float, want: float) -> bool:
    if math.isnan(want):
        return math.isnan(got)
    return got == want and math.copysign(1, got) == math.copysign(1, want)


def datasets(etype):
    """(name, array) cases: the generator's randu on several sizes, a signed
    spread (iota scaled through the oracle's own rounding is avoided: values
    are built from bit patterns), and arrays with repeated extremes."""
    out = []
    for n, s in ((1, 3), (2, 4), (7, 5), (300, 6), (4099, 7)):
        out.append((f"randu{n}", oracle.fill(etype, "randu", n, stream=s)))
    rng = np.random.default_rng(11)
    if etype in HALF:
        bits = rng.integers(0, 1 << 16, 3000, dtype=np.uint32).astype(np.uint16)
        vals = oracle.to_float(etype, bits.view(oracle.DTYPES[etype]))
        # finite, and small enough that squares and sums stay in range
        keep = np.isfinite(vals) & (np.abs(vals) < 64)
        out.append(("signed_bits", bits[keep].view(oracle.DTYPES[etype])))
    else:
        bits = rng.integers(0, 256, 3000, dtype=np.uint32).astype(np.uint8)
        vals = oracle.to_float(etype, bits)
        keep = np.isfinite(vals)
        out.append(("signed_bits", bits[keep]))
    ties = oracle.fill(etype, "randu", 500, stream=9).copy()
    ties[[17, 230, 499]] = ties[[3, 3, 3]]  # a repeated value somewhere in the middle
    out.append(("ties", ties))
    return out


@pytest.mark.parametrize("etype", LOWP)
def test_accu_norm2_minmax(etype):
    for name, a in datasets(etype):
        x = values(etype, a)
        s = sum(x, Fraction(0))
        assert same(result_value(etype, oracle.reduce(etype, "ACCU", a)), rounded(s, etype)), name
        n2 = sum((t * t for t in x), Fraction(0))
        assert same(result_value(etype, oracle.reduce(etype, "NORM2", a)),
                    rounded_sqrt(n2, etype)), name
        mm = oracle.reduce(etype, "MINMAX", a)
        assert result_value(etype, mm[0]) == float(min(x)), name
        assert result_value(etype, mm[1]) == float(max(x)), name
        assert result_value(etype, oracle.reduce(etype, "MIN", a)) == float(min(x)), name
        assert result_value(etype, oracle.reduce(etype, "MAX", a)) == float(max(x)), name


@pytest.mark.parametrize("etype", LOWP)
def test_mean_var_stddev(etype):
    for name, a in datasets(etype):
        x = values(etype, a)
        n = len(x)
        mean = sum(x, Fraction(0)) / n
        var = sum(((t - mean) ** 2 for t in x), Fraction(0)) / (n - 1) if n > 1 else Fraction(0)
        assert same(result_value(etype, oracle.stats(etype, "MEAN", a)), rounded(mean, etype)), name
        assert same(result_value(etype, oracle.stats(etype, "VAR", a)), rounded(var, etype)), name
        assert same(result_value(etype, oracle.stats(etype, "STDDEV", a)),
                    rounded_sqrt(var, etype)), name


@pytest.mark.parametrize("etype", LOWP)
def test_index_min_max_first_occurrence(etype):
    for name, a in datasets(etype):
        x = values(etype, a)
        lo, hi = min(x), max(x)
        assert oracle.stats(etype, "INDEX_MIN", a) == x.index(lo), name  # list.index: first
        assert oracle.stats(etype, "INDEX_MAX", a) == x.index(hi), name
    # hand-made ties: extremes repeated, the first occurrence wins
    b = oracle.fill(etype, "randu", 64, stream=2).copy()
    xs = values(etype, b)
    i_lo, i_hi = xs.index(min(xs)), xs.index(max(xs))
    b[40], b[63] = b[i_lo], b[i_hi]
    assert oracle.stats(etype, "INDEX_MIN", b) == min(i_lo, 40)
    assert oracle.stats(etype, "INDEX_MAX", b) == min(i_hi, 63)


@pytest.mark.parametrize("etype", LOWP)
def test_closed_forms(etype):
    ones = oracle.fill(etype, "ones", 4096)
    # accu(ones(n)) = n; norm2(ones(4^k)) = 2^k; mean(ones) = 1, var(ones) = 0
    assert result_value(etype, oracle.reduce(etype, "ACCU", ones)) == rounded(Fraction(4096), etype)
    assert result_value(etype, oracle.reduce(etype, "NORM2", ones)) == 64.0
    assert result_value(etype, oracle.stats(etype, "MEAN", ones)) == 1.0
    assert result_value(etype, oracle.stats(etype, "VAR", ones)) == 0.0
    assert result_value(etype, oracle.stats(etype, "STDDEV", ones)) == 0.0
    # norm2 of a basis vector e_k is 1
    z = oracle.fill(etype, "zeros", 999).copy()
    z[500] = ones[0]
    assert result_value(etype, oracle.reduce(etype, "NORM2", z)) == 1.0
    assert oracle.stats(etype, "INDEX_MAX", z) == 500 and oracle.stats(etype, "INDEX_MIN", z) == 0


@pytest.mark.parametrize("etype", LOWP)
@pytest.mark.parametrize("shape", [(1, 1), (1, 9), (9, 1), (37, 11), (64, 33)])
def test_sum_dim_exact(etype, shape):
    m, n = shape
    X = oracle.fill(etype, "randu", m * n, stream=12)
    F = values(etype, X)
    col = oracle.sum_dim(etype, 0, X, m, n)
    row = oracle.sum_dim(etype, 1, X, m, n)
    for j in range(n):
        want = rounded(sum(F[j * m:(j + 1) * m], Fraction(0)), etype)
        assert same(result_value(etype, col[j]), want), ("dim0", j)
    for i in range(m):
        want = rounded(sum((F[i + j * m] for j in range(n)), Fraction(0)), etype)
        assert same(result_value(etype, row[i]), want), ("dim1", i)


@pytest.mark.parametrize("etype", LOWP)
def test_sum_dim_index_closed_forms(etype):
    """X(i,j) = j -> dim0[j] = j*m (exact while j*m is representable);
    X(i,j) = i -> dim1[i] = i*n; small enough that every value is exact."""
    m, n = 5, 7
    col = oracle.fill(etype, "colidx", m * n, n_rows=m)
    row = oracle.fill(etype, "rowidx", m * n, n_rows=m)
    d0 = [result_value(etype, v) for v in oracle.sum_dim(etype, 0, col, m, n)]
    d1 = [result_value(etype, v) for v in oracle.sum_dim(etype, 1, row, m, n)]
    assert d0 == [float(j * m) for j in range(n)]
    assert d1 == [float(i * n) for i in range(m)]
