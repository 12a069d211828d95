"""Pins for the oracle's statistics (reading R22): mean, var (n-1
normalisation), stddev, index_min / index_max (first occurrence)."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from exactref import round_fraction, to_np
import mpmath


def exact_var(v):
    xs = [Fraction(float(x)) for x in v]
    n = len(xs)
    mean = sum(xs, Fraction(0)) / n
    return sum(((x - mean) ** 2 for x in xs), Fraction(0)) / (n - 1) if n > 1 else Fraction(0)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_closed_forms(etype):
    dt = oracle.DTYPES[etype]
    for n in (2, 3, 10, 1000, 100001):
        v = np.arange(1, n + 1, dtype=dt)
        assert oracle.stats(etype, "MEAN", v) == dt((n + 1) / 2)
        # var(1..n) = n(n+1)/12 exactly
        want = to_np(round_fraction(Fraction(n * (n + 1), 12), etype), etype)
        assert oracle.stats(etype, "VAR", v) == want
    c = np.full(777, 3.25, dt)
    assert oracle.stats(etype, "VAR", c) == 0 and oracle.stats(etype, "MEAN", c) == dt(3.25)
    assert oracle.stats(etype, "VAR", np.array([1.0, 4.0], dt)) == 4.5  # (a-b)^2/2
    assert oracle.stats(etype, "VAR", np.array([5.0], dt)) == 0        # n == 1
    assert oracle.stats(etype, "STDDEV", np.array([1.0, 4.0, 1.0, 4.0], dt)) == dt(np.sqrt(3.0))


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_var_scale_invariance_far_from_one(etype):
    """var(2^e v) = 2^(2e) var(v) exactly for power-of-two scalings that put the
    deviations' squares outside eT's range (the device's f64 route, R12/R22):
    pins the oracle's squares and sums as wider than eT."""
    dt = oracle.DTYPES[etype]
    v = np.array([1.0, 4.0, 1.0, 4.0, 7.0], dt)          # mean 3.4, var 6.3
    base = oracle.stats(etype, "VAR", v)
    e = 62 if etype == "f32" else 500
    for k in (e, -e):
        s = 2.0 ** k
        got = oracle.stats(etype, "VAR", (v * dt(s)).astype(dt))
        want = to_np(round_fraction(exact_var(v) * Fraction(2) ** (2 * k), etype), etype)
        assert got == want, (k, got, want)
        if np.isfinite(want) and want != 0 and np.isfinite(base * dt(s) * dt(s)):
            assert got == base * dt(s) * dt(s)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_random_against_exact_rationals(etype):
    rng = np.random.default_rng(12)
    dt = oracle.DTYPES[etype]
    for n in (2, 7, 50, 301):
        for shift in (0.0, 1000.0):
            v = (rng.normal(size=n) + shift).astype(dt)
            ev = exact_var(v)
            assert oracle.stats(etype, "VAR", v) == to_np(round_fraction(ev, etype), etype)
            m = sum((Fraction(float(x)) for x in v), Fraction(0)) / n
            assert oracle.stats(etype, "MEAN", v) == to_np(round_fraction(m, etype), etype)
            with mpmath.workprec(300):
                sd = mpmath.sqrt(mpmath.mpf(ev.numerator) / ev.denominator)
                sign, man, exp, _ = sd._mpf_
                f = Fraction(int(man)) * (Fraction(2) ** int(exp))
            assert oracle.stats(etype, "STDDEV", v) == to_np(round_fraction(f, etype), etype)


@pytest.mark.parametrize("etype", ["f32", "f64", "u32", "s64"])
def test_index_min_max_first_occurrence(etype):
    dt = oracle.DTYPES[etype]
    v = np.array([3, 1, 2, 1, 9, 0, 9, 0, 5], dt)
    assert oracle.stats(etype, "INDEX_MIN", v) == 5
    assert oracle.stats(etype, "INDEX_MAX", v) == 4
    rng = np.random.default_rng(3)
    w = rng.integers(0, 50, 10_000).astype(dt)
    assert oracle.stats(etype, "INDEX_MIN", w) == int(np.argmin(w))  # numpy: first occurrence
    assert oracle.stats(etype, "INDEX_MAX", w) == int(np.argmax(w))


def test_stats_errors():
    with pytest.raises(oracle.OracleError):
        oracle.stats("f32", "MEAN", np.zeros(0, np.float32))
    with pytest.raises(oracle.OracleError):
        oracle.stats("u32", "VAR", np.ones(3, np.uint32))
    with pytest.raises(oracle.OracleError):
        oracle.stats("f64", "INDEX_MIN", np.zeros(0))
