"""Pins for the oracle's 8-bit storage types (reading R25): E4M3 / E5M2 values
are decoded exactly, the expression is evaluated as an f32 program, and each
element's value is rounded once (nearest-even, saturating) to the 8-bit format;
reductions return f32.  Checked against torch's float8 dtypes (a library
routine) for decoding and in-range rounding, against the closed-form
saturation rule, against the f32 oracle (pinned separately) composed with
torch's rounding, and against exact rational sums."""
import random
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle
from progs import P, n_operands, random_program

FP8 = {"e4m3": torch.float8_e4m3fn, "e5m2": torch.float8_e5m2}
MAXFIN = {"e4m3": 448.0, "e5m2": 57344.0}


def torch_decode(etype, bits) -> np.ndarray:
    b = torch.from_numpy(np.asarray(bits, dtype=np.uint8).copy())
    return b.view(FP8[etype]).to(torch.float64).numpy()


def torch_round(etype, x) -> np.ndarray:
    """torch's (non-saturating) RNE cast, applied to f32 values."""
    t = torch.from_numpy(np.asarray(x, dtype=np.float32).copy())
    return t.to(FP8[etype]).view(torch.uint8).numpy()


@pytest.mark.parametrize("etype", FP8)
def test_decode_all_patterns(etype):
    mine = oracle.fp8_table(etype)
    ref = torch_decode(etype, np.arange(256))
    assert np.array_equal(np.isnan(mine), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert np.array_equal(mine[ok], ref[ok])
    assert np.nanmax(mine[np.isfinite(mine)]) == MAXFIN[etype]


@pytest.mark.parametrize("etype", FP8)
def test_round_in_range_matches_torch(etype):
    rng = np.random.default_rng(5)
    x = (rng.uniform(-1, 1, 30000) * 2.0 ** rng.integers(-22, 17, 30000)).astype(np.float32)
    # every midpoint between neighbouring finite values, and the values themselves
    vals = np.unique(oracle.fp8_table(etype)[np.isfinite(oracle.fp8_table(etype))])
    mids = ((vals[1:] + vals[:-1]) / 2).astype(np.float32)
    x = np.concatenate([x, vals.astype(np.float32), mids, -mids])
    ref = torch_round(etype, x)
    finite_ref = np.isfinite(torch_decode(etype, ref))
    mine = np.array([oracle.fp8_from_double(etype, float(v)) for v in x], dtype=np.uint8)
    assert np.array_equal(mine[finite_ref], ref[finite_ref])
    # everything torch sends past the format (NaN / inf) saturates here (R25)
    sat = ~finite_ref & ~np.isnan(x)
    assert sat.sum() > 0
    assert np.array_equal(oracle.fp8_table(etype)[mine[sat]], np.sign(x[sat]) * MAXFIN[etype])


@pytest.mark.parametrize("etype", FP8)
def test_special_values(etype):
    f = lambda x: oracle.fp8_from_double(etype, x)  # noqa: E731
    tab = oracle.fp8_table(etype)
    assert f(0.0) == 0 and f(-0.0) == 0x80
    assert np.isnan(tab[f(float("nan"))])
    assert tab[f(float("inf"))] == MAXFIN[etype] and tab[f(-float("inf"))] == -MAXFIN[etype]
    assert tab[f(1e30)] == MAXFIN[etype]
    assert tab[f(1.0)] == 1.0 and tab[f(3.0)] == 3.0
    # ties to even: 1 + half an ulp -> 1 ; 1 + 3 half-ulps -> 1 + 2 ulps
    ulp = 2.0 ** -3 if etype == "e4m3" else 2.0 ** -2
    assert tab[f(1 + ulp / 2)] == 1.0
    assert tab[f(1 + 1.5 * ulp)] == 1 + 2 * ulp
    # smallest subnormal and half of it (tie -> 0)
    tiny = 2.0 ** -9 if etype == "e4m3" else 2.0 ** -16
    assert tab[f(tiny)] == tiny and tab[f(tiny / 2)] == 0.0 and tab[f(tiny * 0.75)] == tiny


@pytest.mark.parametrize("etype", FP8)
def test_fill_randu_grid(etype):
    n = 5000
    got = oracle.to_float(etype, oracle.fill(etype, "randu", n, stream=3))
    shift, scale = (60, 16.0) if etype == "e4m3" else (61, 8.0)
    want = np.array([(oracle.hash64(42, 3, i) >> shift) / scale for i in range(n)])
    assert np.array_equal(got, want)
    ones = oracle.to_float(etype, oracle.fill(etype, "ones", 10))
    assert np.all(ones == 1.0)


@pytest.mark.parametrize("etype", FP8)
def test_programs_are_f32_programs_rounded_once(etype):
    rng = random.Random(11)
    for trial in range(30):
        prog = random_program(rng, 3, "f32", n_ops=3)
        k = n_operands(prog)
        ops = [oracle.fill(etype, "randu", 2000, seed=trial, stream=s) for s in range(k)]
        sc = [2.5, -0.75]
        got = oracle.eval_program(etype, prog, ops, sc)
        dec = [torch_decode(etype, o).astype(np.float32) for o in ops]
        z32 = oracle.eval_program("f32", prog, dec, sc)
        ref = torch_round(etype, z32)
        fin = np.isfinite(torch_decode(etype, ref))
        assert np.array_equal(got[fin], ref[fin]), prog
        nan = np.isnan(z32)
        assert np.all(np.isnan(oracle.to_float(etype, got[nan])))
        sat = ~fin & ~nan
        assert np.array_equal(np.abs(oracle.to_float(etype, got[sat])),
                              np.full(sat.sum(), MAXFIN[etype]))


@pytest.mark.parametrize("etype", FP8)
def test_reductions_exact(etype):
    v = oracle.fill(etype, "randu", 3001, stream=1)
    x = [Fraction(float(t)) for t in oracle.to_float(etype, v)]
    acc = oracle.reduce(etype, "ACCU", v)
    assert acc.dtype == np.float32 and acc == np.float32(float(sum(x)))
    mm = oracle.reduce(etype, "MINMAX", v)
    assert mm[0] == float(min(x)) and mm[1] == float(max(x))
    n2 = oracle.reduce(etype, "NORM2", v)
    assert abs(float(n2) - float(sum(t * t for t in x)) ** 0.5) <= 2.0 ** -23 * float(n2)
    mean = oracle.stats(etype, "MEAN", v)
    assert mean.dtype == np.float32 and mean == np.float32(float(sum(x) / len(x)))
    im = oracle.stats(etype, "INDEX_MAX", v)
    assert x[im] == max(x) and all(t < max(x) for t in x[:im])


@pytest.mark.parametrize("etype", FP8)
def test_sum_dim_exact(etype):
    m, n = 37, 11
    X = oracle.fill(etype, "randu", m * n, stream=2)
    F = oracle.to_float(etype, X).reshape(n, m)  # column-major: column j = row j here
    col = oracle.sum_dim(etype, 0, X, m, n)
    row = oracle.sum_dim(etype, 1, X, m, n)
    assert col.dtype == np.float32 and row.dtype == np.float32
    assert np.array_equal(col, np.array([float(sum(Fraction(t) for t in F[j])) for j in range(n)],
                                        dtype=np.float32))
    assert np.array_equal(row, np.array([float(sum(Fraction(t) for t in F[:, i]))
                                         for i in range(m)], dtype=np.float32))
