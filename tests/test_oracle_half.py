"""Pins for the oracle's 16-bit float types (reading R24): bf16 and f16 values
are rounded once per node from the exact result (round-half-to-even), checked
against exact rational arithmetic / mpmath rounded by tests/exactref.py."""
import math
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
from exactref import _mp_to_fraction, round_fraction
import mpmath

HALF = ("bf16", "f16")


def bits_to_float(etype, b: int) -> float:
    if etype == "bf16":
        return struct.unpack("<f", struct.pack("<I", (int(b) & 0xFFFF) << 16))[0]
    return float(np.array([b], np.uint16).view(np.float16)[0])


def float_to_bits(etype, x: float) -> int:
    """Bits of an exactly representable value (nan -> canonical)."""
    if etype == "bf16":
        if math.isnan(x):
            return 0x7FC0
        return struct.unpack("<I", struct.pack("<f", x))[0] >> 16
    if math.isnan(x):
        return 0x7E00
    return int(np.array([x], np.float16).view(np.uint16)[0])


def exact_round_bits(etype, fr: Fraction, neg_zero=False) -> int:
    return float_to_bits(etype, round_fraction(fr, etype, neg_zero))


def samples(etype, n, seed):
    rng = np.random.default_rng(seed)
    b = rng.integers(0, 1 << 16, n, dtype=np.uint32).astype(np.uint16)
    vals = [bits_to_float(etype, int(x)) for x in b]
    keep = [int(x) for x, v in zip(b, vals) if math.isfinite(v)]
    special = [float_to_bits(etype, v) for v in (0.0, -0.0, 1.0, -1.0, 0.5, 3.0, 1e-3, 100.0)]
    return np.array(special + keep, dtype=np.uint16)


def as_array(etype, bits):
    return np.asarray(bits, dtype=np.uint16).view(oracle.DTYPES[etype])


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("op", ["ADD", "SUB", "MUL", "DIV"])
def test_binary_ops_correctly_rounded(etype, op):
    a = samples(etype, 400, 1)
    b = samples(etype, 400, 2)[: a.size]
    a = a[: b.size]
    got = oracle.eval_program(etype, [("LOAD", 0), ("LOAD", 1), (op, 0)],
                              [as_array(etype, a), as_array(etype, b)]).view(np.uint16)
    for i in range(a.size):
        x, y = bits_to_float(etype, a[i]), bits_to_float(etype, b[i])
        if op == "DIV" and y == 0:
            continue
        fx, fy = Fraction(x), Fraction(y)
        r = {"ADD": fx + fy, "SUB": fx - fy, "MUL": fx * fy, "DIV": fx / fy if y else None}[op]
        if r == 0:  # sign of exact zero per IEEE
            nz = (op == "MUL" or op == "DIV") and (math.copysign(1, x) * math.copysign(1, y) < 0)
            nz = nz or (op == "ADD" and math.copysign(1, x) < 0 and math.copysign(1, y) < 0)
            nz = nz or (op == "SUB" and math.copysign(1, x) < 0 and math.copysign(1, y) > 0)
            want = float_to_bits(etype, -0.0 if nz else 0.0)
        else:
            want = exact_round_bits(etype, r)
        assert int(got[i]) == want, (op, x, y, hex(got[i]), hex(want))


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("op", ["SQRT", "EXP", "LOG", "NEG", "ABS", "SQUARE"])
def test_unary_ops_correctly_rounded(etype, op):
    a = samples(etype, 500, 3)
    got = oracle.eval_program(etype, [("LOAD", 0), (op, 0)], [as_array(etype, a)]).view(np.uint16)
    for i in range(a.size):
        x = bits_to_float(etype, a[i])
        if op == "NEG":
            assert int(got[i]) == int(a[i]) ^ 0x8000
            continue
        if op == "ABS":
            assert int(got[i]) == int(a[i]) & 0x7FFF
            continue
        if op == "SQUARE":
            want = exact_round_bits(etype, Fraction(x) ** 2) if x else float_to_bits(etype, 0.0)
        elif op == "SQRT":
            if x < 0:
                assert math.isnan(bits_to_float(etype, got[i]))
                continue
            if x == 0:
                assert int(got[i]) == int(a[i])
                continue
            with mpmath.workprec(300):
                want = exact_round_bits(etype, _mp_to_fraction(mpmath.sqrt(mpmath.mpf(x))))
        elif op == "EXP":
            if x == 0:
                want = float_to_bits(etype, 1.0)
            elif x > 100 or x < -110:  # certain overflow / underflow for both formats
                want = float_to_bits(etype, math.inf if x > 0 else 0.0)
            else:
                with mpmath.workprec(300):
                    want = exact_round_bits(etype, _mp_to_fraction(mpmath.exp(mpmath.mpf(x))))
        else:  # LOG
            if x < 0 or (x == 0):
                g = bits_to_float(etype, got[i])
                assert math.isnan(g) if x < 0 else g == -math.inf
                continue
            if x == 1:
                want = float_to_bits(etype, 0.0)
            else:
                with mpmath.workprec(300):
                    want = exact_round_bits(etype, _mp_to_fraction(mpmath.log(mpmath.mpf(x))))
        assert int(got[i]) == want, (op, x, hex(got[i]), hex(want))


@pytest.mark.parametrize("etype", HALF)
def test_reductions_rounded_once(etype):
    rng = np.random.default_rng(4)
    for n in (1, 5, 300, 5000):
        a = oracle.fill(etype, "randu", n, stream=rng.integers(0, 9))
        vals = [Fraction(bits_to_float(etype, int(b))) for b in a.view(np.uint16)]
        got = int(np.asarray(oracle.reduce(etype, "ACCU", a)).view(np.uint16))
        assert got == exact_round_bits(etype, sum(vals, Fraction(0)))
        mm = oracle.reduce(etype, "MINMAX", a).view(np.uint16)
        fl = [bits_to_float(etype, int(b)) for b in a.view(np.uint16)]
        assert bits_to_float(etype, mm[0]) == min(fl) and bits_to_float(etype, mm[1]) == max(fl)
        if n > 1:
            m = sum(vals, Fraction(0)) / n
            var = sum(((v - m) ** 2 for v in vals), Fraction(0)) / (n - 1)
            gv = int(np.asarray(oracle.stats(etype, "VAR", a)).view(np.uint16))
            assert gv == exact_round_bits(etype, var)


@pytest.mark.parametrize("etype", HALF)
def test_generator_grid_and_overflow(etype):
    a = oracle.fill(etype, "randu", 100_000)
    v = np.array([bits_to_float(etype, int(b)) for b in a.view(np.uint16)[:2000]])
    step = 2.0 ** (-8 if etype == "bf16" else -11)
    assert np.all(v >= 0) and np.all(v < 1) and np.all(np.floor(v / step) == v / step)
    big = oracle.fill(etype, "iota", 70_000)  # f16 overflows past 65504
    last = bits_to_float(etype, int(big.view(np.uint16)[-1]))
    # f16 overflows past 65504; bf16 has an 8-bit significand: ulp(69999) = 512, 69999 -> 137*512
    assert last == (math.inf if etype == "f16" else 70144.0)


# ---- exhaustive: every one of the 65536 bit patterns ---------------------------
def _round_f64_to(etype, y):
    """Round float64 values to bf16 / f16 (nearest-even, subnormals, overflow
    to inf), vectorised: n = rint(y / 2^q) with q the exponent of one ulp.
    Also returns where y lies within 2^-45 |y| of a rounding midpoint."""
    p, emin, emax = {"bf16": (8, -126, 127), "f16": (11, -14, 15)}[etype]
    a = np.abs(y)
    with np.errstate(all="ignore"):
        e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
        # log2 may be off by one near powers of two: fix e so 2^e <= a < 2^(e+1)
        e = np.where(np.exp2(e) > a, e - 1, e)
        e = np.where(np.exp2(e + 1) <= a, e + 1, e)
        q = np.maximum(e, emin) - (p - 1)
        s = a / np.exp2(q)
        frac = s - np.floor(s)
        near = np.abs(frac - 0.5) <= 2.0 ** -45 * s
        val = np.rint(s) * np.exp2(q)
        val = np.where(val >= 2.0 ** (emax + 1), np.inf, val)
        val = np.where(a == 0, 0.0, val)
        val = np.where(np.isinf(a), np.inf, val)
        out = np.copysign(val, y)
        out = np.where(np.isnan(y), np.nan, out)
    return out, near & np.isfinite(y) & (a > 0)


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("op", ["SQRT", "EXP", "LOG", "NEG", "ABS", "SQUARE"])
def test_unary_ops_exhaustive(etype, op):
    """All 65536 inputs of each unary op: the oracle equals the exact value
    rounded once (reference: numpy f64 value rounded by _round_f64_to, and
    mpmath at 300 bits wherever the f64 value is near a midpoint)."""
    a = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    x = np.array([bits_to_float(etype, int(b)) for b in a])
    got = oracle.eval_program(etype, [("LOAD", 0), (op, 0)], [as_array(etype, a)]).view(np.uint16)
    gotf = np.array([bits_to_float(etype, int(b)) for b in got])
    if op == "NEG":
        assert np.array_equal(got, a ^ 0x8000)
        return
    if op == "ABS":
        assert np.array_equal(got, a & 0x7FFF)
        return
    with np.errstate(all="ignore"):
        y = {"SQRT": np.sqrt, "EXP": np.exp, "LOG": np.log, "SQUARE": np.square}[op](x)
    want, near = _round_f64_to(etype, y)
    mpf = {"SQRT": mpmath.sqrt, "EXP": mpmath.exp, "LOG": mpmath.log,
           "SQUARE": lambda v: v * v}[op]
    for i in np.nonzero(near)[0]:
        with mpmath.workprec(300):
            want[i] = round_fraction(_mp_to_fraction(mpf(mpmath.mpf(float(x[i])))), etype)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(gotf), nan)
    ok = nan | ((gotf == want) & (np.signbit(gotf) == np.signbit(want)))
    bad = np.nonzero(~ok)[0]
    assert bad.size == 0, [(hex(a[i]), x[i], gotf[i], want[i]) for i in bad[:5]]
