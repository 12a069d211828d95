"""Independent exact-arithmetic references used to PIN the oracle.

Nothing here calls the oracle or the CUDA path.  Every value is computed from
its mathematical definition with Python integers / ``fractions.Fraction``
(exact rationals) and ``mpmath`` (arbitrary precision), then rounded to the
IEEE-754 format with an integer round-half-to-even written out below.  A bug
in the oracle's element functions, its rounding, its accumulation or its
program walk therefore shows up as a mismatch against this module.
"""
from __future__ import annotations

import math
import struct
from fractions import Fraction

import mpmath
import numpy as np

# (precision incl. hidden bit, emin, emax)
FMT = {"f32": (24, -126, 127), "f64": (53, -1022, 1023), "bf16": (8, -126, 127),
       "f16": (11, -14, 15)}
MASK = {"u32": (1 << 32) - 1, "s64": (1 << 64) - 1}


def _floor_log2(a: Fraction) -> int:
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while _pow2(e) > a:
        e -= 1
    while _pow2(e + 1) <= a:
        e += 1
    return e


def _pow2(e: int) -> Fraction:
    return Fraction(1 << e) if e >= 0 else Fraction(1, 1 << (-e))


def round_fraction(fr: Fraction, etype: str, neg_zero: bool = False) -> float:
    """Round an exact rational to binary32/binary64, round-half-to-even.

    Returns a Python float (exactly the binary32 value when etype == 'f32').
    ``neg_zero`` selects the sign of an exact zero result (IEEE rules are the
    caller's business)."""
    p, emin, emax = FMT[etype]
    if fr == 0:
        return -0.0 if neg_zero else 0.0
    sign = -1.0 if fr < 0 else 1.0
    a = abs(fr)
    e = _floor_log2(a)
    q = max(e, emin) - (p - 1)
    scaled = a / _pow2(q)
    n = scaled.numerator // scaled.denominator
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    val = Fraction(n) * _pow2(q)
    if val >= _pow2(emax + 1):
        return sign * math.inf
    return sign * float(val)


def to_np(x: float, etype: str):
    return np.float32(x) if etype == "f32" else np.float64(x)


def frac(x) -> Fraction:
    return Fraction(float(x))


def is_neg_zero(x) -> bool:
    return float(x) == 0.0 and math.copysign(1.0, float(x)) < 0


# ---- element-wise float ops, exact then rounded once ---------------------

def f_add(a, b, etype):
    a, b = float(a), float(b)
    if math.isnan(a) or math.isnan(b) or math.isinf(a) or math.isinf(b):
        return to_np(a + b, etype)  # IEEE specials: exact by definition
    s = frac(a) + frac(b)
    nz = s == 0 and is_neg_zero(a) and is_neg_zero(b)
    return to_np(round_fraction(s, etype, nz), etype)


def f_sub(a, b, etype):
    return f_add(a, -float(b), etype)


def f_mul(a, b, etype):
    a, b = float(a), float(b)
    if math.isnan(a) or math.isnan(b) or math.isinf(a) or math.isinf(b):
        return to_np(a * b, etype)
    s = frac(a) * frac(b)
    nz = (math.copysign(1.0, a) * math.copysign(1.0, b)) < 0
    return to_np(round_fraction(s, etype, nz), etype)


def f_div(a, b, etype):
    a, b = float(a), float(b)
    if math.isnan(a) or math.isnan(b) or math.isinf(a) or math.isinf(b) or b == 0.0:
        with np.errstate(all="ignore"):
            return to_np(np.float64(a) / np.float64(b), etype)
    s = frac(a) / frac(b)
    nz = (math.copysign(1.0, a) * math.copysign(1.0, b)) < 0
    return to_np(round_fraction(s, etype, nz), etype)


def _mp_to_fraction(v) -> Fraction:
    sign, man, exp, _ = mpmath.mpf(v)._mpf_
    man = -int(man) if sign else int(man)
    exp = int(exp)
    return Fraction(man) * _pow2(exp) if exp < 0 else Fraction(man << exp)


def f_sqrt(a, etype):
    a = float(a)
    if math.isnan(a) or a < 0 or math.isinf(a) or a == 0.0:
        with np.errstate(all="ignore"):
            return to_np(np.sqrt(np.float64(a)), etype)
    with mpmath.workprec(400):
        r = mpmath.sqrt(mpmath.mpf(a))
        return to_np(round_fraction(_mp_to_fraction(r), etype), etype)


def f_exp(a, etype):
    a = float(a)
    if math.isnan(a):
        return to_np(math.nan, etype)
    if math.isinf(a):
        return to_np(math.inf if a > 0 else 0.0, etype)
    if a == 0.0:
        return to_np(1.0, etype)
    if a > 800:
        return to_np(math.inf, etype)
    if a < -800:
        return to_np(0.0, etype)
    with mpmath.workprec(400):
        r = mpmath.exp(mpmath.mpf(a))
        return to_np(round_fraction(_mp_to_fraction(r), etype), etype)


def f_log(a, etype):
    a = float(a)
    if math.isnan(a) or a < 0:
        return to_np(math.nan, etype)
    if a == 0.0:
        return to_np(-math.inf, etype)
    if math.isinf(a):
        return to_np(math.inf, etype)
    if a == 1.0:
        return to_np(0.0, etype)
    with mpmath.workprec(400):
        r = mpmath.log(mpmath.mpf(a))
        return to_np(round_fraction(_mp_to_fraction(r), etype), etype)


def f_neg(a, etype):
    return to_np(-float(a), etype)


def f_abs(a, etype):
    return to_np(abs(float(a)), etype)


def f_square(a, etype):
    return f_mul(a, a, etype)


def f_min(a, b, etype):
    return to_np(float(b) if float(b) < float(a) else float(a), etype)


def f_max(a, b, etype):
    return to_np(float(b) if float(a) < float(b) else float(a), etype)


# ---- integer ops: textbook modular arithmetic -----------------------------

def _to_int(x, etype) -> int:
    v = int(x)
    return v & MASK[etype]


def _from_int(v: int, etype):
    v &= MASK[etype]
    if etype == "u32":
        return np.uint32(v)
    if v >= 1 << 63:
        v -= 1 << 64
    return np.int64(v)


def _signed(v: int, etype) -> int:
    if etype == "s64" and v >= 1 << 63:
        return v - (1 << 64)
    return v


def i_op(op, a, b, etype):
    x, y = _to_int(a, etype), (_to_int(b, etype) if b is not None else None)
    if op == "ADD":
        return _from_int(x + y, etype)
    if op == "SUB":
        return _from_int(x - y, etype)
    if op == "MUL":
        return _from_int(x * y, etype)
    if op == "MIN":
        return _from_int(y if _signed(y, etype) < _signed(x, etype) else x, etype)
    if op == "MAX":
        return _from_int(y if _signed(x, etype) < _signed(y, etype) else x, etype)
    if op == "NEG":
        return _from_int(-x, etype)
    if op == "ABS":
        return _from_int(abs(_signed(x, etype)), etype)
    if op == "SQUARE":
        return _from_int(x * x, etype)
    raise ValueError(op)


UNARY = ("NEG", "ABS", "SQUARE", "SQRT", "EXP", "LOG")
BINARY = ("ADD", "SUB", "MUL", "DIV", "MIN", "MAX")
INT_ILLEGAL = ("SQRT", "EXP", "LOG", "DIV")

_FUN = {"NEG": f_neg, "ABS": f_abs, "SQUARE": f_square, "SQRT": f_sqrt, "EXP": f_exp,
        "LOG": f_log}
_BFUN = {"ADD": f_add, "SUB": f_sub, "MUL": f_mul, "DIV": f_div, "MIN": f_min, "MAX": f_max}


def elem_op(op, etype, a, b=None):
    if etype in ("u32", "s64"):
        return i_op(op, a, b, etype)
    if op in _FUN:
        return _FUN[op](a, etype)
    return _BFUN[op](a, b, etype)


# ---- recursive per-element evaluator (tree form, not postfix walk) -------

def postfix_to_tree(program):
    st = []
    for op, arg in program:
        if op in ("LOAD", "SCALAR"):
            st.append((op, arg))
        elif op in UNARY:
            a = st.pop()
            st.append((op, a))
        else:
            b = st.pop()
            a = st.pop()
            st.append((op, a, b))
    assert len(st) == 1
    return st[0]


def eval_tree(node, etype, operands, scalars, i):
    op = node[0]
    if op == "LOAD":
        return operands[node[1]][i]
    if op == "SCALAR":
        return scalars[node[1]]
    if op in UNARY:
        return elem_op(op, etype, eval_tree(node[1], etype, operands, scalars, i))
    return elem_op(op, etype, eval_tree(node[1], etype, operands, scalars, i),
                   eval_tree(node[2], etype, operands, scalars, i))


# ---- exact reductions -----------------------------------------------------

def exact_sum(values) -> Fraction:
    s = Fraction(0)
    for v in values:
        s += Fraction(float(v))
    return s


def rounded_sum(values, etype):
    return to_np(round_fraction(exact_sum(values), etype), etype)


def rounded_norm2(values, etype):
    s = Fraction(0)
    for v in values:
        f = Fraction(float(v))
        s += f * f
    if s == 0:
        return to_np(0.0, etype)
    with mpmath.workprec(600):
        r = mpmath.sqrt(mpmath.mpf(s.numerator) / mpmath.mpf(s.denominator))
        return to_np(round_fraction(_mp_to_fraction(r), etype), etype)


def bits(x) -> int:
    x = np.asarray(x)
    if x.dtype == np.float32:
        return struct.unpack("<I", struct.pack("<f", float(x)))[0]
    if x.dtype == np.float64:
        return struct.unpack("<Q", struct.pack("<d", float(x)))[0]
    return int(x)


def same_bits(a, b) -> bool:
    fa, fb = np.asarray(a), np.asarray(b)
    if fa.dtype.kind == "f" and np.isnan(fa) and np.isnan(fb):
        return True
    return bits(a) == bits(b)
