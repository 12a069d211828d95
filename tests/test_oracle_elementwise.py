"""Pins for the oracle's per-element semantics (readings R5-R9).

Each op is checked against exact rational arithmetic (fractions) or mpmath,
rounded to binary32/binary64 by tests/exactref.py's integer round-half-even.
"""
import math

import numpy as np
import pytest

import oracle
from exactref import INT_ILLEGAL, elem_op, same_bits


def _float_samples(etype, n, seed):
    rng = np.random.default_rng(seed)
    dt = np.float32 if etype == "f32" else np.float64
    it = np.uint32 if etype == "f32" else np.uint64
    bits = rng.integers(0, np.iinfo(it).max, size=n, dtype=it, endpoint=True)
    wide = bits.view(dt)
    wide = wide[np.isfinite(wide)]
    unit = rng.random(n).astype(dt)
    special = np.array([0.0, -0.0, 1.0, -1.0, 0.5, 2.0, 3.0, 1e-30, -1e-30, 1e30,
                        np.finfo(dt).tiny, np.finfo(dt).max, -np.finfo(dt).max,
                        np.finfo(dt).tiny / 4, np.finfo(dt).eps], dtype=dt)
    return np.concatenate([special, unit, wide[: n // 2]]).astype(dt)


def _run_unary(etype, op, x):
    return oracle.eval_program(etype, [("LOAD", 0), (op, 0)], [x])


def _run_binary(etype, op, a, b):
    return oracle.eval_program(etype, [("LOAD", 0), ("LOAD", 1), (op, 0)], [a, b])


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("op", ["ADD", "SUB", "MUL", "DIV", "MIN", "MAX"])
def test_float_binary_ops_correctly_rounded(etype, op):
    a = _float_samples(etype, 300, 1)
    b = _float_samples(etype, 300, 2)[: a.size]
    a = a[: b.size]
    got = _run_binary(etype, op, a, b)
    for i in range(a.size):
        want = elem_op(op, etype, a[i], b[i])
        assert same_bits(got[i], want), (op, a[i], b[i], got[i], want)


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("op", ["NEG", "ABS", "SQUARE", "SQRT"])
def test_float_unary_ops_correctly_rounded(etype, op):
    x = _float_samples(etype, 400, 3)
    got = _run_unary(etype, op, x)
    for i in range(x.size):
        want = elem_op(op, etype, x[i])
        assert same_bits(got[i], want), (op, x[i], got[i], want)


def test_f32_exp_correctly_rounded_sampled():
    rng = np.random.default_rng(7)
    x = np.concatenate([
        rng.uniform(-104, 89, 6000), rng.uniform(-1, 1, 3000), rng.uniform(0, 1, 3000),
        np.array([0.0, -0.0, 1.0, -1.0, 88.72, 88.73, -87.3, -103.9, -104.0, -110.0, 89.0, 100.0]),
    ]).astype(np.float32)
    got = _run_unary("f32", "EXP", x)
    for i in range(x.size):
        assert same_bits(got[i], elem_op("EXP", "f32", x[i])), (x[i], got[i])


def test_f32_log_correctly_rounded_sampled():
    rng = np.random.default_rng(8)
    x = np.concatenate([
        rng.uniform(0, 1, 4000), rng.uniform(0, 100, 3000),
        np.exp(rng.uniform(-100, 88, 4000)),
        np.array([1.0, 2.0, 0.5, 1e-45, 1e-38, 3.4e38, 0.0, -1.0, np.inf]),
    ]).astype(np.float32)
    got = _run_unary("f32", "LOG", x)
    for i in range(x.size):
        assert same_bits(got[i], elem_op("LOG", "f32", x[i])), (x[i], got[i])


def test_f64_exp_log_correctly_rounded_sampled():
    rng = np.random.default_rng(9)
    x = np.concatenate([rng.uniform(-700, 700, 1500), rng.uniform(0, 1, 1000)])
    got = _run_unary("f64", "EXP", x)
    for i in range(x.size):
        assert same_bits(got[i], elem_op("EXP", "f64", x[i])), (x[i], got[i])
    y = np.concatenate([np.exp(rng.uniform(-700, 700, 1500)), rng.uniform(0, 1, 1000)])
    got = _run_unary("f64", "LOG", y)
    for i in range(y.size):
        assert same_bits(got[i], elem_op("LOG", "f64", y[i])), (y[i], got[i])


def test_exp_log_special_values():
    one = np.array([0.0, 1.0], np.float32)
    e = _run_unary("f32", "EXP", one)
    assert e[0] == 1.0
    assert float(e[1]) == float.fromhex("0x1.5bf0a8p+1")  # RN_f32(e)
    assert _run_unary("f32", "LOG", np.array([1.0], np.float32))[0] == 0.0
    assert _run_unary("f64", "EXP", np.array([0.0]))[0] == 1.0
    assert _run_unary("f64", "LOG", np.array([1.0]))[0] == 0.0


def _int_samples(etype, n, seed):
    rng = np.random.default_rng(seed)
    if etype == "u32":
        edge = np.array([0, 1, 2, 7, 0xFFFF, 0x10000, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFF,
                         0x24924925], dtype=np.uint32)
        return np.concatenate([edge, rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)])
    edge = np.array([0, 1, -1, 2, 7, 2**62, -2**62, 2**63 - 1, -2**63, 2**32, -2**32 - 1],
                    dtype=np.int64)
    return np.concatenate([edge, rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64)])


@pytest.mark.parametrize("etype", ["u32", "s64"])
@pytest.mark.parametrize("op", ["ADD", "SUB", "MUL", "MIN", "MAX"])
def test_integer_binary_ops_modular(etype, op):
    a = _int_samples(etype, 400, 11)
    b = _int_samples(etype, 400, 12)[::-1].copy()
    got = _run_binary(etype, op, a, b)
    for i in range(a.size):
        assert int(got[i]) == int(elem_op(op, etype, a[i], b[i])), (op, a[i], b[i])


@pytest.mark.parametrize("etype", ["u32", "s64"])
@pytest.mark.parametrize("op", ["NEG", "ABS", "SQUARE"])
def test_integer_unary_ops_modular(etype, op):
    x = _int_samples(etype, 400, 13)
    got = _run_unary(etype, op, x)
    for i in range(x.size):
        assert int(got[i]) == int(elem_op(op, etype, x[i])), (op, x[i])


def test_integer_wrap_cases_R8():
    # u32: 0x10000 * 0x10000 = 2^32 = 0 (mod 2^32); 7 * 0x24924925 = 3 (mod 2^32)
    a = np.array([0x10000, 7], np.uint32)
    b = np.array([0x10000, 0x24924925], np.uint32)
    assert list(_run_binary("u32", "MUL", a, b)) == [0, 3]
    # s64: INT64_MAX + 1 = INT64_MIN; INT64_MAX * 2 = -2; ABS(INT64_MIN) = INT64_MIN
    imax = np.array([2**63 - 1], np.int64)
    assert _run_binary("s64", "ADD", imax, np.array([1], np.int64))[0] == -2**63
    assert _run_binary("s64", "MUL", imax, np.array([2], np.int64))[0] == -2
    assert _run_unary("s64", "ABS", np.array([-2**63], np.int64))[0] == -2**63
    assert _run_unary("u32", "NEG", np.array([1], np.uint32))[0] == 0xFFFFFFFF


@pytest.mark.parametrize("etype", ["u32", "s64"])
@pytest.mark.parametrize("op", INT_ILLEGAL)
def test_integer_illegal_ops_rejected_R9(etype, op):
    x = np.ones(4, dtype=oracle.DTYPES[etype])
    prog = [("LOAD", 0), (op, 0)] if op != "DIV" else [("LOAD", 0), ("LOAD", 0), ("DIV", 0)]
    with pytest.raises(oracle.OracleError):
        oracle.eval_program(etype, prog, [x])


def test_no_fma_contraction_in_oracle():
    # a*b + c with a*b inexact: eager rounding of the product must be visible.
    a = np.array([1 + 2**-12], np.float32)
    c = np.array([-(1 + 2**-11)], np.float32)
    got = oracle.eval_program("f32", [("LOAD", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1),
                                      ("ADD", 0)], [a, c])
    # exact a*a = 1 + 2^-11 + 2^-24 rounds (tie, even) to 1 + 2^-11, so the sum is 0;
    # a fused multiply-add would give 2^-24.
    assert got[0] == 0.0 and not math.copysign(1.0, float(got[0])) < 0
