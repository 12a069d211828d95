"""Pins for the oracle's program walk: SPEC worked examples and brute force
against an independent recursive per-element evaluator (tests/exactref.py)."""
import os
import random

import numpy as np
import pytest

import oracle
from exactref import BINARY, INT_ILLEGAL, UNARY, eval_tree, postfix_to_tree, same_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.txt")

TOKENS = {"S0": ("SCALAR", 0), "S1": ("SCALAR", 1), "L0": ("LOAD", 0), "L1": ("LOAD", 1),
          "L2": ("LOAD", 2)}


def parse_prog(s):
    out = []
    for t in s.split():
        out.append(TOKENS[t] if t in TOKENS else (t, 0))
    return out


def parse_vals(s):
    s = s.strip()
    if ".." in s:
        lo, hi = s.split("..")
        return [float(v) for v in range(int(lo), int(hi) + 1)]
    return [float(v) for v in s.split(",")]


def golden_rows():
    rows = []
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        name, etype, prog, ops, scal, want = [f.strip() for f in line.split("|")]
        rows.append((name, etype, prog, ops, scal, want))
    return rows


@pytest.mark.parametrize("row", golden_rows(), ids=lambda r: r[0])
def test_spec_worked_examples(row):
    name, etype, prog, ops, scal, want = row
    dt = oracle.DTYPES[etype]
    operands = [np.array(parse_vals(o), dtype=dt) for o in ops.split(";")]
    want = np.array(parse_vals(want), dtype=dt)
    if prog == "ACCU":
        got = oracle.reduce(etype, "ACCU", operands[0])
        assert got == want[0]
        return
    scalars = [] if scal == "-" else [float(s) for s in scal.split(",")]
    got = oracle.eval_program(etype, parse_prog(prog), operands, scalars)
    assert np.array_equal(got, want)


def random_tree(rng, depth, etype, n_ops=3, n_sc=2):
    unary = [u for u in UNARY if etype in ("f32", "f64") or u not in INT_ILLEGAL]
    binary = [b for b in BINARY if etype in ("f32", "f64") or b not in INT_ILLEGAL]
    if depth == 0 or rng.random() < 0.25:
        if rng.random() < 0.7:
            return [("LOAD", rng.randrange(n_ops))]
        return [("SCALAR", rng.randrange(n_sc))]
    if rng.random() < 0.35:
        return random_tree(rng, depth - 1, etype) + [(rng.choice(unary), 0)]
    return (random_tree(rng, depth - 1, etype) + random_tree(rng, depth - 1, etype)
            + [(rng.choice(binary), 0)])


def _inputs(etype, n, seed):
    rng = np.random.default_rng(seed)
    if etype in ("f32", "f64"):
        dt = oracle.DTYPES[etype]
        ops = [rng.uniform(-2, 2, n).astype(dt) for _ in range(3)]
        sc = [dt(2.5), dt(-0.75)]
    elif etype == "u32":
        ops = [rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32) for _ in range(3)]
        sc = [np.uint32(7), np.uint32(0xFFFFFFF0)]
    else:
        ops = [rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64) for _ in range(3)]
        sc = [np.int64(7), np.int64(-3)]
    return ops, sc


@pytest.mark.parametrize("etype", ["f32", "f64", "u32", "s64"])
def test_brute_force_depth1_exhaustive(etype):
    """Every op over every leaf pair (depth <= 1), 5x5 inputs, bit-identical."""
    ops, sc = _inputs(etype, 25, 21)
    leaves = [("LOAD", 0), ("LOAD", 1), ("SCALAR", 0)]
    progs = [[leaf] for leaf in leaves]
    for u in UNARY:
        if etype in ("u32", "s64") and u in INT_ILLEGAL:
            continue
        progs += [[leaf, (u, 0)] for leaf in leaves]
    for b in BINARY:
        if etype in ("u32", "s64") and b in INT_ILLEGAL:
            continue
        progs += [[x, y, (b, 0)] for x in leaves for y in leaves]
    for prog in progs:
        if all(o == "SCALAR" for o, _ in prog if o in ("LOAD", "SCALAR")):
            continue  # scalar-only expression has no operand extent
        got = oracle.eval_program(etype, prog, ops, sc)
        tree = postfix_to_tree(prog)
        for i in range(25):
            assert same_bits(got[i], eval_tree(tree, etype, ops, sc, i)), (prog, i)


@pytest.mark.parametrize("etype", ["f32", "f64", "u32", "s64"])
def test_brute_force_random_depth3(etype):
    rng = random.Random(1234 + hash(etype) % 1000)
    ops, sc = _inputs(etype, 25, 22)
    n_checked = 0
    while n_checked < 60:
        prog = random_tree(rng, 3, etype)
        if not any(o == "LOAD" for o, _ in prog):
            continue
        got = oracle.eval_program(etype, prog, ops, sc)
        tree = postfix_to_tree(prog)
        for i in range(25):
            assert same_bits(got[i], eval_tree(tree, etype, ops, sc, i)), (prog, i)
        n_checked += 1


def test_postfix_operand_order_for_noncommutative_ops():
    a = np.array([10.0, 1.0])
    b = np.array([4.0, 8.0])
    assert list(oracle.eval_program("f64", [("LOAD", 0), ("LOAD", 1), ("SUB", 0)], [a, b])) == [6, -7]
    assert list(oracle.eval_program("f64", [("LOAD", 0), ("LOAD", 1), ("DIV", 0)], [a, b])) == [2.5, 0.125]
    assert list(oracle.eval_program("f64", [("LOAD", 1), ("LOAD", 0), ("SUB", 0)], [a, b])) == [-6, 7]


def test_malformed_programs_rejected():
    x = np.ones(3)
    for prog in ([("ADD", 0)], [("LOAD", 0), ("LOAD", 0)], [("LOAD", 5)], [("SCALAR", 0)],
                 [("LOAD", 0), ("NEG", 0), ("SUB", 0)]):
        with pytest.raises(oracle.OracleError):
            oracle.eval_program("f64", prog, [x])


def test_c1_axpy_known_values():
    # axpy x=1, y=2, alpha=2.5 -> 4.5 everywhere (SURVEY §8(c) closed form)
    n = 1000
    x = np.ones(n, np.float32)
    y = np.full(n, 2.0, np.float32)
    got = oracle.eval_program("f32", [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1),
                                      ("ADD", 0)], [x, y], [2.5])
    assert np.all(got == 4.5)
    assert oracle.reduce("f32", "ACCU", got) == np.float32(4.5 * n)
