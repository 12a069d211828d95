"""Brute force over programs (SURVEY §8(c) "Brute-force sizing"; SPEC S:217,
S:653): the oracle's eager postfix walk against an independent
per-element tree evaluator, bit for bit, on 5x5 inputs.

* EXHAUSTIVE to depth 2 over leaves {L0, L1, L2, S0, S1}, the 6 unary and 6
  binary ops, restricted to the ops legal for the type (int: no SQRT / EXP /
  LOG / DIV): 206,465 trees per float type (197,571 that read an operand),
  105,565 per integer type.
* A seeded random sample of 10^5 depth-3 programs per type.

The reference evaluates the TREE (not the postfix stack) vectorised over the
25 elements.  Element semantics, each pinned separately against exact rational
arithmetic in test_oracle_elementwise.py:
  + - * / sqrt neg abs square: IEEE-754 in eT (numpy's own kernels); MIN(a,b) =
  (b < a) ? b : a, MAX(a,b) = (a < b) ? b : a (R13); ints wrap (R8);
  EXP / LOG: correctly rounded — evaluated in a wider type by a DIFFERENT
  library routine than the oracle's (numpy f64 for f32, long double expl /
  logl for f64), and wherever that wide value lies within a generous error
  band of an eT rounding midpoint the value is recomputed with mpmath at 200
  bits and rounded exactly (tests/exactref.py).
"""
import random

import mpmath
import numpy as np
import pytest

import oracle
from exactref import _mp_to_fraction, round_fraction

FLOATS = ("f32", "f64")
TYPES = ("f32", "f64", "u32", "s64")
UNARY = ("NEG", "ABS", "SQUARE", "SQRT", "EXP", "LOG")
BINARY = ("ADD", "SUB", "MUL", "DIV", "MIN", "MAX")
INT_ILLEGAL = ("SQRT", "EXP", "LOG", "DIV")
LEAVES = (("LOAD", 0), ("LOAD", 1), ("LOAD", 2), ("SCALAR", 0), ("SCALAR", 1))
N = 25  # a 5 x 5 matrix


def legal(etype, ops):
    return ops if etype in FLOATS else tuple(o for o in ops if o not in INT_ILLEGAL)


def inputs(etype, seed):
    rng = np.random.default_rng(seed)
    dt = oracle.DTYPES[etype]
    if etype in FLOATS:
        special = np.array([0.0, -0.0, 1.0, -1.0, 0.5], dt)
        ops = [np.concatenate([special[np.roll(np.arange(5), k)],
                               rng.uniform(-2, 2, N - 5).astype(dt)]) for k in range(3)]
        sc = [dt(2.5), dt(-0.75)]
    elif etype == "u32":
        special = np.array([0, 1, 0xFFFFFFFF, 0x80000000, 0x10000], np.uint32)
        ops = [np.concatenate([special[np.roll(np.arange(5), k)],
                               rng.integers(0, 2**32, N - 5, dtype=np.uint64).astype(np.uint32)])
               for k in range(3)]
        sc = [np.uint32(7), np.uint32(0xFFFFFFF0)]
    else:
        special = np.array([0, 1, -1, -2**63, 2**63 - 1], np.int64)
        ops = [np.concatenate([special[np.roll(np.arange(5), k)],
                               rng.integers(-2**63, 2**63 - 1, N - 5, dtype=np.int64)])
               for k in range(3)]
        sc = [np.int64(7), np.int64(-3)]
    return ops, sc


# ---- the reference: a tree evaluator over numpy arrays -----------------------
_MP_FN = {"EXP": mpmath.exp, "LOG": mpmath.log}
_NP_FN = {"EXP": np.exp, "LOG": np.log}


def _mp_round(op, x: float, etype):
    with mpmath.workprec(200):
        return round_fraction(_mp_to_fraction(_MP_FN[op](mpmath.mpf(x))), etype)


def cr_transcendental(op, x, etype):
    """Correctly rounded EXP / LOG of an eT array (see module docstring)."""
    dt = oracle.DTYPES[etype]
    wide, tol = (np.float64, 2.0 ** -45) if etype == "f32" else (np.longdouble, 2.0 ** -58)
    with np.errstate(all="ignore"):
        y = _NP_FN[op](x.astype(wide))
        r = y.astype(dt)
        up = np.nextafter(r, dt(np.inf)).astype(wide)
        dn = np.nextafter(r, dt(-np.inf)).astype(wide)
        rw = r.astype(wide)
        ay = np.abs(y) * wide(tol)
        near = np.isfinite(y) & (y != 0) & (
            (np.abs(y - (rw + up) / 2) <= ay) | (np.abs(y - (rw + dn) / 2) <= ay) |
            ~np.isfinite(r))
    for i in np.nonzero(near)[0]:
        r[i] = dt(_mp_round(op, float(x[i]), etype))
    return r


def ref_unary(op, a, etype):
    dt = oracle.DTYPES[etype]
    with np.errstate(all="ignore"):
        if op == "NEG":
            return (-a).astype(dt) if etype in FLOATS or etype == "s64" else (dt(0) - a).astype(dt)
        if op == "ABS":
            return np.abs(a).astype(dt) if etype != "u32" else a.copy()
        if op == "SQUARE":
            return (a * a).astype(dt)
        if op == "SQRT":
            return np.sqrt(a).astype(dt)
        return cr_transcendental(op, a, etype)


def ref_binary(op, a, b, etype):
    dt = oracle.DTYPES[etype]
    with np.errstate(all="ignore"):
        if op == "ADD":
            r = a + b
        elif op == "SUB":
            r = a - b
        elif op == "MUL":
            r = a * b
        elif op == "DIV":
            r = a / b
        elif op == "MIN":
            r = np.where(b < a, b, a)
        else:
            r = np.where(a < b, b, a)
    return np.asarray(r).astype(dt)


def same_bits_all(got, want, etype):
    """Element-wise bit equality; any NaN matches any NaN."""
    got, want = np.asarray(got), np.asarray(want)
    if etype in FLOATS:
        nan = np.isnan(want)
        ok = (np.isnan(got) == nan)
        ub = np.uint32 if etype == "f32" else np.uint64
        ok &= nan | (got.view(ub) == want.view(ub))
        return ok
    return got == want


# ---- exhaustive depth <= 2 ----------------------------------------------------
def enumerate_depth2(etype, ops, sc):
    """(programs, reference values [len, N]) of every tree of depth <= 2 that
    reads an operand, in a fixed order, the values built from the depth-1
    level by broadcasting (no per-program work)."""
    dt = oracle.DTYPES[etype]
    un, bi = legal(etype, UNARY), legal(etype, BINARY)
    leaf_val = [ops[0], ops[1], ops[2], np.full(N, sc[0], dt), np.full(N, sc[1], dt)]
    leaf_load = [True, True, True, False, False]
    # depth <= 1
    d1_prog, d1_val, d1_load = [], [], []
    for lp, lv, ll in zip(LEAVES, leaf_val, leaf_load):
        d1_prog.append([lp]); d1_val.append(lv); d1_load.append(ll)
    for u in un:
        for lp, lv, ll in zip(LEAVES, leaf_val, leaf_load):
            d1_prog.append([lp, (u, 0)]); d1_val.append(ref_unary(u, lv, etype)); d1_load.append(ll)
    for b in bi:
        for lp, lv, ll in zip(LEAVES, leaf_val, leaf_load):
            for rp, rv, rl in zip(LEAVES, leaf_val, leaf_load):
                d1_prog.append([lp, rp, (b, 0)])
                d1_val.append(ref_binary(b, lv, rv, etype))
                d1_load.append(ll or rl)
    V = np.stack(d1_val)                    # [K, N]
    L = np.array(d1_load)
    K = len(d1_prog)
    progs, vals, loads = [], [], []
    # depth <= 2 = leaves, unary(depth <= 1), binary(depth <= 1, depth <= 1)
    for i in range(len(LEAVES)):
        progs.append(d1_prog[i]); vals.append(V[i:i + 1]); loads.append(L[i:i + 1])
    for u in un:
        for k in range(K):
            progs.append(d1_prog[k] + [(u, 0)])
        vals.append(np.stack([ref_unary(u, V[k], etype) for k in range(K)]))
        loads.append(L)
    for b in bi:
        for k in range(K):
            for j in range(K):
                progs.append(d1_prog[k] + d1_prog[j] + [(b, 0)])
        vals.append(ref_binary(b, V[:, None, :], V[None, :, :], etype).reshape(K * K, N))
        loads.append((L[:, None] | L[None, :]).reshape(-1))
    vals = np.concatenate(vals)
    loads = np.concatenate(loads)
    return [p for p, l in zip(progs, loads) if l], vals[loads], len(progs)


@pytest.mark.parametrize("etype", TYPES)
def test_exhaustive_depth2(etype):
    ops, sc = inputs(etype, 31)
    progs, want, total = enumerate_depth2(etype, ops, sc)
    assert total == (206_465 if etype in FLOATS else 105_565)  # SURVEY §8(c) tree counts
    got = oracle.eval_programs(etype, progs, ops, sc)
    ok = same_bits_all(got, want, etype)
    if not ok.all():
        p, i = np.argwhere(~ok)[0]
        raise AssertionError(f"{etype} {progs[p]} element {i}: oracle {got[p, i]!r} "
                             f"reference {want[p, i]!r} ({(~ok).sum()} mismatches)")


# ---- seeded sample at depth 3 ----------------------------------------------------
def random_tree(rng, depth, etype):
    un, bi = legal(etype, UNARY), legal(etype, BINARY)
    if depth == 0 or rng.random() < 0.15:
        return (rng.choice(LEAVES),)
    if rng.random() < 0.35:
        return (rng.choice(un), random_tree(rng, depth - 1, etype))
    return (rng.choice(bi), random_tree(rng, depth - 1, etype), random_tree(rng, depth - 1, etype))


def to_postfix(t):
    if len(t) == 1:
        return [t[0]]
    return [x for k in t[1:] for x in to_postfix(k)] + [(t[0], 0)]


def reads_operand(t):
    return t[0][0] == "LOAD" if len(t) == 1 else any(reads_operand(k) for k in t[1:])


def ref_tree(t, etype, leaf_val, memo):
    v = memo.get(t)
    if v is not None:
        return v
    if len(t) == 1:
        v = leaf_val[t[0]]
    elif len(t) == 2:
        v = ref_unary(t[0], ref_tree(t[1], etype, leaf_val, memo), etype)
    else:
        v = ref_binary(t[0], ref_tree(t[1], etype, leaf_val, memo),
                       ref_tree(t[2], etype, leaf_val, memo), etype)
    memo[t] = v
    return v


@pytest.mark.parametrize("etype", TYPES)
def test_random_depth3_sample(etype):
    ops, sc = inputs(etype, 32)
    dt = oracle.DTYPES[etype]
    leaf_val = {LEAVES[0]: ops[0], LEAVES[1]: ops[1], LEAVES[2]: ops[2],
                LEAVES[3]: np.full(N, sc[0], dt), LEAVES[4]: np.full(N, sc[1], dt)}
    rng = random.Random(4242 + TYPES.index(etype))
    trees = []
    while len(trees) < 100_000:
        t = random_tree(rng, 3, etype)
        if reads_operand(t):
            trees.append(t)
    memo = {}
    want = np.stack([ref_tree(t, etype, leaf_val, memo) for t in trees])
    progs = [to_postfix(t) for t in trees]
    got = oracle.eval_programs(etype, progs, ops, sc)
    ok = same_bits_all(got, want, etype)
    if not ok.all():
        p, i = np.argwhere(~ok)[0]
        raise AssertionError(f"{etype} {progs[p]} element {i}: oracle {got[p, i]!r} "
                             f"reference {want[p, i]!r} ({(~ok).sum()} mismatches)")
