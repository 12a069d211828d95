"""Shared test helpers: program shapes, random programs, the parity checker.

Nothing here computes the method's arithmetic; the oracle (oracle/) and the
exact references (tests/exactref.py) do that.
"""
from __future__ import annotations

import random

import numpy as np

UNARY = ("NEG", "ABS", "SQUARE", "SQRT", "EXP", "LOG")
BINARY = ("ADD", "SUB", "MUL", "DIV", "MIN", "MAX")
INT_ILLEGAL = ("SQRT", "EXP", "LOG", "DIV")
FLOATS = ("f32", "f64")
INTS = ("u32", "s64")
ALL = FLOATS + INTS


def P(s: str):
    """Parse "L0 L1 MUL EXP S0 L2 MUL ADD" into [(op, arg), ...]."""
    out = []
    for t in s.split():
        if t[0] in "LS" and t[1:].isdigit():
            out.append(("LOAD" if t[0] == "L" else "SCALAR", int(t[1:])))
        else:
            out.append((t, 0))
    return out


# The catalog shapes (paper_2508_11385_b200/csrc/coot_catalog.h) restated.
CATALOG = {
    0: "L0", 1: "S0 L0 MUL L1 ADD", 2: "L0 L1 MUL EXP S0 L2 MUL ADD",
    3: "L0 L1 MUL S0 L2 MUL ADD", 4: "L0 L1 MUL", 5: "L0 L1 ADD", 6: "L0 L1 SUB",
    7: "S0 L0 MUL", 8: "L0 S0 ADD", 9: "L0 L1 DIV",
}
C1_AXPY = P(CATALOG[1])
C2 = P(CATALOG[2])
C4 = P(CATALOG[3])


def n_operands(prog) -> int:
    return 1 + max((a for o, a in prog if o == "LOAD"), default=-1)


def n_scalars(prog) -> int:
    return 1 + max((a for o, a in prog if o == "SCALAR"), default=-1)


def legal(prog, etype) -> bool:
    return etype in FLOATS or not any(o in INT_ILLEGAL for o, _ in prog)


def has_transcendental(prog) -> bool:
    return any(o in ("EXP", "LOG") for o, _ in prog)


def random_program(rng: random.Random, depth: int, etype: str, n_ops: int = 3, n_sc: int = 2):
    unary = [u for u in UNARY if etype in FLOATS or u not in INT_ILLEGAL]
    binary = [b for b in BINARY if etype in FLOATS or b not in INT_ILLEGAL]

    def rec(d):
        if d == 0 or rng.random() < 0.2:
            if rng.random() < 0.75:
                return [("LOAD", rng.randrange(n_ops))]
            return [("SCALAR", rng.randrange(n_sc))]
        if rng.random() < 0.3:
            return rec(d - 1) + [(rng.choice(unary), 0)]
        return rec(d - 1) + rec(d - 1) + [(rng.choice(binary), 0)]

    while True:
        p = rec(depth)
        if any(o == "LOAD" for o, _ in p) and len(p) <= 32 and max_depth(p) <= 8:
            return p


def max_depth(prog) -> int:
    d = m = 0
    for o, _ in prog:
        if o in ("LOAD", "SCALAR"):
            d += 1
        elif o in BINARY:
            d -= 1
        m = max(m, d)
    return m


# ---- parity checker ----------------------------------
def _ordinal(a: np.ndarray) -> np.ndarray:
    if a.dtype == np.float32:
        i = a.view(np.int32).astype(np.int64)
        return np.where(i < 0, np.int64(-(2**31)) - i, i)
    i = a.view(np.int64)
    return np.where(i < 0, np.int64(-(2**63)) - i, i)


def ulp_distance(got: np.ndarray, want: np.ndarray) -> np.ndarray:
    """Ordinal ulp distance; +-0 are 0 apart; NaN vs NaN = 0, NaN vs number = huge."""
    got = np.asarray(got)
    want = np.asarray(want)
    d = np.abs(_ordinal(got) - _ordinal(want))
    gn, wn = np.isnan(got), np.isnan(want)
    d = np.where(gn & wn, 0, d)
    d = np.where(gn ^ wn, np.iinfo(np.int64).max, d)
    gi, wi = np.isinf(got), np.isinf(want)
    d = np.where((gi | wi) & (got != want) & ~(gn | wn), np.iinfo(np.int64).max, d)
    return d


def assert_elementwise(got, want, etype, max_ulp=0):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, (got.shape, want.shape)
    if got.size == 0:
        return
    if etype in INTS:
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, f"{bad.size} integer mismatches, first at {bad[0]}: {got[bad[0]]} vs {want[bad[0]]}"
        return
    d = ulp_distance(got, want)
    worst = int(d.max())
    if worst > max_ulp:
        i = int(np.argmax(d))
        raise AssertionError(f"{etype} element {i}: got {got[i]!r} want {want[i]!r} ({worst} ulp > {max_ulp})")


TOL = {"f32": 1e-5, "f64": 1e-12}


def assert_reduction(got, want, etype, kind, abs_scale=None):
    """Floats: |g - o| <= tol*|o| (1e-5 f32, 1e-12 f64); if o == 0, |g| <= tol*abs_scale.
    Integers and MIN/MAX: exact (min/max return an element)."""
    got = np.atleast_1d(np.asarray(got))
    want = np.atleast_1d(np.asarray(want))
    if etype in INTS or kind in ("MIN", "MAX", "MINMAX"):
        assert np.array_equal(got, want), (got, want)
        return
    tol = TOL[etype]
    for g, o in zip(got.astype(np.float64), want.astype(np.float64)):
        if o == 0:
            # the oracle's sum is exactly 0: only a cancellation residue relative
            # to the magnitudes summed (abs_scale = sum |v_i|) is tolerated, and
            # without that scale the result must be exactly 0
            scale = abs_scale if abs_scale is not None else 0.0
            assert abs(g) <= tol * scale, (g, o)
        else:
            assert abs(g - o) <= tol * abs(o), (g, o, abs(g - o) / abs(o))
