"""Pins for the oracle's reductions: closed forms, exact rational sums,
textbook min/max, modular integer sums, chunked == unchunked."""
import numpy as np
import pytest

import oracle
from exactref import rounded_norm2, rounded_sum, same_bits

C2 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2),
      ("MUL", 0), ("ADD", 0)]
AXPY = [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)]


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_accu_of_ones_is_n(etype):
    for n in (0, 1, 7, 1000, 1 << 20, (1 << 24) + 3):
        v = np.ones(n, oracle.DTYPES[etype])
        assert oracle.reduce(etype, "ACCU", v) == np.float64(n).astype(oracle.DTYPES[etype])


def test_accu_of_iota_closed_form():
    # sum_{i<n} i = n(n-1)/2 exactly; rounded once to eT
    for n in (10, 1000, 123457, 1 << 22):
        v = np.arange(n, dtype=np.float64)
        assert oracle.reduce("f64", "ACCU", v) == n * (n - 1) // 2
        v32 = np.arange(n, dtype=np.float32)  # exact up to 2^24
        assert oracle.reduce("f32", "ACCU", v32) == np.float32(n * (n - 1) // 2)


def test_naive_f32_sum_would_stall_but_oracle_does_not():
    # R10: a running f32 sum of 2^25 ones stalls at 2^24; the oracle returns 2^25.
    v = np.ones(1 << 25, np.float32)
    assert oracle.reduce("f32", "ACCU", v) == np.float32(1 << 25)


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_accu_random_equals_rounded_exact_sum(etype):
    rng = np.random.default_rng(5)
    for n in (1, 2, 17, 100, 999):
        for scale in (1.0, 1e10):
            v = (rng.uniform(-1, 1, n) * scale).astype(oracle.DTYPES[etype])
            assert same_bits(oracle.reduce(etype, "ACCU", v), rounded_sum(v, etype))
            # same-sign data
            w = np.abs(v)
            assert same_bits(oracle.reduce(etype, "ACCU", w), rounded_sum(w, etype))


def test_accu_cancellation_exact():
    # 1e30 + 1 - 1e30 = 1 exactly (a naive float sum returns 0)
    v = np.array([1e30, 1.0, -1e30], np.float64)
    assert oracle.reduce("f64", "ACCU", v) == 1.0
    v32 = np.array([1e30, 1.0, -1e30], np.float32)
    assert oracle.reduce("f32", "ACCU", v32) == 1.0


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_norm2_closed_forms_and_exact(etype):
    dt = oracle.DTYPES[etype]
    for k in range(0, 8):
        assert oracle.reduce(etype, "NORM2", np.ones(4**k, dt)) == 2**k
    e = np.zeros(50, dt)
    e[17] = 1
    assert oracle.reduce(etype, "NORM2", e) == 1
    assert oracle.reduce(etype, "NORM2", np.array([3, 4], dt)) == 5
    assert oracle.reduce(etype, "NORM2", np.zeros(0, dt)) == 0
    rng = np.random.default_rng(6)
    for n in (1, 5, 64, 333):
        v = rng.uniform(-3, 3, n).astype(dt)
        assert same_bits(oracle.reduce(etype, "NORM2", v), rounded_norm2(v, etype))


@pytest.mark.parametrize("etype", ["f32", "f64", "u32", "s64"])
def test_min_max_minmax(etype):
    rng = np.random.default_rng(8)
    dt = oracle.DTYPES[etype]
    if etype in ("f32", "f64"):
        v = rng.normal(size=777).astype(dt)
    elif etype == "u32":
        v = rng.integers(0, 2**32, 777, dtype=np.uint64).astype(np.uint32)
    else:
        v = rng.integers(-2**63, 2**63 - 1, 777, dtype=np.int64)
    lo = min(v.tolist())
    hi = max(v.tolist())
    assert oracle.reduce(etype, "MIN", v) == lo
    assert oracle.reduce(etype, "MAX", v) == hi
    mm = oracle.reduce(etype, "MINMAX", v)
    assert mm[0] == lo and mm[1] == hi
    assert lo in v.tolist() and hi in v.tolist()  # attained


@pytest.mark.parametrize("etype", ["f32", "u32"])
def test_min_of_empty_is_contract_error_R13(etype):
    for kind in ("MIN", "MAX", "MINMAX"):
        with pytest.raises(oracle.OracleError):
            oracle.reduce(etype, kind, np.zeros(0, oracle.DTYPES[etype]))
    assert oracle.reduce(etype, "ACCU", np.zeros(0, oracle.DTYPES[etype])) == 0


def test_integer_accu_modular():
    rng = np.random.default_rng(9)
    u = rng.integers(0, 2**32, 5000, dtype=np.uint64).astype(np.uint32)
    assert int(oracle.reduce("u32", "ACCU", u)) == sum(int(x) for x in u) % 2**32
    s = rng.integers(-2**63, 2**63 - 1, 5000, dtype=np.int64)
    want = sum(int(x) for x in s) % 2**64
    want = want - 2**64 if want >= 2**63 else want
    assert int(oracle.reduce("s64", "ACCU", s)) == want


@pytest.mark.parametrize("etype", ["f32", "f64"])
def test_norm2_scale_invariance_far_from_one(etype):
    """norm2(2^e * v) = 2^e * norm2(v) exactly (power-of-two scaling is exact and
    commutes with the correctly rounded result) for e far outside where v^2 is a
    normal number of eT: pins the oracle's squares as wider than eT."""
    dt = oracle.DTYPES[etype]
    v = np.array([3, 4, 12, 84], dt)                     # norm2 = 85
    big, small = ((2.0 ** 100, 2.0 ** -100) if etype == "f32" else (2.0 ** 600, 2.0 ** -600))
    assert oracle.reduce(etype, "NORM2", v) == 85
    assert oracle.reduce(etype, "NORM2", (v * dt(big)).astype(dt)) == dt(85 * big)
    assert oracle.reduce(etype, "NORM2", (v * dt(small)).astype(dt)) == dt(85 * small)
    for k in range(0, 6):
        assert oracle.reduce(etype, "NORM2", np.full(4**k, small, dt)) == dt(2**k * small)


def test_norm2_rejected_for_integers():
    with pytest.raises(oracle.OracleError):
        oracle.reduce("u32", "NORM2", np.ones(3, np.uint32))


@pytest.mark.parametrize("etype,prog,sc,kind", [
    ("f32", C2, [3.0], "ACCU"), ("f32", AXPY, [2.5], "ACCU"), ("f64", AXPY, [2.5], "NORM2"),
    ("u32", [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("SCALAR", 0), ("LOAD", 2), ("MUL", 0),
             ("ADD", 0)], [7], "MINMAX"),
])
def test_chunked_is_bit_identical_to_unchunked(etype, prog, sc, kind):
    n = 100_003
    k = 1 + max(a for o, a in prog if o == "LOAD")
    fills = ["randu"] * k
    ops = [oracle.fill(etype, "randu", n, stream=s) for s in range(k)]
    z = oracle.eval_program(etype, prog, ops, sc)
    r = oracle.reduce(etype, kind, z)
    r2, z2 = oracle.run_chunked(etype, prog, fills, start=0, count=n, scalars=sc, kind=kind,
                                want_out=True, chunk=4099)
    assert np.array_equal(z.view(np.uint8), z2.view(np.uint8))
    assert np.array_equal(np.atleast_1d(r).view(np.uint8), np.atleast_1d(r2).view(np.uint8))


def test_accumulator_fed_in_chunks_equals_one_shot():
    v = oracle.fill("f32", "randu", 50_000, stream=4)
    acc = oracle.Accumulator("f32", "ACCU")
    for lo in range(0, v.size, 777):
        acc.add(v[lo:lo + 777])
    assert same_bits(acc.final(), oracle.reduce("f32", "ACCU", v))


def test_linearity_invariant():
    # accu(alpha*x + y) ~= alpha*accu(x) + accu(y) (up to the per-element rounding)
    n = 200_000
    x = oracle.fill("f32", "randu", n, stream=0)
    y = oracle.fill("f32", "randu", n, stream=1)
    z = oracle.eval_program("f32", AXPY, [x, y], [2.5])
    lhs = float(oracle.reduce("f32", "ACCU", z))
    rhs = 2.5 * float(oracle.reduce("f64", "ACCU", x.astype(np.float64))) + \
        float(oracle.reduce("f64", "ACCU", y.astype(np.float64)))
    assert abs(lhs - rhs) / rhs < 1e-6
    # statistical wiring check: E[2.5x + y] = 1.75
    assert abs(lhs / n - 1.75) < 0.01
