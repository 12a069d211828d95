"""norm2 and var over the whole f32 / bf16 range, and f64 norm2 over the whole
f64 range (R12, R22).

The device squares f32 / bf16 values in f32 inside a 16-byte unit; a unit with
an element (or, for var, a deviation from the shift) outside [2^-63, 2^62) is
squared and summed in f64 instead.  These cases put whole vectors, or single
units, outside that range — where f32 squares would overflow to inf or flush
to zero — and compare with the oracle (long-double squares) at the reduction
bar: 1e-5 relative for f32, 1 ulp for bf16.  Every driver (TMA, interpreter,
LDG for f32) sees the same inputs."""
import os

import numpy as np
import pytest
import torch

import oracle
from gpu_util import TORCH, half_ulp, requires_gpu, to_dev, to_host
from progs import P, assert_reduction

pytestmark = [pytest.mark.gpu, requires_gpu]


@pytest.fixture(scope="module")
def ctxs():
    import paper_2508_11385_b200 as coot
    from paper_2508_11385_b200 import _native as N
    old = os.environ.get("COOT_DRIVER")
    os.environ["COOT_DRIVER"] = "0"
    try:
        ldg = coot.Context(0)
    finally:
        if old is None:
            os.environ.pop("COOT_DRIVER", None)
        else:
            os.environ["COOT_DRIVER"] = old
    return {"tma": coot.Context(0), "interp": coot.Context(0, flags=N.INIT_FORCE_INTERP),
            "ldg": ldg}


def scaled(etype, n, scale, shift=0.0, stream=0):
    """(randu + shift) * scale, rounded once per node to eT (the oracle's program)."""
    x = oracle.fill(etype, "randu", n, stream=stream)
    return oracle.eval_program(etype, P("L0 S0 ADD S1 MUL"), [x], [shift, scale])


def gpu(ctx, etype, x, kind):
    r = torch.zeros(2, dtype=TORCH[etype], device="cuda")
    ctx.reduce(etype, x.size, 1, P("L0"), [to_dev(x, etype)], [], kind, r)
    torch.cuda.synchronize()
    return to_host(r, etype)[:1]


def want_of(etype, kind, x):
    return oracle.stats(etype, kind, x) if kind in ("VAR", "STDDEV") else \
        oracle.reduce(etype, "NORM2", x)


def check(ctxs, etype, kind, x):
    want = np.atleast_1d(want_of(etype, kind, x))
    assert np.all(np.isfinite(want.astype(np.float64))), want
    for name, ctx in ctxs.items():
        if etype == "bf16" and name == "ldg":
            continue  # 16-bit types run on the TMA driver only
        got = gpu(ctx, etype, x, kind)
        if etype == "bf16":
            assert half_ulp(got, want).max() <= 1, (name, kind, got, want)
        else:
            assert_reduction(got, want, etype, kind), (name, kind)


@pytest.mark.parametrize("etype", ["f32", "bf16"])
@pytest.mark.parametrize("scale", [1e-25, 1e-21, 2.0 ** -63, 2.0 ** 62, 1e25])
@pytest.mark.parametrize("n", [1, 7, 100_003])
def test_norm2_tiny_and_huge(ctxs, etype, scale, n):
    """f32 squares of 1e-25 are 0 and of 1e25 are inf; the f64 route is exact."""
    check(ctxs, etype, "NORM2", scaled(etype, n, scale, shift=0.5))


@pytest.mark.parametrize("etype", ["f32", "bf16"])
def test_norm2_isolated_outliers(ctxs, etype):
    """Mostly in-range units (f32 fast path) with a few out-of-range elements:
    the units holding them switch to f64, the rest stay on the f32 path."""
    x = scaled(etype, 300_007, 1.0, shift=0.25)
    big = oracle.eval_program(etype, P("S0"), [x[:1]], [3e20])[0]
    tiny = oracle.eval_program(etype, P("S0"), [x[:1]], [1e-30])[0]
    for i in (0, 5, 4096, 123_457, 300_006):
        x[i] = big
    for i in (1, 77, 200_000):
        x[i] = tiny
    check(ctxs, etype, "NORM2", x)


@pytest.mark.parametrize("etype", ["f32", "bf16"])
@pytest.mark.parametrize("scale", [2e19, 3e18, 1e-18])
@pytest.mark.parametrize("kind", ["VAR", "STDDEV"])
def test_var_large_and_small_spread(ctxs, etype, scale, kind):
    """(randu - 0.5) * scale: deviations up to 1e19 square past f32's range
    (the old f32 route returned inf); 1e-18 puts some below 2^-63."""
    check(ctxs, etype, kind, scaled(etype, 100_003, scale, shift=-0.5))


@pytest.mark.parametrize("etype", ["f32", "bf16"])
def test_norm2_nonfinite(ctxs, etype):
    x = scaled(etype, 10_001, 1.0)
    for name, ctx in ctxs.items():
        if etype == "bf16" and name == "ldg":
            continue
        y = x.copy()
        y[5000] = np.inf if etype == "f32" else oracle.half_from_double(etype, float("inf"))
        assert np.isinf(oracle.to_float(etype, gpu(ctx, etype, y, "NORM2"))[0]), name
        y[5001] = np.nan if etype == "f32" else oracle.half_from_double(etype, float("nan"))
        assert np.isnan(oracle.to_float(etype, gpu(ctx, etype, y, "NORM2"))[0]), name


# ---- f64 norm2 over the whole f64 range (R12): scaled sum of squares -------
@pytest.mark.parametrize("scale", [1e300, 2.0 ** 600, 1e154, 1e-154, 2.0 ** -600, 1e-300,
                                   2.0 ** -1060, 1.0])
@pytest.mark.parametrize("n", [1, 7, 100_003])
def test_f64_norm2_whole_range(ctxs, scale, n):
    """f64 squares of 1e300 overflow and of 1e-300 flush to 0; the scaled
    accumulator (value = s 2^es) keeps norm2 within 1e-12 of the oracle's
    long-double result, on every driver, down to subnormal inputs."""
    check(ctxs, "f64", "NORM2", scaled("f64", n, scale, shift=0.5))


def test_f64_norm2_isolated_outliers_and_shards(ctxs):
    """Mostly in-range data with a few 1e250 / 1e-300 elements (those units and
    the threads that saw them take the scaled path); also the rank-order
    combine of shard partials carries the scale exponent."""
    import paper_2508_11385_b200 as coot
    x = scaled("f64", 300_007, 1.0, shift=0.25)
    for i in (0, 5, 4096, 123_457, 300_006):
        x[i] = 3e250
    for i in (1, 77, 200_000):
        x[i] = 1e-300
    check(ctxs, "f64", "NORM2", x)
    want = oracle.reduce("f64", "NORM2", x)
    ctx = ctxs["tma"]
    d = to_dev(x, "f64")
    nparts = 5
    parts = torch.zeros(nparts * 4, dtype=torch.int64, device="cuda")
    for r in range(nparts):
        b, e = coot.shard_range(x.size, r, nparts, 16)
        ctx.reduce_partial("f64", e - b, 1, P("L0"), [d[b:e]], [], "NORM2", parts[4 * r:4 * r + 4])
    res = torch.zeros(2, dtype=torch.float64, device="cuda")
    ctx.combine("f64", "NORM2", parts, nparts, 1, res)
    torch.cuda.synchronize()
    assert_reduction(res[0].item(), want, "f64", "NORM2")


def test_f64_norm2_nonfinite(ctxs):
    x = scaled("f64", 10_001, 1e200)
    for name, ctx in ctxs.items():
        y = x.copy()
        y[5000] = np.inf
        assert np.isinf(gpu(ctx, "f64", y, "NORM2")[0]), name
        y[5001] = np.nan
        assert np.isnan(gpu(ctx, "f64", y, "NORM2")[0]), name
