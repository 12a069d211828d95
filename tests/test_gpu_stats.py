"""mean / var / stddev and index_min / index_max
on the GPU against the oracle: one launch each, every driver, shard combine."""
import random

import numpy as np
import pytest
import torch

import oracle
from gpu_util import TORCH, requires_gpu, to_dev, to_host
from progs import ALL, FLOATS, P, assert_reduction, random_program

pytestmark = [pytest.mark.gpu, requires_gpu]
STATS = ["MEAN", "VAR", "STDDEV"]


@pytest.fixture(scope="module")
def coot():
    import paper_2508_11385_b200 as c
    return c


@pytest.fixture(scope="module")
def ctxs(coot):
    import os

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


def gpu_reduce(ctx, etype, prog, ops, sc, kind, offset=0):
    n = ops[0].size
    dev = [to_dev(o, etype, offset) for o in ops]
    dt = torch.int64 if kind.startswith("INDEX") else TORCH[etype]
    r = torch.zeros(2, dtype=dt, device="cuda")
    before = ctx.stats()["launches"]
    ctx.reduce(etype, n, 1, prog, dev, sc, kind, r)
    assert ctx.stats()["launches"] == before + 1
    torch.cuda.synchronize()
    return int(r[0].item()) if kind.startswith("INDEX") else to_host(r, etype)[0]


@pytest.mark.parametrize("etype", FLOATS)
@pytest.mark.parametrize("kind", STATS)
@pytest.mark.parametrize("n", [1, 2, 3, 17, 1000, 100_003, 3_000_001])
def test_statistics_plain(ctxs, etype, kind, n):
    x = oracle.fill(etype, "randu", n, stream=0)
    want = oracle.stats(etype, kind, x)
    for name, ctx in ctxs.items():
        got = gpu_reduce(ctx, etype, P("L0"), [x], [], kind)
        assert_reduction(got, want, etype, "ACCU", abs_scale=1.0), name


@pytest.mark.parametrize("etype", FLOATS)
def test_statistics_closed_forms_and_shift(ctxs, etype):
    dt = oracle.DTYPES[etype]
    ctx = ctxs["tma"]
    n = 1_000_000
    iota = np.arange(1, n + 1, dtype=dt)
    assert gpu_reduce(ctx, etype, P("L0"), [iota], [], "MEAN") == dt((n + 1) / 2)
    var = gpu_reduce(ctx, etype, P("L0"), [iota], [], "VAR")
    assert abs(float(var) - n * (n + 1) / 12) <= {"f32": 1e-5, "f64": 1e-12}[etype] * n * (n + 1) / 12
    const = np.full(123_457, 7.5, dt)
    assert gpu_reduce(ctx, etype, P("L0"), [const], [], "VAR") == 0
    # a large offset with a small spread: the shifted sums keep the variance
    x = (oracle.fill(etype, "randu", 200_003, stream=3) + dt(1e4)).astype(dt)
    want = oracle.stats(etype, "VAR", x)
    assert_reduction(gpu_reduce(ctx, etype, P("L0"), [x], [], "VAR"), want, etype, "ACCU")


@pytest.mark.parametrize("etype", FLOATS)
@pytest.mark.parametrize("kind", STATS)
def test_statistics_of_fused_expressions(ctxs, etype, kind):
    rng = random.Random(5)
    n = 70_001
    for trial in range(6):
        prog = random_program(rng, 3, etype, n_ops=3)
        ops = [oracle.fill(etype, "randu", n, stream=s) + oracle.DTYPES[etype](0.25)
               for s in range(3)]
        z = oracle.eval_program(etype, prog, ops, [2.5, -0.75])
        if not np.all(np.isfinite(z)):
            continue
        want = oracle.stats(etype, kind, z)
        for name, ctx in ctxs.items():
            got = gpu_reduce(ctx, etype, prog, ops, [2.5, -0.75], kind)
            assert_reduction(got, want, etype, "ACCU", abs_scale=1.0), (name, prog)


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("kind", ["INDEX_MIN", "INDEX_MAX"])
@pytest.mark.parametrize("offset", [0, 1])
def test_index_min_max_first_occurrence(ctxs, etype, kind, offset):
    rng = np.random.default_rng(9)
    n = 1_000_003
    dt = oracle.DTYPES[etype]
    x = rng.integers(0, 1000, n).astype(dt)  # many ties: the FIRST index must win
    want = oracle.stats(etype, kind, x)
    for name, ctx in ctxs.items():
        assert gpu_reduce(ctx, etype, P("L0"), [x], [], kind, offset) == want, name
    # extreme value at both ends and in the middle
    x[:] = dt(500)
    for pos in (n - 1, 0, n // 2):
        x[pos] = dt(7) if kind == "INDEX_MIN" else dt(999)
        assert gpu_reduce(ctxs["tma"], etype, P("L0"), [x], [], kind) == oracle.stats(etype, kind, x)


def test_index_of_expression_and_all_equal(ctxs):
    x = np.full(1 << 20, np.uint32(0xFFFFFFFF))  # identity value everywhere
    assert gpu_reduce(ctxs["tma"], "u32", P("L0"), [x], [], "INDEX_MIN") == 0
    assert gpu_reduce(ctxs["tma"], "u32", P("L0"), [x], [], "INDEX_MAX") == 0
    a = oracle.fill("f32", "randu", 500_000, stream=1)
    b = oracle.fill("f32", "randu", 500_000, stream=2)
    z = oracle.eval_program("f32", P("L0 L1 SUB ABS"), [a, b], [])
    for kind in ("INDEX_MIN", "INDEX_MAX"):
        want = oracle.stats("f32", kind, z)
        for ctx in ctxs.values():
            assert gpu_reduce(ctx, "f32", P("L0 L1 SUB ABS"), [a, b], [], kind) == want


@pytest.mark.parametrize("kind", ["MEAN", "VAR", "STDDEV", "INDEX_MIN", "INDEX_MAX"])
def test_statistics_shard_combine(coot, ctxs, kind):
    ctx = ctxs["tma"]
    n = 2_000_003
    x = oracle.fill("f64", "randu", n, stream=6)
    d = to_dev(x, "f64")
    want = oracle.stats("f64", kind, x)
    for nparts in (1, 3, 8):
        parts = torch.zeros(nparts * 4, dtype=torch.int64, device="cuda")
        for r in range(nparts):
            b, e = coot.shard_range(n, r, nparts, 16)
            ctx.reduce_partial("f64", e - b, 1, P("L0"), [d[b:e]], [], kind, parts[4 * r:4 * r + 4])
        dt = torch.int64 if kind.startswith("INDEX") else torch.float64
        res = torch.zeros(2, dtype=dt, device="cuda")
        ctx.combine("f64", kind, parts, nparts, 1, res)
        torch.cuda.synchronize()
        if kind.startswith("INDEX"):
            assert int(res[0].item()) == want
        else:
            assert_reduction(res[0].item(), want, "f64", "ACCU")


def test_statistics_errors(coot, ctxs):
    ctx = ctxs["tma"]
    u = torch.ones(10, dtype=torch.uint32, device="cuda")
    r = torch.zeros(2, dtype=torch.uint32, device="cuda")
    for kind in ("MEAN", "VAR", "STDDEV"):
        with pytest.raises(coot.CootError):
            ctx.reduce("u32", 10, 1, P("L0"), [u], [], kind, r)
    e = torch.empty(0, device="cuda")
    for kind in ("MEAN", "VAR", "INDEX_MIN"):
        with pytest.raises(coot.CootError):
            ctx.reduce("f32", 0, 1, P("L0"), [e], [], kind, torch.zeros(2, device="cuda"))


def test_builder_statistics(coot, ctxs):
    A = coot.Mat.randu(1000, 300, "f64", stream=2, ctx=ctxs["tma"])
    h = oracle.fill("f64", "randu", 300_000, stream=2, n_rows=1000)
    assert_reduction(coot.mean(A).item(), oracle.stats("f64", "MEAN", h), "f64", "ACCU")
    assert_reduction(coot.var(2 * A).item(),
                     oracle.stats("f64", "VAR", oracle.eval_program("f64", P("S0 L0 MUL"), [h], [2.0])),
                     "f64", "ACCU")
    assert coot.index_max(A).item() == oracle.stats("f64", "INDEX_MAX", h)
