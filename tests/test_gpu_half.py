"""bf16 / f16 element types (reading R24) on the GPU vs
the oracle: element-wise results bit-exact (every node correctly rounded on
both sides), reductions within 1 ulp of the format, min/max/index exact."""
import random

import numpy as np
import pytest
import torch

import oracle
from gpu_util import TORCH, half_ulp, requires_gpu, to_dev, to_host
from progs import CATALOG, P, n_operands, n_scalars, random_program

pytestmark = [pytest.mark.gpu, requires_gpu]
HALF = ("bf16", "f16")


@pytest.fixture(scope="module")
def coot():
    import paper_2508_11385_b200 as c
    return c


@pytest.fixture(scope="module")
def ctxs(coot):
    from paper_2508_11385_b200 import _native as N
    return {"tma": coot.Context(0), "interp": coot.Context(0, flags=N.INIT_FORCE_INTERP)}


def inputs(etype, n, k, seed=42):
    # randu shifted to [0.25, 1.25): log/sqrt/div stay in-domain
    shift = P("L0 S0 ADD")
    return [oracle.eval_program(etype, shift, [oracle.fill(etype, "randu", n, seed=seed, stream=s)],
                                [0.25]) for s in range(k)]


def bits(a):
    return np.asarray(a).view(np.uint16)


def run(ctx, etype, prog, ops, sc, kind=None, n_out=True):
    n = ops[0].size
    dev = [to_dev(o, etype) for o in ops]
    out = torch.empty(n, dtype=TORCH[etype], device="cuda") if n_out else None
    if kind is None:
        ctx.eval(etype, n, 1, prog, dev, sc, out)
        torch.cuda.synchronize()
        return to_host(out, etype)
    dt = torch.int64 if kind.startswith("INDEX") else TORCH[etype]
    r = torch.zeros(2, dtype=dt, device="cuda")
    ctx.reduce(etype, n, 1, prog, dev, sc, kind, r, out)
    torch.cuda.synchronize()
    if kind.startswith("INDEX"):
        return int(r[0].item())
    h = to_host(r, etype)
    return h[:2] if kind == "MINMAX" else h[:1]


@pytest.mark.parametrize("etype", HALF)
def test_generator_matches_oracle(ctxs, etype):
    t = torch.empty(100_003, dtype=TORCH[etype], device="cuda")
    ctxs["tma"].fill(t, "randu", stream=4, start=77)
    torch.cuda.synchronize()
    assert np.array_equal(bits(to_host(t, etype)), bits(oracle.fill(etype, "randu", 100_003,
                                                                    stream=4, start=77)))


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("cat", sorted(CATALOG))
def test_catalog_programs_bit_exact(ctxs, etype, cat):
    prog = P(CATALOG[cat])
    n = 70_001
    ops = inputs(etype, n, n_operands(prog))
    sc = [2.5, 3.0][:n_scalars(prog)]
    want = oracle.eval_program(etype, prog, ops, sc)
    for name, ctx in ctxs.items():
        got = run(ctx, etype, prog, ops, sc)
        d = half_ulp(got, want)
        assert d.max() == 0, (name, cat, int(np.argmax(d)))


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("op", ["EXP", "LOG", "SQRT", "SQUARE"])
def test_unary_exhaustive(ctxs, etype, op):
    """Every one of the 65536 bit patterns through each rounding unary op: covers
    the f32 fast path and the f64 fallback near rounding midpoints (R24)."""
    pats = np.arange(1 << 16, dtype=np.uint16)
    x = pats if etype == "bf16" else pats.view(np.float16)
    prog = P(f"L0 {op}")
    want = oracle.eval_program(etype, prog, [x])
    for name, ctx in ctxs.items():
        got = run(ctx, etype, prog, [x], [])
        nan_w = np.isnan(oracle.to_float(etype, want))
        assert np.array_equal(nan_w, np.isnan(oracle.to_float(etype, got))), name
        assert np.array_equal(bits(got)[~nan_w], bits(want)[~nan_w]), (
            name, int(np.nonzero(bits(got)[~nan_w] != bits(want)[~nan_w])[0][0]))


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("op", ["ADD", "SUB", "MUL", "DIV"])
def test_binary_dense_sample(ctxs, etype, op):
    """One operand exhaustive (all finite patterns), the other a fixed spread of
    magnitudes: subnormal, overflow and tie cases of the single rounding.  The
    subnormal b (2^-130 bf16, 2^-20 f16) makes ADD / SUB of two subnormals
    exact-or-tie cases that a flush-to-zero packed instruction would get wrong."""
    pats = np.arange(1 << 16, dtype=np.uint16)
    a = pats if etype == "bf16" else pats.view(np.float16)
    sub = 2.0 ** -130 if etype == "bf16" else 2.0 ** -20
    for bval in (3.0, -0.375, 1.0 / 3.0, 1e-3, 300.0, sub, -3 * sub):
        b = np.full(a.size, oracle.half_from_double(etype, bval), dtype=np.uint16)
        b = b if etype == "bf16" else b.view(np.float16)
        prog = P(f"L0 L1 {op}")
        want = oracle.eval_program(etype, prog, [a, b])
        got = run(ctxs["tma"], etype, prog, [a, b], [])
        nan_w = np.isnan(oracle.to_float(etype, want))
        assert np.array_equal(nan_w, np.isnan(oracle.to_float(etype, got)))
        assert np.array_equal(bits(got)[~nan_w], bits(want)[~nan_w]), (op, bval)


@pytest.mark.parametrize("etype", HALF)
def test_random_programs_bit_exact(ctxs, etype):
    rng = random.Random(77 + len(etype))
    for trial in range(25):
        prog = random_program(rng, 3, "f32", n_ops=3)   # the full float op set
        ops = inputs(etype, 3001, n_operands(prog), seed=trial)
        sc = [2.5, -0.75]
        want = oracle.eval_program(etype, prog, ops, sc)
        for name, ctx in ctxs.items():
            got = run(ctx, etype, prog, ops, sc)
            nan_w = np.isnan(oracle.to_float(etype, want))
            nan_g = np.isnan(oracle.to_float(etype, got))
            assert np.array_equal(nan_w, nan_g), (name, prog)
            # +-0 compare equal (ordinal distance 0); everything else bit-exact
            assert half_ulp(got[~nan_w], want[~nan_w]).max(initial=0) == 0, (name, prog)


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("kind", ["ACCU", "NORM2", "MEAN", "VAR", "STDDEV", "MINMAX",
                                  "INDEX_MIN", "INDEX_MAX"])
@pytest.mark.parametrize("n", [1, 7, 1000, 300_007])
def test_reductions(ctxs, etype, kind, n):
    prog = P("L0 L1 MUL S0 L2 MUL ADD")
    ops = inputs(etype, n, 3)
    z = oracle.eval_program(etype, prog, ops, [3.0])
    if kind in ("MEAN", "VAR", "STDDEV", "INDEX_MIN", "INDEX_MAX"):
        want = oracle.stats(etype, kind, z)
    else:
        want = oracle.reduce(etype, kind, z)
    for name, ctx in ctxs.items():
        got = run(ctx, etype, prog, ops, [3.0], kind, n_out=False)
        if kind.startswith("INDEX"):
            assert got == want, name
        elif kind == "MINMAX":
            assert np.array_equal(bits(got), bits(want)), name
        else:
            assert half_ulp(got, np.atleast_1d(want)).max() <= 1, (name, got, want)


# (1000, 333): the row tile (1024 rows) exceeds m, scalar path; (4096, 1000)
# and (2048, 4099): whole row tiles and several column chunks (vector path)
DIM_SHAPES = [(1000, 333), (4096, 1000), (2048, 4099)]


@pytest.mark.parametrize("etype", HALF)
@pytest.mark.parametrize("dim", [0, 1])
@pytest.mark.parametrize("shape", DIM_SHAPES)
@pytest.mark.parametrize("which", ["tma", "interp"])
def test_sum_dims(ctxs, etype, dim, shape, which):
    m, n = shape
    X = oracle.fill(etype, "randu", m * n, stream=8)
    want = oracle.sum_dim(etype, dim, X, m, n)
    dev = to_dev(X, etype)
    r = torch.zeros(n if dim == 0 else m, dtype=TORCH[etype], device="cuda")
    ctxs[which].reduce(etype, m, n, P("L0"), [dev], [], f"SUM_DIM{dim}", r)
    torch.cuda.synchronize()
    assert half_ulp(to_host(r, etype), want).max() <= 1


def test_builder_half(coot, ctxs):
    A = coot.Mat.randu(512, 300, "bf16", stream=1, ctx=ctxs["tma"])
    B = coot.Mat.randu(512, 300, "bf16", stream=2, ctx=ctxs["tma"])
    Z = coot.exp(A % B) + 3 * B
    out = Z.eval(ctxs["tma"])
    torch.cuda.synchronize()
    ha = oracle.fill("bf16", "randu", 512 * 300, stream=1, n_rows=512)
    hb = oracle.fill("bf16", "randu", 512 * 300, stream=2, n_rows=512)
    want = oracle.eval_program("bf16", P("L0 L1 MUL EXP S0 L1 MUL ADD"), [ha, hb], [3.0])
    assert np.array_equal(bits(to_host(out.data, "bf16")), bits(want))
