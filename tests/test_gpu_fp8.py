"""E4M3 / E5M2 storage types (SURVEY §8(f) row 3 "fp8 storage", reading R25) on
the GPU vs the oracle: element-wise results bit-exact (f32 program, one
saturating rounding), reductions (f32 results) within the f32 bar, min/max and
indices exact, dim sums, generator, views, builder."""
import random

import numpy as np
import pytest
import torch

import oracle
from gpu_util import RTORCH, TORCH, requires_gpu, to_dev, to_host
from progs import CATALOG, P, assert_reduction, n_operands, n_scalars, random_program

pytestmark = [pytest.mark.gpu, requires_gpu]
FP8 = ("e4m3", "e5m2")


@pytest.fixture(scope="module")
def ctxs():
    import paper_2508_11385_b200 as c
    from paper_2508_11385_b200 import _native as N
    return {"tma": c.Context(0), "interp": c.Context(0, flags=N.INIT_FORCE_INTERP)}


def run(ctx, etype, prog, ops, sc, kind=None, store=True, shape=None):
    n = ops[0].size
    m, c = shape or (n, 1)
    dev = [to_dev(o, etype) for o in ops]
    out = torch.empty(n, dtype=TORCH[etype], device="cuda") if store else None
    if kind is None:
        ctx.eval(etype, m, c, prog, dev, sc, out)
        torch.cuda.synchronize()
        return to_host(out, etype)
    if kind.startswith("INDEX"):
        r = torch.zeros(2, dtype=torch.int64, device="cuda")
    else:
        rl = c if kind == "SUM_DIM0" else (m if kind == "SUM_DIM1" else 2)
        r = torch.zeros(rl, dtype=RTORCH[etype], device="cuda")
    ctx.reduce(etype, m, c, prog, dev, sc, kind, r, out)
    torch.cuda.synchronize()
    res = int(r[0].item()) if kind.startswith("INDEX") else r.cpu().numpy()
    return res, (to_host(out, etype) if store else None)


def same_bits(etype, got, want):
    nan_w = np.isnan(oracle.to_float(etype, want))
    assert np.array_equal(nan_w, np.isnan(oracle.to_float(etype, got)))
    # +-0 compare equal; everything else bit-exact
    g, w = oracle.to_float(etype, got[~nan_w]), oracle.to_float(etype, want[~nan_w])
    assert np.array_equal(g, w)


@pytest.mark.parametrize("etype", FP8)
def test_generator_matches_oracle(ctxs, etype):
    t = torch.empty(100_003, dtype=TORCH[etype], device="cuda")
    ctxs["tma"].fill(t, "randu", stream=4, start=77)
    torch.cuda.synchronize()
    assert np.array_equal(to_host(t, etype), oracle.fill(etype, "randu", 100_003, stream=4, start=77))
    ctxs["tma"].fill(t, "iota")
    torch.cuda.synchronize()
    assert np.array_equal(to_host(t, etype), oracle.fill(etype, "iota", 100_003))


@pytest.mark.parametrize("etype", FP8)
@pytest.mark.parametrize("op", ["NEG", "ABS", "SQUARE", "SQRT", "EXP", "LOG"])
def test_unary_all_patterns(ctxs, etype, op):
    x = np.tile(np.arange(256, dtype=np.uint8), 13)  # several tiles + a ragged tail
    prog = P(f"L0 {op}")
    want = oracle.eval_program(etype, prog, [x])
    for name, ctx in ctxs.items():
        same_bits(etype, run(ctx, etype, prog, [x], []), want)


@pytest.mark.parametrize("etype", FP8)
@pytest.mark.parametrize("op", ["ADD", "SUB", "MUL", "DIV", "MIN", "MAX"])
def test_binary_all_pairs(ctxs, etype, op):
    a = np.repeat(np.arange(256, dtype=np.uint8), 256)  # every (a, b) pair
    b = np.tile(np.arange(256, dtype=np.uint8), 256)
    prog = P(f"L0 L1 {op}")
    want = oracle.eval_program(etype, prog, [a, b])
    same_bits(etype, run(ctxs["tma"], etype, prog, [a, b], []), want)


@pytest.mark.parametrize("etype", FP8)
@pytest.mark.parametrize("cat", sorted(CATALOG))
def test_catalog_programs(ctxs, etype, cat):
    prog = P(CATALOG[cat])
    ops = [oracle.fill(etype, "randu", 70_001, stream=s) for s in range(n_operands(prog))]
    sc = [2.5, 3.0][:n_scalars(prog)]
    want = oracle.eval_program(etype, prog, ops, sc)
    for name, ctx in ctxs.items():
        same_bits(etype, run(ctx, etype, prog, ops, sc), want)


@pytest.mark.parametrize("etype", FP8)
def test_random_programs(ctxs, etype):
    rng = random.Random(5 + len(etype))
    for trial in range(25):
        prog = random_program(rng, 3, "f32", n_ops=3)
        ops = [oracle.fill(etype, "randu", 4099, seed=trial, stream=s)
               for s in range(n_operands(prog))]
        sc = [2.5, -0.75]
        want = oracle.eval_program(etype, prog, ops, sc)
        for name, ctx in ctxs.items():
            same_bits(etype, run(ctx, etype, prog, ops, sc), want)


@pytest.mark.parametrize("etype", FP8)
@pytest.mark.parametrize("kind", ["ACCU", "NORM2", "MINMAX", "MEAN", "VAR", "STDDEV",
                                  "INDEX_MIN", "INDEX_MAX"])
@pytest.mark.parametrize("n", [1, 15, 1000, 300_007])
def test_reductions(ctxs, etype, kind, n):
    prog = P("L0 L1 MUL S0 L2 MUL ADD")
    ops = [oracle.fill(etype, "randu", n, stream=s) for s in range(3)]
    z = oracle.eval_program(etype, prog, ops, [3.0])
    stats = kind in ("MEAN", "VAR", "STDDEV", "INDEX_MIN", "INDEX_MAX")
    want = oracle.stats(etype, kind, z) if stats else oracle.reduce(etype, kind, z)
    for name, ctx in ctxs.items():
        got, zd = run(ctx, etype, prog, ops, [3.0], kind)
        assert np.array_equal(zd, z), name  # Z stored in the same pass
        if kind.startswith("INDEX"):
            assert got == want, name
        else:
            assert got.dtype == np.float32
            assert_reduction(got[:2] if kind == "MINMAX" else got[:1], want, "f32", kind,
                             abs_scale=float(np.abs(oracle.to_float(etype, z)).sum()) or 1.0)


# (1000, 333): scalar paths (m % 16 != 0); (4096, 1000) and (2048, 4099): m a
# multiple of the row tile with several column chunks, so dim1_kernel_b8's
# vector path (widen + pairwise f32 over a 16-byte unit) and the chunk combine run
DIM_SHAPES = [(1000, 333), (4096, 1000), (2048, 4099)]


@pytest.mark.parametrize("etype", FP8)
@pytest.mark.parametrize("dim", [0, 1])
@pytest.mark.parametrize("shape", DIM_SHAPES)
@pytest.mark.parametrize("which", ["tma", "interp"])
def test_sum_dims(ctxs, etype, dim, shape, which):
    m, n = shape
    X = oracle.fill(etype, "randu", m * n, stream=8)
    want = oracle.sum_dim(etype, dim, X, m, n)
    got, _ = run(ctxs[which], etype, P("L0"), [X], [], f"SUM_DIM{dim}", store=False,
                 shape=(m, n))
    assert got.dtype == np.float32
    np.testing.assert_allclose(got, want, rtol=1e-6, atol=0)


def test_builder_and_view(ctxs):
    import paper_2508_11385_b200 as coot
    ctx = ctxs["tma"]
    A = coot.Mat.randu(300, 200, "e4m3", stream=1, ctx=ctx)
    B = coot.Mat.randu(300, 200, "e4m3", stream=2, ctx=ctx)
    Z = (coot.exp(A % B) + 3 * B).eval(ctx)
    s = coot.accu(coot.exp(A % B) + 3 * B, ctx)
    torch.cuda.synchronize()
    assert s.dtype == torch.float32
    ha = oracle.fill("e4m3", "randu", 300 * 200, stream=1, n_rows=300)
    hb = oracle.fill("e4m3", "randu", 300 * 200, stream=2, n_rows=300)
    z = oracle.eval_program("e4m3", P("L0 L1 MUL EXP S0 L1 MUL ADD"), [ha, hb], [3.0])
    assert np.array_equal(to_host(Z.data, "e4m3"), z)
    assert_reduction(s.cpu().numpy()[:1], oracle.reduce("e4m3", "ACCU", z), "f32", "ACCU")
    # in-place diagonal update Z.diag() += 400: values past 448 saturate (R25)
    d = Z.diag()
    d += 400.0
    torch.cuda.synchronize()
    zz = z.copy()
    diag = np.arange(200) * 301
    zz[diag] = oracle.eval_program("e4m3", P("L0 S0 ADD"), [z[diag]], [400.0])
    assert np.array_equal(to_host(Z.data, "e4m3"), zz)
    assert np.all(oracle.to_float("e4m3", zz[diag]) <= 448.0)


@pytest.mark.parametrize("etype", FP8)
@pytest.mark.parametrize("scalar", [3.0, -1.5, 0.0078125])
def test_c2_every_input_triple(ctxs, etype, scalar):
    """Catalog c2 (exp(A % B) + s*C) on EVERY (a, b, c) triple of 8-bit patterns
    (2^24 elements, NaNs included): the fast path (cheap expf + a proof that the
    8-bit rounding cannot change, exact program otherwise) is bit-identical to
    the oracle's exact f32 program + one rounding, on the catalog kernel and on
    the interpreter; the accu of Z too."""
    i = np.arange(1 << 24, dtype=np.uint32)
    a, b, c = (i & 255).astype(np.uint8), ((i >> 8) & 255).astype(np.uint8), (i >> 16).astype(np.uint8)
    prog = P(CATALOG[2])
    want = oracle.eval_program(etype, prog, [a, b, c], [scalar])
    for name, ctx in ctxs.items():
        res, z = run(ctx, etype, prog, [a, b, c], [scalar], kind="MINMAX")
        same_bits(etype, z, want)
