"""GPU parity of the fused element-wise pass + terminal reductions (K1/K2)
against the oracle, through the C ABI.  Sizes span several tiles and ragged
tails; pointer offsets exercise the head/tail and misaligned paths."""
import random

import numpy as np
import pytest
import torch

import oracle
from gpu_util import TORCH, empty_dev, requires_gpu, to_dev, to_host
from progs import (ALL, CATALOG, C2, FLOATS, INTS, P, assert_elementwise, assert_reduction,
                   legal, n_operands, n_scalars, random_program)

pytestmark = [pytest.mark.gpu, requires_gpu]


@pytest.fixture(scope="module")
def coot():
    import paper_2508_11385_b200 as c
    return c


@pytest.fixture(scope="module")
def ctx(coot):
    return coot.Context(0)


@pytest.fixture(scope="module")
def ctx_interp(coot):
    from paper_2508_11385_b200 import _native as N
    return coot.Context(0, flags=N.INIT_FORCE_INTERP)


SCAL = {"f32": [2.5, 3.0, -0.75], "f64": [2.5, 3.0, -0.75], "u32": [7, 0xFFFFFFF0, 3],
        "s64": [7, -3, 2**40 + 1]}


def make_inputs(etype, n, k, *, seed=42, positive=True):
    if etype in FLOATS and positive:
        # randu in [0,1) shifted to [0.25, 1.25): keeps log/sqrt/div in-domain
        ops = [oracle.fill(etype, "randu", n, seed=seed, stream=s) + oracle.DTYPES[etype](0.25)
               for s in range(k)]
    else:
        ops = [oracle.fill(etype, "randu", n, seed=seed, stream=s) for s in range(k)]
    return [np.ascontiguousarray(o, dtype=oracle.DTYPES[etype]) for o in ops]


def run_eval(ctx, etype, prog, host_ops, scalars, offsets=None):
    n = host_ops[0].size
    offsets = offsets or [0] * (len(host_ops) + 1)
    dev = [to_dev(o, etype, offsets[i]) for i, o in enumerate(host_ops)]
    out = empty_dev(n, etype, offsets[-1])
    ctx.eval(etype, n, 1, prog, dev, scalars, out)
    torch.cuda.synchronize()
    return to_host(out, etype)


def run_reduce(ctx, etype, prog, host_ops, scalars, kind, with_out=False, offsets=None):
    n = host_ops[0].size
    offsets = offsets or [0] * (len(host_ops) + 1)
    dev = [to_dev(o, etype, offsets[i]) for i, o in enumerate(host_ops)]
    res = torch.zeros(2, dtype=TORCH[etype], device="cuda")
    out = empty_dev(n, etype, offsets[-1]) if with_out else None
    ctx.reduce(etype, n, 1, prog, dev, scalars, kind, res, out)
    torch.cuda.synchronize()
    r = to_host(res, etype)
    r = r[:2] if kind == "MINMAX" else r[0]
    return (r, to_host(out, etype)) if with_out else r


def oracle_reduce(etype, kind, z):
    return oracle.reduce(etype, kind, z)


def abs_scale(z):
    return float(np.sum(np.abs(z.astype(np.float64))))


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("cat", sorted(CATALOG))
def test_catalog_programs_eval_and_reduce(ctx, etype, cat):
    prog = P(CATALOG[cat])
    if not legal(prog, etype):
        pytest.skip("op not defined for integers (R9)")
    n = 100_003
    ops = make_inputs(etype, n, n_operands(prog))
    sc = SCAL[etype][:n_scalars(prog)]
    want = oracle.eval_program(etype, prog, ops, sc)
    got = run_eval(ctx, etype, prog, ops, sc)
    assert ctx.stats()["last_path"] == cat
    assert_elementwise(got, want, etype, max_ulp=0)
    kinds = ["ACCU", "MIN", "MAX", "MINMAX"] + (["NORM2"] if etype in FLOATS else [])
    for kind in kinds:
        r = run_reduce(ctx, etype, prog, ops, sc, kind)
        assert_reduction(r, oracle_reduce(etype, kind, want), etype, kind, abs_scale(want))


@pytest.mark.parametrize("etype", ALL)
def test_interpreter_random_programs(ctx, etype):
    rng = random.Random(2024 + ALL.index(etype))
    n = 5003
    for trial in range(40):
        depth = 2 + trial % 3
        nops = 3 if trial % 4 else 6
        prog = random_program(rng, depth, etype, n_ops=nops, n_sc=2)
        ops = make_inputs(etype, n, max(nops, n_operands(prog)), seed=trial)
        ops = ops[:n_operands(prog)]
        sc = SCAL[etype][:2]
        want = oracle.eval_program(etype, prog, ops, sc)
        got = run_eval(ctx, etype, prog, ops, sc)
        # every node is correctly rounded (EXP / LOG included, R6): bit-exact
        assert_elementwise(got, want, etype, max_ulp=0)
        if np.all(np.isfinite(want.astype(np.float64))) or etype in INTS:
            kind = "ACCU" if trial % 2 else "MINMAX"
            r = run_reduce(ctx, etype, prog, ops, sc, kind)
            assert_reduction(r, oracle_reduce(etype, kind, want), etype, kind, abs_scale(want))


@pytest.mark.parametrize("etype", ALL)
def test_interpreter_large_class_deep_and_wide(ctx, etype):
    # 8 operands, stack depth 8: L0 L1 ... L7 then 7 binary ops
    ops_names = ["ADD", "MUL", "SUB", "MAX", "ADD", "MIN", "MUL"]
    prog = [("LOAD", k) for k in range(8)] + [(o, 0) for o in ops_names]
    n = 70_001
    ops = make_inputs(etype, n, 8)
    want = oracle.eval_program(etype, prog, ops, [])
    got = run_eval(ctx, etype, prog, ops, [])
    assert ctx.stats()["last_path"] == -1
    assert_elementwise(got, want, etype, max_ulp=0)
    r = run_reduce(ctx, etype, prog, ops, [], "ACCU")
    assert_reduction(r, oracle_reduce(etype, "ACCU", want), etype, "ACCU", abs_scale(want))


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 255, 256, 257, 1023, 1025,
                               256 * 8 * 148 + 3, (1 << 20) + 5])
def test_sizes_and_ragged_tails(ctx, etype, n):
    prog = P(CATALOG[3])  # X % Y + s*Z
    ops = make_inputs(etype, n, 3)
    sc = SCAL[etype][:1]
    want = oracle.eval_program(etype, prog, ops, sc)
    r, got = run_reduce(ctx, etype, prog, ops, sc, "ACCU", with_out=True)
    assert_elementwise(got, want, etype, max_ulp=0)
    assert_reduction(r, oracle_reduce(etype, "ACCU", want), etype, "ACCU", abs_scale(want))


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("offsets", [(0, 0, 0, 0), (1, 1, 1, 1), (3, 3, 3, 3), (0, 1, 2, 3),
                                     (2, 2, 2, 0), (1, 0, 1, 1)])
def test_pointer_offsets(ctx, etype, offsets):
    prog = P(CATALOG[3])
    n = 30_011
    ops = make_inputs(etype, n, 3)
    sc = SCAL[etype][:1]
    want = oracle.eval_program(etype, prog, ops, sc)
    r, got = run_reduce(ctx, etype, prog, ops, sc, "MINMAX", with_out=True, offsets=list(offsets))
    assert_elementwise(got, want, etype, max_ulp=0)
    assert_reduction(r, oracle_reduce(etype, "MINMAX", want), etype, "MINMAX")
    r = run_reduce(ctx, etype, prog, ops, sc, "ACCU", offsets=list(offsets))
    assert_reduction(r, oracle_reduce(etype, "ACCU", want), etype, "ACCU", abs_scale(want))


@pytest.mark.parametrize("etype", ALL)
def test_k1_equals_k2_bitwise(ctx, ctx_interp, etype):
    n = 200_003
    for cat, s in sorted(CATALOG.items()):
        prog = P(s)
        if not legal(prog, etype):
            continue
        ops = make_inputs(etype, n, n_operands(prog))
        sc = SCAL[etype][:n_scalars(prog)]
        a = run_eval(ctx, etype, prog, ops, sc)
        b = run_eval(ctx_interp, etype, prog, ops, sc)
        assert ctx_interp.stats()["last_path"] == -1
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), f"catalog {cat} eval differs"
        for kind in ["ACCU", "MINMAX"] + (["NORM2"] if etype in FLOATS else []):
            ra = run_reduce(ctx, etype, prog, ops, sc, kind)
            rb = run_reduce(ctx_interp, etype, prog, ops, sc, kind)
            assert np.array_equal(np.atleast_1d(ra).view(np.uint8),
                                  np.atleast_1d(rb).view(np.uint8)), (cat, kind, ra, rb)


@pytest.mark.parametrize("etype", ALL)
def test_determinism_run_to_run(ctx, etype):
    prog = C2 if etype in FLOATS else P(CATALOG[3])
    n = 1_000_003
    ops = make_inputs(etype, n, 3)
    sc = SCAL[etype][:1]
    dev = [to_dev(o, etype) for o in ops]
    res = [torch.zeros(2, dtype=TORCH[etype], device="cuda") for _ in range(3)]
    for r in res:
        ctx.reduce(etype, n, 1, prog, dev, sc, "ACCU", r)
    torch.cuda.synchronize()
    h = [to_host(r, etype) for r in res]
    assert all(np.array_equal(h[0].view(np.uint8), x.view(np.uint8)) for x in h[1:])


def test_one_launch_per_call_and_none_before_assignment(coot, ctx):
    n = 1 << 16
    A = coot.Mat.randu(n, 1, "f32", stream=0, ctx=ctx)
    B = coot.Mat.randu(n, 1, "f32", stream=1, ctx=ctx)
    before = ctx.stats()["launches"]
    e = coot.exp(A % B) + 3 * A - B / 2.0  # building: no launch
    assert ctx.stats()["launches"] == before
    e.eval(ctx)
    assert ctx.stats()["launches"] == before + 1
    coot.accu(e, ctx)
    assert ctx.stats()["launches"] == before + 2
    coot.minmax(e, ctx)
    assert ctx.stats()["launches"] == before + 3
    Z = coot.Mat.empty(n, 1, "f32")
    coot.accu(e, ctx, out=Z)  # Z = e; accu(Z) fused: still one launch
    assert ctx.stats()["launches"] == before + 4


def test_in_place_axpy_alias(coot, ctx):
    # B += 3 * A: out aliases operand B exactly
    n = 100_001
    a = oracle.fill("f32", "randu", n, stream=0)
    b = oracle.fill("f32", "randu", n, stream=1)
    A = coot.Col(to_dev(a, "f32"))
    B = coot.Col(to_dev(b, "f32"))
    B += 3 * A
    torch.cuda.synchronize()
    want = oracle.eval_program("f32", P("S0 L0 MUL L1 ADD"), [a, b], [3.0])
    assert_elementwise(to_host(B.data, "f32"), want, "f32", max_ulp=0)


def test_empty_inputs(coot, ctx):
    e0 = torch.empty(0, dtype=torch.float32, device="cuda")
    before = ctx.stats()["launches"]
    ctx.eval("f32", 0, 5, P("L0 L1 ADD"), [e0, e0], [], e0)
    assert ctx.stats()["launches"] == before  # zero launches
    r = torch.full((2,), 7.0, device="cuda")
    ctx.reduce("f32", 0, 1, P("L0"), [e0], [], "ACCU", r)
    torch.cuda.synchronize()
    assert r[0].item() == 0.0
    ctx.reduce("f32", 0, 1, P("L0"), [e0], [], "NORM2", r)
    torch.cuda.synchronize()
    assert r[0].item() == 0.0
    with pytest.raises(coot.CootError) as ei:
        ctx.reduce("f32", 0, 1, P("L0"), [e0], [], "MIN", r)
    assert ei.value.status == "CONTRACT"


def test_contract_errors_before_enqueue(coot, ctx):
    x = torch.zeros(1000, device="cuda")
    y = torch.zeros(1000, device="cuda")
    r = torch.zeros(2, device="cuda")
    before = ctx.stats()["launches"]
    with pytest.raises(coot.CootError) as ei:  # partial overlap of out with an operand
        ctx.eval("f32", 999, 1, P("L0 L1 ADD"), [x[:999], y[:999]], [], x[1:])
    assert ei.value.status == "CONTRACT"
    with pytest.raises(coot.CootError) as ei:  # result inside an operand
        ctx.reduce("f32", 999, 1, P("L0"), [x[:999]], [], "ACCU", x[10:12])
    assert ei.value.status == "CONTRACT"
    xi = torch.zeros(10, dtype=torch.int64, device="cuda")
    with pytest.raises(coot.CootError) as ei:
        ctx.reduce("s64", 10, 1, P("L0"), [xi], [], "NORM2", torch.zeros(2, dtype=torch.int64, device="cuda"))
    assert ei.value.status == "CONTRACT"
    with pytest.raises(coot.CootError) as ei:
        ctx.eval("f32", 10, 100, P("L0 L1 ADD"), [(x.data_ptr(), 10, 100), (y.data_ptr(), 10, 99)], [], r)
    assert ei.value.status == "CONFORM" and "10x99" in str(ei.value)
    assert ctx.stats()["launches"] == before


@pytest.mark.parametrize("etype", FLOATS)
def test_closed_forms_exact(ctx, etype):
    n = (1 << 24) + 3 if etype == "f64" else (1 << 24)
    ones = torch.ones(n, dtype=TORCH[etype], device="cuda")
    r = torch.zeros(2, dtype=TORCH[etype], device="cuda")
    ctx.reduce(etype, n, 1, P("L0"), [ones], [], "ACCU", r)
    assert r[0].item() == n                                # accu(ones) = n
    ctx.reduce(etype, n, 1, P("L0 L1 MUL"), [ones, ones], [], "ACCU", r)
    assert r[0].item() == n                                # dot(ones, ones) = n
    m = 4 ** 10
    ctx.reduce(etype, m, 1, P("L0"), [ones[:m]], [], "NORM2", r)
    assert r[0].item() == 2 ** 10                          # norm2(ones(4^k)) = 2^k
    iota = torch.arange(1 << 20, dtype=TORCH[etype], device="cuda")
    ctx.reduce(etype, 1 << 20, 1, P("L0"), [iota], [], "ACCU", r)
    nn = 1 << 20
    assert r[0].item() == nn * (nn - 1) // 2               # sum of i < n
    x = torch.ones(4096, dtype=TORCH[etype], device="cuda")
    y = torch.full((4096,), 2.0, dtype=TORCH[etype], device="cuda")
    out = torch.empty(4096, dtype=TORCH[etype], device="cuda")
    ctx.reduce(etype, 4096, 1, P("S0 L0 MUL L1 ADD"), [x, y], [2.5], "ACCU", r, out)
    assert torch.all(out == 4.5).item() and r[0].item() == 4.5 * 4096  # axpy closed form


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("kind", ["ACCU", "MINMAX", "NORM2", "MIN"])
def test_simulated_shards_partial_combine(coot, ctx, etype, kind):
    """Contiguous shards of one array -> reduce_partial each -> combine in rank order."""
    if kind == "NORM2" and etype in INTS:
        pytest.skip("NORM2 is float-only")
    prog = P(CATALOG[1])
    n = 1_000_003
    ops = make_inputs(etype, n, 2)
    sc = SCAL[etype][:1]
    dev = [to_dev(o, etype) for o in ops]
    want_z = oracle.eval_program(etype, prog, ops, sc)
    want = oracle.reduce(etype, kind, want_z)
    for nparts in (1, 2, 3, 8):
        parts = torch.zeros(nparts * 4, dtype=torch.int64, device="cuda")
        for r in range(nparts):
            b, e = coot.shard_range(n, r, nparts, 16)
            ctx.reduce_partial(etype, e - b, 1, prog, [d[b:e] for d in dev], sc, kind,
                               parts[4 * r:4 * r + 4])
        res = torch.zeros(2, dtype=TORCH[etype], device="cuda")
        ctx.combine(etype, kind, parts, nparts, 1, res)
        torch.cuda.synchronize()
        got = to_host(res, etype)
        got = got[:2] if kind == "MINMAX" else got[0]
        assert_reduction(got, want, etype, kind, abs_scale(want_z))


@pytest.fixture(scope="module")
def ctx_ldg(coot):
    """A ctx on the register-pipelined LDG driver (COOT_DRIVER=0 at coot_init)."""
    import os
    old = os.environ.get("COOT_DRIVER")
    os.environ["COOT_DRIVER"] = "0"
    try:
        c = coot.Context(0)
    finally:
        if old is None:
            os.environ.pop("COOT_DRIVER", None)
        else:
            os.environ["COOT_DRIVER"] = old
    return c


@pytest.mark.parametrize("etype", ALL)
def test_ldg_driver_parity(ctx_ldg, etype):
    n = 300_007
    for cat, s in sorted(CATALOG.items()):
        prog = P(s)
        if not legal(prog, etype):
            continue
        ops = make_inputs(etype, n, n_operands(prog))
        sc = SCAL[etype][:n_scalars(prog)]
        want = oracle.eval_program(etype, prog, ops, sc)
        r, got = run_reduce(ctx_ldg, etype, prog, ops, sc, "ACCU", with_out=True)
        assert_elementwise(got, want, etype, max_ulp=0)
        assert_reduction(r, oracle_reduce(etype, "ACCU", want), etype, "ACCU", abs_scale(want))
    rng = random.Random(77)
    for trial in range(10):
        prog = random_program(rng, 3, etype, n_ops=3)
        ops = make_inputs(etype, 4001, n_operands(prog), seed=trial)
        want = oracle.eval_program(etype, prog, ops, SCAL[etype][:2])
        got = run_eval(ctx_ldg, etype, prog, ops, SCAL[etype][:2])
        assert_elementwise(got, want, etype, max_ulp=0)


# Fused-operand dispatch (runtime.cu fill_program): every ADD / SUB / MUL whose
# right operand is a LOAD or SCALAR push, at every depth the small (<= 4) and
# large (<= 8) interpreter classes reach, the commutative "S k L j OP" swap, and
# non-commutative forms that must NOT be swapped (s - x, s / x, min/max).
FUSED_FORMS = [
    "L0 L1 ADD", "L0 L1 SUB", "L0 L1 MUL", "L0 S0 ADD", "L0 S0 SUB", "L0 S1 MUL",
    "S0 L0 ADD", "S0 L0 MUL", "S0 L0 SUB", "S1 L1 MAX", "S0 L1 MIN",
    "L0 L1 L2 SUB SUB", "L0 L1 L2 L3 SUB S0 MUL SUB L2 MUL SUB",
    "L0 S0 L1 MUL SUB", "L2 S1 L0 ADD L1 SUB MUL", "L0 L1 L2 S0 L3 MUL ADD ADD SUB",
    "L0 L1 L2 L3 L4 L5 L6 S0 SUB L7 MUL ADD SUB MUL ADD SUB MUL",
    "L0 L1 L2 L3 L4 L5 L6 S1 ADD L7 SUB MUL SUB ADD MUL SUB ADD",
    "S0 L0 L1 L2 SUB MUL SUB S1 L3 MUL ADD",
]


@pytest.mark.parametrize("etype", ["f32", "f64", "u32", "s64", "bf16"])
def test_interpreter_fused_operand_forms(ctx_interp, etype):
    n = 4099
    sc = {"f32": [2.5, -0.75], "f64": [2.5, -0.75], "u32": [7, 3], "s64": [7, -3],
          "bf16": [2.5, -0.75]}[etype]
    for form in FUSED_FORMS:
        prog = P(form)
        k = n_operands(prog)
        if etype == "bf16":
            ops = [oracle.fill(etype, "randu", n, stream=s) for s in range(k)]
        else:
            ops = make_inputs(etype, n, k, seed=len(form))
        want = oracle.eval_program(etype, prog, ops, sc)
        got = run_eval(ctx_interp, etype, prog, ops, sc)
        if etype == "bf16":
            w, g = np.asarray(want).view(np.uint16), np.asarray(got).view(np.uint16)
            nan_w = np.isnan(oracle.to_float(etype, want))
            assert np.array_equal(nan_w, np.isnan(oracle.to_float(etype, got))), form
            assert np.array_equal(g[~nan_w], w[~nan_w]), form
        else:
            assert_elementwise(got, want, etype, max_ulp=0), form
