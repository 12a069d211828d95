"""GPU parity of sum(X,0) / sum(X,1) (K4/K5) against the oracle (R3)."""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import TORCH, requires_gpu, to_dev, to_host
from progs import ALL, FLOATS, P, assert_reduction

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


SHAPES = [(1, 1), (1, 7), (7, 1), (5, 3), (33, 17), (64, 4099), (1000, 37), (2047, 11),
          (2048, 9), (4099, 5), (20000, 3), (3, 20000), (1 << 17, 4), (513, 513), (4096, 1000)]


def _check_vec(got, want, etype, X, m, n, dim):
    if etype not in FLOATS:
        assert np.array_equal(got, want)
        return
    Xm = np.abs(X.astype(np.float64)).reshape(n, m)
    scale = Xm.sum(axis=1) if dim == 0 else Xm.sum(axis=0)
    for i in range(got.size):
        assert_reduction(got[i], want[i], etype, "ACCU", abs_scale=scale[i] + 1e-300)


def run_dim(ctx, etype, prog, ops, sc, m, n, dim, offset=0):
    dev = [to_dev(o, etype, offset) for o in ops]
    res = torch.zeros(n if dim == 0 else m, dtype=TORCH[etype], device="cuda")
    ctx.reduce(etype, m, n, prog, dev, sc, "SUM_DIM0" if dim == 0 else "SUM_DIM1", res)
    torch.cuda.synchronize()
    return to_host(res, etype)


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dim", [0, 1])
def test_sum_dim_plain(ctx, etype, shape, dim):
    m, n = shape
    X = oracle.fill(etype, "randu", m * n, stream=5)
    want = oracle.sum_dim(etype, dim, X, m, n)
    got = run_dim(ctx, etype, P("L0"), [X], [], m, n, dim)
    _check_vec(got, want, etype, X, m, n, dim)


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("dim", [0, 1])
@pytest.mark.parametrize("offset", [1, 2])
def test_sum_dim_misaligned(ctx, etype, dim, offset):
    m, n = 3001, 77
    X = oracle.fill(etype, "randu", m * n, stream=5)
    want = oracle.sum_dim(etype, dim, X, m, n)
    got = run_dim(ctx, etype, P("L0"), [X], [], m, n, dim, offset)
    _check_vec(got, want, etype, X, m, n, dim)


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("dim", [0, 1])
def test_sum_dim_of_fused_expression(ctx, ctx_interp, etype, dim):
    m, n = 2500, 301
    prog = P("L0 L1 MUL S0 L2 MUL ADD")
    ops = [oracle.fill(etype, "randu", m * n, stream=s) for s in range(3)]
    sc = [3]
    Z = oracle.eval_program(etype, prog, ops, sc)
    want = oracle.sum_dim(etype, dim, Z, m, n)
    got = run_dim(ctx, etype, prog, ops, sc, m, n, dim)
    _check_vec(got, want, etype, Z, m, n, dim)
    got2 = run_dim(ctx_interp, etype, prog, ops, sc, m, n, dim)
    _check_vec(got2, want, etype, Z, m, n, dim)


@pytest.mark.parametrize("etype", ALL)
def test_sum_dim_closed_forms(ctx, etype):
    m, n = 3000, 2001
    col = oracle.fill(etype, "colidx", m * n, n_rows=m)  # X(i,j) = j
    row = oracle.fill(etype, "rowidx", m * n, n_rows=m)  # X(i,j) = i
    assert np.array_equal(run_dim(ctx, etype, P("L0"), [col], [], m, n, 0), np.arange(n) * m)
    assert np.array_equal(run_dim(ctx, etype, P("L0"), [row], [], m, n, 1), np.arange(m) * n)
    assert np.all(run_dim(ctx, etype, P("L0"), [col], [], m, n, 1) == n * (n - 1) // 2)
    assert np.all(run_dim(ctx, etype, P("L0"), [row], [], m, n, 0) == m * (m - 1) // 2)


def test_sum_dim_2x2_convention(ctx):
    X = np.array([1, 3, 2, 4], np.float64)  # [[1,2],[3,4]] column-major
    assert list(run_dim(ctx, "f64", P("L0"), [X], [], 2, 2, 0)) == [4, 6]
    assert list(run_dim(ctx, "f64", P("L0"), [X], [], 2, 2, 1)) == [3, 7]


def test_sum_dim_empty_gives_zeros(ctx):
    e = torch.empty(0, dtype=torch.float64, device="cuda")
    r = torch.full((4,), 9.0, dtype=torch.float64, device="cuda")
    ctx.reduce("f64", 0, 4, P("L0"), [e], [], "SUM_DIM0", r)
    torch.cuda.synchronize()
    assert torch.all(r == 0).item()


def test_sum_dim_deterministic_and_one_launch(ctx):
    m, n = 4096, 1500
    X = to_dev(oracle.fill("f32", "randu", m * n), "f32")
    rs = []
    for dim in (0, 1, 0, 1):
        before = ctx.stats()["launches"]
        r = torch.zeros(n if dim == 0 else m, device="cuda")
        ctx.reduce("f32", m, n, P("L0"), [X], [], f"SUM_DIM{dim}", r)
        assert ctx.stats()["launches"] == before + 1
        rs.append(r)
    torch.cuda.synchronize()
    assert torch.equal(rs[0], rs[2]) and torch.equal(rs[1], rs[3])


@pytest.mark.parametrize("dim", [0, 1])
def test_sum_dim_partial_combine_column_shards(coot, ctx, dim):
    """Column-block shards: dim 0 is local, dim 1 needs the vector combine."""
    m, n = 3000, 999
    X = oracle.fill("f64", "randu", m * n, stream=3)
    want = oracle.sum_dim("f64", dim, X, m, n)
    Xd = to_dev(X, "f64")
    P_ = 4
    if dim == 1:
        parts = torch.zeros(P_ * m, dtype=torch.float64, device="cuda")
        for r in range(P_):
            c0, c1 = coot.shard_range(n, r, P_, 1)
            ctx.reduce_partial("f64", m, c1 - c0, P("L0"), [Xd[c0 * m:c1 * m]], [], "SUM_DIM1",
                               parts[r * m:(r + 1) * m])
        res = torch.zeros(m, dtype=torch.float64, device="cuda")
        ctx.combine("f64", "SUM_DIM1", parts, P_, m, res)
        torch.cuda.synchronize()
        _check_vec(to_host(res, "f64"), want, "f64", X, m, n, 1)
    else:
        res = torch.zeros(n, dtype=torch.float64, device="cuda")
        for r in range(P_):
            c0, c1 = coot.shard_range(n, r, P_, 1)
            ctx.reduce("f64", m, c1 - c0, P("L0"), [Xd[c0 * m:c1 * m]], [], "SUM_DIM0", res[c0:c1])
        torch.cuda.synchronize()
        _check_vec(to_host(res, "f64"), want, "f64", X, m, n, 0)


@pytest.fixture(scope="module")
def ctx_tma(coot):
    """A ctx on the TMA-staged dim kernels (COOT_DIM_TMA=1, read at coot_init)."""
    import os
    old = os.environ.get("COOT_DIM_TMA")
    os.environ["COOT_DIM_TMA"] = "1"
    try:
        c = coot.Context(0)
    finally:
        if old is None:
            os.environ.pop("COOT_DIM_TMA", None)
        else:
            os.environ["COOT_DIM_TMA"] = old
    return c


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("shape", [(4096, 1000), (20000, 3), (513, 513), (2048, 9), (1024, 77),
                                   (8192, 33)])
@pytest.mark.parametrize("dim", [0, 1])
def test_sum_dim_tma_kernels(ctx_tma, etype, shape, dim):
    m, n = shape
    X = oracle.fill(etype, "randu", m * n, stream=6)
    want = oracle.sum_dim(etype, dim, X, m, n)
    got = run_dim(ctx_tma, etype, P("L0"), [X], [], m, n, dim)
    _check_vec(got, want, etype, X, m, n, dim)


@pytest.mark.parametrize("etype", ["f32", "u32"])
@pytest.mark.parametrize("dim", [0, 1])
def test_sum_dim_tma_fused_expression(ctx_tma, etype, dim):
    m, n = 4096, 203
    prog = P("L0 L1 MUL S0 L2 MUL ADD")
    ops = [oracle.fill(etype, "randu", m * n, stream=s) for s in range(3)]
    Z = oracle.eval_program(etype, prog, ops, [3])
    want = oracle.sum_dim(etype, dim, Z, m, n)
    got = run_dim(ctx_tma, etype, prog, ops, [3], m, n, dim)
    _check_vec(got, want, etype, Z, m, n, dim)
