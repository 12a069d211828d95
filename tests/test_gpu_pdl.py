"""Back-to-back dependent calls: every fused / dim kernel is launched as a
programmatic dependent of the previous kernel on the stream (coot_launch.cuh
launch_k) and waits in pdl_wait() before touching memory.  These chains make
each call read what the previous call wrote — in place, through a reduction
result, and fused pass -> dim sum — eagerly and under CUDA-graph capture, and
compare the end state with the oracle applying the same calls one by one."""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import requires_gpu, to_dev, to_host
from progs import P, assert_elementwise

pytestmark = [pytest.mark.gpu, requires_gpu]

AXPY = P("S0 L0 MUL L1 ADD")


@pytest.fixture(scope="module")
def coot():
    import paper_2508_11385_b200 as c
    return c


@pytest.fixture(scope="module")
def ctx(coot):
    return coot.Context(0)


def _oracle_axpy_chain(x, y, alpha, k):
    for _ in range(k):
        y = oracle.eval_program("f32", AXPY, [x, y], [alpha])
    return y


@pytest.mark.parametrize("n", [1000, 1_000_003, 4_194_304 + 17])
def test_in_place_chain_eager(ctx, n):
    # y <- 0.5 x + y, 8 times in a row, each call reading the previous one's y;
    # every call also reduces (so the finish / ticket path is chained too)
    x = oracle.fill("f32", "randu", n, stream=0)
    y = oracle.fill("f32", "randu", n, stream=1)
    X, Y = to_dev(x, "f32"), to_dev(y, "f32")
    res = torch.zeros(8, 2, dtype=torch.float32, device="cuda")
    for i in range(8):
        ctx.reduce("f32", n, 1, AXPY, [X, Y], [0.5], "ACCU", res[i], Y)
    torch.cuda.synchronize()
    want = y
    for i in range(8):
        want = oracle.eval_program("f32", AXPY, [x, want], [0.5])
        r = float(res[i, 0].item())
        o = float(oracle.reduce("f32", "ACCU", want))
        assert abs(r - o) <= 1e-5 * abs(o), (i, r, o)
    assert_elementwise(to_host(Y, "f32"), want, "f32", max_ulp=0)


def test_in_place_chain_cuda_graph(ctx):
    n = 1_000_000
    x = oracle.fill("f32", "randu", n, stream=0)
    y = oracle.fill("f32", "randu", n, stream=1)
    X, Y = to_dev(x, "f32"), to_dev(y, "f32")
    res = torch.zeros(2, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    main = ctx.stream
    ctx.set_stream(s)
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(5):
                ctx.reduce("f32", n, 1, AXPY, [X, Y], [0.25], "ACCU", res, Y)
    finally:
        ctx.set_stream(main)
    # capture does not execute: Y is still y; replay twice = 10 dependent calls
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    want = _oracle_axpy_chain(x, y, 0.25, 10)
    assert_elementwise(to_host(Y, "f32"), want, "f32", max_ulp=0)
    o = float(oracle.reduce("f32", "ACCU", want))
    assert abs(float(res[0].item()) - o) <= 1e-5 * abs(o)


def test_fused_then_dim_sums_chain(ctx):
    # Z = exp(A % B) + 3 C (fused pass, stored), then sum(Z, 0) and sum(Z, 1)
    # (dim kernels reading Z), then A <- Z - A (fused, reads Z), then sum(A, 1)
    m, ncol = 3000, 517
    n = m * ncol
    a, b, c = (oracle.fill("f32", "randu", n, stream=s) for s in range(3))
    A, B, C = (to_dev(v, "f32") for v in (a, b, c))
    Z = torch.empty(n, dtype=torch.float32, device="cuda")
    d0 = torch.empty(ncol, dtype=torch.float32, device="cuda")
    d1 = torch.empty(m, dtype=torch.float32, device="cuda")
    d1b = torch.empty(m, dtype=torch.float32, device="cuda")
    c2 = P("L0 L1 MUL EXP S0 L2 MUL ADD")
    ctx.eval("f32", m, ncol, c2, [A, B, C], [3.0], Z)
    ctx.reduce("f32", m, ncol, P("L0"), [Z], [], "SUM_DIM0", d0)
    ctx.reduce("f32", m, ncol, P("L0"), [Z], [], "SUM_DIM1", d1)
    ctx.eval("f32", m, ncol, P("L0 L1 SUB"), [Z, A], [], A)
    ctx.reduce("f32", m, ncol, P("L0"), [A], [], "SUM_DIM1", d1b)
    torch.cuda.synchronize()
    z = oracle.eval_program("f32", c2, [a, b, c], [3.0])
    assert_elementwise(to_host(Z, "f32"), z, "f32", max_ulp=0)
    zz = to_host(Z, "f32")  # the device's Z feeds the rest (exp may differ by an ulp)
    a2 = oracle.eval_program("f32", P("L0 L1 SUB"), [zz, a], [])
    assert_elementwise(to_host(A, "f32"), a2, "f32", max_ulp=0)
    for got, want in ((d0, oracle.sum_dim("f32", 0, zz, m, ncol)),
                      (d1, oracle.sum_dim("f32", 1, zz, m, ncol)),
                      (d1b, oracle.sum_dim("f32", 1, a2, m, ncol))):
        g = to_host(got, "f32").astype(np.float64)
        w = np.asarray(want, dtype=np.float64)
        assert np.all(np.abs(g - w) <= 1e-5 * np.abs(w)), np.max(np.abs(g - w) / np.abs(w))
