"""Views with the 16- and 8-bit element types (row 3):
strided diagonal update, submatrix expressions through the column-streaming
TMA path (shared misalignment) into a view destination, and reductions over a
view — element results bit-exact vs the oracle, reductions within the type's
bar (1 ulp for bf16/f16, 1e-5 relative f32 result for fp8)."""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import RTORCH, half_ulp, requires_gpu, to_dev, to_host
from progs import P

pytestmark = [pytest.mark.gpu, requires_gpu]
NARROW = ("bf16", "f16", "e4m3", "e5m2")


@pytest.fixture(scope="module")
def coot():
    import paper_2508_11385_b200 as c
    return c


@pytest.fixture(scope="module")
def ctx(coot):
    return coot.default_ctx(0)


def dev_mat(coot, etype, m, n, stream):
    host = oracle.fill(etype, "randu", m * n, stream=stream)
    return coot.Mat(to_dev(host, etype), m, n), host.reshape(n, m).T.copy()


def same(etype, got, want):
    g, w = oracle.to_float(etype, got), oracle.to_float(etype, want)
    assert np.array_equal(np.isnan(g), np.isnan(w))
    assert np.array_equal(g[~np.isnan(w)], w[~np.isnan(w)])


def check_red(etype, got, want):
    if etype in ("bf16", "f16"):
        assert half_ulp(np.atleast_1d(got), np.atleast_1d(want)).max() <= 1, (got, want)
    else:
        g, w = float(np.atleast_1d(got)[0]), float(np.atleast_1d(want)[0])
        assert abs(g - w) <= 1e-5 * abs(w), (g, w)


@pytest.mark.parametrize("etype", NARROW)
def test_diag_update(coot, ctx, etype):
    m, n = 37, 29
    Z, H = dev_mat(coot, etype, m, n, 0)
    d = Z.diag(2)
    rows, cols = np.arange(27), np.arange(27) + 2
    d += 3.0
    torch.cuda.synchronize()
    want = H.copy()
    want[rows, cols] = oracle.eval_program(etype, P("L0 S0 ADD"), [H[rows, cols].copy()], [3.0])
    same(etype, to_host(Z.data, etype).reshape(n, m).T, want)


@pytest.mark.parametrize("etype", NARROW)
@pytest.mark.parametrize("r0", [16, 3])  # aligned columns / shared misalignment
def test_submatrix_into_view_and_reductions(coot, ctx, etype, r0):
    m, n = 1024, 256
    A, HA = dev_mat(coot, etype, m, n, 6)
    B, HB = dev_mat(coot, etype, m, n, 7)
    Z, HZ = dev_mat(coot, etype, m, n, 8)
    a = A.submat(r0, 3, r0 + 799, 202)  # 800 x 200
    b = B.submat(r0 + 32, 50, r0 + 831, 249)
    z = Z.submat(r0 + 64, 20, r0 + 863, 219)
    sa = HA[r0:r0 + 800, 3:203].T.reshape(-1)
    sb = HB[r0 + 32:r0 + 832, 50:250].T.reshape(-1)
    want = oracle.eval_program(etype, P("S0 L0 MUL L1 ADD"), [sa, sb], [3.0])
    z.assign(3 * a + b)
    torch.cuda.synchronize()
    got = to_host(Z.data, etype).reshape(n, m).T
    same(etype, got[r0 + 64:r0 + 864, 20:220].T.reshape(-1), want)
    keep = np.ones(got.shape, dtype=bool)
    keep[r0 + 64:r0 + 864, 20:220] = False
    assert np.array_equal(got[keep], HZ[keep])
    r = coot.accu(3 * a + b, ctx)
    torch.cuda.synchronize()
    assert r.dtype == RTORCH[etype]
    check_red(etype, to_host(r, etype)[:1], oracle.reduce(etype, "ACCU", want))
    i = coot.index_max(3 * a + b, ctx)
    torch.cuda.synchronize()
    assert int(i[0].item()) == oracle.stats(etype, "INDEX_MAX", want)
