"""Strided views (PAPER.md P:177 `Z.diag() += 100`
diagonal / submatrix views): views as operands, as assignment targets and
under every reduction, against the oracle on the gathered view elements."""
import os

import numpy as np
import pytest
import torch

import oracle
from gpu_util import TORCH, requires_gpu, to_dev, to_host
from progs import ALL, FLOATS, P, assert_elementwise, assert_reduction

pytestmark = [pytest.mark.gpu, requires_gpu]
GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_diag.txt")


@pytest.fixture(scope="module")
def coot():
    import paper_2508_11385_b200 as c
    return c


@pytest.fixture(scope="module")
def ctx(coot):
    return coot.default_ctx(0)


def dev_mat(coot, etype, m, n, stream):
    host = oracle.fill(etype, "randu", m * n, stream=stream)
    if etype in FLOATS:
        host = host + oracle.DTYPES[etype](0.5)
    return coot.Mat(to_dev(host, etype), m, n), host.reshape(n, m).T.copy()  # host (m x n)


def test_spec_diag_example(coot, ctx):
    g = {}
    for line in open(GOLD):
        if line.strip() and not line.startswith("#"):
            k, *v = line.split()
            g[k] = [float(x) for x in v]
    Z = coot.Mat(torch.tensor(g["before"], dtype=torch.float64, device="cuda"), 2, 2)
    d = Z.diag()
    d += 100  # Z.diag() += 100
    torch.cuda.synchronize()
    assert Z.data.cpu().tolist() == g["after"]


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("k", [0, 3, -5])
def test_diag_in_place_update(coot, ctx, etype, k):
    m, n = 37, 29
    Z, H = dev_mat(coot, etype, m, n, 0)
    d = Z.diag(k)
    idx = np.arange(len(np.diagonal(H, k)))
    rows = idx + max(0, -k)
    cols = idx + max(0, k)
    diag = H[rows, cols].copy()
    before = ctx.stats()["launches"]
    d += 100
    assert ctx.stats()["launches"] == before + 1 and ctx.stats()["last_path"] == -4
    torch.cuda.synchronize()
    want = H.copy()
    want[rows, cols] = oracle.eval_program(etype, P("L0 S0 ADD"), [diag], [100])
    got = to_host(Z.data, etype).reshape(n, m).T
    assert np.array_equal(got, want)  # untouched elements unchanged, diagonal exact


@pytest.mark.parametrize("etype", ALL)
def test_submatrix_expression_into_dense_and_into_view(coot, ctx, etype):
    m, n = 300, 300
    A, HA = dev_mat(coot, etype, m, n, 1)
    B, HB = dev_mat(coot, etype, m, n, 2)
    a = A.submat(10, 20, 109, 139)  # 100 x 120
    b = B.submat(50, 5, 149, 124)
    sa = HA[10:110, 20:140].T.reshape(-1)  # column-major gather
    sb = HB[50:150, 5:125].T.reshape(-1)
    prog = P("S0 L0 MUL L1 ADD")
    want = oracle.eval_program(etype, prog, [sa, sb], [3])
    Z = (3 * a + b).eval(ctx)  # dense destination
    torch.cuda.synchronize()
    assert_elementwise(to_host(Z.data, etype), want, etype, max_ulp=0)
    # the same expression written INTO another submatrix view of B (disjoint span)
    c = B.submat(160, 150, 259, 269)
    c.assign(3 * a + b.parent.submat(50, 5, 149, 124))
    torch.cuda.synchronize()
    got = to_host(B.data, etype).reshape(n, m).T
    assert np.array_equal(got[160:260, 150:270].T.reshape(-1), want)
    assert np.array_equal(got[:160, :], HB[:160, :])


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("kind", ["ACCU", "MINMAX", "NORM2"])
def test_reductions_over_views(coot, ctx, etype, kind):
    if kind == "NORM2" and etype not in FLOATS:
        pytest.skip("NORM2 is float-only")
    m, n = 500, 300
    A, HA = dev_mat(coot, etype, m, n, 3)
    views = {"sub": (A.submat(7, 9, 406, 258), HA[7:407, 9:259]),
             "diag": (A.diag(), np.diagonal(HA).reshape(-1, 1)),
             "row": (A.row(123), HA[123:124, :])}
    for name, (v, h) in views.items():
        flat = np.ascontiguousarray(h.T.reshape(-1))
        want = oracle.reduce(etype, kind, flat)
        got = {"ACCU": coot.accu, "MINMAX": coot.minmax, "NORM2": coot.norm2}[kind](v, ctx)
        torch.cuda.synchronize()
        g = to_host(got, etype)
        g = g[:2] if kind == "MINMAX" else g[0]
        assert_reduction(g, want, etype, kind, float(np.abs(flat.astype(np.float64)).sum()))


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("dim", [0, 1])
def test_sum_dim_over_views(coot, ctx, etype, dim):
    m, n = 400, 300
    A, HA = dev_mat(coot, etype, m, n, 4)
    v = A.submat(11, 13, 310, 212)
    h = HA[11:311, 13:213]
    r = coot.sum(v, dim, ctx)
    torch.cuda.synchronize()
    got = to_host(r.data, etype)
    want = oracle.sum_dim(etype, dim, np.ascontiguousarray(h.T.reshape(-1)), 300, 200)
    for i in range(got.size):
        assert_reduction(got[i], want[i], etype, "ACCU", 1.0)


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("r0", [4, 1])  # 16-byte aligned columns / shared misalignment
def test_contiguous_column_views_tma_path(coot, ctx, etype, r0):
    """Submatrix views whose columns share one misalignment (incl. the
    destination) take the column-streaming TMA path; results must match."""
    m, n = 1024, 512
    A, HA = dev_mat(coot, etype, m, n, 6)
    B, HB = dev_mat(coot, etype, m, n, 7)
    Z, HZ = dev_mat(coot, etype, m, n, 8)
    a = A.submat(r0, 3, r0 + 999, 402)     # 1000 x 400
    b = B.submat(r0 + 16, 50, r0 + 1015, 449)
    z = Z.submat(r0 + 8, 100, r0 + 1007, 499)
    sa = HA[r0:r0 + 1000, 3:403].T.reshape(-1)
    sb = HB[r0 + 16:r0 + 1016, 50:450].T.reshape(-1)
    prog = P("S0 L0 MUL L1 ADD")
    want = oracle.eval_program(etype, prog, [sa, sb], [3])
    z.assign(3 * a + b)
    torch.cuda.synchronize()
    got = to_host(Z.data, etype).reshape(n, m).T
    assert np.array_equal(got[r0 + 8:r0 + 1008, 100:500].T.reshape(-1), want)
    keep = np.ones_like(HZ, dtype=bool)
    keep[r0 + 8:r0 + 1008, 100:500] = False
    assert np.array_equal(got[keep], HZ[keep])
    for kind in ["ACCU", "MINMAX", "INDEX_MAX"] + (["VAR"] if etype in FLOATS else []):
        fn = {"ACCU": coot.accu, "MINMAX": coot.minmax, "INDEX_MAX": coot.index_max,
              "VAR": coot.var}[kind]
        r = fn(3 * a + b, ctx)
        torch.cuda.synchronize()
        if kind == "INDEX_MAX":
            assert int(r[0].item()) == oracle.stats(etype, kind, want)
        elif kind == "VAR":
            assert_reduction(to_host(r, etype)[0], oracle.stats(etype, kind, want), etype, "ACCU")
        else:
            g = to_host(r, etype)
            g = g[:2] if kind == "MINMAX" else g[0]
            assert_reduction(g, oracle.reduce(etype, kind, want), etype, kind,
                             float(np.abs(want.astype(np.float64)).sum()))


def test_view_alias_rules(coot, ctx):
    m, n = 64, 64
    A, _ = dev_mat(coot, "f32", m, n, 5)
    # destination overlapping (not identical to) an operand view -> contract error
    with pytest.raises(coot.CootError) as ei:
        A.submat(1, 1, 10, 10).assign(A.submat(0, 0, 9, 9) + 1)
    assert ei.value.status == "CONTRACT"
    # a self-overlapping destination view -> contract error
    from paper_2508_11385_b200.api import View
    bad = View(A, 0, 8, 8, ld=4, inc=1)
    with pytest.raises(coot.CootError) as ei:
        bad.assign(A.submat(20, 20, 27, 27) * 2)
    assert ei.value.status == "CONTRACT"
    # identical view in place is fine
    s = A.submat(3, 3, 40, 50)
    s *= 2


@pytest.mark.parametrize("etype", ALL)
@pytest.mark.parametrize("prog", ["S0 L0 MUL L1 ADD", "L0 L1 MUL EXP S0 L2 MUL ADD",
                                  "L0 L1 MUL S0 L2 MUL ADD"])
def test_column_views_catalog_equals_interpreter(coot, etype, prog):
    """Column-streamed submatrix views: a catalog program's own instance (K1)
    and the interpreter (K2) give the same bits, element-wise and reduced, and
    match the oracle."""
    from paper_2508_11385_b200 import _native as N
    p = P(prog)
    if etype in ("u32", "s64") and "EXP" in prog:
        pytest.skip("EXP is float-only (R9)")
    m, n = 2048, 96
    mats = [dev_mat(coot, etype, m, n, 10 + k) for k in range(3)]
    views = [M.submat(4, 2 + k, 4 + 1999, 2 + k + 80) for k, (M, _) in enumerate(mats)]
    hs = [H[4:2004, 2 + k:83 + k].T.reshape(-1) for k, (_, H) in enumerate(mats)]  # 2000 x 81
    k = 1 + max(a for o, a in p if o == "LOAD")
    sc = [3] if etype in ("u32", "s64") else [2.5]
    want = oracle.eval_program(etype, p, hs[:k], sc)
    outs = []
    for flags in (0, N.INIT_FORCE_INTERP):
        c = coot.Context(0, flags=flags)
        out = torch.empty(2000 * 81, dtype=TORCH[etype], device="cuda")
        r = torch.zeros(2, dtype=TORCH[etype], device="cuda")
        ops = [v.operand() for v in views[:k]]
        c.reduce(etype, 2000, 81, p, ops, sc, "ACCU", r, out)
        torch.cuda.synchronize()
        outs.append((to_host(out, etype), to_host(r, etype)))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[0][0], want) if etype in ("u32", "s64") else \
        np.array_equal(outs[0][0].view(np.uint8), want.view(np.uint8))
