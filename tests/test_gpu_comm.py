"""The libcoot communicator (coot_comm_unique_id / coot_comm_init, SURVEY §8(b),
§8(e)) on ONE GPU: a single-rank NCCL communicator (NCCL does not let two
ranks share a device, so the >1-rank transport runs only on a multi-GPU box).
With the communicator bound, coot_reduce runs partial -> ncclAllGather ->
rank-order combine on the ctx stream; with one rank that must give the same
bits as the plain single-launch reduction, for every kind, and SUM_DIM along
the unsharded dimension must stay local."""
import numpy as np
import pytest
import torch

from gpu_util import requires_gpu

pytestmark = [pytest.mark.gpu, requires_gpu]

C2 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2),
      ("MUL", 0), ("ADD", 0)]


@pytest.fixture(scope="module")
def ctxs():
    import paper_2508_11385_b200 as coot
    plain = coot.Context(0)
    uid = coot.Context.comm_unique_id()
    assert len(uid) == 128
    cols = coot.Context(0)
    cols.comm_init(1, 0, uid, "cols")
    rows = coot.Context(0)
    rows.comm_init(1, 0, coot.Context.comm_unique_id(), "rows")
    yield plain, cols, rows
    cols.comm_destroy()
    rows.comm_destroy()


def _ops(ctx, etype, n, k):
    from paper_2508_11385_b200.api import TORCH_DTYPE
    ops = [torch.empty(n, dtype=TORCH_DTYPE[etype], device="cuda") for _ in range(k)]
    for s, t in enumerate(ops):
        ctx.fill(t, "randu", stream=s)
    return ops


@pytest.mark.parametrize("etype,kinds", [
    ("f32", ["ACCU", "NORM2", "MIN", "MAX", "MINMAX", "MEAN", "VAR", "STDDEV", "INDEX_MIN",
             "INDEX_MAX"]),
    ("f64", ["ACCU", "NORM2", "MINMAX", "VAR"]),
    ("u32", ["ACCU", "MINMAX", "INDEX_MAX"]),
    ("s64", ["ACCU", "MINMAX"]),
    ("bf16", ["ACCU", "NORM2", "MINMAX"]),
])
def test_single_rank_comm_equals_plain_reduce(ctxs, etype, kinds):
    from paper_2508_11385_b200.api import RESULT_DTYPE
    plain, cols, _ = ctxs
    n = 2_000_003
    if etype in ("u32", "s64"):
        prog, sc = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("SCALAR", 0), ("LOAD", 2), ("MUL", 0),
                    ("ADD", 0)], [7]
    else:
        prog, sc = C2, [3.0]
    ops = _ops(plain, etype, n, 3)
    for kind in kinds:
        dt = torch.int64 if kind.startswith("INDEX") else RESULT_DTYPE[etype]
        a = torch.zeros(2, dtype=dt, device="cuda")
        b = torch.zeros(2, dtype=dt, device="cuda")
        plain.reduce(etype, n, 1, prog, ops, sc, kind, a)
        cols.reduce(etype, n, 1, prog, ops, sc, kind, b)
        torch.cuda.synchronize()
        w = 2 if kind == "MINMAX" else 1
        assert torch.equal(a[:w].view(torch.uint8), b[:w].view(torch.uint8)), (kind, a, b)


def test_sum_dims_local_or_exchanged(ctxs):
    plain, cols, rows = ctxs
    m, n = 3000, 777
    X = _ops(plain, "f64", m * n, 1)
    for kind, length in (("SUM_DIM0", n), ("SUM_DIM1", m)):
        want = torch.zeros(length, dtype=torch.float64, device="cuda")
        plain.reduce("f64", m, n, [("LOAD", 0)], X, [], kind, want)
        for c in (cols, rows):  # one rank: exchanged or local, the same bits
            got = torch.zeros(length, dtype=torch.float64, device="cuda")
            c.reduce("f64", m, n, [("LOAD", 0)], X, [], kind, got)
            torch.cuda.synchronize()
            assert torch.equal(got, want), kind


def test_eval_and_store_with_comm(ctxs):
    """Element-wise evaluation never communicates; Z stored in the same pass."""
    plain, cols, _ = ctxs
    n = 1_000_000
    ops = _ops(plain, "f32", n, 3)
    z0 = torch.empty(n, device="cuda")
    z1 = torch.empty(n, device="cuda")
    r0 = torch.zeros(1, device="cuda")
    r1 = torch.zeros(1, device="cuda")
    plain.reduce("f32", n, 1, C2, ops, [3.0], "ACCU", r0, z0)
    cols.reduce("f32", n, 1, C2, ops, [3.0], "ACCU", r1, z1)
    torch.cuda.synchronize()
    assert torch.equal(z0, z1) and torch.equal(r0, r1)


def test_comm_init_errors(ctxs):
    import paper_2508_11385_b200 as coot
    _, cols, _ = ctxs
    with pytest.raises(coot.CootError):
        cols.comm_init(1, 0, coot.Context.comm_unique_id())  # already bound
    c = coot.Context(0)
    with pytest.raises(coot.CootError):
        c.comm_init(2, 2, coot.Context.comm_unique_id())  # rank out of range
    with pytest.raises(coot.CootError):
        c.comm_init(1, 0, coot.Context.comm_unique_id(), "diagonal")  # unknown shard
