"""The N>1 path end to end on ONE GPU: two processes (gloo, host-staged
exchange) share cuda:0, each owns a contiguous block (R17), runs the fused
partial kernel, all-gathers the 32-byte partial records and combines them in
rank order with the combine kernel (paper_2508_11385_b200.dist.DistReducer).
The result must be identical on both ranks and match the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gpu_util import requires_gpu

pytestmark = [pytest.mark.gpu, requires_gpu]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2508_11385_b200 as coot
        from paper_2508_11385_b200.dist import DistReducer, column_block
        ctx = coot.Context(0)
        red = DistReducer(ctx)
        out = {}
        # c2-shaped f32 expression over a row-block-sharded Col
        n = 3_000_017
        b, e = coot.shard_range(n, rank, world, 16)
        ops = [torch.empty(e - b, dtype=torch.float32, device="cuda") for _ in range(3)]
        for s, t in enumerate(ops):
            ctx.fill(t, "randu", stream=s, start=b)
        lw = coot.lower(coot.exp(coot.Col(ops[0]) % coot.Col(ops[1])) + 3 * coot.Col(ops[2]))
        out["accu"] = float(red.reduce(lw, "ACCU")[0].item())
        # u32 c4 expression, MINMAX: bit-exact
        uo = [torch.empty(e - b, dtype=torch.uint32, device="cuda") for _ in range(3)]
        for s, t in enumerate(uo):
            ctx.fill(t, "randu", stream=s, start=b)
        U = [coot.Col(t) for t in uo]
        lw = coot.lower(U[0] % U[1] + 7 * U[2])
        mm = red.reduce(lw, "MINMAX")
        out["minmax"] = [int(v) for v in mm.cpu().view(torch.int32).numpy().view(np.uint32)]
        # sum(X, 1) with column blocks
        m, ncols = 1000, 301
        c0, c1 = column_block(ncols, rank, world)
        X = torch.empty(m * (c1 - c0), dtype=torch.float64, device="cuda")
        ctx.fill(X, "randu", stream=4, start=c0 * m, n_rows=m)
        rows = red.sum_dim1_columns(coot.lower(coot.Mat(X, m, c1 - c0)))
        out["rows"] = rows.cpu().numpy()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as exc:
        import traceback
        q.put((rank, traceback.format_exc() + repr(exc)))


@pytest.mark.timeout(600)
def test_two_ranks_on_one_gpu_match_oracle():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
    # identical bits on every rank (rank-order combine)
    assert res[0]["accu"] == res[1]["accu"]
    assert res[0]["minmax"] == res[1]["minmax"]
    assert np.array_equal(res[0]["rows"], res[1]["rows"])
    n = 3_000_017
    prog = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2),
            ("MUL", 0), ("ADD", 0)]
    acc, _ = oracle.run_chunked("f32", prog, ["randu"] * 3, start=0, count=n, scalars=[3.0],
                                kind="ACCU")
    assert abs(res[0]["accu"] - float(acc)) <= 1e-5 * abs(float(acc))
    prog4 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("SCALAR", 0), ("LOAD", 2), ("MUL", 0),
             ("ADD", 0)]
    mm, _ = oracle.run_chunked("u32", prog4, ["randu"] * 3, start=0, count=n, scalars=[7],
                               kind="MINMAX")
    assert res[0]["minmax"] == [int(mm[0]), int(mm[1])]
    m, ncols = 1000, 301
    X = oracle.fill("f64", "randu", m * ncols, stream=4)
    want = oracle.sum_dim("f64", 1, X, m, ncols)
    assert np.all(np.abs(res[0]["rows"] - want) <= 1e-12 * np.abs(want))
