"""Multi-process (world size 2, gloo on CPU) coverage of the N>1 host path:
partitioning (coot_shard_range), the partial all-gather in rank order
(paper_2508_11385_b200.dist.allgather_partials) and the rank-order combine
semantics, checked against the oracle on the global array.  The device
kernels of the same path are covered by tests/test_gpu_fused.py
(simulated shards) and tests/test_gpu_dist.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


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
        import oracle
        import paper_2508_11385_b200 as coot
        from paper_2508_11385_b200.dist import allgather_partials, column_block

        out = {}
        # 1) accu of axpy over a row-block-sharded Col (R17)
        n = 1_000_003
        b, e = coot.shard_range(n, rank, world, 16)
        prog = [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)]
        x = oracle.fill("f32", "randu", e - b, stream=0, start=b)
        y = oracle.fill("f32", "randu", e - b, stream=1, start=b)
        z = oracle.eval_program("f32", prog, [x, y], [2.5])
        part = torch.tensor([float(oracle.reduce("f64", "ACCU", z.astype(np.float64)))],
                            dtype=torch.float64)
        g = allgather_partials(part)
        out["parts"] = g.tolist()
        out["range"] = (b, e)
        # 2) integer min/max partials (bit-exact after combine)
        u = oracle.fill("u32", "randu", e - b, stream=2, start=b)
        mm = torch.tensor([int(u.min()), int(u.max())], dtype=torch.int64)
        out["mm"] = allgather_partials(mm).tolist()
        # 3) column blocks of a matrix for sum(X, 1)
        m, ncols = 300, 77
        c0, c1 = column_block(ncols, rank, world)
        X = oracle.fill("f64", "randu", m * (c1 - c0), stream=3, start=c0 * m)
        rows = torch.from_numpy(oracle.sum_dim("f64", 1, X, m, c1 - c0).astype(np.float64))
        out["rows"] = allgather_partials(rows).numpy()
        out["cols"] = (c0, c1)
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as exc:  # surface the failure to the parent
        q.put((rank, repr(exc)))


@pytest.mark.timeout(300)
def test_two_rank_gloo_partials_and_combine():
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
    # every rank gathered the same partials, in rank order
    assert res[0]["parts"] == res[1]["parts"]
    assert res[0]["range"][1] == res[1]["range"][0]
    # combine in rank order == the global oracle within the f32 tolerance
    n = 1_000_003
    prog = [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)]
    x = oracle.fill("f32", "randu", n, stream=0)
    y = oracle.fill("f32", "randu", n, stream=1)
    want = float(oracle.reduce("f32", "ACCU", oracle.eval_program("f32", prog, [x, y], [2.5])))
    got = float(np.float32(sum(res[0]["parts"])))
    assert abs(got - want) <= 1e-5 * abs(want)
    # integer min/max: exact
    u = oracle.fill("u32", "randu", n, stream=2)
    mm = res[0]["mm"]
    assert min(mm[0::2]) == int(u.min()) and max(mm[1::2]) == int(u.max())
    # sum(X,1) over column blocks: rank-order sum of the row partials
    m, ncols = 300, 77
    X = oracle.fill("f64", "randu", m * ncols, stream=3)
    want_rows = oracle.sum_dim("f64", 1, X, m, ncols)
    g = res[0]["rows"].reshape(world, m)
    got_rows = g[0] + g[1]
    assert np.all(np.abs(got_rows - want_rows) <= 1e-12 * np.abs(want_rows))
    assert res[0]["cols"][1] == res[1]["cols"][0]
