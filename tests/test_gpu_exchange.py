"""In-kernel exchange (coot_reduce_exchange, SURVEY §8(e) upgrade path / §8(f)
row 4): the fused kernel publishes its partial into every peer's mailbox over
peer memory and combines in rank order.  On one GPU: (1) a single rank
(mailbox = its own), (2) two processes sharing cuda:0 whose mailboxes are
mapped through CUDA IPC.  Results must be bit-identical to the host-staged
partial -> all-gather -> combine path (same records, same order) and match
the oracle; repeated calls exercise the epoch / parity protocol; an empty
shard publishes the identity."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from gpu_util import requires_gpu
from progs import P, assert_reduction

pytestmark = [pytest.mark.gpu, requires_gpu]
C2 = P("L0 L1 MUL EXP S0 L2 MUL ADD")
C4 = P("L0 L1 MUL S0 L2 MUL ADD")


def test_single_rank_exchange_equals_reduce():
    import paper_2508_11385_b200 as coot
    ctx = coot.Context(0)
    mine, _ = ctx.mailbox_create()
    n = 1_000_003
    ops = [torch.empty(n, device="cuda") for _ in range(3)]
    for s, t in enumerate(ops):
        ctx.fill(t, "randu", stream=s)
    try:
        for epoch, kind in enumerate(["ACCU", "MINMAX", "NORM2", "MEAN", "VAR", "INDEX_MAX",
                                      "ACCU"], start=1):
            dt = torch.int64 if kind.startswith("INDEX") else torch.float32
            a = torch.zeros(2, dtype=dt, device="cuda")
            b = torch.zeros(2, dtype=dt, device="cuda")
            ctx.reduce_exchange("f32", n, 1, C2, ops, [3.0], kind, [mine], 0, epoch, a)
            ctx.reduce("f32", n, 1, C2, ops, [3.0], kind, b)
            torch.cuda.synchronize()
            assert torch.equal(a, b), (kind, a, b)
        # contract checks happen before anything is enqueued
        with pytest.raises(coot.CootError):
            ctx.reduce_exchange("f32", n, 1, C2, ops, [3.0], "SUM_DIM0", [mine], 0, 9, a)
        with pytest.raises(coot.CootError):
            ctx.reduce_exchange("f32", n, 1, C2, ops, [3.0], "ACCU", [mine], 1, 9, a)
        with pytest.raises(coot.CootError):
            ctx.reduce_exchange("f32", n, 1, C2, ops, [3.0], "ACCU", [mine], 0, 0, a)
    finally:
        ctx.mailbox_destroy(mine)


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
        from paper_2508_11385_b200.dist import DistReducer, MailboxExchange
        ctx = coot.Context(0)
        red, mx = DistReducer(ctx), MailboxExchange(ctx)
        out = {}
        n = 2_000_017
        b, e = coot.shard_range(n, rank, world, 16)
        f = [torch.empty(e - b, dtype=torch.float32, device="cuda") for _ in range(3)]
        u = [torch.empty(e - b, dtype=torch.uint32, device="cuda") for _ in range(3)]
        for s in range(3):
            ctx.fill(f[s], "randu", stream=s, start=b)
            ctx.fill(u[s], "randu", stream=s, start=b)
        lf = coot.lower(coot.exp(coot.Col(f[0]) % coot.Col(f[1])) + 3 * coot.Col(f[2]))
        U = [coot.Col(t) for t in u]
        lu = coot.lower(U[0] % U[1] + 7 * U[2])
        for it in range(3):  # several epochs: parity double-buffering
            for name, lw, kind in (("accu", lf, "ACCU"), ("var", lf, "VAR"),
                                   ("imax", lf, "INDEX_MAX"), ("minmax", lu, "MINMAX")):
                k = 2 if kind == "MINMAX" else 1  # result words the kind writes
                a = mx.reduce(lw, kind)[:k]
                h = red.reduce(lw, kind)[:k]
                torch.cuda.synchronize()
                assert torch.equal(a, h), (name, a, h)
                v = a.cpu()
                out[name] = (v.view(torch.int32).numpy().view(np.uint32).tolist()
                             if v.dtype == torch.uint32 else v.tolist())
        # an empty shard on rank 0 (n < align): identity record, still one kernel
        b2, e2 = coot.shard_range(10, rank, world, 16)
        t = torch.empty(max(e2 - b2, 0), dtype=torch.float32, device="cuda")
        ctx.fill(t, "randu", stream=0, start=b2)
        out["small"] = mx.reduce(coot.lower(coot.Col(t)), "ACCU")[:1].cpu().tolist()
        mx.close()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as exc:
        import traceback
        q.put((rank, traceback.format_exc() + repr(exc)))


@pytest.mark.timeout(600)
def test_two_ranks_exchange_in_kernel():
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=500) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
    assert res[0] == res[1]  # identical bits on every rank
    n = 2_000_017
    acc, _ = oracle.run_chunked("f32", C2, ["randu"] * 3, start=0, count=n, scalars=[3.0],
                                kind="ACCU")
    assert_reduction(np.float32(res[0]["accu"][0]), acc, "f32", "ACCU")
    z = oracle.run_chunked("f32", C2, ["randu"] * 3, start=0, count=n, scalars=[3.0],
                           want_out=True)[1]
    assert res[0]["imax"][0] == oracle.stats("f32", "INDEX_MAX", z)
    assert_reduction(np.float32(res[0]["var"][0]), oracle.stats("f32", "VAR", z), "f32", "ACCU")
    mm, _ = oracle.run_chunked("u32", C4, ["randu"] * 3, start=0, count=n, scalars=[7],
                               kind="MINMAX")
    assert res[0]["minmax"] == [int(mm[0]), int(mm[1])]
    small = oracle.reduce("f32", "ACCU", oracle.fill("f32", "randu", 10, stream=0))
    assert res[0]["small"][0] == float(small)
