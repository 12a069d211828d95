"""In-kernel exchange (coot_reduce_exchange, SURVEY §8(e) upgrade path / §8(f)
row 4): the fused kernel publishes its partial into every peer's mailbox over
peer memory, raises its flag there, waits for every rank's flag in its own
mailbox and combines the records in rank order.

One GPU cannot run ranks whose kernels wait on one another (nothing makes two
such launches run at the same time — on B200 two processes doing so raised a
context-switch timeout), so the P-rank protocol is emulated SEQUENTIALLY in one
process: the ranks' kernels run one after another, and before rank r's launch
the host writes the records of the ranks that have not run yet (r+1..P-1,
computed by coot_reduce_partial on their shards) with their flags into rank r's
mailbox, exactly as those peers' kernels would.  Every launch thus finds its
wait already satisfied; everything else — the remote record stores into every
mailbox, the flags, the epoch tags, the parity halves, the rank-order combine —
is the real device path.  Results must be bit-identical on every rank, equal to
the host-staged partial -> combine path, and match the oracle."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from gpu_util import requires_gpu
from progs import P, assert_reduction

pytestmark = [pytest.mark.gpu, requires_gpu]
C2 = P("L0 L1 MUL EXP S0 L2 MUL ADD")
C4 = P("L0 L1 MUL S0 L2 MUL ADD")
MAX_RANKS, REC = 8, 32
FLAG_OFF = 2 * MAX_RANKS * REC  # mailbox: Rec slot[2][MAX_RANKS], then u64 flag[MAX_RANKS]
_cudart = ctypes.CDLL("libcudart.so.12")


def poke(ptr: int, data: bytes):
    buf = ctypes.create_string_buffer(data, len(data))
    assert _cudart.cudaMemcpy(ctypes.c_void_p(ptr), buf, ctypes.c_size_t(len(data)), 1) == 0


def peek(ptr: int, n: int) -> bytes:
    buf = ctypes.create_string_buffer(n)
    assert _cudart.cudaMemcpy(buf, ctypes.c_void_p(ptr), ctypes.c_size_t(n), 2) == 0
    return buf.raw


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


def _emulated_ranks(ctx, mailboxes, shards, elem, prog, sc, kind, epoch):
    """One exchange step of len(shards) ranks, run sequentially (see module doc).
    shards[r] = operand list of rank r.  Returns (per-rank results, partials)."""
    import paper_2508_11385_b200 as coot
    nr = len(shards)
    n_of = [int(s[0].numel()) for s in shards]
    dtype = torch.int64 if kind.startswith("INDEX") else coot.api.RESULT_DTYPE[elem]
    parts = torch.zeros(nr * 4, dtype=torch.int64, device="cuda")
    for q in range(nr):
        ctx.reduce_partial(elem, n_of[q], 1, prog, shards[q], sc, kind, parts[4 * q:4 * q + 4])
    torch.cuda.synchronize()
    recs = parts.cpu().numpy().reshape(nr, 4)
    half = (epoch & 1) * MAX_RANKS
    results = []
    for r in range(nr):
        for q in range(r + 1, nr):  # peers that have not run yet: their record + flag
            rec = recs[q].copy()
            rec[3] = epoch
            poke(mailboxes[r] + (half + q) * REC, rec.astype(np.int64).tobytes())
            poke(mailboxes[r] + FLAG_OFF + 8 * q, np.array([epoch], np.uint64).tobytes())
        res = torch.zeros(2, dtype=dtype, device="cuda")
        ctx.reduce_exchange(elem, n_of[r], 1, prog, shards[r], sc, kind, mailboxes, r, epoch, res)
        torch.cuda.synchronize()  # done before the next rank's launch: nothing waits
        results.append(res.cpu())
    # the records the kernels published are the partials (rank 0's, in the last mailbox)
    pub = np.frombuffer(peek(mailboxes[-1] + half * REC, REC * nr), np.int64).reshape(nr, 4)
    for q in range(nr - 1):
        assert np.array_equal(pub[q][:3], recs[q][:3]) and pub[q][3] == epoch
    comb = torch.zeros(2, dtype=dtype, device="cuda")
    ctx.combine(elem, kind, parts, nr, 1, comb)
    torch.cuda.synchronize()
    return results, comb.cpu()


@pytest.mark.parametrize("nranks", [2, 3])
def test_emulated_ranks_exchange_in_kernel(nranks):
    import paper_2508_11385_b200 as coot
    ctx = coot.Context(0)
    mailboxes = [ctx.mailbox_create()[0] for _ in range(nranks)]
    n = 2_000_017
    f = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(3)]
    u = [torch.empty(n, dtype=torch.uint32, device="cuda") for _ in range(3)]
    for s in range(3):
        ctx.fill(f[s], "randu", stream=s)
        ctx.fill(u[s], "randu", stream=s)
    blocks = [coot.shard_range(n, r, nranks, 16) for r in range(nranks)]
    fs = [[t[b:e] for t in f] for b, e in blocks]
    us = [[t[b:e] for t in u] for b, e in blocks]
    z = oracle.run_chunked("f32", C2, ["randu"] * 3, start=0, count=n, scalars=[3.0],
                           want_out=True)[1]
    want = {"ACCU": oracle.reduce("f32", "ACCU", z), "VAR": oracle.stats("f32", "VAR", z),
            "INDEX_MAX": oracle.stats("f32", "INDEX_MAX", z)}
    mm, _ = oracle.run_chunked("u32", C4, ["randu"] * 3, start=0, count=n, scalars=[7],
                               kind="MINMAX")
    try:
        epoch = 0
        for it in range(3):  # several epochs: both parity halves, twice
            for kind in ("ACCU", "VAR", "INDEX_MAX", "MINMAX"):
                epoch += 1
                if kind == "MINMAX":
                    res, comb = _emulated_ranks(ctx, mailboxes, us, "u32", C4, [7], kind, epoch)
                else:
                    res, comb = _emulated_ranks(ctx, mailboxes, fs, "f32", C2, [3.0], kind, epoch)
                k = 2 if kind == "MINMAX" else 1
                for r in range(nranks):  # identical bits on every rank = host-staged combine
                    assert torch.equal(res[r][:k], comb[:k]), (kind, r, res[r], comb)
                if kind == "MINMAX":
                    got = res[0][:2].view(torch.int32).numpy().view(np.uint32)
                    assert [int(got[0]), int(got[1])] == [int(mm[0]), int(mm[1])]
                elif kind == "INDEX_MAX":
                    assert int(res[0][0]) == want[kind]
                else:
                    assert_reduction(np.float32(res[0][0].item()), want[kind], "f32", "ACCU")
        # an empty shard (rank 0 owns nothing): the identity record, still one kernel
        epoch += 1
        t = torch.empty(10, dtype=torch.float32, device="cuda")
        ctx.fill(t, "randu", stream=0)
        parts = [[t[b:e]] for b, e in (coot.shard_range(10, r, nranks, 16) for r in range(nranks))]
        res, comb = _emulated_ranks(ctx, mailboxes, parts, "f32", [("LOAD", 0)], [], "ACCU", epoch)
        small = oracle.reduce("f32", "ACCU", oracle.fill("f32", "randu", 10, stream=0))
        assert all(float(r[0]) == float(small) for r in res)
    finally:
        for mbx in mailboxes:
            ctx.mailbox_destroy(mbx)


VHDR = 256  # vector mailbox: u64 flag[MAX_RANKS] @0, u64 tag[2][MAX_RANKS] @64, data @256


def _emulated_sum_dim1(ctx, vboxes, cap, elem, m, blocks, epoch):
    """sum(X,1) of column blocks `blocks[r]` (device tensors, m rows each) with
    the in-kernel vector exchange, ranks run sequentially (module doc): before
    rank r's launch the host writes the partial vectors, tags and flags of ranks
    r+1.. into rank r's mailbox.  Returns (per-rank results, host-staged combine)."""
    import paper_2508_11385_b200 as coot
    nr = len(blocks)
    ncol = [b.numel() // m for b in blocks]
    parts = torch.zeros(nr * m, dtype=torch.int64, device="cuda")  # 8-byte partial words
    for q in range(nr):
        ctx.reduce_partial(elem, m, ncol[q], [("LOAD", 0)], [blocks[q]], [], "SUM_DIM1",
                           parts[q * m:(q + 1) * m])
    torch.cuda.synchronize()
    host = parts.cpu().numpy().reshape(nr, m)
    half = (epoch & 1) * MAX_RANKS
    rdt = coot.api.RESULT_DTYPE[elem]
    results = []
    for r in range(nr):
        for q in range(r + 1, nr):
            poke(vboxes[r] + VHDR + ((half + q) * cap) * 8, host[q].tobytes())
            poke(vboxes[r] + 64 + (half + q) * 8, np.array([epoch], np.uint64).tobytes())
            poke(vboxes[r] + 8 * q, np.array([epoch], np.uint64).tobytes())
        res = torch.zeros(m, dtype=rdt, device="cuda")
        ctx.sum_dim_exchange(elem, m, ncol[r], [("LOAD", 0)], [blocks[r]], [], "SUM_DIM1",
                             vboxes, r, epoch, cap, res)
        torch.cuda.synchronize()
        results.append(res.cpu())
    comb = torch.zeros(m, dtype=rdt, device="cuda")
    ctx.combine(elem, "SUM_DIM1", parts, nr, m, comb)
    torch.cuda.synchronize()
    return results, comb.cpu()


@pytest.mark.parametrize("nranks", [1, 2, 3])
@pytest.mark.parametrize("elem,m,ncols", [("f64", 1000, 301), ("f64", 4096, 2000),
                                          ("f32", 4096, 1203), ("bf16", 777, 64),
                                          ("u32", 1000, 37), ("e4m3", 2048, 100),
                                          ("f64", 5, 2)])
def test_emulated_ranks_sum_dim1_vector_exchange(nranks, elem, m, ncols):
    """sum(X,1) over column shards with the exchange inside the dim-1 kernel
    (LDG and TMA kernels, single- and multi-chunk tiles, a rank with NO
    columns when ncols < nranks): identical bits on every rank, equal to the
    host-staged combine, and the oracle's row sums (exact for u32)."""
    import paper_2508_11385_b200 as coot
    from gpu_util import TORCH, to_host
    from paper_2508_11385_b200.dist import column_block
    from progs import TOL
    ctx = coot.Context(0)
    cap = m + 7
    vboxes = [ctx.vec_mailbox_create(cap)[0] for _ in range(nranks)]
    X = torch.empty(m * ncols, dtype=TORCH[elem], device="cuda")
    ctx.fill(X, "randu", stream=4, n_rows=m)
    torch.cuda.synchronize()
    want = oracle.sum_dim(elem, 1, to_host(X, elem), m, ncols)
    blocks = []
    for r in range(nranks):
        c0, c1 = column_block(ncols, r, nranks)
        blocks.append(X[c0 * m:c1 * m])
    try:
        for epoch in range(1, 4):  # both parity halves
            res, comb = _emulated_sum_dim1(ctx, vboxes, cap, elem, m, blocks, epoch)
            for r in range(nranks):
                assert torch.equal(res[r], comb), (elem, r)
            got = to_host(res[0], elem) if elem in ("u32", "bf16") else res[0].numpy()
            if elem == "u32":
                assert np.array_equal(got, want)
            elif elem == "bf16":
                # 1 bf16 ulp (DESIGN R24: the exact sum rounded once vs one more rounding)
                g = got.astype(np.int64)
                w = want.view(np.uint16).astype(np.int64)
                assert np.abs(g - w).max() <= 1
            else:
                tol = TOL["f64" if elem == "f64" else "f32"]
                assert np.all(np.abs(got - want) <= tol * np.abs(want)), elem
    finally:
        for b in vboxes:
            ctx.mailbox_destroy(b)


def test_sum_dim_exchange_contract_errors():
    import paper_2508_11385_b200 as coot
    ctx = coot.Context(0)
    b, _ = ctx.vec_mailbox_create(100)
    X = torch.empty(200 * 3, dtype=torch.float64, device="cuda")
    r = torch.empty(200, dtype=torch.float64, device="cuda")
    try:
        with pytest.raises(coot.CootError):  # more rows than the capacity
            ctx.sum_dim_exchange("f64", 200, 3, [("LOAD", 0)], [X], [], "SUM_DIM1", [b], 0, 1, 100, r)
        with pytest.raises(coot.CootError):  # SUM_DIM0 is not exchanged in the kernel
            ctx.sum_dim_exchange("f64", 100, 6, [("LOAD", 0)], [X], [], "SUM_DIM0", [b], 0, 1, 100, r)
        with pytest.raises(coot.CootError):  # epoch 0
            ctx.sum_dim_exchange("f64", 100, 6, [("LOAD", 0)], [X], [], "SUM_DIM1", [b], 0, 0, 100, r)
        with pytest.raises(coot.CootError):
            ctx.vec_mailbox_create(0)
    finally:
        ctx.mailbox_destroy(b)
