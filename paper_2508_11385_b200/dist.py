"""Multi-GPU sharding of the fused path (one process per GPU).

Partitioning (reading R17): a long Col / Mat is split into contiguous blocks
of the global linear index — for a column-major Mat, blocks of whole columns —
with ``coot_shard_range``.  Each rank evaluates its block with ONE fused
kernel that writes an UNROUNDED partial (``coot_reduce_partial``: a 32-byte
record, or an f64/u64 vector for sum(X,1) over column shards).  The only
exchange step of the method is the all-gather of those partials
(torch.distributed, NCCL over NVLink/NVSwitch on B200; gloo on CPU / for
host-staged tests), followed by ``coot_combine``: a kernel that merges the
partials in rank order 0..P-1 and rounds once, so every rank holds the same
bits and the result does not depend on collective algorithm choice.
Element-wise evaluation alone needs no communication.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .api import RESULT_DTYPE, Context, Lowered, partial_bytes, shard_range

__all__ = ["shard_range", "column_block", "allgather_partials", "DistReducer",
           "MailboxExchange"]


def column_block(n_cols: int, rank: int, world: int) -> tuple[int, int]:
    """Columns [c0, c1) of a column-major Mat owned by `rank`."""
    return shard_range(n_cols, rank, world, 1)


def allgather_partials(local: torch.Tensor, group=None) -> torch.Tensor:
    """Gather every rank's partial (same byte length) into one tensor laid out
    in rank order.  NCCL: device all_gather_into_tensor on the current stream.
    Other backends (gloo): staged through host memory."""
    world = dist.get_world_size(group)
    flat = local.reshape(-1)
    if world == 1:
        return flat.clone()
    backend = dist.get_backend(group)
    if backend == "nccl" and flat.is_cuda:
        out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
        dist.all_gather_into_tensor(out, flat, group=group)
        return out
    host = flat.detach().cpu()
    parts = [torch.empty_like(host) for _ in range(world)]
    dist.all_gather(parts, host, group=group)
    out = torch.cat(parts)
    return out.to(flat.device, non_blocking=False) if flat.is_cuda else out


class DistReducer:
    """Global reductions over rank-sharded operands: partial -> gather -> combine."""

    def __init__(self, ctx: Context, group=None):
        self.ctx = ctx
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = ctx.device
        self._rec = torch.zeros(partial_bytes("ACCU") // 8, dtype=torch.int64, device=dev)

    def reduce(self, lw: Lowered, kind: str, out: torch.Tensor | None = None,
               kernel_events: list | None = None) -> torch.Tensor:
        """Full reduction (ACCU/MIN/MAX/MINMAX/NORM2) of this rank's block;
        returns the GLOBAL result (1 or 2 eT) on every rank."""
        if kernel_events is not None:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(self.ctx.stream)
        self.ctx.reduce_partial(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands,
                                lw.scalars, kind, self._rec, out)
        if kernel_events is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(self.ctx.stream)
            kernel_events.append((e0, e1))
        parts = allgather_partials(self._rec, self.group)
        dtype = torch.int64 if kind.startswith("INDEX") else RESULT_DTYPE[lw.elem]
        res = torch.empty(2, dtype=dtype, device=self.ctx.device)
        self.ctx.combine(lw.elem, kind, parts, self.world, 1, res)
        return res

    def sum_dim1_columns(self, lw: Lowered, total_rows: int | None = None) -> torch.Tensor:
        """sum(X, 1) when ranks own column blocks: every rank's row-sum partial
        (n_rows f64/u64) is gathered and combined in rank order."""
        m = lw.n_rows
        words = partial_bytes("SUM_DIM1", m) // 8
        part = torch.zeros(words, dtype=torch.int64, device=self.ctx.device)
        self.ctx.reduce_partial(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands,
                                lw.scalars, "SUM_DIM1", part)
        parts = allgather_partials(part, self.group)
        res = torch.empty(m, dtype=RESULT_DTYPE[lw.elem], device=self.ctx.device)
        self.ctx.combine(lw.elem, "SUM_DIM1", parts, self.world, m, res)
        return res

    def sum_dim0_columns(self, lw: Lowered) -> torch.Tensor:
        """sum(X, 0) when ranks own column blocks: purely local (no exchange);
        returns this rank's slice of the Row."""
        res = torch.empty(lw.n_cols, dtype=RESULT_DTYPE[lw.elem], device=self.ctx.device)
        self.ctx.reduce(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands, lw.scalars,
                        "SUM_DIM0", res)
        return res


class MailboxExchange:
    """Global scalar reductions with the exchange INSIDE the fused kernel
    (coot_reduce_exchange; SURVEY §8(e) upgrade path, §8(f) row 4): every rank
    allocates a mailbox, the CUDA IPC handles are all-gathered once (host
    objects over the process group), and each reduce is ONE kernel per rank
    that writes its partial into every peer's mailbox over peer memory
    (NVLink P2P), waits for all of them and combines in rank order — no host
    round trip, no collective call per reduction.  Same bits as DistReducer
    (same records, same rank-order combine)."""

    def __init__(self, ctx: Context, group=None, vec_capacity: int = 0):
        """vec_capacity > 0 also sets up vector mailboxes for sum(X,1) over column
        shards of up to that many rows (sum_dim1)."""
        self.ctx = ctx
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.mine, self.mailboxes, ok = self._setup(ctx.mailbox_create())
        self.vec_capacity = vec_capacity
        self.vmine, self.vmailboxes = None, None
        if vec_capacity > 0:
            self.vmine, self.vmailboxes, vok = self._setup(ctx.vec_mailbox_create(vec_capacity))
            ok = ok and vok
        oks = [None] * self.world
        dist.all_gather_object(oks, ok, group=self.group)
        self.ok = all(oks)  # usable only if EVERY rank mapped every peer
        self.epoch = 0
        self.vepoch = 0
        # no rank may release its mailbox while a peer could still write into it
        dist.barrier(group)

    def _setup(self, created):
        mine, handle = created
        handles = [None] * self.world
        dist.all_gather_object(handles, handle, group=self.group)
        boxes, mapped = [], True
        for r, h in enumerate(handles):
            if r == self.rank:
                boxes.append(mine)
                continue
            try:
                boxes.append(self.ctx.mailbox_open(h))
            except Exception:  # e.g. no peer access between these devices
                boxes.append(None)
                mapped = False
        return mine, boxes, mapped

    @classmethod
    def try_create(cls, ctx: Context, group=None, vec_capacity: int = 0):
        """Collective: a MailboxExchange if every rank could map every peer's
        mailbox, else None on every rank (the caller then uses DistReducer)."""
        mx = cls(ctx, group, vec_capacity)
        if mx.ok:
            return mx
        mx.close()
        return None

    def reduce(self, lw: Lowered, kind: str, out: torch.Tensor | None = None) -> torch.Tensor:
        """Full scalar reduction of this rank's block; the GLOBAL result on every
        rank.  Every rank must call it the same number of times."""
        if not self.ok:
            raise RuntimeError("MailboxExchange: some rank could not map every peer's mailbox")
        dtype = torch.int64 if kind.startswith("INDEX") else RESULT_DTYPE[lw.elem]
        res = torch.empty(2, dtype=dtype, device=self.ctx.device)
        # the epoch advances only once the kernel is enqueued: a call rejected on
        # the host (validation) leaves it unchanged, so a retry reuses it and a
        # peer waiting at this epoch is never released by a later one
        self.ctx.reduce_exchange(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands,
                                 lw.scalars, kind, self.mailboxes, self.rank, self.epoch + 1,
                                 res, out)
        self.epoch += 1
        return res

    def sum_dim1(self, lw: Lowered) -> torch.Tensor:
        """sum(X, 1) of a Mat sharded by column blocks (this rank's block `lw`):
        the GLOBAL row sums on every rank, exchanged inside the dim-1 kernel
        (coot_sum_dim_exchange).  Every rank must call it the same number of times."""
        if not self.ok or not self.vec_capacity:
            raise RuntimeError("MailboxExchange: no usable vector mailboxes (vec_capacity=0?)")
        res = torch.empty(lw.n_rows, dtype=RESULT_DTYPE[lw.elem], device=self.ctx.device)
        self.ctx.sum_dim_exchange(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands,
                                  lw.scalars, "SUM_DIM1", self.vmailboxes, self.rank,
                                  self.vepoch + 1, self.vec_capacity, res)
        self.vepoch += 1
        return res

    def close(self):
        torch.cuda.synchronize(self.ctx.device)
        dist.barrier(self.group)  # every rank's last kernel has finished writing
        for boxes in (self.mailboxes, self.vmailboxes or []):
            for r, p in enumerate(boxes):
                if r != self.rank and p is not None:
                    self.ctx.mailbox_close(p)
        dist.barrier(self.group)
        self.ctx.mailbox_destroy(self.mine)
        if self.vmine is not None:
            self.ctx.mailbox_destroy(self.vmine)
