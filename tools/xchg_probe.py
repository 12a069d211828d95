"""Single-rank cost of the in-kernel exchange: c2 stored 2^30 via coot_reduce
vs coot_reduce_exchange (own mailbox), interleaved.
usage: python tools/xchg_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_11385_b200 as coot  # noqa: E402

C2 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2),
      ("MUL", 0), ("ADD", 0)]


def timed(fn, reps=60):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ctx = coot.Context(0)
    n = 1 << 30
    ops = [torch.empty(n, device="cuda") for _ in range(3)]
    for s, t in enumerate(ops):
        ctx.fill(t, "randu", stream=s)
    z = torch.empty(n, device="cuda")
    r = torch.empty(2, device="cuda")
    mbox, _ = ctx.mailbox_create()
    ep = [0]

    def plain():
        ctx.reduce("f32", n, 1, C2, ops, [3.0], "ACCU", r, z)

    def xchg():
        ep[0] += 1
        ctx.reduce_exchange("f32", n, 1, C2, ops, [3.0], "ACCU", [mbox], 0, ep[0], r, z)

    for rnd in range(3):
        for name, fn in (("plain", plain), ("exchange", xchg)):
            ms = timed(fn)
            print(f"round {rnd} {name:9s} {ms * 1e3:8.1f} us", flush=True)
    ctx.mailbox_destroy(mbox)


if __name__ == "__main__":
    main()
