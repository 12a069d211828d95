"""Small-problem latency: axpy + accu (c1 shape) for several n, per driver,
timed as CUDA-graph replays of 100 back-to-back calls (device time per call;
inputs L2-resident).  usage: python tools/small_n.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_11385_b200 as coot  # noqa: E402

AXPY = [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)]


def mkctx(**env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        return coot.Context(0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def per_call_us(ctx, n, reps=100):
    x = torch.empty(n, device="cuda")
    y = torch.empty(n, device="cuda")
    ctx.fill(x, "randu", stream=0)
    ctx.fill(y, "randu", stream=1)
    r = torch.empty(2, device="cuda")

    def call():
        ctx.reduce("f32", n, 1, AXPY, [x, y], [2.5], "ACCU", r, y)

    call()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    main = ctx.stream
    ctx.set_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            call()
    ctx.set_stream(main)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, ctx.stats()["last_grid"]


def torch_us(n, reps=100):
    """floor reference: torch's own axpy + sum kernels (two launches) on the same n"""
    x = torch.rand(n, device="cuda")
    y = torch.rand(n, device="cuda")
    r = torch.empty((), device="cuda")
    s = torch.cuda.Stream()
    out = {}
    for name, fn in (("torch_axpy", lambda: y.add_(x, alpha=2.5)),
                     ("torch_sum", lambda: r.copy_(torch.sum(y))),
                     ("torch_copy", lambda: y.copy_(x))):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps * 1e3
    return out


def main():
    ctxs = {"tma": mkctx(), "tma1cta": mkctx(COOT_TMA_CTAS=1), "ldg": mkctx(COOT_DRIVER=0),
            "ldg4": mkctx(COOT_DRIVER=0, COOT_BLOCKS_PER_SM=4)}
    for n in (10_000, 100_000, 1_000_000, 4_000_000, 16_000_000):
        row = []
        for name, ctx in ctxs.items():
            us, grid = per_call_us(ctx, n)
            row.append(f"{name}={us:7.2f}us(g{grid})")
        t = torch_us(n)
        row += [f"{k}={v:7.2f}us" for k, v in t.items()]
        print(f"n={n:>10d} " + " ".join(row), flush=True)


if __name__ == "__main__":
    main()
