"""Fixed per-call cost of the fused pass: eval-only vs reduce-only vs
eval + reduce (axpy, f32), CUDA-graph replays of back-to-back calls, per
driver.  usage: python tools/latency_parts.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

from small_n import AXPY, mkctx  # noqa: E402


S = None


def graph_us(fn, reps=200):
    s = S
    with torch.cuda.stream(s):
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
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    global S
    S = torch.cuda.Stream()
    tiny = torch.zeros(16, device="cuda")
    print(f"torch tiny fill_: {graph_us(lambda: tiny.fill_(1.0)):.2f} us")
    for name, env in (("tma", {}), ("tma_nopdl", {"COOT_PDL": 0}), ("ldg", {"COOT_DRIVER": 0})):
        ctx = mkctx(**env)
        for n in (1000, 10_000, 1_000_000):
            x = torch.rand(n, device="cuda")
            y = torch.rand(n, device="cuda")
            z = torch.empty(n, device="cuda")
            r = torch.empty(2, device="cuda")
            ctx.set_stream(S)
            ev = graph_us(lambda: ctx.eval("f32", n, 1, AXPY, [x, y], [2.5], z))
            ro = graph_us(lambda: ctx.reduce("f32", n, 1, AXPY, [x, y], [2.5], "ACCU", r))
            er = graph_us(lambda: ctx.reduce("f32", n, 1, AXPY, [x, y], [2.5], "ACCU", r, z))
            mm = graph_us(lambda: ctx.reduce("f32", n, 1, AXPY, [x, y], [2.5], "MAX", r))
            print(f"{name} n={n:>8d} eval={ev:6.2f} reduce={ro:6.2f} eval+reduce={er:6.2f} "
                  f"max={mm:6.2f} us", flush=True)


if __name__ == "__main__":
    main()
