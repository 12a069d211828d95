"""Per-launch fixed cost of the fused pass: time c2 (Z stored + accu) and c2
reduce-only at several sizes, back-to-back calls (as bench.py runs them), and
fit t(n) = t0 + n / BW.  usage: python tools/size_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_11385_b200 as coot  # noqa: E402

C2 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2),
      ("MUL", 0), ("ADD", 0)]
SIZES = [int(v) for v in os.environ.get("SIZES", "25000000,50000000,100000000,200000000,400000000").split(",")]


def timed(fn, reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    ctx = coot.Context(0)
    nmax = max(SIZES)
    a = [torch.empty(nmax, device="cuda") for _ in range(3)]
    z = torch.empty(nmax, device="cuda")
    r = torch.empty(2, device="cuda")
    for s, t in enumerate(a):
        ctx.fill(t, "randu", stream=s)
    for form, store in (("eval+accu", True), ("reduce", False)):
        pts = []
        for n in SIZES:
            ops = [t[:n] for t in a]
            reps = max(20, int(1e8 / n * 400))
            us = timed(lambda: ctx.reduce("f32", n, 1, C2, ops, [3.0], "ACCU", r, z[:n] if store else None), reps)
            b = (16 if store else 12) * n
            pts.append((n, us))
            print(f"c2 {form:9s} n={n:11d} {us:9.1f} us {b / us / 1e3:7.1f} GB/s", flush=True)
        # least-squares t = t0 + n * k
        import statistics
        xs, ys = [p[0] for p in pts], [p[1] for p in pts]
        mx, my = statistics.mean(xs), statistics.mean(ys)
        k = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
        t0 = my - k * mx
        print(f"  fit: t0 = {t0:.1f} us, asymptotic {(16 if store else 12) / k / 1e3:.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
