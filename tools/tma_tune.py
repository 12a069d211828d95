"""TMA ring geometry sweep (COOT_TMA_TILE units per tile, COOT_TMA_SMEM_KB ring
budget per CTA, COOT_TMA_CTAS CTAs per SM) on the bench workload and two
bandwidth probes.  usage: python tools/tma_tune.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_11385_b200 as coot  # noqa: E402

C2 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2),
      ("MUL", 0), ("ADD", 0)]
AXPY = [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)]
DOT = [("LOAD", 0), ("LOAD", 1), ("MUL", 0)]
CONFIGS = [(0, 0, 2), (512, 96, 2), (0, 0, 2), (512, 96, 2), (1024, 64, 2), (0, 0, 2)]
if len(sys.argv) > 1:  # tile,kb,ctas ...
    CONFIGS = [tuple(int(v) for v in c.split(",")) for c in sys.argv[1:]]


def mkctx(tile, kb, ctas):
    # tile = kb = 0: the library's default policy
    env = {"COOT_TMA_TILE": tile, "COOT_TMA_SMEM_KB": kb, "COOT_TMA_CTAS": ctas}
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


def timed(fn, reps=30):
    for _ in range(3):
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
    n1 = 100_000_000
    a = [torch.empty(n1, device="cuda") for _ in range(3)]
    z = torch.empty(n1, device="cuda")
    n2 = 1 << 30
    x = torch.empty(n2, device="cuda")
    y = torch.empty(n2, device="cuda")
    r = torch.empty(2, device="cuda")
    base = coot.Context(0)
    for s, t in enumerate(a + [x, y]):
        base.fill(t, "randu", stream=s)
    ctxs = [mkctx(*c) for c in CONFIGS]
    rounds = int(os.environ.get("TUNE_ROUNDS", "3"))
    res = {}
    for rnd in range(rounds):  # interleaved rounds: clock / power drift hits every config alike
        for c, ctx in zip(CONFIGS, ctxs):
            t_c2 = timed(lambda: ctx.reduce("f32", n1, 1, C2, a, [3.0], "ACCU", r, z), 400)
            t_ro = timed(lambda: ctx.reduce("f32", n1, 1, C2, a, [3.0], "ACCU", r), 400)
            t_ax = timed(lambda: ctx.reduce("f32", n2, 1, AXPY, [x, y], [2.5], "ACCU", r, y), 50)
            t_dot = timed(lambda: ctx.reduce("f32", n2, 1, DOT, [x, y], [], "ACCU", r), 50)
            t_acc = timed(lambda: ctx.reduce("f32", n2, 1, [("LOAD", 0)], [x], [], "ACCU", r), 50)
            res.setdefault(c, []).append((16 * n1 / t_c2 / 1e6, 12 * n1 / t_ro / 1e6,
                                          12 * n2 / t_ax / 1e6, 8 * n2 / t_dot / 1e6,
                                          4 * n2 / t_acc / 1e6))
    for (tile, kb, ctas), v in res.items():
        med = [sorted(col)[len(col) // 2] for col in zip(*v)]
        print(f"tile={tile:5d} kb={kb:3d} ctas={ctas}  c2 eval+accu {med[0]:7.1f}"
              f"  c2 reduce {med[1]:7.1f}  axpy {med[2]:7.1f}  dot {med[3]:7.1f}  accu {med[4]:7.1f}"
              f" GB/s (median of {len(v)})", flush=True)


if __name__ == "__main__":
    main()
