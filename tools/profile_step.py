"""Run a few launches of one workload's fused kernel (for ncu captures).

usage: python tools/profile_step.py [c1|c2|c2ro|c2i|axpy|c3d0|c3d1|c4u|c4s|dot|norm2] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_11385_b200 as coot  # noqa: E402
from paper_2508_11385_b200 import api  # noqa: E402

P = lambda s: [(t, 0) if not (t[0] in "LS" and t[1:].isdigit()) else  # noqa: E731
               ("LOAD" if t[0] == "L" else "SCALAR", int(t[1:])) for t in s.split()]

WL = {
    "c2": ("f32", 10000, 10000, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True),
    "c2ro": ("f32", 10000, 10000, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False),
    # interpreter (K2) on the c2 program: the ctx is created with COOT_INIT_FORCE_INTERP
    "c2i": ("f32", 10000, 10000, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True),
    "c1": ("f32", 1_000_000, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", True),
    "c2ro_bf16": ("bf16", 1 << 15, 1 << 15, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False),
    "c2ro_e4m3": ("e4m3", 1 << 15, 1 << 16, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False),
    "c3d1_e4m3": ("e4m3", 65536, 32768, "L0", [], "SUM_DIM1", False),
    "c3d1_bf16": ("bf16", 32768, 32768, "L0", [], "SUM_DIM1", False),
    "var": ("f32", 1 << 30, 1, "L0", [], "VAR", False),
    "c2ro_f64": ("f64", 1 << 14, 1 << 15, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False),
    "var_bf16": ("bf16", 1 << 31, 1, "L0", [], "VAR", False),
    "c3d1_f32": ("f32", 32768, 32768, "L0", [], "SUM_DIM1", False),
    "c1g": ("f32", 1_000_000, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", True),
    "imin": ("f32", 1 << 30, 1, "L0", [], "INDEX_MIN", False),
    "axpy": ("f32", 1 << 30, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", True),
    "c3d0": ("f64", 32768, 32768, "L0", [], "SUM_DIM0", False),
    "c3d1": ("f64", 32768, 32768, "L0", [], "SUM_DIM1", False),
    "c4u": ("u32", 1 << 28, 1, "L0 L1 MUL S0 L2 MUL ADD", [7], "MINMAX", False),
    "c4s": ("s64", 1 << 28, 1, "L0 L1 MUL S0 L2 MUL ADD", [7], "MINMAX", False),
    "dot": ("f32", 1 << 30, 1, "L0 L1 MUL", [], "ACCU", False),
    "norm2": ("f32", 1 << 30, 1, "L0", [], "NORM2", False),
}

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
elem, m, n, prog, sc, kind, store = WL[name]
prog = P(prog)
ctx = coot.Context(0, flags=2 if name in ("c2i",) else 0)  # 2 = COOT_INIT_FORCE_INTERP
k = 1 + max(a for o, a in prog if o == "LOAD")
ops = [torch.empty(m * n, dtype=api.TORCH_DTYPE[elem], device="cuda") for _ in range(k)]
for s, t in enumerate(ops):
    ctx.fill(t, "randu", stream=s, n_rows=m)
out = torch.empty(m * n, dtype=api.TORCH_DTYPE[elem], device="cuda") if store else None
rlen = n if kind == "SUM_DIM0" else (m if kind == "SUM_DIM1" else 2)
res = torch.empty(rlen, dtype=torch.int64 if kind.startswith("INDEX") else api.RESULT_DTYPE[elem],
                  device="cuda")
torch.cuda.synchronize()
for _ in range(reps):
    ctx.reduce(elem, m, n, prog, ops, sc, kind, res, out)
torch.cuda.synchronize()
print(name, "ok", ctx.stats())
