"""Throughput sweep over the workloads of BASELINE.json (tuning aid).

usage: python tools/sweep.py [--reps R] [--only name,name] [--json out.json]
Prints algorithmic GB/s (each distinct input read once, each output written
once) and elements/s per workload, CUDA-event timed, inputs >> L2.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2508_11385_b200 as coot  # noqa: E402
from paper_2508_11385_b200 import _native as N  # noqa: E402
from paper_2508_11385_b200 import api  # noqa: E402


def P(s):
    return [(t, 0) if not (t[0] in "LS" and t[1:].isdigit()) else
            ("LOAD" if t[0] == "L" else "SCALAR", int(t[1:])) for t in s.split()]


# name: (elem, m, n, program, scalars, kind or None (eval), store, interp)
WL = {
    "c2_eval_accu": ("f32", 10000, 10000, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True, False),
    "c2_reduce": ("f32", 10000, 10000, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False, False),
    "c2_interp": ("f32", 10000, 10000, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True, True),
    "c2_eval": ("f32", 10000, 10000, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], None, True, False),
    "axpy_interp_2p30": ("f32", 1 << 30, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", True, True),
    "poly_interp_2p30": ("f32", 1 << 30, 1, "L0 L1 MUL L2 ADD L0 MUL S0 SUB ABS SQRT", [0.5], "ACCU", True, True),
    "f64_c2_interp_2p29": ("f64", 1 << 29, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False, True),
    "f64_c2_2p29": ("f64", 1 << 29, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False, False),
    "f64_log_2p29": ("f64", 1 << 29, 1, "L0 LOG L1 ADD", [], "ACCU", False, False),
    "f64_log_interp_2p29": ("f64", 1 << 29, 1, "L0 LOG L1 ADD", [], "ACCU", False, True),
    "f32_log_interp_2p30": ("f32", 1 << 30, 1, "L0 LOG L1 ADD", [], "ACCU", False, True),
    "hl_c2_2p30": ("f32", 1 << 30, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False, False),
    "axpy_accu_2p30": ("f32", 1 << 30, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", True, False),
    "axpy_reduce_2p30": ("f32", 1 << 30, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", False, False),
    "accu_2p30": ("f32", 1 << 30, 1, "L0", [], "ACCU", False, False),
    "dot_2p30": ("f32", 1 << 30, 1, "L0 L1 MUL", [], "ACCU", False, False),
    "norm2_2p30": ("f32", 1 << 30, 1, "L0", [], "NORM2", False, False),
    "c4_u32": ("u32", 1 << 28, 1, "L0 L1 MUL S0 L2 MUL ADD", [7], "MINMAX", False, False),
    "c4_s64": ("s64", 1 << 28, 1, "L0 L1 MUL S0 L2 MUL ADD", [7], "MINMAX", False, False),
    "c4_u32_store": ("u32", 1 << 28, 1, "L0 L1 MUL S0 L2 MUL ADD", [7], "MINMAX", True, False),
    "c3_dim0": ("f64", 32768, 32768, "L0", [], "SUM_DIM0", False, False),
    "c3_dim1": ("f64", 32768, 32768, "L0", [], "SUM_DIM1", False, False),
    "c1_axpy_1e6": ("f32", 1_000_000, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", True, False),
    "mean_2p30": ("f32", 1 << 30, 1, "L0", [], "MEAN", False, False),
    "var_2p30": ("f32", 1 << 30, 1, "L0", [], "VAR", False, False),
    "var_f64_2p29": ("f64", 1 << 29, 1, "L0", [], "VAR", False, False),
    "imin_2p30": ("f32", 1 << 30, 1, "L0", [], "INDEX_MIN", False, False),
    "norm2_f64_2p29": ("f64", 1 << 29, 1, "L0", [], "NORM2", False, False),
    "diag_add_1e4": ("f32", 10_000, 1, "L0 S0 ADD", [100.0], None, "diag", False),
    "submat_axpy": ("f32", 8192, 8192, "S0 L0 MUL L1 ADD", [2.5], "ACCU", "submat", False),
    "bf16_c2_2p31": ("bf16", 1 << 31, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False, False),
    "bf16_c2_eval_2p30": ("bf16", 1 << 30, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True, False),
    "bf16_dot_2p31": ("bf16", 1 << 31, 1, "L0 L1 MUL", [], "ACCU", False, False),
    "f16_c2_2p31": ("f16", 1 << 31, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False, False),
    "f16_axpy_eval_2p30": ("f16", 1 << 30, 1, "S0 L0 MUL L1 ADD", [2.5], None, True, False),
    "bf16_var_2p31": ("bf16", 1 << 31, 1, "L0", [], "VAR", False, False),
    "f16_var_2p31": ("f16", 1 << 31, 1, "L0", [], "VAR", False, False),
    "e4m3_var_2p32": ("e4m3", 1 << 32, 1, "L0", [], "VAR", False, False),
    "bf16_norm2_2p31": ("bf16", 1 << 31, 1, "L0", [], "NORM2", False, False),
    "bf16_dim0": ("bf16", 32768, 32768, "L0", [], "SUM_DIM0", False, False),
    "bf16_dim1": ("bf16", 32768, 32768, "L0", [], "SUM_DIM1", False, False),
    "e4m3_dim0": ("e4m3", 65536, 32768, "L0", [], "SUM_DIM0", False, False),
    "f32_dim1": ("f32", 32768, 32768, "L0", [], "SUM_DIM1", False, False),
    "e4m3_c2_2p32": ("e4m3", 1 << 32, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", False, False),
    "e4m3_c2_eval_2p31": ("e4m3", 1 << 31, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True, False),
    "e5m2_axpy_eval_2p31": ("e5m2", 1 << 31, 1, "S0 L0 MUL L1 ADD", [2.5], None, True, False),
    "e4m3_dot_2p32": ("e4m3", 1 << 32, 1, "L0 L1 MUL", [], "ACCU", False, False),
    "e4m3_dim1": ("e4m3", 65536, 32768, "L0", [], "SUM_DIM1", False, False),
    "s64_interp_c4": ("s64", 1 << 28, 1, "L0 L1 MUL S0 L2 MUL SUB", [7], "MINMAX", False, True),
    "e4m3_interp_c2": ("e4m3", 1 << 31, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True, True),
    "f16_interp_axpy": ("f16", 1 << 30, 1, "S0 L0 MUL L1 ADD", [2.5], "ACCU", True, True),
    "bf16_interp_c2":("bf16", 1 << 30, 1, "L0 L1 MUL EXP S0 L2 MUL ADD", [3.0], "ACCU", True, True),
}


def run(name, reps, ctxs):
    elem, m, n, prog, sc, kind, store, interp = WL[name]
    prog = P(prog)
    ctx = ctxs[1] if interp else ctxs[0]
    k = 1 + max(a for o, a in prog if o == "LOAD")
    dt = api.TORCH_DTYPE[elem]
    es = api.ESIZE[elem]
    if store in ("diag", "submat"):  # strided views of 10000 x 10000 parents
        P_ = 10000
        parents = [torch.empty(P_ * P_, dtype=dt, device="cuda") for _ in range(k)]
        for s, t in enumerate(parents):
            ctx.fill(t, "randu", stream=s, n_rows=P_)
        if store == "diag":
            ops = [(t.data_ptr(), m, 1, m, P_ + 1) for t in parents]
        else:
            ops = [(t.data_ptr() + (100 + 200 * P_) * es, m, n, P_, 1) for t in parents]
        out = None
    else:
        ops = [torch.empty(m * n, dtype=dt, device="cuda") for _ in range(k)]
        for s, t in enumerate(ops):
            ctx.fill(t, "randu", stream=s, n_rows=m)
        out = torch.empty(m * n, dtype=dt, device="cuda") if store else None
    rlen = n if kind == "SUM_DIM0" else (m if kind == "SUM_DIM1" else 2)
    res = torch.empty(rlen, dtype=torch.int64 if kind and kind.startswith("INDEX")
                      else api.RESULT_DTYPE[elem],
                      device="cuda")

    def call():
        if store == "diag":
            ctx.eval_view(elem, m, n, prog, ops, sc, ops[0])
        elif kind is None:
            ctx.eval(elem, m, n, prog, ops, sc, out)
        else:
            ctx.reduce(elem, m, n, prog, ops, sc, kind, res, out)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if ms < 0.05:
        # launch-bound sizes: host marshalling would starve the GPU between
        # calls, so time device work as CUDA-graph replays of `reps` calls
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
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
    rbytes = (n if kind == "SUM_DIM0" else m if kind == "SUM_DIM1" else 0) * res.element_size()
    alg = m * n * es * (k + (1 if store in (True, "diag") else 0)) + rbytes
    st = ctx.stats()
    del ops, out
    if store in ("diag", "submat"):
        del parents
    torch.cuda.empty_cache()
    return {"name": name, "ms": ms, "GBps": alg / ms / 1e6, "Gelem_s": m * n / ms / 1e6,
            "grid": st["last_grid"], "path": st["last_path"]}


def stream_copy(reps):
    a = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    a.fill_(1)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"name": "torch_copy_2p30", "ms": ms, "GBps": 8 * (1 << 30) / ms / 1e6}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    ctxs = (coot.Context(0), coot.Context(0, flags=N.INIT_FORCE_INTERP))
    names = [x for x in args.only.split(",") if x] or list(WL)
    rows = [stream_copy(args.reps)]
    for nm in names:
        rows.append(run(nm, args.reps, ctxs))
    for r in rows:
        print(f"{r['name']:>20s} {r['ms']*1e3:10.1f} us {r['GBps']:9.1f} GB/s "
              f"{r.get('Gelem_s', 0):8.1f} Gel/s grid={r.get('grid', '')} path={r.get('path', '')}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"lib": N.LIB_PATH, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
