"""Small-shape exercise of every libcoot kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  usage:
    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
Checks results against the oracle so a sanitizer-clean run is also correct."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2508_11385_b200 as coot  # noqa: E402
from paper_2508_11385_b200 import _native as N  # noqa: E402


def P(s):
    return [(t, 0) if not (t[0] in "LS" and t[1:].isdigit()) else
            ("LOAD" if t[0] == "L" else "SCALAR", int(t[1:])) for t in s.split()]


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


def check(got, want, tol):
    got, want = float(got), float(want)
    assert abs(got - want) <= tol * max(abs(want), 1e-30), (got, want)


def main():
    ctxs = {"tma": coot.Context(0), "interp": coot.Context(0, flags=N.INIT_FORCE_INTERP),
            "ldg": mkctx(COOT_DRIVER=0), "dimtma": mkctx(COOT_DIM_TMA=1)}
    n = 70_003
    c2 = P("L0 L1 MUL EXP S0 L2 MUL ADD")
    host = [oracle.fill("f32", "randu", n, stream=s) for s in range(3)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    want_z = oracle.eval_program("f32", c2, host, [3.0])
    want = oracle.reduce("f32", "ACCU", want_z)
    for name, ctx in ctxs.items():
        for off in (0, 1):
            ops = [d[off:] for d in dev]
            z = torch.empty(n - off, device="cuda")
            r = torch.zeros(2, device="cuda")
            ctx.reduce("f32", n - off, 1, c2, ops, [3.0], "ACCU", r, z)
            torch.cuda.synchronize()
            w = oracle.reduce("f32", "ACCU", want_z[off:])
            check(r[0].item(), w, 1e-5)
        for kind in ("MINMAX", "NORM2"):
            r = torch.zeros(2, device="cuda")
            ctx.reduce("f32", n, 1, c2, dev, [3.0], kind, r)
        ctx.eval("f32", n, 1, c2, dev, [3.0], torch.empty(n, device="cuda"))
        # dim sums (LDG and TMA kernels)
        for m, cols in ((4096, 17), (512, 130), (3000, 7)):
            X = torch.from_numpy(oracle.fill("f64", "randu", m * cols, stream=4)).cuda()
            for dim in (0, 1):
                res = torch.zeros(cols if dim == 0 else m, dtype=torch.float64, device="cuda")
                ctx.reduce("f64", m, cols, P("L0"), [X], [], f"SUM_DIM{dim}", res)
                torch.cuda.synchronize()
                ref = oracle.sum_dim("f64", dim, X.cpu().numpy(), m, cols)
                assert np.allclose(res.cpu().numpy(), ref, rtol=1e-12, atol=0)
    # 16- and 8-bit element types: fused reductions with Z stored (TMA catalog
    # and interpreter), statistics / index kinds, dim sums
    for et in ("bf16", "f16", "e4m3", "e5m2"):
        tctx = ctxs["tma"]
        ops = [coot.Mat.randu(n, 1, et, stream=s, ctx=tctx).data for s in range(3)]
        z = torch.empty(n, dtype=ops[0].dtype, device="cuda")
        for kind in ("ACCU", "VAR", "INDEX_MAX", "MINMAX", "NORM2"):
            dt = torch.int64 if kind.startswith("INDEX") else coot.api.RESULT_DTYPE[et]
            r = torch.zeros(2, dtype=dt, device="cuda")
            for c in (ctxs["tma"], ctxs["interp"]):
                c.reduce(et, n, 1, c2, ops, [3.0], kind, r, z)
        X = coot.Mat.randu(700, 130, et, stream=5, ctx=tctx)
        for dim in (0, 1):
            res = torch.zeros(130 if dim == 0 else 700, dtype=coot.api.RESULT_DTYPE[et],
                              device="cuda")
            tctx.reduce(et, 700, 130, P("L0"), [X.data], [], f"SUM_DIM{dim}", res)
        torch.cuda.synchronize()
        zr = oracle.eval_program(et, c2, [oracle.fill(et, "randu", n, stream=s) for s in range(3)],
                                 [3.0])
        zh = z.cpu().view(torch.int16 if z.element_size() == 2 else torch.uint8).numpy()
        assert np.array_equal(zh.view(zr.dtype), zr), et
    # views: strided diagonal update and a column-streamed submatrix expression
    M = coot.Mat.randu(300, 300, "f32", stream=6, ctx=ctxs["tma"])
    d = M.diag()
    d += 100.0
    sub = M.submat(10, 20, 200, 250)
    sub.assign(2.5 * sub + 1.0, ctx=ctxs["tma"])
    torch.cuda.synchronize()
    # partial + combine, fill
    ctx = ctxs["tma"]
    parts = torch.zeros(3 * 4, dtype=torch.int64, device="cuda")
    for r_ in range(3):
        b, e = coot.shard_range(n, r_, 3, 16)
        ctx.reduce_partial("f32", e - b, 1, c2, [d[b:e] for d in dev], [3.0], "ACCU",
                           parts[4 * r_:4 * r_ + 4])
    res = torch.zeros(2, device="cuda")
    ctx.combine("f32", "ACCU", parts, 3, 1, res)
    torch.cuda.synchronize()
    check(res[0].item(), want, 1e-5)
    u = torch.empty(1000, dtype=torch.int64, device="cuda")
    ctx.fill(u, "randu")
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
