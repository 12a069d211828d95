#!/usr/bin/env python
"""Benchmark of the fused element-wise expression + reduction path.

Workload (BASELINE.json configs[1], the config `metric` is quoted on):
    Z = exp(A % B) + 3*C ; accu(Z)      A, B, C: 10000 x 10000 f32, fill::randu
One STEP = one pass of the whole hot path: expression capture (delayed
evaluation) -> validate/lower -> ONE fused kernel that writes Z and reduces it
-> (N > 1) exchange of the 32-byte partials + rank-order combine.  Weak
scaling: every rank owns a 10000 x 10000 column block of a 10000 x (10000 N)
global matrix (generated on the device from the global element index, so the
global data do not depend on N).

At N > 1 the line also carries `scaling_configs`: BASELINE configs[4] (c5:
dot / norm2 over a 2^32-element f32 Col) and the three north-star 2^30 forms,
STRONG-scaled (the global size fixed, row-block shards, R17), each timed with
both exchange transports (libcoot's NCCL communicator and the in-kernel
mailbox exchange) as the max over ranks.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl coot|reference]
With --gpus N > 1 and no torchrun environment, bench.py launches N ranks
itself (torch.distributed.run, 127.0.0.1); under torchrun WORLD_SIZE must
equal N.  Rank 0 prints ONE JSON line.  COOT_BENCH_SHARE_GPU=1 is a one-GPU
dry run of the N > 1 code path (every rank on cuda:0, gloo for the host-side
collectives).  COOT_BENCH_EXCHANGE=mailbox|nccl|torch picks the main line's
exchange (default mailbox where every rank maps its peers, else nccl).
`--impl reference` times the CPU oracle (oracle/, the reference arm of this
tier) on the same workload, a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

M_ROWS, N_COLS = 10_000, 10_000
PROGRAM = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2),
           ("MUL", 0), ("ADD", 0)]
SCALARS = [3.0]
BYTES_PER_ELEM = 16  # 3 f32 reads + 1 f32 write (Z stored), SURVEY §8(d) / DESIGN.md
METRIC = "fused-expression GB/s and elements/s vs HBM peak at 1/2/4/8 B200; vs CPU oracle"
WORKLOAD = ("c2: Z = exp(A % B) + 3*C then accu(Z), 10000x10000 f32 Mat per GPU "
            "(BASELINE.json configs[1])")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic():
    """dram read+write bytes per launch of the fused kernel from the committed
    ncu --set full capture (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        return t.get("c2_eval_accu", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """NVML SM clock, power and clock-event (throttle) reasons, sampled every
    `period` s on a background thread while the GPU works; windows (e.g. the
    timed region) are marked by wall-clock timestamps."""

    BAD = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")

    def __init__(self, cuda_index: int, period: float = 0.005):
        self.period = period
        self.samples = []  # (t, sm_mhz, reason_bits, power_w)
        self.windows = {}
        self.err = None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml
            import torch
            self.nv = pynvml
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(cuda_index).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            g = lambda n: getattr(pynvml, "nvmlClocksEventReason" + n,  # noqa: E731
                                  getattr(pynvml, "nvmlClocksThrottleReason" + n, 0))
            self.bits = {"hw_slowdown": g("HwSlowdown"), "hw_thermal_slowdown": g("HwThermalSlowdown"),
                         "sw_thermal_slowdown": g("SwThermalSlowdown"), "sw_power_cap": g("SwPowerCap"),
                         "hw_power_brake": g("HwPowerBrakeSlowdown")}
            self.get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        except Exception as exc:  # noqa: BLE001
            self.err = f"nvml unavailable: {exc}"[:200]

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rb = self.get_reasons(self.h)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((time.perf_counter(), sm, rb, pw))
            except Exception as exc:  # noqa: BLE001
                self.err = str(exc)[:200]
                return
            time.sleep(self.period)

    def start(self):
        if self.err is None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def mark(self, name, begin=True):
        w = self.windows.setdefault(name, [None, None])
        w[0 if begin else 1] = time.perf_counter()

    def stop(self):
        self._stop.set()
        if self._th:
            self._th.join(timeout=2)

    def summary(self, window=None):
        if self.err is not None and not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err]}
        rows = self.samples
        if window and window in self.windows and None not in self.windows[window]:
            t0, t1 = self.windows[window]
            rows = [r for r in rows if t0 <= r[0] <= t1] or rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None),
                    "reasons": ["no samples"]}
        pw = sorted(r[3] for r in rows)
        cut = pw[len(pw) // 2]  # under-load samples: the upper half of observed power
        sm = sorted(r[1] for r in rows if r[3] >= cut) or sorted(r[1] for r in rows)
        reasons = sorted({k for r in rows for k, b in self.bits.items() if b and (r[2] & b)})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(rows), "period_ms": self.period * 1e3,
                "power_w_max": pw[-1], "throttled": any(x in self.BAD for x in reasons)}


def run_reference(args):
    """Reference arm: the CPU oracle, as it stands, on the same workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np

    import oracle
    total = args.steps + args.warmup
    # calibrate ns/element of the oracle on this host, then size each step so the
    # whole --steps/--warmup run stays within ~90 s of CPU work
    cal_n = 1 << 20
    cal = [oracle.fill("f32", "randu", cal_n, stream=s) for s in range(3)]
    t0 = time.perf_counter()
    z = oracle.eval_program("f32", PROGRAM, cal, SCALARS)
    oracle.reduce("f32", "ACCU", z)
    ns_per_el = (time.perf_counter() - t0) / cal_n * 1e9
    budget_s = float(os.environ.get("COOT_REF_BUDGET_S", "90"))
    per_step = int(min(M_ROWS * N_COLS, max(1 << 16, budget_s / total / (ns_per_el * 1e-9))))
    per_step = per_step // M_ROWS * M_ROWS or M_ROWS  # whole columns of the matrix
    ops = [oracle.fill("f32", "randu", per_step, stream=s) for s in range(3)]
    times = []
    for i in range(total):
        t0 = time.perf_counter()
        z = oracle.eval_program("f32", PROGRAM, ops, SCALARS)
        r = oracle.reduce("f32", "ACCU", z)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t = sum(times) / len(times)
    gbs = per_step * BYTES_PER_ELEM / t / 1e9
    sample = (f"first {per_step // M_ROWS} of 10000 columns ({per_step} elements) of the c2 "
              f"workload per step, single-threaded oracle, generation untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_rows": M_ROWS, "n_cols": N_COLS,
                   "mode": "eval+accu (Z stored)"},
        "elements_per_s": per_step / t,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "result_sample": float(r),
    }
    print(json.dumps(line), file=_OUT, flush=True)
    return 0


# The other BASELINE.json configurations (and the north-star 2^30 forms), timed
# at N=1 after the headline: (name, elem, n_rows, n_cols, program, scalars,
# reduce kind or None, Z stored?, algorithmic bytes per element, stream mix
# (reads, writes) for the mix-matched roofline).  Informational lines beside
# the contract line; parity for each is in tests/test_gpu_configs.py.
AXPY = [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)]
C4 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("SCALAR", 0), ("LOAD", 2), ("MUL", 0), ("ADD", 0)]
OTHER_CONFIGS = [
    ("c1 axpy y=2.5x+y in place + accu, f32 n=1e6", "f32", 1_000_000, 1, AXPY, [2.5], "ACCU",
     "inplace", 12, (2, 1)),
    ("c2 reduce-only accu(exp(A%B)+3C), 1e4x1e4 f32", "f32", 10_000, 10_000, PROGRAM, SCALARS,
     "ACCU", None, 12, (3, 0)),
    ("c3 sum(X,0), 32768^2 f64", "f64", 32768, 32768, [("LOAD", 0)], [], "SUM_DIM0", None, 8, (1, 0)),
    ("c3 sum(X,1), 32768^2 f64", "f64", 32768, 32768, [("LOAD", 0)], [], "SUM_DIM1", None, 8, (1, 0)),
    ("c4 minmax(X%Y+7Z), u32 2^28", "u32", 1 << 28, 1, C4, [7], "MINMAX", None, 12, (3, 0)),
    ("c4 minmax(X%Y+7Z), s64 2^28", "s64", 1 << 28, 1, C4, [7], "MINMAX", None, 24, (3, 0)),
    ("c5 dot(x,y), f32 2^32", "f32", 1 << 32, 1, [("LOAD", 0), ("LOAD", 1), ("MUL", 0)], [],
     "ACCU", None, 8, (2, 0)),
    ("c5 norm2(x), f32 2^32", "f32", 1 << 32, 1, [("LOAD", 0)], [], "NORM2", None, 4, (1, 0)),
    ("headline accu(exp(A%B)+3C), f32 2^30", "f32", 1 << 30, 1, PROGRAM, SCALARS, "ACCU", None, 12,
     (3, 0)),
    ("headline exp(A%B)+3C stored + accu, f32 2^30", "f32", 1 << 30, 1, PROGRAM, SCALARS, "ACCU",
     "out", 16, (3, 1)),
    ("headline y=2.5x+y in place + accu, f32 2^30", "f32", 1 << 30, 1, AXPY, [2.5], "ACCU",
     "inplace", 12, (2, 1)),
]
NOMINAL_GBS = 8000.0  # B200 HBM3e nominal (BASELINE north_star "roughly 8 TB/s")
MIXES = [(1, 0), (2, 0), (3, 0), (0, 1), (1, 1), (2, 1), (3, 1)]


def mix_name(m):
    return f"{m[0]}R{m[1]}W" if m[1] else f"{m[0]}R"


def measure_mix_peaks(ctx, n=1 << 30, reps=10):
    """Same-run stream microbenchmarks: the best of `reps`
    launches of libcoot's trivial stream kernel for every read:write mix over
    2^30-element f32 arrays (4 GiB each, >> L2)."""
    import torch
    bufs = [torch.empty(n, dtype=torch.float32, device=ctx.device) for _ in range(4)]
    for s, t in enumerate(bufs):
        ctx.fill(t, "randu", stream=s)
    sink = torch.zeros(1, dtype=torch.float32, device=ctx.device)
    out = {}
    for r, w in MIXES:
        best = None
        for _ in range(reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            ctx.stream_mix(bufs[:r], bufs[3] if w else None, n, sink)
            e1.record(ctx.stream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[mix_name((r, w))] = n * 4 * (r + w) / (best * 1e-3) / 1e9
    del bufs
    torch.cuda.empty_cache()
    return out


def time_calls(call, stream, min_ms=200.0, min_reps=10, graph_below=1 << 22, n=0):
    """Average device time of call() over >= min_ms and >= min_reps back-to-back
    calls (CUDA events on the launching stream).  Small problems are launch-
    bound: their calls are captured in a CUDA graph so the device time is
    measured, not the Python submission rate."""
    import torch
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    call()
    e1.record(stream)
    e1.synchronize()
    one = max(e0.elapsed_time(e1), 1e-3)
    reps = max(min_reps, int(min_ms / one) + 1)
    if n and n <= graph_below:
        return None, reps  # caller times a graph
    e0.record(stream)
    for _ in range(reps):
        call()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps, reps


def measure_other_configs(coot, ctx, peak, mix_peaks, clocks):
    import torch
    from paper_2508_11385_b200.api import TORCH_DTYPE
    out = []
    for name, elem, m, n, prog, sc, kind, store, bpe, mix in OTHER_CONFIGS:
        k = 1 + max(a for o, a in prog if o == "LOAD")
        ops = [torch.empty(m * n, dtype=TORCH_DTYPE[elem], device="cuda") for _ in range(k)]
        for s, t in enumerate(ops):
            ctx.fill(t, "randu", stream=s, n_rows=m)
        z = ops[1] if store == "inplace" else (
            torch.empty(m * n, dtype=TORCH_DTYPE[elem], device="cuda") if store == "out" else None)
        rlen = n if kind == "SUM_DIM0" else (m if kind == "SUM_DIM1" else 2)
        res = torch.empty(rlen, dtype=TORCH_DTYPE[elem], device="cuda")

        def call():
            ctx.reduce(elem, m, n, prog, ops, sc, kind, res, z)

        if clocks:
            clocks.mark(name)
        ms, reps = time_calls(call, ctx.stream, n=m * n)
        if ms is None:
            s_ = torch.cuda.Stream()
            main_stream = ctx.stream
            ctx.set_stream(s_)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s_):
                for _ in range(reps):
                    call()
            ctx.set_stream(main_stream)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
        if clocks:
            clocks.mark(name, begin=False)
        gbs = m * n * bpe / (ms * 1e-3) / 1e9
        mp = mix_peaks.get(mix_name(mix)) if mix_peaks else None
        rec = {"config": name, "ms": ms, "reps": reps, "GBps": gbs,
               "elements_per_s": m * n / (ms * 1e-3), "frac_of_peak": gbs / peak,
               "frac_of_nominal_8TBs": gbs / NOMINAL_GBS, "mix": mix_name(mix),
               "mix_peak_GBps": mp, "frac_of_mix_peak": (gbs / mp) if mp else None,
               "path": ctx.stats()["last_path"]}
        if m * n <= (1 << 22):
            rec["note"] = "L2-resident, CUDA-graph timed: HBM fraction not meaningful"
        if clocks:
            rec["clocks"] = clocks.summary(name)
        out.append(rec)
        del ops, z, res
        torch.cuda.empty_cache()
    return out


# Strong-scaled configurations timed at N > 1 (global sizes fixed; row-block
# shards of the global index, R17): (name, elem, n_global, program, scalars,
# kind, store, bytes/element)
SCALING_CONFIGS = [
    ("c5 dot(x,y), f32 2^32", "f32", 1 << 32, [("LOAD", 0), ("LOAD", 1), ("MUL", 0)], [], "ACCU",
     None, 8),
    ("c5 norm2(x), f32 2^32", "f32", 1 << 32, [("LOAD", 0)], [], "NORM2", None, 4),
    ("headline accu(exp(A%B)+3C), f32 2^30", "f32", 1 << 30, PROGRAM, SCALARS, "ACCU", None, 12),
    ("headline exp(A%B)+3C stored + accu, f32 2^30", "f32", 1 << 30, PROGRAM, SCALARS, "ACCU",
     "out", 16),
    ("headline y=2.5x+y in place + accu, f32 2^30", "f32", 1 << 30, AXPY, [2.5], "ACCU", "inplace",
     12),
]


def measure_scaling_configs(coot, ctx, comm_ctx, mailbox, rank, world, dist, dev):
    """Every rank owns a contiguous block of the global index; each call is the
    fused kernel over the block + the exchange + the rank-order combine.  Timed
    per transport over >= 200 ms (>= 10 calls), per-rank CUDA events, max over
    ranks.  The transports must agree bit for bit (same records, same combine)."""
    import torch
    from paper_2508_11385_b200.api import TORCH_DTYPE
    out = []
    for name, elem, n, prog, sc, kind, store, bpe in SCALING_CONFIGS:
        b, e = coot.shard_range(n, rank, world, 16)
        k = 1 + max(a for o, a in prog if o == "LOAD")
        ops = [torch.empty(e - b, dtype=TORCH_DTYPE[elem], device=dev) for _ in range(k)]
        for s, t in enumerate(ops):
            ctx.fill(t, "randu", stream=s, start=b)
        z = ops[1] if store == "inplace" else (
            torch.empty(e - b, dtype=TORCH_DTYPE[elem], device=dev) if store == "out" else None)
        lw = coot.api.Lowered(elem, e - b, 1, prog, ops, sc, dev)
        rec = {"config": name, "global_elements": n, "elements_per_rank_max": max(
            coot.shard_range(n, r, world, 16)[1] - coot.shard_range(n, r, world, 16)[0]
            for r in range(world))}
        results = {}
        transports = []
        if comm_ctx is not None:
            res_c = torch.zeros(2, dtype=TORCH_DTYPE[elem], device=dev)
            transports.append(("nccl", lambda: comm_ctx.reduce(elem, e - b, 1, prog, ops, sc, kind,
                                                               res_c, z), lambda: res_c))
        if mailbox is not None:
            box = {}
            transports.append(("mailbox", lambda: box.__setitem__("r", mailbox.reduce(lw, kind, out=z)),
                               lambda: box["r"]))
        # two rounds in opposite orders (A B B A), best per transport: the
        # compute-heavy forms run at the power cap, so whichever went second lost clock
        for tname, call, get in transports + transports[::-1]:
            dist.barrier()
            torch.cuda.synchronize()
            ms, reps = time_calls(call, ctx.stream)
            tt = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = float(tt[0])
            if tname in rec and rec[tname]["ms"] <= ms:
                continue
            rec[tname] = {"ms": ms, "reps": reps, "GBps": n * bpe / (ms * 1e-3) / 1e9,
                          "elements_per_s": n / (ms * 1e-3)}
            if store != "inplace":  # in place: the data change every call
                results[tname] = get()[:1].clone()
        if len(results) == 2:
            a_, b_ = results.values()
            rec["transports_bit_identical"] = bool(torch.equal(a_.view(torch.uint8), b_.view(torch.uint8)))
        best = min((rec[t]["ms"] for t, _, _ in transports), default=None)
        if best:
            rec["GBps"] = n * bpe / (best * 1e-3) / 1e9
            rec["elements_per_s"] = n / (best * 1e-3)
        out.append(rec)
        del ops, z, lw
        torch.cuda.empty_cache()
    out.append(measure_c3_dim1_scaling(coot, ctx, comm_ctx, mailbox, rank, world, dist, dev))
    return out


C3_ROWS = C3_COLS = 32768


def measure_c3_dim1_scaling(coot, ctx, comm_ctx, mailbox, rank, world, dist, dev):
    """BASELINE configs[2] at N > 1: sum(X,1) of the 32768 x 32768 f64 Mat, strong-
    scaled over column blocks (each rank sums its columns for every row; the
    n_rows partial vectors are exchanged and combined in rank order).  Transports:
    the in-kernel vector exchange (one dim-1 kernel per rank, partial vectors
    stored into every rank's mailbox over NVLink) and libcoot's NCCL
    communicator (partial kernel -> ncclAllGather -> combine kernel)."""
    import torch
    from paper_2508_11385_b200.dist import column_block
    m, ncols = C3_ROWS, C3_COLS
    c0, c1 = column_block(ncols, rank, world)
    X = torch.empty(m * (c1 - c0), dtype=torch.float64, device=dev)
    ctx.fill(X, "randu", stream=0, start=c0 * m, n_rows=m)
    lw = coot.lower(coot.Mat(X, m, c1 - c0))
    rec = {"config": "c3 sum(X,1), 32768^2 f64, column blocks", "global_elements": m * ncols}
    results = {}
    transports = []
    if comm_ctx is not None:
        res_c = torch.zeros(m, dtype=torch.float64, device=dev)
        transports.append(("nccl", lambda: comm_ctx.reduce("f64", m, c1 - c0, lw.program, lw.operands,
                                                           [], "SUM_DIM1", res_c), lambda: res_c))
    if mailbox is not None and mailbox.vec_capacity >= m:
        box = {}
        transports.append(("mailbox", lambda: box.__setitem__("r", mailbox.sum_dim1(lw)),
                           lambda: box["r"]))
    for tname, call, get in transports + transports[::-1]:  # A B B A, best per transport
        dist.barrier()
        torch.cuda.synchronize()
        ms, reps = time_calls(call, ctx.stream)
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt[0])
        if tname in rec and rec[tname]["ms"] <= ms:
            continue
        rec[tname] = {"ms": ms, "reps": reps, "GBps": m * ncols * 8 / (ms * 1e-3) / 1e9}
        results[tname] = get().clone()
    if len(results) == 2:
        a_, b_ = results.values()
        rec["transports_bit_identical"] = bool(torch.equal(a_, b_))
    best = min((rec[t]["ms"] for t, _, _ in transports), default=None)
    if best:
        rec["GBps"] = m * ncols * 8 / (best * 1e-3) / 1e9
    del X, lw
    torch.cuda.empty_cache()
    return rec


def cpu_baseline_oracle(n=M_ROWS * N_COLS, what="full c2 workload on rank 0's block"):
    """The oracle timed on this host on the c2 workload (by default all 1e8
    elements of rank 0's block), single-threaded; input generation untimed.
    Returns (record, accu)."""
    import numpy as np

    import oracle
    ops = [oracle.fill("f32", "randu", n, stream=s) for s in range(3)]
    t0 = time.perf_counter()
    z = oracle.eval_program("f32", PROGRAM, ops, SCALARS)
    r = oracle.reduce("f32", "ACCU", z)
    dt = time.perf_counter() - t0
    del z
    gbs = n * BYTES_PER_ELEM / dt / 1e9
    rec = {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle",
           "sample": f"{what} ({n} elements), one pass, "
                     f"{dt:.2f} s single-threaded, generation untimed",
           "elements_per_s": n / dt}
    # SURVEY §8(d) variant (ii): the same oracle on T host threads over
    # contiguous chunks (the C calls release the GIL), chunk sums combined in
    # chunk order in f64 — context only; parity uses the 1-thread result
    try:
        import concurrent.futures as cf
        T = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        T = max(1, min(T or 1, 64))
        bounds = [(n * k // T, n * (k + 1) // T) for k in range(T)]

        def chunk(b):
            lo, hi = b
            zz = oracle.eval_program("f32", PROGRAM, [o[lo:hi] for o in ops], SCALARS)
            return float(oracle.reduce("f64", "ACCU", zz.astype(np.float64)))

        with cf.ThreadPoolExecutor(max_workers=T) as ex:
            t0 = time.perf_counter()
            parts = list(ex.map(chunk, bounds))
            dtm = time.perf_counter() - t0
        tot = 0.0
        for p_ in parts:
            tot += p_
        rec["threads"] = {"value": n * BYTES_PER_ELEM / dtm / 1e9, "unit": "GB/s", "cores": T,
                          "seconds": dtm, "speedup_vs_1_thread": dt / dtm,
                          "accu_rel_diff_vs_1_thread": abs(tot - float(r)) / abs(float(r))}
    except Exception as exc:  # informational only
        rec["threads"] = {"error": str(exc)[:200]}
    del ops
    return rec, float(r)


_OUT = sys.stdout


def _claim_stdout():
    """Reserve the real stdout for the ONE JSON line; anything else written to
    fd 1 (NCCL banners, library chatter) is redirected to stderr."""
    sys.stdout.flush()
    fd = os.dup(1)
    os.dup2(2, 1)
    return os.fdopen(fd, "w")


def _free_port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: start N ranks here (one
    process per GPU, torch.distributed.run on 127.0.0.1); rank 0's JSON line
    goes to this process's stdout."""
    share = os.environ.get("COOT_BENCH_SHARE_GPU") == "1"
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        have = 0
    if not share and have < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible\n")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="coot", choices=["coot", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "coot" and "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    global _OUT
    _OUT = _claim_stdout()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    share = os.environ.get("COOT_BENCH_SHARE_GPU") == "1"  # one-GPU dry run of N > 1
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        return 2
    if share:
        local = 0
    torch.cuda.set_device(local)
    force_dist = os.environ.get("COOT_BENCH_FORCE_DIST", "0") == "1"
    if world > 1 or force_dist:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2508_11385_b200 as coot
    from paper_2508_11385_b200 import dist as cdist

    stream = torch.cuda.current_stream()
    ctx = coot.Context(local, stream=stream)
    n = M_ROWS * N_COLS
    start = rank * n  # global element index of this rank's column block
    dev = torch.device("cuda", local)
    data = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(3)]
    for s, t in enumerate(data):
        ctx.fill(t, "randu", seed=42, stream=s, start=start, n_rows=M_ROWS)
    A, B, C = (coot.Mat(t, M_ROWS, N_COLS) for t in data)
    Z = coot.Mat.empty(M_ROWS, N_COLS, "f32", device=dev)
    multi = world > 1 or force_dist
    # N > 1 transports: the in-kernel mailbox exchange (one kernel per rank:
    # partial -> peers' mailboxes over NVLink -> rank-order combine), libcoot's
    # NCCL communicator (partial -> ncclAllGather -> combine kernel, all inside
    # libcoot), or torch.distributed's all-gather between the two libcoot
    # kernels (DistReducer; the host-staged path under gloo)
    exchange = os.environ.get("COOT_BENCH_EXCHANGE", "mailbox")
    # the in-kernel mailbox exchange makes each rank's kernel wait for its
    # peers: never with several ranks on one GPU (nothing runs those launches
    # at the same time), so the shared-GPU dry run uses the host-staged path
    mailbox = (cdist.MailboxExchange.try_create(ctx, vec_capacity=C3_ROWS)
               if multi and not share else None)
    comm_ctx = None
    if multi and not share:
        # libcoot's communicator; any failure (e.g. NCCL not loadable by
        # libcoot) leaves every rank on the other transports
        try:
            uid = [coot.Context.comm_unique_id() if rank == 0 else None]
        except Exception as exc:  # noqa: BLE001
            sys.stderr.write(f"bench.py: coot_comm_unique_id failed: {exc}\n")
            uid = [None]
        dist.broadcast_object_list(uid, src=0)
        if uid[0] is not None:
            comm_ctx = coot.Context(local, stream=stream)
            try:
                comm_ctx.comm_init(world, rank, uid[0], "cols")
            except Exception as exc:  # noqa: BLE001
                sys.stderr.write(f"bench.py: coot_comm_init failed: {exc}\n")
                comm_ctx = None
            ok = torch.tensor([1 if comm_ctx is not None else 0], device=dev)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()) == 0:
                comm_ctx = None
    reducer = cdist.DistReducer(ctx) if multi else None
    if exchange == "mailbox" and mailbox is None:
        exchange = "nccl" if comm_ctx is not None else "torch"
    if exchange == "nccl" and comm_ctx is None:
        exchange = "torch"

    kern_ev = []

    def step(record=False):
        # a1: expression capture (delayed evaluation); a2-a4: one fused launch
        e = coot.exp(A % B) + 3 * C
        lw = coot.lower(e)
        if record:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if not multi or exchange in ("mailbox", "nccl"):
            if not multi:
                res = torch.empty(1, dtype=torch.float32, device=dev)
                ctx.reduce(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands, lw.scalars,
                           "ACCU", res, Z.data)
            elif exchange == "mailbox":
                # a3-a6 in ONE kernel: reduce, publish to the peers' mailboxes, combine
                res = mailbox.reduce(lw, "ACCU", out=Z.data)
            else:
                # a3-a6 inside libcoot: partial kernel, ncclAllGather, combine kernel
                res = torch.empty(1, dtype=torch.float32, device=dev)
                comm_ctx.reduce(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands,
                                lw.scalars, "ACCU", res, Z.data)
            if record:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                kern_ev.append((e0, e1))
            return res
        # a6 via torch.distributed: partial -> all-gather -> rank-order combine kernel
        return reducer.reduce(lw, "ACCU", out=Z.data, kernel_events=kern_ev if record else None)

    peak, peak_kind = _peaks()
    clocks = ClockSampler(local).start() if rank == 0 else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.stats()["launches"] + (comm_ctx.stats()["launches"] if comm_ctx else 0)
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.mark("timed")
    t_begin.record(stream)
    last = None
    for _ in range(args.steps):
        last = step(record=True)
    t_end.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.mark("timed", begin=False)
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    launches = (ctx.stats()["launches"] + (comm_ctx.stats()["launches"] if comm_ctx else 0)
                - launches0)
    elapsed_ms = t_begin.elapsed_time(t_end)
    kern_ms = sum(a.elapsed_time(b) for a, b in kern_ev) / max(1, len(kern_ev))
    if multi:
        tt = torch.tensor([elapsed_ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms, kern_ms = float(tt[0]), float(tt[1])
    ms_per_step = elapsed_ms / args.steps
    total_elems = n * world
    value = total_elems * BYTES_PER_ELEM / (ms_per_step * 1e-3) / 1e9
    accu = float(last[0].item())

    # reduce-only variant (12 B/el), informational
    torch.cuda.synchronize()
    ro_res = torch.empty(1, dtype=torch.float32, device=dev)
    lw = coot.lower(coot.exp(A % B) + 3 * C)
    ro_ms, _ = time_calls(lambda: ctx.reduce(lw.elem, lw.n_rows, lw.n_cols, lw.program,
                                             lw.operands, lw.scalars, "ACCU", ro_res), stream,
                          min_ms=50.0)

    # e2e: the same step through the public API with HOST inputs (pinned) — the
    # H2D copies of A, B, C and the D2H read of accu are inside the timed region
    e2e = None
    if args.e2e_steps > 0:
        host = [t.cpu().pin_memory() for t in data]
        r_host = torch.empty(1, dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()

        def e2e_step():
            for h, d in zip(host, data):
                d.copy_(h, non_blocking=True)
            r = step()
            r_host.copy_(r[:1], non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if multi:
            dist.barrier()
        x0 = torch.cuda.Event(enable_timing=True)
        x1 = torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        x1.record(stream)
        torch.cuda.synchronize()
        e_ms = x0.elapsed_time(x1) / args.e2e_steps
        if multi:
            tt = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt[0])
        e2e = {"value": total_elems * BYTES_PER_ELEM / (e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 3 * n * 4, "d2h_bytes_per_step": 4,
               "ms_per_step": e_ms}
        del host

    # same-run stream microbenchmarks: the roofline denominator per read:write mix
    mix_peaks = None
    if rank == 0 and not args.no_other_configs:
        del data, A, B, C, Z
        torch.cuda.empty_cache()
        mix_peaks = measure_mix_peaks(ctx)

    scaling = None
    if multi and not args.no_other_configs:
        if rank != 0:
            del data, A, B, C, Z
            torch.cuda.empty_cache()
        scaling = measure_scaling_configs(coot, ctx, comm_ctx, mailbox, rank, world, dist, dev)

    if mailbox is not None:
        mailbox.close()  # collective: every rank is here
    if rank != 0:
        if comm_ctx is not None:
            comm_ctx.comm_destroy()
        if multi and dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()
        return 0

    cpu = None
    parity = None
    others = None
    if not args.no_cpu_baseline:
        if world == 1:
            cpu, ref_accu = cpu_baseline_oracle()
            parity = {"accu": accu, "oracle_accu": ref_accu,
                      "rel_err": abs(accu - ref_accu) / abs(ref_accu)}
        else:  # N > 1: a bounded sample (the first 2000 columns of rank 0's block)
            cpu, _ = cpu_baseline_oracle(2000 * M_ROWS, "first 2000 of rank 0's 10000 columns")
    if world == 1 and not args.no_other_configs:
        others = measure_other_configs(coot, ctx, peak, mix_peaks, clocks)
    if clocks:
        clocks.stop()

    alg_bytes = n * BYTES_PER_ELEM
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    mp = mix_peaks.get("3R1W") if mix_peaks else None
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_rows": M_ROWS, "n_cols": N_COLS,
                   "global_elements": total_elems, "mode": "eval+accu (Z stored)",
                   "parallelism": f"dp{world} (column blocks)",
                   "exchange": ("none (one rank)" if not multi else
                                "in-kernel mailboxes (CUDA IPC peer memory)" if exchange == "mailbox" else
                                "libcoot NCCL communicator: partial + ncclAllGather + combine kernel"
                                if exchange == "nccl" else
                                "torch.distributed all_gather of 32-byte partials + combine kernel"),
                   "shared_gpu_dry_run": share,
                   "l2": "inputs 1.2 GB + output 0.4 GB per GPU >> 126 MB L2; no flush needed"},
        "elements_per_s": total_elems / (ms_per_step * 1e-3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": _traffic(),
                     "peak_kind": peak_kind,
                     "mix": "3R1W", "mix_peak": mp, "frac_of_mix_peak": (achieved / mp) if mp else None,
                     "frac_of_nominal_8TBs": achieved / NOMINAL_GBS,
                     "kernel": "fused_tma_kernel<float, ACC_SUM, catalog 2> (c2 program)",
                     "alg_bytes_per_launch": alg_bytes, "kernel_ms": kern_ms},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary("timed") if clocks else None,
        "clocks_whole_run": clocks.summary() if clocks else None,
        "variants": {"reduce_only_GBps": n * 12 / (ro_ms * 1e-3) / 1e9,
                     "reduce_only_ms": ro_ms},
        "parity": parity,
        "mix_peaks_GBps": mix_peaks,
        "other_configs": others,
        "scaling_configs": scaling,
    }
    print(json.dumps(line), file=_OUT, flush=True)
    if comm_ctx is not None:
        comm_ctx.comm_destroy()
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
