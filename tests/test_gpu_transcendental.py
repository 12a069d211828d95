"""The device EXP / LOG against the correctly rounded oracle (reading R6,
coot_crmath.cuh): bit for bit, in every float type.

* f32: EXHAUSTIVE over every f32 in [0, 1) for EXP (1.07e9 inputs) and every
  f32 in (0, 89] for LOG (1.12e9), plus every 61st bit pattern of all 2^32
  for both (every sign, exponent, subnormals, inf, NaN).  The oracle's f32
  EXP / LOG are themselves pinned against binary128 over all 2^32 patterns
  (tests/test_oracle_cr_sweep.py).
* f64: random inputs over the whole domain (including the subnormal-result
  range of EXP, subnormal inputs of LOG, tiny |x| next to 1) and the classic
  hard cases e^(2^-k), log(1 + 2^-k), against the oracle's binary128 values.
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest
import torch

import oracle
from gpu_util import requires_gpu, to_dev, to_host

pytestmark = [pytest.mark.gpu, requires_gpu]


@pytest.fixture(scope="module")
def ctx():
    import paper_2508_11385_b200 as coot
    return coot.Context(0)


THREADS = max(1, min(64, len(os.sched_getaffinity(0))))


def oracle_unary(etype, op, x):
    """The oracle on `x`, split over the host's cores (the C calls release the GIL)."""
    n = x.size
    parts = [(n * k // THREADS, n * (k + 1) // THREADS) for k in range(THREADS)]
    out = np.empty_like(x)

    def run(b):
        lo, hi = b
        if hi > lo:
            out[lo:hi] = oracle.eval_program(etype, [("LOAD", 0), (op, 0)], [x[lo:hi]])
    with cf.ThreadPoolExecutor(THREADS) as ex:
        list(ex.map(run, parts))
    return out


def same_bits(got, want):
    """Bool mask: bit-identical, or both NaN."""
    u = np.uint32 if got.dtype == np.float32 else np.uint64
    nan = np.isnan(want)
    return (np.isnan(got) == nan) & (nan | (got.view(u) == want.view(u)))


def gpu_unary(ctx, etype, op, d_in):
    out = torch.empty_like(d_in)
    ctx.eval(etype, d_in.numel(), 1, [("LOAD", 0), (op, 0)], [d_in], [], out)
    return out


def sweep_f32(ctx, op, lo_bits, hi_bits, stride=1, chunk=1 << 26):
    """Compare the device with the oracle on the f32 bit patterns lo, lo +
    stride, ... < hi; returns (checked, first mismatches)."""
    checked, bad = 0, []
    pos = np.arange(0, chunk, dtype=np.int64)
    total = (hi_bits - lo_bits + stride - 1) // stride
    for c0 in range(0, total, chunk):
        n = min(chunk, total - c0)
        b = lo_bits + (c0 + pos[:n]) * stride
        x = b.astype(np.uint32).view(np.float32)
        d = torch.from_numpy(b.astype(np.uint32).view(np.int32)).cuda().view(torch.float32)
        got = gpu_unary(ctx, "f32", op, d).cpu().numpy()
        want = oracle_unary("f32", op, x)
        ok = same_bits(got, want)
        if not ok.all():
            i = np.nonzero(~ok)[0][:5]
            bad += [(hex(int(b[k])), float(x[k]), float(got[k]), float(want[k])) for k in i]
        checked += n
    return checked, bad


def test_f32_exp_exhaustive_unit_interval(ctx):
    checked, bad = sweep_f32(ctx, "EXP", 0x00000000, 0x3F800000)  # every f32 in [0, 1)
    assert checked == 0x3F800000 and not bad, bad


def test_f32_log_exhaustive_to_89(ctx):
    hi = int(np.float32(89.0).view(np.uint32)) + 1  # every f32 in (0, 89]
    checked, bad = sweep_f32(ctx, "LOG", 0x00000001, hi)
    assert checked == hi - 1 and not bad, bad


@pytest.mark.parametrize("op", ["EXP", "LOG"])
def test_f32_all_patterns_strided(ctx, op):
    checked, bad = sweep_f32(ctx, op, 0, 1 << 32, stride=61)
    assert checked == -(-(1 << 32) // 61) and not bad, bad


def f64_inputs(op, n, seed):
    rng = np.random.default_rng(seed)
    if op == "EXP":
        parts = [rng.uniform(-1, 1, n), rng.uniform(-745.2, 709.8, n), rng.uniform(-30, 30, n),
                 rng.uniform(-745.2, -700, n // 4), rng.uniform(700, 709.8, n // 4),
                 np.exp2(rng.uniform(-60, -20, n // 4)) * rng.choice([-1.0, 1.0], n // 4)]
        k = np.arange(1, 64, dtype=np.float64)
        hard = np.concatenate([2.0 ** -k, -(2.0 ** -k), 3 * 2.0 ** -k, 2.0 ** -k * (1 + 2.0 ** -52),
                               np.arange(-745, 710, dtype=np.float64)])
        special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 709.782712893384,
                            709.7827128933841, -745.1332191019411, -745.1332191019412,
                            -708.3964185322641, 5e-324, -5e-324, 1e-300])
    else:
        parts = [rng.uniform(0, 2, n), 1 + rng.uniform(-1e-3, 1e-3, n),
                 np.exp2(rng.uniform(-1020, 1023, n)) * rng.uniform(1, 2, n),
                 rng.uniform(0, 1, n // 4) * 2.0 ** -1022]
        k = np.arange(1, 54, dtype=np.float64)
        hard = np.concatenate([1 + 2.0 ** -k, 1 - 2.0 ** -k, np.arange(1, 100_000, dtype=np.float64),
                               2.0 ** np.arange(-1074, 1024, dtype=np.float64)])
        special = np.array([0.0, -0.0, -1.0, np.inf, -np.inf, np.nan, 1.0, 5e-324,
                            1.7976931348623157e308, 0.75, 1.5, 1.4999999999999998,
                            0.7499999999999999])
    return np.concatenate(parts + [hard, special])


@pytest.mark.parametrize("op", ["EXP", "LOG"])
def test_f64_correctly_rounded(ctx, op):
    x = f64_inputs(op, 1_000_000, 5 + (op == "LOG"))
    want = oracle_unary("f64", op, x)
    got = to_host(gpu_unary(ctx, "f64", op, to_dev(x, "f64")), "f64")
    ok = same_bits(got, want)
    bad = np.nonzero(~ok)[0][:5]
    assert ok.all(), [(x[i].hex(), got[i].hex(), want[i].hex()) for i in bad]


@pytest.mark.parametrize("etype", ["f32", "f64"])
@pytest.mark.parametrize("op", ["EXP", "LOG"])
def test_interpreter_and_catalog_agree_in_a_program(ctx, etype, op):
    """EXP / LOG inside longer programs on the interpreter: every node bit-exact."""
    from paper_2508_11385_b200 import _native as N
    import paper_2508_11385_b200 as coot
    ictx = coot.Context(0, flags=N.INIT_FORCE_INTERP)
    rng = np.random.default_rng(9)
    n = 1_000_003
    dt = oracle.DTYPES[etype]
    a, b = rng.uniform(-3, 3, n).astype(dt), rng.uniform(0.1, 3, n).astype(dt)
    prog = ([("LOAD", 0), ("LOAD", 1), ("MUL", 0), (op, 0), ("SCALAR", 0), ("SUB", 0)]
            if op == "EXP" else
            [("LOAD", 1), (op, 0), ("LOAD", 0), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("SUB", 0)])
    want = oracle.eval_program(etype, prog, [a, b], [1.0])
    for c in (ctx, ictx):
        out = torch.empty(n, dtype=torch.float32 if etype == "f32" else torch.float64, device="cuda")
        c.eval(etype, n, 1, prog, [to_dev(a, etype), to_dev(b, etype)], [1.0], out)
        got = to_host(out, etype)
        ok = same_bits(got, want)
        assert ok.all(), np.nonzero(~ok)[0][:5]
