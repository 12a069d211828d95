"""Run under AddressSanitizer + UndefinedBehaviorSanitizer (tests/test_sanitizers.py
starts it with LD_PRELOAD=libasan/libubsan, COOT_LIB_PATH = the sanitized
host-runtime build of libcoot, ORACLE_LIB_PATH = the sanitized oracle).  No
torch, no GPU: the host halves of both libraries — libcoot's validation,
lowering checks and error paths (every coot_* call that does not reach a
kernel), and every oracle entry point on every element type."""
import ctypes
import importlib.util
import os
import random
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

spec = importlib.util.spec_from_file_location(
    "_native_san", os.path.join(ROOT, "paper_2508_11385_b200", "_native.py"))
N = importlib.util.module_from_spec(spec)
spec.loader.exec_module(N)
assert N.LIB_PATH == os.environ["COOT_LIB_PATH"]

import oracle  # noqa: E402
from progs import ALL, random_program  # noqa: E402


def libcoot_host():
    lib = N.lib
    rng = random.Random(1)
    names = list(N.OP)
    n_ok = n_err = 0
    for it in range(20000):  # random (often malformed) descriptors through coot_validate
        e = N.Expr()
        e.abi_version = 1 if rng.random() < 0.95 else rng.randrange(5)
        e.elem = rng.randrange(10)
        e.n_rows = rng.choice([0, 1, 7, 1 << 20, (1 << 63) + 5])
        e.n_cols = rng.choice([0, 1, 3, 1 << 40])
        e.n_operands = rng.randrange(11)
        e.n_scalars = rng.randrange(11)
        e.n_instr = rng.randrange(36)
        e.reserved = 0 if rng.random() < 0.9 else 1
        for k in range(N.MAX_OPERANDS):
            e.operands[k].ptr = rng.choice([0, 0x1000, 0x1004, 0x7f0000000010])
            e.operands[k].n_rows = e.n_rows if rng.random() < 0.9 else rng.randrange(9)
            e.operands[k].n_cols = e.n_cols if rng.random() < 0.9 else rng.randrange(9)
            e.operands[k].ld = rng.choice([0, 0, 1, e.n_rows, e.n_rows + 3])
            e.operands[k].inc = rng.choice([0, 0, 1, 2])
        for k in range(N.MAX_SCALARS):
            e.scalars[k].bits = rng.getrandbits(64)
        for i in range(N.MAX_INSTR):
            e.prog[i].op = rng.randrange(16)
            e.prog[i].arg = rng.randrange(12)
        rc = lib.coot_validate(ctypes.byref(e))
        msg = lib.coot_last_error()
        assert rc == 0 or msg, rc
        n_ok += rc == 0
        n_err += rc != 0
    for et in ("f32", "f64", "u32", "s64", "bf16", "f16", "e4m3", "e5m2"):  # well-formed programs
        for d in range(6):
            p = random_program(rng, d, et if et in ALL else "f32")
            e = N.Expr()
            e.abi_version, e.elem, e.n_rows, e.n_cols = 1, N.ELEM[et], 100, 3
            e.n_operands, e.n_scalars, e.n_instr = 3, 2, len(p)
            for k in range(3):
                e.operands[k].ptr, e.operands[k].n_rows, e.operands[k].n_cols = 0x10000 * (k + 1), 100, 3
            for i, (op, a) in enumerate(p):
                e.prog[i].op, e.prog[i].arg = N.OP[op], a
            lib.coot_validate(ctypes.byref(e))
    nb = ctypes.c_uint64()
    for kind in range(14):
        lib.coot_partial_bytes(kind, 12345, ctypes.byref(nb))
    b, en = ctypes.c_uint64(), ctypes.c_uint64()
    for n in (0, 1, 15, 16, 1000003, 1 << 32):
        for P in (1, 2, 3, 8, 9):
            for r in range(P + 1):
                lib.coot_shard_range(n, r, P, 16, ctypes.byref(b), ctypes.byref(en))
    for code in range(-2, 9):
        lib.coot_status_string(code)
    h = ctypes.c_void_p()
    rc = lib.coot_init(ctypes.byref(h), 0, None, 0)  # no GPU in this container: a device error
    if rc == 0:
        lib.coot_destroy(h)
    assert lib.coot_destroy(None) == 0  # NULL is a no-op (coot.h)
    mb = (ctypes.c_void_p * 2)(None, None)
    e = N.Expr()
    for kind in (5, 6, 99):  # SUM_DIM0 / SUM_DIM1 / junk: rejected before any CUDA call
        assert lib.coot_sum_dim_exchange(None, ctypes.byref(e), kind, mb, 2, 0, 1, 10, None) != 0
    assert lib.coot_vec_mailbox_create(None, 0, None, None) != 0
    for fn, args in (("coot_sync", [None]), ("coot_stats", [None, None]),
                     ("coot_eval", [None, None, None]), ("coot_comm_destroy", [None])):
        assert getattr(lib, fn)(*args) != 0, fn
    return n_ok, n_err


def oracle_all():
    rng = random.Random(2)
    for et in ("f32", "f64", "u32", "s64", "bf16", "f16", "e4m3", "e5m2"):
        n = 1237
        ops = [oracle.fill(et, "randu", n, stream=s) for s in range(3)]
        base = et if et in ALL else "f32"
        for d in range(5):
            p = random_program(rng, d, base)
            z = oracle.eval_program(et, p, ops, [1.5, 0.25] if et not in ("u32", "s64") else [3, 5])
            for kind in ("ACCU", "MIN", "MAX", "MINMAX") + (("NORM2",) if et not in ("u32", "s64") else ()):
                oracle.reduce(et, kind, z)
                acc = oracle.Accumulator(et, kind)
                acc.add(z[:500])
                acc.add(z[500:])
                acc.final()
        if et not in ("u32", "s64"):
            for k in ("MEAN", "VAR", "STDDEV"):
                oracle.stats(et, k, ops[0])
        for k in ("INDEX_MIN", "INDEX_MAX"):
            oracle.stats(et, k, ops[1])
        for dim in (0, 1):
            oracle.sum_dim(et, dim, ops[0][:1200], 40, 30)
        rs = oracle.RowSums(et, 40)
        rs.add_rows_of(ops[0][:1200], 40, 0, 17)
        rs.add_rows_of(ops[0][:1200], 40, 17, 23)
        rs.final()
        del rs
        prog = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("LOAD", 2), ("ADD", 0)]
        oracle.run_chunked(et, prog, ["randu"] * 3, start=77, count=5000, kind="ACCU",
                           want_out=True, chunk=999)
        for _ in oracle.stream_chunks(et, prog, ["randu"] * 3, start=5, count=3000, chunk=1000,
                                      threads=2):
            pass
    return True


if __name__ == "__main__":
    ok, err = libcoot_host()
    oracle_all()
    print(f"sanitize host driver ok: {ok} valid / {err} rejected descriptors")
