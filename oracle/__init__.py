"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, unfused CPU reference for the fused element-wise expression +
reduction path (see coot_oracle.c for the per-function paper citations).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the
product package ``paper_2508_11385_b200`` never does, and shares no code
with it.

Programs are lists of ``(op_name, arg)`` tuples in postfix order, e.g.
``[("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0),
("LOAD", 2), ("MUL", 0), ("ADD", 0)]`` for ``exp(A % B) + 3*C``.
Arrays are numpy 1-D arrays holding the column-major element order.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

TYPES = {"f32": 0, "f64": 1, "u32": 2, "s64": 3, "bf16": 4, "f16": 5, "e4m3": 6, "e5m2": 7}
# bf16 / fp8 arrays are carried as their bit patterns (numpy has no such dtypes)
DTYPES = {"f32": np.float32, "f64": np.float64, "u32": np.uint32, "s64": np.int64,
          "bf16": np.uint16, "f16": np.float16, "e4m3": np.uint8, "e5m2": np.uint8}
FP8 = ("e4m3", "e5m2")
# reduction / dim-sum / statistics result dtype: eT, f32 for the fp8 storage types (R25)
RDTYPES = dict(DTYPES, e4m3=np.float32, e5m2=np.float32)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float32."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def fp8_table(etype: str) -> np.ndarray:
    """The 256 exact values of an fp8 format, indexed by bit pattern."""
    return np.array([lib().orc_fp8_to_double(TYPES[etype], b) for b in range(256)])


def to_float(etype: str, a: np.ndarray) -> np.ndarray:
    """Exact float64 values of an array of any float element type."""
    if etype == "bf16":
        return bf16_to_f32(a).astype(np.float64)
    if etype in FP8:
        return fp8_table(etype)[np.asarray(a, dtype=np.uint8)]
    return np.asarray(a).astype(np.float64)
OPS = {
    "LOAD": 0, "SCALAR": 1, "NEG": 2, "ABS": 3, "SQUARE": 4, "SQRT": 5, "EXP": 6,
    "LOG": 7, "ADD": 8, "SUB": 9, "MUL": 10, "DIV": 11, "MIN": 12, "MAX": 13,
}
KINDS = {"ACCU": 0, "MIN": 1, "MAX": 2, "MINMAX": 3, "NORM2": 4}
FILLS = {"randu": 0, "ones": 1, "iota": 2, "modk": 3, "colidx": 4, "rowidx": 5, "zeros": 6}

_lib = None


def lib():
    global _lib
    if _lib is None:
        # ORACLE_LIB_PATH: a prebuilt variant (the sanitizer build of tests/test_sanitizers.py)
        path = os.environ.get("ORACLE_LIB_PATH") or _build.build()
        L = ctypes.CDLL(path)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        L.orc_half_from_double.restype = ctypes.c_uint16
        L.orc_half_from_double.argtypes = [i32, ctypes.c_double]
        L.orc_fp8_from_double.restype = ctypes.c_uint8
        L.orc_fp8_from_double.argtypes = [i32, ctypes.c_double]
        L.orc_fp8_to_double.restype = ctypes.c_double
        L.orc_fp8_to_double.argtypes = [i32, ctypes.c_uint8]
        L.orc_hash.restype = u64
        L.orc_hash.argtypes = [u64, u64, u64]
        L.orc_fill.restype = i32
        L.orc_fill.argtypes = [i32, i32, u64, u64, u64, u64, u64, u64, vp]
        L.orc_eval.restype = i32
        L.orc_eval.argtypes = [i32, u64, ctypes.POINTER(vp), i32, vp, i32,
                               ctypes.POINTER(i32), ctypes.POINTER(i32), i32, vp]
        L.orc_eval_batch.restype = i32
        L.orc_eval_batch.argtypes = [i32, u64, ctypes.POINTER(vp), i32, vp, i32, vp, vp, vp,
                                     ctypes.c_int64, vp]
        L.orc_acc_size.restype = ctypes.c_size_t
        L.orc_acc_init.restype = i32
        L.orc_acc_init.argtypes = [vp, i32, i32]
        L.orc_acc_add.restype = i32
        L.orc_acc_add.argtypes = [vp, u64, vp]
        L.orc_acc_final.restype = i32
        L.orc_acc_final.argtypes = [vp, vp]
        L.orc_reduce.restype = i32
        L.orc_reduce.argtypes = [i32, i32, u64, vp, vp]
        L.orc_stats.restype = i32
        L.orc_stats.argtypes = [i32, i32, u64, vp, vp]
        L.orc_sum_dim.restype = i32
        L.orc_sum_dim.argtypes = [i32, i32, u64, u64, vp, vp]
        L.orc_rows_new.restype = vp
        L.orc_rows_new.argtypes = [i32, u64]
        L.orc_rows_free.restype = None
        L.orc_rows_free.argtypes = [vp]
        L.orc_rows_add.restype = i32
        L.orc_rows_add.argtypes = [vp, u64, u64, u64, u64, vp]
        L.orc_rows_final.restype = i32
        L.orc_rows_final.argtypes = [vp, vp]
        L.orc_run_chunked.restype = i32
        L.orc_run_chunked.argtypes = [i32, u64, u64, u64, i32, ctypes.POINTER(i32), u64, u64,
                                      vp, i32, ctypes.POINTER(i32), ctypes.POINTER(i32), i32,
                                      u64, vp, vp]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(f"oracle {what} failed with code {rc}")


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def hash64(seed: int, stream: int, i: int) -> int:
    return int(lib().orc_hash(seed, stream, i))


def fill(etype: str, kind: str, count: int, *, seed: int = 42, stream: int = 0,
         start: int = 0, n_rows: int = 1, k: int = 1) -> np.ndarray:
    """Generate elements [start, start+count) of a (global) operand."""
    out = np.empty(count, dtype=DTYPES[etype])
    _check(lib().orc_fill(TYPES[etype], FILLS[kind], seed, stream, start, count, n_rows, k,
                          _ptr(out)), "fill")
    return out


def _encode_program(program):
    n = len(program)
    ops = (ctypes.c_int * max(n, 1))(*[OPS[o] for o, _ in program])
    args = (ctypes.c_int * max(n, 1))(*[int(a) for _, a in program])
    return ops, args, n


def _scalar_array(etype: str, scalars):
    if etype in ("bf16", "f16"):  # R4: the scalar rounded once to the 16-bit format
        bits = [lib().orc_half_from_double(TYPES[etype], float(s)) for s in (scalars or [0])]
        return np.array(bits, dtype=np.uint16).view(DTYPES[etype])
    if etype in FP8:  # R25: the arithmetic type is f32, so scalars are f32
        return np.array(list(scalars) if scalars else [0], dtype=np.float32)
    return np.array(list(scalars) if scalars else [0], dtype=DTYPES[etype])


def half_from_double(etype: str, x: float) -> int:
    """Bits of x rounded (nearest-even) to bf16 / f16."""
    return int(lib().orc_half_from_double(TYPES[etype], float(x)))


def fp8_from_double(etype: str, x: float) -> int:
    """Bits of x rounded (nearest-even, saturating) to e4m3 / e5m2."""
    return int(lib().orc_fp8_from_double(TYPES[etype], float(x)))


def eval_program(etype: str, program, operands, scalars=()) -> np.ndarray:
    """Eager op-by-op evaluation: each node a new temporary."""
    dt = DTYPES[etype]
    ops_ = [np.ascontiguousarray(o, dtype=dt) for o in operands]
    n = ops_[0].size if ops_ else 0
    for o in ops_:
        if o.size != n:
            raise ValueError("operands must have the same number of elements")
    ptrs = (ctypes.c_void_p * max(len(ops_), 1))(*[o.ctypes.data for o in ops_])
    sc = _scalar_array(etype, scalars)
    opc, argc, ni = _encode_program(program)
    out = np.empty(n, dtype=dt)
    _check(lib().orc_eval(TYPES[etype], n, ptrs, len(ops_), _ptr(sc), len(scalars), opc, argc,
                          ni, _ptr(out)), "eval")
    return out


def eval_programs(etype: str, programs, operands, scalars=()) -> np.ndarray:
    """eval_program for many programs over the same operands (one C call);
    returns an array of shape (len(programs), n)."""
    dt = DTYPES[etype]
    ops_ = [np.ascontiguousarray(o, dtype=dt) for o in operands]
    n = ops_[0].size
    ptrs = (ctypes.c_void_p * max(len(ops_), 1))(*[o.ctypes.data for o in ops_])
    sc = _scalar_array(etype, scalars)
    lens = np.array([len(p) for p in programs], dtype=np.int64)
    offs = np.zeros(len(programs) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    flat = [x for p in programs for x in p]
    opc = np.array([OPS[o] for o, _ in flat], dtype=np.int32)
    argc = np.array([int(a) for _, a in flat], dtype=np.int32)
    out = np.empty((len(programs), n), dtype=dt)
    _check(lib().orc_eval_batch(TYPES[etype], n, ptrs, len(ops_), _ptr(sc), len(scalars),
                                _ptr(opc), _ptr(argc), _ptr(offs), len(programs), _ptr(out)),
           "eval_batch")
    return out


def reduce(etype: str, kind: str, v: np.ndarray):
    """Full reduction; returns a numpy scalar of eT (f32 for fp8), or a 2-array
    for MINMAX."""
    dt = DTYPES[etype]
    v = np.ascontiguousarray(v, dtype=dt)
    out = np.zeros(2, dtype=RDTYPES[etype])
    _check(lib().orc_reduce(TYPES[etype], KINDS[kind], v.size, _ptr(v), _ptr(out)), "reduce")
    return out.copy() if kind == "MINMAX" else out[0]


STATS = {"MEAN": 0, "VAR": 1, "STDDEV": 2, "INDEX_MIN": 3, "INDEX_MAX": 4}


def stats(etype: str, kind: str, v: np.ndarray):
    """MEAN / VAR / STDDEV (floats; eT result) or INDEX_MIN / INDEX_MAX (int)."""
    dt = DTYPES[etype]
    v = np.ascontiguousarray(v, dtype=dt)
    if kind.startswith("INDEX"):
        out = np.zeros(1, dtype=np.uint64)
    else:
        out = np.zeros(1, dtype=RDTYPES[etype])
    _check(lib().orc_stats(TYPES[etype], STATS[kind], v.size, _ptr(v), _ptr(out)), "stats")
    return int(out[0]) if kind.startswith("INDEX") else out[0]


class Accumulator:
    """Chunk-fed reduction state (bit-identical to a one-shot reduce)."""

    def __init__(self, etype: str, kind: str):
        self.etype, self.kind = etype, kind
        self._buf = ctypes.create_string_buffer(int(lib().orc_acc_size()))
        _check(lib().orc_acc_init(self._buf, TYPES[etype], KINDS[kind]), "acc_init")

    def add(self, v: np.ndarray):
        v = np.ascontiguousarray(v, dtype=DTYPES[self.etype])
        _check(lib().orc_acc_add(self._buf, v.size, _ptr(v)), "acc_add")

    def final(self):
        out = np.zeros(2, dtype=RDTYPES[self.etype])
        _check(lib().orc_acc_final(self._buf, _ptr(out)), "acc_final")
        return out.copy() if self.kind == "MINMAX" else out[0]


def sum_dim(etype: str, dim: int, X: np.ndarray, n_rows: int, n_cols: int) -> np.ndarray:
    """sum(X, dim) of a column-major n_rows x n_cols matrix stored as 1-D."""
    dt = DTYPES[etype]
    X = np.ascontiguousarray(X, dtype=dt).reshape(-1)
    if X.size != n_rows * n_cols:
        raise ValueError("X size mismatch")
    out = np.empty(n_cols if dim == 0 else n_rows, dtype=RDTYPES[etype])
    _check(lib().orc_sum_dim(TYPES[etype], dim, n_rows, n_cols, _ptr(X), _ptr(out)), "sum_dim")
    return out


def run_chunked(etype: str, program, fills, *, start: int, count: int, n_rows: int = 1,
                seed: int = 42, modk: int = 1, scalars=(), kind: str | None = None,
                want_out: bool = False, chunk: int = 1 << 24):
    """Evaluate `program` over global indices [start, start+count) with operands
    regenerated per chunk (operand k uses stream k and fill kind fills[k]).
    Returns (reduction result or None, element-wise result or None)."""
    dt = DTYPES[etype]
    fk = (ctypes.c_int * max(len(fills), 1))(*[FILLS[f] for f in fills])
    sc = _scalar_array(etype, scalars)
    opc, argc, ni = _encode_program(program)
    acc = Accumulator(etype, kind) if kind else None
    out = np.empty(count, dtype=dt) if want_out else None
    _check(lib().orc_run_chunked(TYPES[etype], start, count, n_rows, len(fills), fk, seed, modk,
                                 _ptr(sc), len(scalars), opc, argc, ni, chunk,
                                 acc._buf if acc else None,
                                 _ptr(out) if out is not None else None), "run_chunked")
    return (acc.final() if acc else None), out


class RowSums:
    """sum(X, 1) fed a block of columns at a time (orc_rows_*): the per-row
    state of orc_sum_dim's dim-1 loop kept between calls.  add(X, i0) takes a
    column-major block (rows x ncols, element (i, j) at X[i + j*rows]) of rows
    i0..; blocks must arrive in column order for each row.  Bit-identical to a
    one-shot sum_dim(..., 1, ...) (tested); calls on disjoint row ranges may run
    on different threads."""

    def __init__(self, etype: str, n_rows: int):
        self.etype, self.m = etype, n_rows
        self._h = lib().orc_rows_new(TYPES[etype], n_rows)
        if not self._h:
            raise OracleError("orc_rows_new failed")

    def add(self, X: np.ndarray, i0: int = 0, rows: int | None = None, ld: int | None = None):
        X = np.ascontiguousarray(X, dtype=DTYPES[self.etype]).reshape(-1)
        ld = ld if ld is not None else (rows if rows is not None else self.m)
        rows = rows if rows is not None else ld
        ncols = X.size // ld if ld else 0
        _check(lib().orc_rows_add(self._h, i0, rows, ncols, ld, _ptr(X)), "rows_add")

    def add_rows_of(self, X: np.ndarray, ld: int, i0: int, rows: int):
        """Add rows i0..i0+rows-1 of a column-major block with leading dimension ld."""
        X = np.ascontiguousarray(X, dtype=DTYPES[self.etype]).reshape(-1)
        ncols = X.size // ld
        base = X[i0:]  # element (i0 + i, j) at base[i + j*ld]
        _check(lib().orc_rows_add(self._h, i0, rows, ncols, ld, _ptr(base)), "rows_add")

    def final(self) -> np.ndarray:
        out = np.empty(self.m, dtype=RDTYPES[self.etype])
        _check(lib().orc_rows_final(self._h, _ptr(out)), "rows_final")
        return out

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_rows_free(self._h)
            self._h = None


def stream_chunks(etype: str, program, fills, *, start: int, count: int, n_rows: int = 1,
                  seed: int = 42, modk: int = 1, scalars=(), chunk: int = 1 << 24,
                  threads: int | None = None):
    """Yield (offset, z) for consecutive chunks of [start, start+count) IN INDEX
    ORDER, z = the program's element-wise result over that chunk (each chunk is
    orc_run_chunked's own regenerate + eval, so bit-identical to one run).  The
    chunks are computed ahead on `threads` worker threads (ctypes releases the
    GIL); the caller consumes them in order, e.g. feeding an Accumulator, so a
    reduction sees exactly the sequential index order."""
    import concurrent.futures as cf
    threads = threads or max(1, min(32, os.cpu_count() or 1))
    offs = list(range(0, count, chunk))

    def one(off):
        _, z = run_chunked(etype, program, fills, start=start + off,
                           count=min(chunk, count - off), n_rows=n_rows, seed=seed, modk=modk,
                           scalars=scalars, want_out=True, chunk=chunk)
        return z

    with cf.ThreadPoolExecutor(threads) as ex:
        pending = {}
        nxt = 0
        for k, off in enumerate(offs):
            while nxt < len(offs) and nxt < k + 2 * threads:
                pending[nxt] = ex.submit(one, offs[nxt])
                nxt += 1
            yield off, pending.pop(k).result()
