"""ctypes binding of libcoot.so (include/coot.h).  Argument marshalling only.

The library is built in-tree (``paper_2508_11385_b200/libcoot.so``).  There is
no fallback: if it is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("COOT_LIB_PATH") or os.path.join(HERE, "libcoot.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "coot.h")

ABI_VERSION = 1
MAX_OPERANDS = 8
MAX_SCALARS = 8
MAX_INSTR = 32
MAX_STACK = 8
PARTIAL_BYTES = 32

ELEM = {"f32": 0, "f64": 1, "u32": 2, "s64": 3, "bf16": 4, "f16": 5, "e4m3": 6, "e5m2": 7}
OP = {"LOAD": 0, "SCALAR": 1, "NEG": 2, "ABS": 3, "SQUARE": 4, "SQRT": 5, "EXP": 6, "LOG": 7,
      "ADD": 8, "SUB": 9, "MUL": 10, "DIV": 11, "MIN": 12, "MAX": 13}
KIND = {"ACCU": 0, "MIN": 1, "MAX": 2, "MINMAX": 3, "NORM2": 4, "SUM_DIM0": 5, "SUM_DIM1": 6,
        "MEAN": 7, "VAR": 8, "STDDEV": 9, "INDEX_MIN": 10, "INDEX_MAX": 11}
FILL = {"randu": 0, "ones": 1, "iota": 2, "modk": 3, "colidx": 4, "rowidx": 5, "zeros": 6}
STATUS = {0: "OK", 1: "CONFIG", 2: "CONFORM", 3: "BOUNDS", 4: "RESOURCE", 5: "CONTRACT", 6: "DEVICE"}
INIT_PRINT_INFO = 1
INIT_FORCE_INTERP = 2


class Instr(ctypes.Structure):
    _fields_ = [("op", ctypes.c_uint8), ("arg", ctypes.c_uint8)]


class Scalar(ctypes.Union):
    _fields_ = [("f32", ctypes.c_float), ("f64", ctypes.c_double), ("u32", ctypes.c_uint32),
                ("s64", ctypes.c_int64), ("bits", ctypes.c_uint64)]


class Operand(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("n_rows", ctypes.c_uint64),
                ("n_cols", ctypes.c_uint64), ("ld", ctypes.c_uint64), ("inc", ctypes.c_uint64)]


def make_operand(o) -> Operand:
    """(ptr, n_rows, n_cols[, ld, inc]) -> coot_operand (ld/inc 0 = dense)."""
    op = Operand()
    op.ptr = o[0]
    op.n_rows, op.n_cols = o[1], o[2]
    op.ld = o[3] if len(o) > 3 else 0
    op.inc = o[4] if len(o) > 4 else 0
    return op


class Expr(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("elem", ctypes.c_uint32),
                ("n_rows", ctypes.c_uint64), ("n_cols", ctypes.c_uint64),
                ("n_operands", ctypes.c_uint32), ("n_scalars", ctypes.c_uint32),
                ("n_instr", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("operands", Operand * MAX_OPERANDS), ("scalars", Scalar * MAX_SCALARS),
                ("prog", Instr * MAX_INSTR)]


class Stats(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_uint64), ("last_path", ctypes.c_int32),
                ("last_grid", ctypes.c_uint32), ("last_alg_bytes", ctypes.c_uint64),
                ("sm_count", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class CootError(RuntimeError):
    """A non-OK coot_status; ``.status`` is the category name."""

    def __init__(self, code: int, message: str):
        self.code = code
        self.status = STATUS.get(code, str(code))
        super().__init__(f"[{self.status}] {message}")


_u32, _u64, _i32, _vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
_SIGS = {
    "coot_abi_version": (_u32, []),
    "coot_last_error": (ctypes.c_char_p, []),
    "coot_status_string": (ctypes.c_char_p, [_i32]),
    "coot_validate": (_i32, [ctypes.POINTER(Expr)]),
    "coot_init": (_i32, [ctypes.POINTER(_vp), _i32, _vp, _u32]),
    "coot_destroy": (_i32, [_vp]),
    "coot_set_stream": (_i32, [_vp, _vp]),
    "coot_eval": (_i32, [_vp, ctypes.POINTER(Expr), _vp]),
    "coot_eval_view": (_i32, [_vp, ctypes.POINTER(Expr), ctypes.POINTER(Operand)]),
    "coot_reduce": (_i32, [_vp, ctypes.POINTER(Expr), _u32, _vp, _vp]),
    "coot_reduce_partial": (_i32, [_vp, ctypes.POINTER(Expr), _u32, _vp, _vp]),
    "coot_combine": (_i32, [_vp, _u32, _u32, _vp, _u32, _u64, _vp]),
    "coot_partial_bytes": (_i32, [_u32, _u64, ctypes.POINTER(_u64)]),
    "coot_shard_range": (_i32, [_u64, _u32, _u32, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64)]),
    "coot_fill": (_i32, [_vp, _u32, _u32, _u64, _u64, _u64, _u64, _u64, _u64, _vp]),
    "coot_sync": (_i32, [_vp]),
    "coot_stream_mix": (_i32, [_vp, _u32, _u32, _u64, ctypes.POINTER(_vp), _vp, _vp]),
    "coot_stats": (_i32, [_vp, ctypes.POINTER(Stats)]),
    "coot_comm_unique_id": (_i32, [_vp]),
    "coot_comm_init": (_i32, [_vp, _u32, _u32, _vp, _u32]),
    "coot_comm_destroy": (_i32, [_vp]),
    "coot_mailbox_create": (_i32, [_vp, ctypes.POINTER(_vp), _vp]),
    "coot_mailbox_open": (_i32, [_vp, _vp, ctypes.POINTER(_vp)]),
    "coot_mailbox_close": (_i32, [_vp, _vp]),
    "coot_mailbox_destroy": (_i32, [_vp, _vp]),
    "coot_reduce_exchange": (_i32, [_vp, ctypes.POINTER(Expr), _u32, ctypes.POINTER(_vp), _u32,
                                    _u32, _u64, _vp, _vp]),
    "coot_vec_mailbox_create": (_i32, [_vp, _u64, ctypes.POINTER(_vp), _vp]),
    "coot_sum_dim_exchange": (_i32, [_vp, ctypes.POINTER(Expr), _u32, ctypes.POINTER(_vp), _u32,
                                     _u32, _u64, _u64, _vp]),
}
MAX_RANKS = 8
IPC_HANDLE_BYTES = 64
COMM_ID_BYTES = 128
SHARD = {"none": 0, "cols": 1, "rows": 2}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libcoot.so not found at {LIB_PATH}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.coot_abi_version() != ABI_VERSION:
        raise ImportError("libcoot ABI version mismatch")
    return lib


lib = _load()


def check(code: int):
    if code != 0:
        raise CootError(code, lib.coot_last_error().decode())


def header_functions() -> list[str]:
    """Names of every function declared in include/coot.h."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(coot_[a-z_0-9]+)\s*\(", src)))


def make_expr(elem: str, n_rows: int, n_cols: int, program, operands, scalars=()) -> Expr:
    """Fill a coot_expr.  ``operands`` are (ptr, n_rows, n_cols) triples or
    objects with ``data_ptr()`` (then the expression dims are used);
    ``scalars`` are python numbers converted to eT (reading R4)."""
    e = Expr()
    e.abi_version = ABI_VERSION
    e.elem = ELEM[elem]
    e.n_rows, e.n_cols = n_rows, n_cols
    if len(operands) > MAX_OPERANDS or len(scalars) > MAX_SCALARS or len(program) > MAX_INSTR:
        # let the library report the precise bounds error
        pass
    e.n_operands = len(operands)
    e.n_scalars = len(scalars)
    e.n_instr = len(program)
    for k, o in enumerate(operands[:MAX_OPERANDS]):
        if not isinstance(o, tuple):
            o = (o.data_ptr(), n_rows, n_cols)
        e.operands[k] = make_operand(o)
    for k, s in enumerate(list(scalars)[:MAX_SCALARS]):
        set_scalar(e.scalars[k], elem, s)
    for i, (op, arg) in enumerate(list(program)[:MAX_INSTR]):
        e.prog[i].op = OP[op] if isinstance(op, str) else int(op)
        e.prog[i].arg = int(arg)
    return e


HALF_FMT = {"bf16": (8, 7), "f16": (5, 10)}  # (exponent bits, stored mantissa bits)


def half_bits(value: float, elem: str) -> int:
    """value rounded to nearest-even in bf16 / f16, as its 16-bit pattern."""
    import math
    from fractions import Fraction
    ebits, mbits = HALF_FMT[elem]
    bias = (1 << (ebits - 1)) - 1
    emask = ((1 << ebits) - 1) << mbits
    x = float(value)
    if math.isnan(x):
        return emask | (1 << (mbits - 1))
    sign = 0x8000 if math.copysign(1.0, x) < 0 else 0
    a = abs(x)
    if math.isinf(a):
        return sign | emask
    if a == 0:
        return sign
    e = math.frexp(a)[1] - 1                 # 2^e <= a < 2^(e+1)
    qe = max(e, 1 - bias) - mbits            # exponent of one unit in the last place
    scaled = Fraction(a) / (Fraction(2) ** qe)
    n = scaled.numerator // scaled.denominator
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    if n < (1 << mbits):
        return sign | n                      # subnormal
    if n == (2 << mbits):
        n >>= 1
        qe += 1
    field = qe + mbits + bias
    if field >= (1 << ebits) - 1:
        return sign | emask                  # overflow
    return sign | (field << mbits) | (n - (1 << mbits))


def set_scalar(slot: Scalar, elem: str, value):
    """Store a scalar AS the element type (R4); reject lossy integer scalars."""
    if elem in ("f32", "e4m3", "e5m2"):  # 8-bit storage types compute in f32 (R25)
        slot.bits = 0
        slot.f32 = float(value)
    elif elem == "f64":
        slot.f64 = float(value)
    elif elem in HALF_FMT:
        slot.bits = half_bits(value, elem)
    else:
        if isinstance(value, float) and not value.is_integer():
            raise CootError(5, f"contract: scalar {value!r} is not integral for a {elem} expression")
        iv = int(value)
        if elem == "u32":
            slot.bits = 0
            slot.u32 = iv & 0xFFFFFFFF
        else:
            iv &= (1 << 64) - 1
            slot.bits = iv
