"""Python front end: a ctx wrapper and an Armadillo/Bandicoot-style expression
builder with delayed evaluation.

Delayed evaluation (§3): operators only build an
expression tree (the analogue of the eOp/eGlue compound types);
nothing runs on the device until the expression is assigned (``eval``,
``assign``) or reduced (``accu``, ``sum``, ``dot``, ``norm2``, ``min``,
``max``).  At that point the tree is lowered to a postfix ``coot_expr`` and
handed to ONE libcoot call.  Matrices are dense column-major
(R2); ``Col`` is n x 1 and ``Row`` is 1 x n.

torch is used only for device memory and streams; every element of every
step is computed by libcoot's CUDA kernels.
"""
from __future__ import annotations

import builtins
import ctypes
import numbers

import torch

from . import _native as N
from ._native import CootError, check, lib

TORCH_DTYPE = {"f32": torch.float32, "f64": torch.float64, "u32": torch.uint32,
               "s64": torch.int64, "bf16": torch.bfloat16, "f16": torch.float16,
               "e4m3": torch.float8_e4m3fn, "e5m2": torch.float8_e5m2}
ELEM_OF = {v: k for k, v in TORCH_DTYPE.items()}
ESIZE = {"f32": 4, "f64": 8, "u32": 4, "s64": 8, "bf16": 2, "f16": 2, "e4m3": 1, "e5m2": 1}
# reduction / dim-sum result dtype: eT, f32 for the 8-bit storage types (R25)
RESULT_DTYPE = dict(TORCH_DTYPE, e4m3=torch.float32, e5m2=torch.float32)


def elem_of(t: torch.Tensor) -> str:
    try:
        return ELEM_OF[t.dtype]
    except KeyError:
        raise CootError(5, f"contract: unsupported dtype {t.dtype}") from None


# ============================================================================
# ctx
# ============================================================================
class Context:
    """A libcoot ctx bound to (device, stream) — coot_init."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None,
                 flags: int = 0):
        self.device_index = int(device)
        self.device = torch.device("cuda", self.device_index)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        check(lib.coot_init(ctypes.byref(h), self.device_index,
                            ctypes.c_void_p(self.stream.cuda_stream), flags))
        self._h = h

    @property
    def handle(self):
        if self._h is None:
            raise CootError(1, "configuration: ctx is closed")
        return self._h

    def close(self):
        if getattr(self, "_h", None) is not None:
            check(lib.coot_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_stream(self, stream: torch.cuda.Stream):
        check(lib.coot_set_stream(self.handle, ctypes.c_void_p(stream.cuda_stream)))
        self.stream = stream

    # ---- program-level entry points (what tests and bench.py call) --------
    def eval(self, elem, n_rows, n_cols, program, operands, scalars, out: torch.Tensor):
        e = N.make_expr(elem, n_rows, n_cols, program, operands, scalars)
        check(lib.coot_eval(self.handle, ctypes.byref(e), ctypes.c_void_p(out.data_ptr())))

    def eval_view(self, elem, n_rows, n_cols, program, operands, scalars, out: tuple):
        """Assign into a strided destination view (ptr, n_rows, n_cols, ld, inc)."""
        e = N.make_expr(elem, n_rows, n_cols, program, operands, scalars)
        o = N.make_operand(out)
        check(lib.coot_eval_view(self.handle, ctypes.byref(e), ctypes.byref(o)))

    def reduce(self, elem, n_rows, n_cols, program, operands, scalars, kind,
               result: torch.Tensor, out: torch.Tensor | None = None):
        e = N.make_expr(elem, n_rows, n_cols, program, operands, scalars)
        check(lib.coot_reduce(self.handle, ctypes.byref(e), N.KIND[kind],
                              ctypes.c_void_p(result.data_ptr()),
                              ctypes.c_void_p(out.data_ptr() if out is not None else 0)))

    def reduce_partial(self, elem, n_rows, n_cols, program, operands, scalars, kind,
                       partial: torch.Tensor, out: torch.Tensor | None = None):
        e = N.make_expr(elem, n_rows, n_cols, program, operands, scalars)
        check(lib.coot_reduce_partial(self.handle, ctypes.byref(e), N.KIND[kind],
                                      ctypes.c_void_p(partial.data_ptr()),
                                      ctypes.c_void_p(out.data_ptr() if out is not None else 0)))

    def combine(self, elem, kind, partials: torch.Tensor, nparts: int, length: int,
                result: torch.Tensor):
        check(lib.coot_combine(self.handle, N.ELEM[elem], N.KIND[kind],
                               ctypes.c_void_p(partials.data_ptr()), nparts, length,
                               ctypes.c_void_p(result.data_ptr())))

    # ---- communicator (coot.h "Communicator") ---------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        """A fresh NCCL unique id (one rank creates it, every rank gets a copy)."""
        b = ctypes.create_string_buffer(N.COMM_ID_BYTES)
        check(lib.coot_comm_unique_id(b))
        return b.raw

    def comm_init(self, nranks: int, rank: int, uid: bytes, shard: str = "cols"):
        """Bind this ctx to an NCCL communicator (collective over nranks ranks):
        from then on ``reduce`` returns GLOBAL results over the ranks' shards."""
        if shard not in N.SHARD:
            raise CootError(5, f"contract: unknown shard kind {shard!r} (none / cols / rows)")
        b = ctypes.create_string_buffer(bytes(uid), N.COMM_ID_BYTES)
        check(lib.coot_comm_init(self.handle, nranks, rank, b, N.SHARD[shard]))

    def comm_destroy(self):
        check(lib.coot_comm_destroy(self.handle))

    # ---- in-kernel exchange (coot.h "In-kernel exchange") -------------------
    def mailbox_create(self) -> tuple[int, bytes]:
        """A zeroed mailbox on this device: (device pointer, CUDA IPC handle)."""
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(N.IPC_HANDLE_BYTES)
        check(lib.coot_mailbox_create(self.handle, ctypes.byref(p), h))
        return int(p.value), h.raw

    def vec_mailbox_create(self, capacity: int) -> tuple[int, bytes]:
        """A zeroed vector mailbox for sum(X,1) partials of up to `capacity` rows:
        (device pointer, CUDA IPC handle)."""
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(N.IPC_HANDLE_BYTES)
        check(lib.coot_vec_mailbox_create(self.handle, capacity, ctypes.byref(p), h))
        return int(p.value), h.raw

    def sum_dim_exchange(self, elem, n_rows, n_cols, program, operands, scalars, kind,
                         mailboxes, rank: int, epoch: int, capacity: int, result: torch.Tensor):
        e = N.make_expr(elem, n_rows, n_cols, program, operands, scalars)
        mb = (ctypes.c_void_p * len(mailboxes))(*mailboxes)
        check(lib.coot_sum_dim_exchange(self.handle, ctypes.byref(e), N.KIND[kind], mb,
                                        len(mailboxes), rank, epoch, capacity,
                                        ctypes.c_void_p(result.data_ptr())))

    def mailbox_open(self, ipc_handle: bytes) -> int:
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(bytes(ipc_handle), N.IPC_HANDLE_BYTES)
        check(lib.coot_mailbox_open(self.handle, h, ctypes.byref(p)))
        return int(p.value)

    def mailbox_close(self, ptr: int):
        check(lib.coot_mailbox_close(self.handle, ctypes.c_void_p(ptr)))

    def mailbox_destroy(self, ptr: int):
        check(lib.coot_mailbox_destroy(self.handle, ctypes.c_void_p(ptr)))

    def reduce_exchange(self, elem, n_rows, n_cols, program, operands, scalars, kind,
                        mailboxes, rank: int, epoch: int, result: torch.Tensor,
                        out: torch.Tensor | None = None):
        e = N.make_expr(elem, n_rows, n_cols, program, operands, scalars)
        mb = (ctypes.c_void_p * len(mailboxes))(*mailboxes)
        check(lib.coot_reduce_exchange(self.handle, ctypes.byref(e), N.KIND[kind], mb,
                                       len(mailboxes), rank, epoch,
                                       ctypes.c_void_p(result.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr() if out is not None else 0)))

    def fill(self, out: torch.Tensor, kind: str = "randu", *, seed: int = 42, stream: int = 0,
             start: int = 0, n_rows: int = 1, k: int = 1):
        check(lib.coot_fill(self.handle, N.ELEM[elem_of(out)], N.FILL[kind], seed, stream, start,
                            out.numel(), n_rows, k, ctypes.c_void_p(out.data_ptr())))

    def stream_mix(self, ins: list, out: torch.Tensor | None, n: int, sink: torch.Tensor):
        """Measurement kernel (coot_stream_mix): stream n f32 from `ins` into `out`."""
        arr = (ctypes.c_void_p * builtins.max(1, len(ins)))(*[t.data_ptr() for t in ins])
        check(lib.coot_stream_mix(self.handle, len(ins), 1 if out is not None else 0, n, arr,
                                  ctypes.c_void_p(out.data_ptr() if out is not None else 0),
                                  ctypes.c_void_p(sink.data_ptr())))

    def sync(self):
        check(lib.coot_sync(self.handle))

    def stats(self) -> dict:
        s = N.Stats()
        check(lib.coot_stats(self.handle, ctypes.byref(s)))
        return {"launches": s.launches, "last_path": s.last_path, "last_grid": s.last_grid,
                "last_alg_bytes": s.last_alg_bytes, "sm_count": s.sm_count}


_default: dict[int, Context] = {}


def init(device: int = 0, print_info: bool = False) -> Context:
    """coot_init analogue: the default ctx for `device`."""
    if device not in _default:
        _default[device] = Context(device, flags=N.INIT_PRINT_INFO if print_info else 0)
    return _default[device]


def default_ctx(device: int | None = None) -> Context:
    """The default ctx for `device`, re-bound to torch's CURRENT stream on every
    call: work issued inside ``with torch.cuda.stream(s)`` is enqueued on s, in
    order with the torch ops that produced its operands.  (An explicitly passed
    Context keeps the stream it was created with / set_stream'ed to.)"""
    if device is None:
        device = torch.cuda.current_device()
    ctx = init(device)
    cur = torch.cuda.current_stream(ctx.device)
    if cur.cuda_stream != ctx.stream.cuda_stream:
        ctx.set_stream(cur)
    return ctx


def partial_bytes(kind: str, length: int = 1) -> int:
    b = ctypes.c_uint64()
    check(lib.coot_partial_bytes(N.KIND[kind], length, ctypes.byref(b)))
    return int(b.value)


def shard_range(n: int, rank: int, nranks: int, align: int = 1) -> tuple[int, int]:
    """Contiguous block of [0, n) owned by `rank` (reading R17)."""
    b, e = ctypes.c_uint64(), ctypes.c_uint64()
    check(lib.coot_shard_range(n, rank, nranks, align, ctypes.byref(b), ctypes.byref(e)))
    return int(b.value), int(e.value)


def validate(elem, n_rows, n_cols, program, operands, scalars=()):
    """Host-only descriptor validation (no GPU needed)."""
    e = N.make_expr(elem, n_rows, n_cols, program, operands, scalars)
    check(lib.coot_validate(ctypes.byref(e)))


# ============================================================================
# expression builder (delayed evaluation)
# ============================================================================
class Expr:
    """Base of every matrix / vector / expression object (cf. Base<eT,T1>)."""

    elem: str
    n_rows: int
    n_cols: int

    # element-wise binary (eGlue) and scalar (eOp) operators
    def __add__(self, o):
        return _binary("ADD", self, o)

    def __radd__(self, o):
        return _binary("ADD", o, self)

    def __sub__(self, o):
        return _binary("SUB", self, o)

    def __rsub__(self, o):
        return _binary("SUB", o, self)

    def __mul__(self, o):
        if isinstance(o, Expr):
            raise NotImplementedError(
                "matrix product (Glue<...,glue_times>) is out of scope; use % for the Schur product")
        return _binary("MUL", self, o)

    def __rmul__(self, o):
        if isinstance(o, Expr):
            raise NotImplementedError("matrix product is out of scope")
        return _binary("MUL", o, self)

    def __mod__(self, o):  # Schur product (reading R1)
        return _binary("MUL", self, o)

    def __rmod__(self, o):
        return _binary("MUL", o, self)

    def __truediv__(self, o):
        return _binary("DIV", self, o)

    def __rtruediv__(self, o):
        return _binary("DIV", o, self)

    def __neg__(self):
        return Node("NEG", (self,))

    @property
    def n_elem(self) -> int:
        return self.n_rows * self.n_cols

    # ---- evaluation ------------------------------------------------------
    def eval(self, ctx: Context | None = None, out: "Mat | View | None" = None):
        """Assign the expression to a (new or given) matrix or view: ONE launch."""
        lw = lower(self)
        ctx = ctx or default_ctx(lw.device_index())
        if out is None:
            out = Mat.empty(lw.n_rows, lw.n_cols, lw.elem, device=lw.device())
        elif (out.n_rows, out.n_cols, out.elem) != (lw.n_rows, lw.n_cols, lw.elem):
            raise CootError(2, f"conformability: assignment target is {out.n_rows}x{out.n_cols} "
                               f"{out.elem}, expression is {lw.n_rows}x{lw.n_cols} {lw.elem}")
        if isinstance(out, View):
            ctx.eval_view(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands, lw.scalars,
                          out.operand())
        else:
            ctx.eval(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands, lw.scalars, out.data)
        return out


class Mat(Expr):
    """Dense column-major matrix held in a flat device tensor (Mat<eT>)."""

    def __init__(self, data: torch.Tensor, n_rows: int, n_cols: int):
        if data.dim() != 1 or not data.is_contiguous():
            raise CootError(5, "contract: Mat data must be a contiguous 1-D tensor "
                               "(column-major element order)")
        if data.numel() != n_rows * n_cols:
            raise CootError(2, f"conformability: {data.numel()} elements for {n_rows}x{n_cols}")
        self.data = data
        self.elem = elem_of(data)
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)

    @classmethod
    def empty(cls, n_rows, n_cols, elem="f32", device="cuda"):
        return cls(torch.empty(n_rows * n_cols, dtype=TORCH_DTYPE[elem], device=device),
                   n_rows, n_cols)

    @classmethod
    def from_torch(cls, t: torch.Tensor):
        """Copy a (rows x cols) torch matrix (or 1-D vector -> Col) into column-major."""
        if t.dim() == 1:
            return cls(t.contiguous(), t.numel(), 1)
        r, c = t.shape
        return cls(t.t().contiguous().reshape(-1), r, c)

    @classmethod
    def randu(cls, n_rows, n_cols, elem="f32", *, seed=42, stream=0, ctx: Context | None = None,
              device=None):
        """fill::randu: uniform [0,1) from the counter-based recipe."""
        ctx = ctx or default_ctx(device)
        m = cls.empty(n_rows, n_cols, elem, device=ctx.device)
        ctx.fill(m.data, "randu", seed=seed, stream=stream, n_rows=n_rows)
        return m

    @classmethod
    def fill(cls, n_rows, n_cols, kind, elem="f32", *, seed=42, stream=0, k=1,
             ctx: Context | None = None, device=None):
        ctx = ctx or default_ctx(device)
        m = cls.empty(n_rows, n_cols, elem, device=ctx.device)
        ctx.fill(m.data, kind, seed=seed, stream=stream, n_rows=n_rows, k=k)
        return m

    def to_torch(self) -> torch.Tensor:
        """(rows x cols) row-major view copy of the column-major data."""
        return self.data.reshape(self.n_cols, self.n_rows).t()

    # ---- views (P:177 `Z.diag() += 100`, P:255 diagonal / submatrix views) -----
    def diag(self, k: int = 0) -> "View":
        """k-th diagonal as an n x 1 Col view (k > 0 above, k < 0 below the main)."""
        m, n = self.n_rows, self.n_cols
        # (this module defines coot's own min/max; use the builtins here)
        if k >= 0:
            length, off = builtins.max(0, builtins.min(m, n - k)), k * m
        else:
            length, off = builtins.max(0, builtins.min(m + k, n)), -k
        if length == 0:
            raise CootError(3, f"bounds: diagonal {k} of a {m}x{n} matrix is empty")
        return View(self, off, length, 1, ld=length, inc=m + 1)

    def submat(self, r0: int, c0: int, r1: int, c1: int) -> "View":
        """Rows r0..r1, columns c0..c1 (inclusive, Armadillo convention)."""
        if not (0 <= r0 <= r1 < self.n_rows and 0 <= c0 <= c1 < self.n_cols):
            raise CootError(3, f"bounds: submat({r0},{c0},{r1},{c1}) of {self.n_rows}x{self.n_cols}")
        return View(self, r0 + c0 * self.n_rows, r1 - r0 + 1, c1 - c0 + 1, ld=self.n_rows, inc=1)

    def col(self, j: int) -> "View":
        return self.submat(0, j, self.n_rows - 1, j)

    def row(self, i: int) -> "View":
        return self.submat(i, 0, i, self.n_cols - 1)

    def operand(self) -> tuple:
        return (self.data.data_ptr(), self.n_rows, self.n_cols, self.n_rows, 1)

    def assign(self, e: Expr, ctx: Context | None = None) -> "Mat":
        """self = e (exact aliasing with an operand is allowed: B += 3*A)."""
        return as_expr(e, self.elem).eval(ctx, out=self)

    def __iadd__(self, o):
        return self.assign(self + o)

    def __isub__(self, o):
        return self.assign(self - o)

    def __imod__(self, o):
        return self.assign(self % o)

    def __imul__(self, o):
        return self.assign(self * o)

    def __itruediv__(self, o):
        return self.assign(self / o)


class View(Expr):
    """A strided view of a Mat: element (i, j) at parent.data[offset + i*inc + j*ld].
    Usable as an operand anywhere, and as an assignment target (`d = Z.diag();
    d += 100` evaluates [L0 S0 ADD] into the diagonal in one launch)."""

    def __init__(self, parent: Mat, offset: int, n_rows: int, n_cols: int, ld: int, inc: int):
        self.parent = parent
        self.offset = int(offset)
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.ld, self.inc = int(ld), int(inc)
        self.elem = parent.elem

    @property
    def data(self):
        raise CootError(5, "contract: a View has no dense storage; use to_torch()")

    def operand(self) -> tuple:
        ptr = self.parent.data.data_ptr() + self.offset * ESIZE[self.elem]
        return (ptr, self.n_rows, self.n_cols, self.ld, self.inc)

    def to_torch(self) -> torch.Tensor:
        """(rows x cols) copy of the viewed elements."""
        t = torch.as_strided(self.parent.data, (self.n_cols, self.n_rows), (self.ld, self.inc),
                             self.offset)
        return t.t().contiguous()

    def assign(self, e: Expr, ctx: Context | None = None) -> "View":
        return as_expr(e).eval(ctx, out=self)

    def __iadd__(self, o):
        return self.assign(self + o)

    def __isub__(self, o):
        return self.assign(self - o)

    def __imod__(self, o):
        return self.assign(self % o)

    def __imul__(self, o):
        return self.assign(self * o)

    def __itruediv__(self, o):
        return self.assign(self / o)


def Col(data: torch.Tensor) -> Mat:
    return Mat(data, data.numel(), 1)


def Row(data: torch.Tensor) -> Mat:
    return Mat(data, 1, data.numel())


class ScalarLeaf(Expr):
    def __init__(self, value):
        self.value = value
        self.elem = None
        self.n_rows = self.n_cols = None


class Node(Expr):
    def __init__(self, op: str, kids: tuple):
        self.op = op
        self.kids = kids
        mats = [k for k in kids if not isinstance(k, ScalarLeaf)]
        ref = mats[0]
        self.elem = ref.elem
        self.n_rows, self.n_cols = ref.n_rows, ref.n_cols
        for k in mats[1:]:
            if k.elem != ref.elem:
                raise CootError(5, f"contract: mixed element types {ref.elem} and {k.elem} in {op}")
        self._mats = mats


def as_expr(x, elem=None):
    if isinstance(x, Expr):
        return x
    if isinstance(x, numbers.Number):
        return ScalarLeaf(x)
    raise TypeError(f"cannot use {type(x).__name__} in a coot expression")


def _binary(op, a, b):
    a, b = as_expr(a), as_expr(b)
    if isinstance(a, ScalarLeaf) and isinstance(b, ScalarLeaf):
        raise TypeError("scalar-only expression")
    return Node(op, (a, b))


def _unary(op, a):
    a = as_expr(a)
    if isinstance(a, ScalarLeaf):
        raise TypeError("scalar-only expression")
    return Node(op, (a,))


def exp(x): return _unary("EXP", x)
def log(x): return _unary("LOG", x)
def sqrt(x): return _unary("SQRT", x)
def abs(x): return _unary("ABS", x)  # noqa: A001
def square(x): return _unary("SQUARE", x)


class Lowered:
    """A lowered expression: postfix program + operands (dense tensors or view
    tuples (ptr, n_rows, n_cols, ld, inc)) + scalars."""

    def __init__(self, elem, n_rows, n_cols, program, operands, scalars, dev=None):
        self.elem, self.n_rows, self.n_cols = elem, n_rows, n_cols
        self.program, self.operands, self.scalars = program, operands, scalars
        self.dev = dev

    def device(self):
        return self.dev

    def device_index(self):
        return self.dev.index


def lower(e: Expr) -> Lowered:
    """Tree -> postfix program.  Operands are deduplicated by identity of their
    storage (each distinct array is loaded once); scalars by value."""
    if isinstance(e, ScalarLeaf):
        raise TypeError("scalar-only expression")
    operands: list = []
    op_index: dict = {}
    scalars: list = []
    program: list[tuple[str, int]] = []
    elem, nr, nc = e.elem, e.n_rows, e.n_cols
    dev = [None]

    def visit(x):
        if isinstance(x, (Mat, View)):
            if (x.n_rows, x.n_cols) != (nr, nc):
                raise CootError(2, f"conformability: operand is {x.n_rows}x{x.n_cols}, "
                                   f"expression is {nr}x{nc}")
            key = x.operand()
            if key not in op_index:
                op_index[key] = len(operands)
                operands.append(x.data if isinstance(x, Mat) else key)
                dev[0] = dev[0] or (x.data.device if isinstance(x, Mat) else x.parent.data.device)
            program.append(("LOAD", op_index[key]))
        elif isinstance(x, ScalarLeaf):
            v = x.value
            if elem in ("u32", "s64") and isinstance(v, float) and not float(v).is_integer():
                raise CootError(5, f"contract: scalar {v!r} is not integral for a {elem} expression")
            for i, s in enumerate(scalars):
                if type(s) is type(v) and s == v:
                    program.append(("SCALAR", i))
                    break
            else:
                scalars.append(v)
                program.append(("SCALAR", len(scalars) - 1))
        else:
            if (x.n_rows, x.n_cols) != (nr, nc):
                raise CootError(2, f"conformability: {x.op} operand is {x.n_rows}x{x.n_cols}, "
                                   f"expression is {nr}x{nc}")
            for k in x.kids:
                visit(k)
            program.append((x.op, 0))

    visit(e)
    return Lowered(elem, nr, nc, program, operands, scalars, dev[0])


# ---- terminal reductions ----------------------------------------------------
def _reduce(e, kind, ctx=None, out: Mat | None = None):
    lw = lower(as_expr(e))
    ctx = ctx or default_ctx(lw.device_index())
    shape = {"MINMAX": (2,), "SUM_DIM0": (lw.n_cols,), "SUM_DIM1": (lw.n_rows,)}.get(kind, (1,))
    dtype = torch.int64 if kind.startswith("INDEX") else RESULT_DTYPE[lw.elem]
    result = torch.empty(shape, dtype=dtype, device=lw.device())
    ctx.reduce(lw.elem, lw.n_rows, lw.n_cols, lw.program, lw.operands, lw.scalars, kind, result,
               out.data if out is not None else None)
    return result


def accu(e, ctx=None, out: Mat | None = None) -> torch.Tensor:
    """Sum of all elements (``float result = sum(A)``); 1-element device tensor."""
    return _reduce(e, "ACCU", ctx, out)


def sum(e, dim: int | None = None, ctx=None):  # noqa: A001
    """Armadillo sum: dim 0 -> column sums (Row), dim 1 -> row sums (Col) (R3);
    for a vector with dim=None the sum of all elements."""
    e = as_expr(e)
    if dim is None:
        if e.n_rows == 1 or e.n_cols == 1:
            return accu(e, ctx)
        dim = 0
    r = _reduce(e, "SUM_DIM0" if dim == 0 else "SUM_DIM1", ctx)
    return Mat(r, 1, r.numel()) if dim == 0 else Mat(r, r.numel(), 1)


def dot(a, b, ctx=None):
    """dot(x, y) = accu(x % y) with eT-rounded products (reading R11)."""
    return accu(as_expr(a) % as_expr(b), ctx)


def norm2(e, ctx=None):
    return _reduce(e, "NORM2", ctx)


def min(a, b=None, ctx=None):  # noqa: A001
    """min(X): smallest element (reduction); min(A, B): element-wise."""
    if b is not None:
        return _binary("MIN", a, b)
    return _reduce(a, "MIN", ctx)


def max(a, b=None, ctx=None):  # noqa: A001
    if b is not None:
        return _binary("MAX", a, b)
    return _reduce(a, "MAX", ctx)


def minmax(e, ctx=None):
    return _reduce(e, "MINMAX", ctx)


# ---- statistics ("mean, variance"; Armadillo semantics, R22) ----------
def mean(e, ctx=None):
    """Mean of all elements (floats), one launch."""
    return _reduce(e, "MEAN", ctx)


def var(e, ctx=None):
    """Variance with n-1 normalisation (Armadillo default), one pass, one launch."""
    return _reduce(e, "VAR", ctx)


def stddev(e, ctx=None):
    return _reduce(e, "STDDEV", ctx)


def index_min(e, ctx=None):
    """Column-major linear index of the first smallest element (int64 tensor)."""
    return _reduce(e, "INDEX_MIN", ctx)


def index_max(e, ctx=None):
    return _reduce(e, "INDEX_MAX", ctx)
