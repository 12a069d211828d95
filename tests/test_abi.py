"""Host-only checks of the C ABI (no GPU needed): the library loads, exports
every function include/coot.h declares, its struct layout matches the header,
and validation reports the SPEC error taxonomy before any CUDA call."""
import ctypes
import os
import subprocess
import tempfile

import pytest

import paper_2508_11385_b200 as coot
from paper_2508_11385_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_function():
    names = N.header_functions()
    assert len(names) >= 16
    missing = [f for f in names if not hasattr(N.lib, f)]
    assert missing == []


def test_abi_version_and_status_strings():
    assert N.lib.coot_abi_version() == N.ABI_VERSION == 1
    for code, name in N.STATUS.items():
        assert N.lib.coot_status_string(code).decode().upper().startswith(
            {"CONFORM": "CONFORMABILITY", "CONFIG": "CONFIGURATION"}.get(name, name)[:4])


def test_struct_layout_matches_header():
    src = r"""
#include <stddef.h>
#include <stdio.h>
#include "coot.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(coot_expr), offsetof(coot_expr, operands),
         offsetof(coot_expr, scalars), offsetof(coot_expr, prog), sizeof(coot_operand),
         sizeof(coot_scalar), sizeof(coot_instr), sizeof(coot_stats_t), offsetof(coot_expr, n_operands));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(c, "w").write(src)
        subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        got = [int(x) for x in subprocess.check_output([exe]).split()]
    want = [ctypes.sizeof(N.Expr), N.Expr.operands.offset, N.Expr.scalars.offset, N.Expr.prog.offset,
            ctypes.sizeof(N.Operand), ctypes.sizeof(N.Scalar), ctypes.sizeof(N.Instr),
            ctypes.sizeof(N.Stats), N.Expr.n_operands.offset]
    assert got == want


def _v(prog, operands, scalars=(), elem="f32", m=10, n=10):
    return coot.validate(elem, m, n, prog, operands, scalars)


def _err(prog, operands, scalars=(), elem="f32", m=10, n=10):
    with pytest.raises(coot.CootError) as ei:
        _v(prog, operands, scalars, elem, m, n)
    return ei.value


A = (1 << 20, 10, 10)
B = (1 << 21, 10, 10)


def test_valid_descriptors_pass():
    _v([("LOAD", 0)], [A])
    _v([("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)], [A, B], [2.5])
    _v([("LOAD", k) for k in range(8)] + [("ADD", 0)] * 7, [(1 << 20 + k, 10, 10) for k in range(8)])
    _v([("LOAD", 0)], [(0, 0, 10)], m=0)  # empty operand may be NULL


@pytest.mark.parametrize("prog,ops,sc,status,frag", [
    ([("LOAD", 0), ("LOAD", 1), ("ADD", 0)], [A, (1 << 21, 10, 9)], (), "CONFORM", "10x9"),
    ([("LOAD", 0), ("ADD", 0)], [A], (), "CONTRACT", "underflow"),
    ([("LOAD", 0), ("LOAD", 0)], [A], (), "CONTRACT", "leaves 2"),
    ([("LOAD", 3)], [A], (), "CONTRACT", "LOAD 3"),
    ([("SCALAR", 0)], [A], (), "CONTRACT", "SCALAR 0"),
    ([("SCALAR", 0)], [A], (1.0,), "CONTRACT", "reads no operand"),
    ([("LOAD", 0), (99, 0)], [A], (), "CONTRACT", "opcode"),
    ([("LOAD", 0)] * 9 + [("ADD", 0)] * 8, [A], (), "BOUNDS", "stack depth 9"),
    ([("LOAD", 0)] * 17 + [("ADD", 0)] * 16, [A], (), "BOUNDS", "instructions"),
    ([("LOAD", 0)], [A] * 9, (), "BOUNDS", "operands"),
    ([("LOAD", 0)], [A], (1.0,) * 9, "BOUNDS", "scalars"),
    ([("LOAD", 0)], [(0, 10, 10)], (), "CONTRACT", "NULL"),
    ([("LOAD", 0)], [(1 << 20 | 2, 10, 10)], (), "CONTRACT", "aligned"),
])
def test_validation_errors(prog, ops, sc, status, frag):
    e = _err(prog, ops, sc)
    assert e.status == status, str(e)
    assert frag in str(e), str(e)


@pytest.mark.parametrize("op", ["SQRT", "EXP", "LOG", "DIV"])
def test_integer_illegal_ops_are_contract_errors(op):
    prog = [("LOAD", 0), (op, 0)] if op != "DIV" else [("LOAD", 0), ("LOAD", 0), ("DIV", 0)]
    e = _err(prog, [A], elem="u32")
    assert e.status == "CONTRACT" and "integer" in str(e)


def test_abi_version_mismatch_is_config_error():
    e = N.make_expr("f32", 10, 10, [("LOAD", 0)], [A])
    e.abi_version = 2
    assert N.lib.coot_validate(ctypes.byref(e)) == 1
    assert "abi_version" in N.lib.coot_last_error().decode()


def test_strided_view_operands_validate():
    # submatrix (ld > n_rows) and diagonal (inc = ld + 1) views are legal operands
    e = N.make_expr("f32", 10, 10, [("LOAD", 0), ("LOAD", 1), ("ADD", 0)],
                    [(1 << 20, 10, 10, 16, 1), (1 << 22, 10, 10)])
    assert N.lib.coot_validate(ctypes.byref(e)) == 0
    e = N.make_expr("f64", 7, 1, [("LOAD", 0), ("SCALAR", 0), ("ADD", 0)],
                    [(1 << 20, 7, 1, 7, 8)], [100.0])
    assert N.lib.coot_validate(ctypes.byref(e)) == 0
    # a view whose dims disagree is still a conformability error
    e = N.make_expr("f32", 10, 10, [("LOAD", 0)], [(1 << 20, 10, 9, 16, 1)])
    assert N.lib.coot_validate(ctypes.byref(e)) == 2


def test_integer_scalar_must_be_integral_R4():
    with pytest.raises(coot.CootError):
        _v([("SCALAR", 0), ("LOAD", 0), ("MUL", 0)], [A], [2.5], elem="s64")
    _v([("SCALAR", 0), ("LOAD", 0), ("MUL", 0)], [A], [7.0], elem="s64")


def test_calls_without_ctx_fail_cleanly():
    e = N.make_expr("f32", 10, 10, [("LOAD", 0)], [A])
    assert N.lib.coot_eval(None, ctypes.byref(e), ctypes.c_void_p(1 << 22)) == 1
    assert N.lib.coot_sync(None) == 1


def test_init_without_gpu_is_config_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    assert N.lib.coot_init(ctypes.byref(h), 0, None, 0) == 1
    assert "no CUDA device" in N.lib.coot_last_error().decode()


@pytest.mark.parametrize("n,P,align", [(0, 1, 1), (10, 3, 1), (100, 3, 16), (1000003, 8, 16),
                                       (2**32, 8, 16), (7, 8, 1), (5, 2, 4)])
def test_shard_range_partitions_exactly(n, P, align):
    cuts = [coot.shard_range(n, r, P, align) for r in range(P)]
    assert cuts[0][0] == 0 and cuts[-1][1] == n
    for (b0, e0), (b1, e1) in zip(cuts, cuts[1:]):
        assert e0 == b1 and b0 <= e0
    for b, e in cuts[1:]:
        assert b % align == 0 or b == n
    # blocks are balanced to within one alignment unit
    sizes = [e - b for b, e in cuts]
    if n >= P * align:
        assert max(sizes) - min(sizes) <= 2 * align


def test_partial_bytes():
    assert coot.partial_bytes("ACCU") == 32
    assert coot.partial_bytes("MINMAX") == 32
    assert coot.partial_bytes("SUM_DIM1", 1000) == 8000
