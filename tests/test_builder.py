"""The delayed-evaluation builder: building an expression
does nothing but record a tree; lowering produces the postfix program the C
ABI consumes.  Runs on CPU tensors (no device work happens before eval)."""
import pytest
import torch

import paper_2508_11385_b200 as coot
from progs import P


def M(n=6, m=1, dtype=torch.float32):
    return coot.Mat(torch.zeros(n * m, dtype=dtype), n, m)


def test_c2_expression_lowers_to_catalog_program():
    A, B, C = M(), M(), M()
    lw = coot.lower(coot.exp(A % B) + 3 * C)
    assert lw.program == P("L0 L1 MUL EXP S0 L2 MUL ADD")
    assert lw.scalars == [3]
    assert len(lw.operands) == 3


def test_axpy_and_in_place_forms():
    x, y = M(), M()
    assert coot.lower(2.5 * x + y).program == P("S0 L0 MUL L1 ADD")
    assert coot.lower(y + x * 2.5).program == P("L0 L1 S0 MUL ADD")


def test_operands_deduplicated_scalars_by_value():
    A, B = M(), M()
    lw = coot.lower(A % A + 2 * B - 2 * A)
    assert len(lw.operands) == 2
    assert lw.scalars == [2]
    assert lw.program == P("L0 L0 MUL S0 L1 MUL ADD S0 L0 MUL SUB")


def test_noncommutative_order_and_unary():
    A, B = M(), M()
    assert coot.lower(A - B).program == P("L0 L1 SUB")
    assert coot.lower(1 - A).program == P("S0 L0 SUB")
    assert coot.lower(A / B).program == P("L0 L1 DIV")
    assert coot.lower(-coot.sqrt(coot.abs(A))).program == P("L0 ABS SQRT NEG")
    assert coot.lower(coot.min(A, B)).program == P("L0 L1 MIN")


def test_conformability_checked_at_lowering():
    A, B = M(6), M(5)
    e = A + B  # building is allowed (delayed)
    with pytest.raises(coot.CootError) as ei:
        coot.lower(e)
    assert ei.value.status == "CONFORM"


def test_matrix_product_is_out_of_scope():
    with pytest.raises(NotImplementedError):
        M() * M()


def test_mixed_element_types_rejected():
    with pytest.raises(coot.CootError):
        M() + M(dtype=torch.float64)


def test_integer_expressions_reject_fractional_scalars_R4():
    X = M(dtype=torch.int64)
    with pytest.raises(coot.CootError):
        coot.lower(2.5 * X)
    assert coot.lower(7 * X).scalars == [7]


def test_views_lower_to_strided_operands():
    A = coot.Mat(torch.zeros(7 * 5, dtype=torch.float32), 7, 5)
    base = A.data.data_ptr()
    d = A.diag()
    assert (d.n_rows, d.n_cols) == (5, 1)
    lw = coot.lower(d + 100)
    assert lw.program == P("L0 S0 ADD")
    assert lw.operands[0] == (base, 5, 1, 5, 8)  # inc = ld + 1
    assert coot.lower(A.diag(2) * 1).operands[0] == (base + 2 * 7 * 4, 5 - 2, 1, 3, 8)
    assert coot.lower(A.diag(-3) * 1).operands[0] == (base + 3 * 4, 4, 1, 4, 8)
    s = A.submat(1, 2, 4, 3)  # rows 1..4, cols 2..3
    assert coot.lower(s * 2).operands[0] == (base + (1 + 2 * 7) * 4, 4, 2, 7, 1)
    r = A.row(6)
    assert coot.lower(r + r).operands == [(base + 6 * 4, 1, 5, 7, 1)]  # one operand, loaded twice
    with pytest.raises(coot.CootError):
        A.submat(0, 0, 7, 1)  # out of bounds


def test_mat_layout_is_column_major():
    t = torch.arange(6, dtype=torch.float64).reshape(2, 3)  # [[0,1,2],[3,4,5]]
    m = coot.Mat.from_torch(t)
    assert (m.n_rows, m.n_cols) == (2, 3)
    assert m.data.tolist() == [0, 3, 1, 4, 2, 5]
    assert torch.equal(m.to_torch(), t)
