"""The oracle and its generator against the seed-42 golden vectors of SURVEY.md
§8(c) (SURVEY.md:709; tests/golden/survey_seed42.txt), computed in the survey
session with the §8(c) semantics and the §8(d) recipe — an external pin of the
generator, of the c1 / c2 / c4 programs and of their reductions."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "survey_seed42.txt")


def golden():
    d = {}
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, etype, vals = [f.strip() for f in line.split("|")]
        d[key] = (etype, vals.split())
    return d


def as_array(etype, vals, as_bits=False):
    if etype == "f32" and as_bits:
        return np.array([int(v, 16) for v in vals], np.uint32).view(np.float32)
    if etype in ("f32", "f64"):
        return np.array([float.fromhex(v) for v in vals], oracle.DTYPES[etype])
    if etype == "u32":
        return np.array([int(v, 16) for v in vals], np.uint32)
    out = [int(v, 16) if v.startswith("0x") else int(v) for v in vals]
    return np.array([(x - (1 << 64)) if x >= (1 << 63) else x for x in out], np.int64)


G = golden()
C2 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("EXP", 0), ("SCALAR", 0), ("LOAD", 2), ("MUL", 0),
      ("ADD", 0)]
C1 = [("SCALAR", 0), ("LOAD", 0), ("MUL", 0), ("LOAD", 1), ("ADD", 0)]
C4 = [("LOAD", 0), ("LOAD", 1), ("MUL", 0), ("SCALAR", 0), ("LOAD", 2), ("MUL", 0), ("ADD", 0)]


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.dtype == b.dtype and np.array_equal(a.view(f"u{a.itemsize}"), b.view(f"u{b.itemsize}"))


def test_generator_f32_and_f64():
    for key, s in (("A_f32", 0), ("B_f32", 1), ("C_f32", 2)):
        assert bits_equal(oracle.fill("f32", "randu", 4, seed=42, stream=s), as_array("f32", G[key][1]))
    assert bits_equal(oracle.fill("f64", "randu", 2, seed=42, stream=0), as_array("f64", G["A_f64"][1]))


def test_c2_z_and_accu():
    A, B, C = (oracle.fill("f32", "randu", 4, seed=42, stream=s) for s in range(3))
    Z = oracle.eval_program("f32", C2, [A, B, C], [3.0])
    assert bits_equal(Z, as_array("f32", G["c2_Z_bits"][1], as_bits=True))
    assert bits_equal(oracle.reduce("f32", "ACCU", Z), as_array("f32", G["c2_accu"][1])[0])


def test_c1_axpy_and_accu():
    A, B = (oracle.fill("f32", "randu", 4, seed=42, stream=s) for s in range(2))
    y = oracle.eval_program("f32", C1, [A, B], [2.5])
    assert bits_equal(y, as_array("f32", G["c1_y"][1]))
    assert bits_equal(oracle.reduce("f32", "ACCU", y), as_array("f32", G["c1_accu"][1])[0])


@pytest.mark.parametrize("etype", ["u32", "s64"])
def test_c4_bitwise_and_minmax(etype):
    X, Y, Z = (oracle.fill(etype, "randu", 4, seed=42, stream=s) for s in range(3))
    r = oracle.eval_program(etype, C4, [X, Y, Z], [7])
    assert np.array_equal(r, as_array(etype, G[f"c4_{etype}"][1]))
    mm = oracle.reduce(etype, "MINMAX", r)
    assert mm[0] == as_array(etype, G[f"c4_{etype}_min"][1])[0]
    assert mm[1] == as_array(etype, G[f"c4_{etype}_max"][1])[0]
