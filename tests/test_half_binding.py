"""CPU: the binding's scalar rounding to bf16/f16 (reading R4 + R24) agrees with
numpy's float16 cast (a library routine) and with the oracle's independent
integer rounding, including ties, subnormals, overflow and signed zero."""
import math
import random

import numpy as np
import pytest

import oracle
from paper_2508_11385_b200 import _native as N

SPECIAL = [0.0, -0.0, 1.0, -1.0, 65504.0, 65520.0, 65519.99, 1e-8, 2.0 ** -24, 2.0 ** -25,
           3 * 2.0 ** -26, 2.0 ** -14, 1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, 1 + 2.0 ** -8,
           1 + 3 * 2.0 ** -8, 3.3895313892515355e38, 3.4e38, 1e-40, float("inf"), -float("inf")]


def _samples(n=4000, seed=3):
    rng = random.Random(seed)
    out = list(SPECIAL)
    for _ in range(n):
        out.append(rng.uniform(-1, 1) * 2.0 ** rng.randint(-140, 130))
    return out


def test_f16_matches_numpy_cast():
    for x in _samples():
        want = int(np.array([x], dtype=np.float64).astype(np.float16).view(np.uint16)[0])
        assert N.half_bits(x, "f16") == want, x


@pytest.mark.parametrize("etype", ["bf16", "f16"])
def test_matches_oracle(etype):
    for x in _samples():
        assert N.half_bits(x, etype) == oracle.half_from_double(etype, x), (etype, x)


def test_bf16_special_values():
    assert N.half_bits(1.0, "bf16") == 0x3F80
    assert N.half_bits(-2.0, "bf16") == 0xC000
    assert N.half_bits(1 + 2.0 ** -8, "bf16") == 0x3F80          # tie -> even
    assert N.half_bits(1 + 3 * 2.0 ** -8, "bf16") == 0x3F82      # tie -> even (up)
    assert N.half_bits(3.4e38, "bf16") == 0x7F80                 # overflow -> inf
    assert N.half_bits(math.nan, "bf16") & 0x7F80 == 0x7F80
    assert N.half_bits(-0.0, "bf16") == 0x8000
