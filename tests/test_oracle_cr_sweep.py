"""Correct rounding of the oracle's f32 EXP and LOG over the f32 bit patterns
(SURVEY §8(c) "EXP/LOG" pin; R6), checked by tests/native/cr_sweep.c
against binary128 expq / logq (libquadmath), with a long-double prefilter that
falls back to binary128 near every f32 rounding midpoint (see the helper's
header).

Default suite: every 61st bit pattern over all 2^32 (7.0e7 inputs per
function: every sign, exponent and range end).  The exhaustive sweep of all
2^32 patterns takes ~3 min per function on 8 cores: it runs with COOT_SLOW=1
(`-m slow`), and its last run is recorded in profiles/r02_oracle_cr_sweep.txt.
"""
import os
import re
import subprocess

import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "native", "cr_sweep.c")


@pytest.fixture(scope="module")
def sweep(tmp_path_factory):
    lib = oracle.lib()._name  # builds liboracle.so if needed
    d = os.path.dirname(lib)
    exe = str(tmp_path_factory.mktemp("crsweep") / "cr_sweep")
    subprocess.check_call(["gcc", "-O2", "-o", exe, SRC, f"-L{d}", "-loracle",
                           f"-Wl,-rpath,{d}", "-lquadmath", "-lm", "-pthread"])
    threads = str(max(1, len(os.sched_getaffinity(0))))

    def run(op, mode, lo, hi, stride=1):
        out = subprocess.run([exe, op, mode, hex(lo), hex(hi), threads, str(stride)],
                             capture_output=True, text=True, check=True).stdout
        m = re.match(r"checked (\d+) mismatches (\d+) quad_fallbacks (\d+)(.*)", out)
        assert m, out
        return int(m.group(1)), int(m.group(2)), out
    return run


@pytest.mark.parametrize("op", ["EXP", "LOG"])
def test_strided_all_patterns(sweep, op):
    checked, bad, out = sweep(op, "filtered", 0, 1 << 32, 61)
    assert checked == -(-(1 << 32) // 61)
    assert bad == 0, out


@pytest.mark.parametrize("op", ["EXP", "LOG"])
def test_quad_everywhere_agrees_on_a_binade(sweep, op):
    """The unfiltered binary128 mode on one full binade [0.5, 1) and its negation."""
    for lo in (0x3F000000, 0xBF000000):
        checked, bad, out = sweep(op, "quad", lo, lo + (1 << 23))
        assert checked == 1 << 23 and bad == 0, out


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("COOT_SLOW") != "1", reason="exhaustive: set COOT_SLOW=1")
@pytest.mark.parametrize("op", ["EXP", "LOG"])
def test_exhaustive_all_patterns(sweep, op):
    checked, bad, out = sweep(op, "filtered", 0, 1 << 32)
    assert checked == 1 << 32 and bad == 0, out
