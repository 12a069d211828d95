"""Build the oracle shared library (TEST INFRASTRUCTURE ONLY).

gcc, -O2, no FP contraction, no fast-math, x86-64 SSE2 default (FLT_EVAL_METHOD
== 0), linked with libquadmath for the correctly-rounded f64 exp/log.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "coot_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = [
        "gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math",
        "-fexcess-precision=standard", "-fPIC", "-shared", "-Wall", "-Wextra",
        "-Wno-unused-parameter", SRC, "-o", LIB + ".tmp", "-lquadmath", "-lm",
    ]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
