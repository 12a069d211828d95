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
# AddressSanitizer + UndefinedBehaviorSanitizer build for tests/test_sanitizers.py
LIB_SAN = os.path.join(HERE, "liboracle_san.so")
SAN_FLAGS = ["-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
             "-fno-omit-frame-pointer", "-g"]


def build(force: bool = False, sanitize: bool = False) -> str:
    lib = LIB_SAN if sanitize else LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= os.path.getmtime(SRC):
        return lib
    cmd = [
        "gcc", "-std=gnu11", "-O2", "-ffp-contract=off", "-fno-fast-math",
        "-fexcess-precision=standard", "-fPIC", "-shared", "-Wall", "-Wextra",
        "-Wno-unused-parameter", *(SAN_FLAGS if sanitize else []), SRC, "-o", lib + ".tmp",
        "-lquadmath", "-lm",
    ]
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
