"""AddressSanitizer + UndefinedBehaviorSanitizer builds of the host code (CPU
suite, no GPU): libcoot's host runtime (validation, lowering checks, error
paths; kernels stubbed out — COOT_DEV_TYPES=none) and the oracle, exercised by
tests/sanitize_host_driver.py in a subprocess with the sanitizer runtimes
preloaded.  Any ASan report or UBSan runtime error fails the test."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# (nvcc splits -Xcompiler values at commas: one sanitizer per flag)
SAN = "-Xcompiler -fsanitize=address -Xcompiler -fsanitize=undefined"


def _runtime(name):
    p = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return p if os.path.isabs(p) and os.path.exists(p) else None


def _build_libcoot_san():
    env = dict(os.environ, COOT_DEV_TYPES="none", COOT_LIB_NAME="libcoot_san.so",
               COOT_EXTRA_FLAGS=f"{SAN} -Xcompiler -fno-sanitize-recover=undefined "
                                "-Xcompiler -fno-omit-frame-pointer -g",
               COOT_EXTRA_LDFLAGS=SAN)
    code = ("import importlib.util; s = importlib.util.spec_from_file_location('b', "
            f"{os.path.join(ROOT, 'paper_2508_11385_b200', 'build.py')!r}); "
            "b = importlib.util.module_from_spec(s); s.loader.exec_module(b); print(b.build())")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.timeout(1200)
def test_host_code_under_asan_ubsan():
    asan, ubsan = _runtime("libasan.so"), _runtime("libubsan.so")
    if not asan or not ubsan:
        pytest.skip("gcc sanitizer runtimes not installed")
    from oracle import build as ob
    orc = ob.build(sanitize=True)
    coot = _build_libcoot_san()
    env = dict(os.environ, LD_PRELOAD=f"{asan}:{ubsan}", COOT_LIB_PATH=coot, ORACLE_LIB_PATH=orc,
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=0:halt_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_host_driver.py")],
                         env=env, capture_output=True, text=True, timeout=900)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-4000:]
    assert "AddressSanitizer" not in log and "runtime error" not in log, log[-4000:]
    assert "sanitize host driver ok" in out.stdout


@pytest.mark.timeout(600)
def test_sanitizer_catches_a_planted_overflow():
    """The preload really instruments the oracle: reading past a numpy buffer
    through orc_rows_add (ncols larger than a malloc-backed buffer holds) is reported."""
    asan, ubsan = _runtime("libasan.so"), _runtime("libubsan.so")
    if not asan or not ubsan:
        pytest.skip("gcc sanitizer runtimes not installed")
    from oracle import build as ob
    orc = ob.build(sanitize=True)
    code = ("import ctypes, numpy as np; L = ctypes.CDLL(%r); L.orc_rows_new.restype = ctypes.c_void_p; "
            "L.orc_rows_new.argtypes = [ctypes.c_int, ctypes.c_uint64]; "
            "L.orc_rows_add.argtypes = [ctypes.c_void_p] + [ctypes.c_uint64] * 4 + [ctypes.c_void_p]; "
            "h = L.orc_rows_new(1, 8); x = (ctypes.c_double * 1024)(); "
            "L.orc_rows_add(h, 0, 8, 200, 8, ctypes.cast(x, ctypes.c_void_p))" % orc)
    env = dict(os.environ, LD_PRELOAD=f"{asan}:{ubsan}", ASAN_OPTIONS="detect_leaks=0")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode != 0 and "AddressSanitizer" in out.stderr, out.stderr[-2000:]
