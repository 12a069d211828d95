"""Build libcoot.so in-tree for sm_100a (nvcc; no torch extension machinery).

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, and the
numerics contract of DESIGN.md R5/R7: -fmad=false (no FMA contraction),
-ftz=false, -prec-div=true, -prec-sqrt=true.  cudart is linked statically so
the library only needs the driver at run time.

Incremental: a translation unit is recompiled when its source or any header
(or this file) is newer than its object; each object is stamped with the time
its compile STARTED, so an edit made while a build is running is never masked.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# COOT_LIB_NAME / COOT_EXTRA_FLAGS build tuning variants side by side.
_VARIANT = os.environ.get("COOT_LIB_NAME", "libcoot.so")
BUILD = os.path.join(HERE, "build", os.path.splitext(_VARIANT)[0])
LIB = os.path.join(HERE, _VARIANT)
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-fmad=false", "-ftz=false",
         "-prec-div=true", "-prec-sqrt=true", "--expt-relaxed-constexpr", "-I", INCLUDE,
         "-Xptxas", "-warn-spills"] + os.environ.get("COOT_EXTRA_FLAGS", "").split()


# COOT_EXTRA_LDFLAGS: extra link flags (the sanitizer build, tests/test_sanitizers.py).
# COOT_DEV_TYPES=f32[,f64...]: a development build with the kernels of the
# listed element types only (the other types' launchers are stubs returning
# cudaErrorNotSupported) — ~1/8 of the compile time, for kernel iteration.
# Use it with COOT_LIB_NAME (a side-by-side library) and COOT_LIB_PATH.
# COOT_DEV_TYPES=none: no kernels at all (the host runtime alone).
_DEV_TYPES = [t for t in os.environ.get("COOT_DEV_TYPES", "").split(",") if t]
_ALL_TYPES = {"f32": "float", "f64": "double", "u32": "uint32_t", "s64": "s64", "bf16": "bf16",
              "f16": "f16", "e4m3": "e4m3", "e5m2": "e5m2"}


def _stub_source() -> str:
    path = os.path.join(BUILD, "dev_stubs.cu")
    lines = ['#include "coot_internal.h"', '#include "coot_device.cuh"', "namespace coot {"]
    for t, ct in _ALL_TYPES.items():
        if t in _DEV_TYPES:
            continue
        ct = ct if ct in ("float", "double", "uint32_t") else ct
        lines += [
            f"template <> cudaError_t launch_fused_t<{ct}>(const FusedPlan&, const FusedArgs&, cudaStream_t) {{ return cudaErrorNotSupported; }}",
            f"template <> cudaError_t launch_dim_t<{ct}>(const DimPlan&, const DimArgs&, cudaStream_t) {{ return cudaErrorNotSupported; }}",
            f"template <> cudaError_t launch_combine_t<{ct}>(uint32_t, int, const void*, uint32_t, unsigned long long, void*, unsigned, cudaStream_t) {{ return cudaErrorNotSupported; }}",
            f"template <> cudaError_t launch_empty_rec_t<{ct}>(int, void*, cudaStream_t, const Exchange*, uint32_t) {{ return cudaErrorNotSupported; }}",
            f"template <> cudaError_t launch_fill_t<{ct}>(uint32_t, unsigned long long, unsigned long long, unsigned long long, unsigned long long, unsigned long long, unsigned long long, void*, unsigned, cudaStream_t) {{ return cudaErrorNotSupported; }}",
        ]
    lines.append("}  // namespace coot")
    src = "\n".join(lines) + "\n"
    os.makedirs(BUILD, exist_ok=True)
    if not os.path.exists(path) or open(path).read() != src:
        with open(path, "w") as f:
            f.write(src)
    return path


def _sources():
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if not _DEV_TYPES:
        return srcs
    keep = [s for s in srcs if not os.path.basename(s).startswith("kernels_")
            or os.path.basename(s)[len("kernels_"):].split("_")[0].split(".")[0] in _DEV_TYPES]
    return keep + [_stub_source()]


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(CSRC, "*.inc"))
            + [os.path.join(INCLUDE, "coot.h"), os.path.abspath(__file__)])


def _obj(src: str) -> str:
    return os.path.join(BUILD, os.path.basename(src) + ".o")


def _stale(src: str, newest_header: float) -> bool:
    obj = _obj(src)
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return os.path.getmtime(src) > t or newest_header > t


STAMP = LIB + ".objs.json"  # object mtimes the library was linked from


def _obj_times() -> dict:
    return {os.path.basename(s): os.path.getmtime(_obj(s)) for s in _sources()}


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    srcs = _sources()
    if os.path.exists(STAMP) and all(os.path.exists(_obj(s)) for s in srcs):
        hdr = max(os.path.getmtime(h) for h in _headers())
        with open(STAMP) as f:
            linked = json.load(f)
        return not any(_stale(s, hdr) for s in srcs) and linked == _obj_times()
    # no object tree (e.g. a copy of the repo without build/): compare sources
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in srcs + _headers())


def _compile(src: str) -> str:
    obj = _obj(src)
    started = time.time()
    cmd = [NVCC, *ARCH, *FLAGS, "-I", CSRC, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    os.utime(obj, (started, started))  # an edit during this compile stays "newer"
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    hdr = max(os.path.getmtime(h) for h in _headers())
    todo = [s for s in srcs if force or _stale(s, hdr)]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 4))) as ex:
            list(ex.map(_compile, todo))
    objs = [_obj(s) for s in srcs]
    tmp = LIB + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC",
                           *os.environ.get("COOT_EXTRA_LDFLAGS", "").split()])
    # the library is stamped as old as its oldest object, so a header edited
    # during this build still makes up_to_date() false next time
    oldest = min(os.path.getmtime(o) for o in objs)
    os.replace(tmp, LIB)
    os.utime(LIB, (oldest, oldest))
    with open(STAMP, "w") as f:
        json.dump(_obj_times(), f)
    if verbose:
        print(f"built {LIB} ({len(todo)} of {len(srcs)} units compiled)")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
