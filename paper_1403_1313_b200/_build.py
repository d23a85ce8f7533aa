"""Build libpms_b200.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_RELEASE = os.path.join(PKG, "libpms_b200.so")
LIB_DEBUG = os.path.join(PKG, "libpms_b200_debug.so")  # -DPMS_DEBUG_CHECKS (bounds counters)
# PMS_DEBUG_LIB=1 selects the bounds-checked build for this process
LIB = LIB_DEBUG if os.environ.get("PMS_DEBUG_LIB") == "1" else LIB_RELEASE
# PMS_LIB_OVERRIDE=build/variants/NAME/libpms_b200.so loads a variant build of
# this source tree (tuning experiments, scripts/variants.py); nothing else is
# accepted
VARIANTS = os.path.join(ROOT, "build", "variants")
_ovr = os.environ.get("PMS_LIB_OVERRIDE")
if _ovr:
    _real = os.path.realpath(_ovr)
    if not (_real.startswith(os.path.realpath(VARIANTS) + os.sep) and
            os.path.basename(_real) == "libpms_b200.so"):
        raise RuntimeError(f"PMS_LIB_OVERRIDE must name build/variants/*/libpms_b200.so, got {_ovr!r}")
    LIB = _real
# pms.cu: 32-bit-word kernels + host code; pms64.cu: 64-bit-word kernels (l <= 31);
# pms_slice.cu / pms_slice_ht.cu / pms_slice_wide.cu (l = 17..31) / pms_roof.cu: the
# slice family's kernels and roofline kernels
SOURCES = [os.path.join(CSRC, f) for f in ("pms.cu", "pms64.cu", "pms_slice.cu",
                                              "pms_slice_ht.cu", "pms_slice_wide.cu", "pms_roof.cu")]
DEPS = SOURCES + [os.path.join(CSRC, h) for h in ("pms_device.cuh", "pms_kernels.cuh",
                                                    "pms_slice.cuh")] + \
    [os.path.join(ROOT, "include", "pms.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-O3"]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in DEPS)


def _compile(lib: str, extra: list[str], verbose: bool) -> None:
    """nvcc -c of every translation unit in parallel, then one nvcc -shared link."""
    tag = f".tmp{os.getpid()}"
    objs, procs = [], []
    for src in SOURCES:
        obj = lib + "." + os.path.splitext(os.path.basename(src))[0] + tag + ".o"
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
               "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        objs.append(obj)
        procs.append((cmd, subprocess.Popen(cmd)))
    try:
        for cmd, pr in procs:
            if pr.wait() != 0:
                raise subprocess.CalledProcessError(pr.returncode, cmd)
        tmp = lib + tag
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", tmp]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        os.replace(tmp, lib)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)


def build(force: bool = False, verbose: bool = False, debug: bool | None = None) -> str:
    """Build the library this process loads (release, or the bounds-checked
    debug build when PMS_DEBUG_LIB=1 or debug=True)."""
    want_debug = (LIB == LIB_DEBUG) if debug is None else debug
    lib = LIB_DEBUG if want_debug else LIB_RELEASE
    if force or stale(lib):
        _compile(lib, ["-DPMS_DEBUG_CHECKS"] if want_debug else [], verbose)
    return lib


if __name__ == "__main__":
    build(force=True, verbose=True, debug=False)
    build(force=True, verbose=True, debug=True)
