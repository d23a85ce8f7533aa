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
SOURCES = [os.path.join(CSRC, "pms.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "pms_device.cuh"), os.path.join(ROOT, "include", "pms.h")]

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-O3"]


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
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *SOURCES, "-o", tmp]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, lib)


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
