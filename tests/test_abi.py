"""CPU-only checks of the C-ABI library (no compute calls need a GPU)."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

import paper_1403_1313_b200 as pms

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pms.h")


def header_functions() -> list[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pms_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    pms.build()
    return pms.load()


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("pms_find", "pms_find_ex", "pms_find64", "pms_find64_ex", "pms_plan_execute64",
              "pms_plan_create", "pms_plan_execute", "pms_plan_wait",
              "pms_plan_destroy", "pms_roofline", "pms_strerror", "pms_device_info"):
        assert f in fns


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", pms.LIB], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for f in header_functions():
        assert f in exported, f
        assert hasattr(lib, f)


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", pms.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_sass_uses_tma_bulk_and_popc(lib):
    sass = subprocess.run(["cuobjdump", "-sass", pms.LIB], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass          # cp.async.bulk (TMA bulk copy) staging the table
    assert "SYNCS.ARRIVE.TRANS64" in sass  # mbarrier expect_tx
    assert "POPC" in sass and "VIMNMX3" in sass


def test_strerror_and_host_argument_checks(lib):
    assert pms.strerror(pms.E_CHAR).startswith("byte outside")
    s = np.full((2, 8), ord("A"), np.uint8)
    # argument errors are detected on the host before any device work
    assert pms.find_ex(s, 0, 1).status == pms.E_ARG
    assert pms.find_ex(s, 17, 1).status == pms.E_ARG
    assert pms.find_ex(s, 9, 1).status == pms.E_ARG      # l > t
    assert pms.find_ex(s, 3, -1).status == pms.E_ARG
    assert pms.find_ex(s, 3, 1, lo=10, hi=5).status == pms.E_ARG
    # 64-bit codes: l <= 31
    s40 = np.full((2, 40), ord("A"), np.uint8)
    assert pms.find64_ex(s40, 32, 1).status == pms.E_ARG
    assert pms.find64_ex(s40, 0, 1).status == pms.E_ARG
    assert pms.find64_ex(s, 9, 1).status == pms.E_ARG    # l > t
    assert pms.find64_ex(s40, 20, -1).status == pms.E_ARG
    assert pms.find64_ex(s40, 20, 1, lo=10, hi=5).status == pms.E_ARG


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_device(lib):
    s = np.full((2, 8), ord("A"), np.uint8)
    r = pms.find_ex(s, 3, 1)
    assert r.status == pms.E_CUDA
    with pytest.raises(pms.PmsError):
        pms.find(s, 3, 1)
    s = np.full((2, 40), ord("A"), np.uint8)
    assert pms.find64_ex(s, 20, 2, lo=0, hi=100).status == pms.E_CUDA
    with pytest.raises(pms.PmsError):
        pms.find64(s, 20, 2, lo=0, hi=100)
