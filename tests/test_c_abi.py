"""The boundary as a C program sees it (include/pms.h):
tests/c/abi_smoke.c is compiled by gcc as C against include/pms.h and linked
to libpms_b200.so.  The compile/link check runs anywhere; the run (-m gpu)
compares its pms_find / pms_find64 output with the CPU oracle."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

import fmgen
import paper_1403_1313_b200 as pms

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "abi_smoke.c")


def build_smoke(tmp_path) -> str:
    pms.build()
    exe = str(tmp_path / "abi_smoke")
    libdir = os.path.dirname(pms.LIB)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    SRC, "-o", exe, f"-L{libdir}", "-l:" + os.path.basename(pms.LIB),
                    f"-Wl,-rpath,{libdir}"], check=True)
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    exe = build_smoke(tmp_path)
    assert os.path.exists(exe)
    out = subprocess.run(["nm", "-u", exe], capture_output=True, text=True, check=True).stdout
    for f in ("pms_find", "pms_find64", "pms_strerror"):
        assert f in out


@pytest.mark.gpu
def test_c_consumer_matches_oracle(tmp_path, orc):
    exe = build_smoke(tmp_path)
    for (n, t, l, d, seed) in [(20, 600, 11, 3, 1), (8, 120, 8, 2, 5), (4, 40, 6, 1, 9)]:
        s, _ = fmgen.generate_fm(n, t, l, d, seed)
        f = tmp_path / f"seqs_{seed}.txt"
        with open(f, "wb") as fh:
            fh.write(f"{n} {t}\n".encode())
            fh.write(s.tobytes())
        out = subprocess.run([exe, str(f), str(l), str(d)], capture_output=True, text=True,
                             check=True, timeout=120).stdout.splitlines()
        want = orc.find(s, l, d)
        find = out[0].split()
        assert find[0] == "find" and int(find[1]) == 0 and int(find[2]) == want.count
        assert [int(x) for x in find[3:]] == want.codes.tolist()
        find64 = out[1].split()
        assert int(find64[1]) == 0 and [int(x) for x in find64[3:]] == want.codes.tolist()
        errs = [int(x) for x in out[2].split()[1:]]
        assert errs[:6] == [pms.E_ARG] * 6
        assert errs[6] == (pms.E_TRUNCATED if want.count else pms.OK)
        assert out[3].startswith("strerror byte outside")


@pytest.mark.gpu
def test_north_star_signatures_via_ctypes(orc):
    """pms_find(seqs, n, t, l, d, out_codes, max_out, &count) and pms_find64
    called directly (no _ex wrapper): the exact north-star entry points."""
    import ctypes
    lib = pms.load()
    s, rec = fmgen.generate_fm(20, 600, 13, 3, 2)
    want = orc.find(s, 13, 3)
    out = np.zeros(1024, np.uint32)
    cnt = ctypes.c_uint64()
    st = lib.pms_find(s.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 20, 600, 13, 3,
                      out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), 1024, ctypes.byref(cnt))
    assert st == pms.OK and cnt.value == want.count
    assert out[:cnt.value].tolist() == want.codes.tolist()
    out64 = np.zeros(1024, np.uint64)
    st = lib.pms_find64(s.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 20, 600, 13, 3,
                        out64.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), 1024,
                        ctypes.byref(cnt))
    assert st == pms.OK and out64[:cnt.value].tolist() == want.codes.tolist()
    # max_out = 0: a size query (count exact, status TRUNCATED)
    st = lib.pms_find(s.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), 20, 600, 13, 3,
                      None, 0, ctypes.byref(cnt))
    assert st == pms.E_TRUNCATED and cnt.value == want.count


def test_too_large_rejected_before_any_read():
    """n * t > 2^31 bytes: PMS_E_TOO_LARGE from the host checks, before the
    (untouched, never-faulted-in) buffer is read or any device work starts."""
    big = np.empty((2, (1 << 30) + 1), dtype=np.uint8)  # 2 GiB virtual, not touched
    r = pms.find_ex(big, 8, 1, max_out=16)
    assert r.status == pms.E_TOO_LARGE and r.count == 0
    r = pms.find64_ex(big, 20, 5, max_out=16)
    assert r.status == pms.E_TOO_LARGE
