"""CPU oracle for Skip-Brute-Force planted (l,d) motif search.

TEST INFRASTRUCTURE ONLY.  Only ``tests/`` (including the hand-run tools in
``tests/tools/``), ``__graft_entry__.smoke()``, ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs and ``scripts/make_golden.py``
(which writes the stored golden sets) may import this package.  The product (``paper_1403_1313_b200``) never imports it, and this
package imports nothing from the product.

The arithmetic lives in ``pms_oracle.c`` (plain C, character compares, see
its header for the passages of PAPER.md / SPEC.md each function follows).
This module only compiles it with gcc and marshals arguments with ctypes.

Pin status: every function here is pinned by ``tests/test_oracle.py``
(SPEC worked examples, closed forms, brute force on tiny inputs, an
independent Hamming-ball algorithm, planted recovery, metamorphic
relations).  Completeness at large l has no pin beyond those relations --
see DESIGN.md section 3 ("parity unpinned except by the oracle" row).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pms_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_pms.so")

OK, E_ARG, E_CHAR, E_TOO_LARGE, E_CUDA, E_TRUNCATED, E_NOMEM = 0, -1, -2, -3, -4, -5, -6

_lib = None


def build(force: bool = False) -> str:
    """Compile pms_oracle.c into liboracle_pms.so (gcc, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC",
                               "-pthread", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u8p, u32p, u64p = (ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_uint32),
                           ctypes.POINTER(ctypes.c_uint64))
        i32, u64 = ctypes.c_int32, ctypes.c_uint64
        for name in ("oracle_find", "oracle_naive_find"):
            f = getattr(lib, name)
            f.argtypes = [u8p, i32, i32, i32, i32, u64, u64, i32, u32p, u64, u64p, u64p]
            f.restype = ctypes.c_int
        lib.oracle_find64.argtypes = [u8p, i32, i32, i32, i32, u64, u64, i32, u64p, u64, u64p,
                                      u64p]
        lib.oracle_find64.restype = ctypes.c_int
        lib.oracle_ball_find.argtypes = [u8p, i32, i32, i32, i32, u32p, u64, u64p]
        lib.oracle_ball_find.restype = ctypes.c_int
        lib.oracle_verify_motif.argtypes = [u8p, i32, i32, i32, i32, u64]
        lib.oracle_verify_motif.restype = ctypes.c_int
        lib.oracle_decode.argtypes = [u64, i32, ctypes.c_char_p]
        lib.oracle_decode.restype = None
        lib.oracle_hamming.argtypes = [ctypes.c_char_p, ctypes.c_char_p, i32]
        lib.oracle_hamming.restype = i32
        lib.oracle_partition.argtypes = [u64, u64, i32, u64p]
        lib.oracle_partition.restype = None
        _lib = lib
    return _lib


@dataclass
class OracleResult:
    status: int
    codes: np.ndarray      # uint32, ascending (first min(count, max_out) entries)
    count: int             # exact total number of motifs
    c_alg: int             # windows compared (first-match stop), 0 if not computed


def _as_rows(seqs) -> tuple[np.ndarray, int, int]:
    a = np.ascontiguousarray(np.asarray(seqs, dtype=np.uint8))
    if a.ndim != 2:
        raise ValueError("seqs must be a 2-D uint8 array [n, t]")
    return a, int(a.shape[0]), int(a.shape[1])


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _call(fname, seqs, l, d, lo, hi, threads, max_out):
    lib = _load()
    a, n, t = _as_rows(seqs)
    if hi is None:
        hi = 4 ** l if 1 <= l <= 16 else 0
    out = np.zeros(max(int(max_out), 1), dtype=np.uint32)
    cnt, work = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = getattr(lib, fname)(
        a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)) if a.size else
        ctypes.cast(ctypes.c_void_p(1), ctypes.POINTER(ctypes.c_uint8)),
        n, t, l, d, lo, hi, threads if threads else default_threads(),
        out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), int(max_out),
        ctypes.byref(cnt), ctypes.byref(work))
    k = min(int(cnt.value), int(max_out))
    return OracleResult(st, out[:k].copy(), int(cnt.value), int(work.value))


def find(seqs, l: int, d: int, lo: int = 0, hi: int | None = None,
         threads: int | None = None, max_out: int = 1 << 22) -> OracleResult:
    """Skip-BF over ranks [lo, hi) with the paper's static partition
    over `threads` workers.  Returns every rank whose l-mer has a
    <= d mismatch window in all n sequences, ascending."""
    return _call("oracle_find", seqs, l, d, lo, hi, threads, max_out)


def find64(seqs, l: int, d: int, lo: int = 0, hi: int | None = None,
           threads: int | None = None, max_out: int = 1 << 22) -> OracleResult:
    """Skip-BF for l <= 31 with 64-bit codes; same algorithm as
    find().  Use [lo, hi) ranges: 4^l candidates are far too many for a CPU
    at large l."""
    lib = _load()
    a, n, t = _as_rows(seqs)
    if hi is None:
        hi = 4 ** l if 1 <= l <= 31 else 0
    out = np.empty(max(int(max_out), 1), dtype=np.uint64)
    cnt, work = ctypes.c_uint64(0), ctypes.c_uint64(0)
    st = lib.oracle_find64(a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), n, t, l, d, lo, hi,
                           threads if threads else default_threads(),
                           out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), int(max_out),
                           ctypes.byref(cnt), ctypes.byref(work))
    k = min(int(cnt.value), int(max_out)) if st in (OK, E_TRUNCATED) else 0
    return OracleResult(st, out[:k].copy(), int(cnt.value), int(work.value))


def naive_find(seqs, l: int, d: int, lo: int = 0, hi: int | None = None,
               threads: int | None = 1, max_out: int = 1 << 22) -> OracleResult:
    """Plain brute force (no skip rule, no early abort)."""
    return _call("oracle_naive_find", seqs, l, d, lo, hi, threads, max_out)


def ball_find(seqs, l: int, d: int, max_out: int = 1 << 24) -> OracleResult:
    """Independent algorithm: intersection over sequences of the union of
    Hamming balls of radius d around each window (l <= 12)."""
    lib = _load()
    a, n, t = _as_rows(seqs)
    out = np.zeros(max(int(max_out), 1), dtype=np.uint32)
    cnt = ctypes.c_uint64(0)
    st = lib.oracle_ball_find(a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), n, t, l, d,
                              out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)),
                              int(max_out), ctypes.byref(cnt))
    k = min(int(cnt.value), int(max_out))
    return OracleResult(st, out[:k].copy(), int(cnt.value), 0)


def verify_motif(seqs, l: int, d: int, rank: int) -> bool:
    """S:251 verify_motif: full Hamming re-check of one rank (no early abort)."""
    lib = _load()
    a, n, t = _as_rows(seqs)
    r = lib.oracle_verify_motif(a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), n, t, l, d,
                                int(rank))
    if r < 0:
        raise ValueError(f"verify_motif: status {r}")
    return bool(r)


def decode(rank: int, l: int) -> str:
    """S:66-74 decode_lmer."""
    buf = ctypes.create_string_buffer(l + 1)
    _load().oracle_decode(int(rank), l, buf)
    return buf.value.decode()


def hamming(a: str, b: str) -> int:
    """S:86-94 hamming_distance on equal-length strings."""
    if len(a) != len(b):
        raise ValueError("LengthMismatch")
    return int(_load().oracle_hamming(a.encode(), b.encode(), len(a)))


def partition(lo: int, hi: int, workers: int) -> list[tuple[int, int]]:
    """S:295-303 make_partition (floor/remainder contiguous split)."""
    starts = (ctypes.c_uint64 * (workers + 1))()
    _load().oracle_partition(lo, hi, workers, starts)
    return [(int(starts[w]), int(starts[w + 1])) for w in range(workers)]
