"""B200-native Skip-Brute-Force planted (l,d) motif search (arxiv 1403.1313).

Thin ctypes binding over ``libpms_b200.so`` (include/pms.h): argument
marshalling only -- every step of the search runs in the library's CUDA
kernels.  There is no CPU fallback: if the library is missing or no CUDA
device is usable, calls raise.  PyTorch is used only by callers that want to
pass device tensors and streams (``Plan.execute``).
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

from ._build import LIB, build

OK, E_ARG, E_CHAR, E_TOO_LARGE, E_CUDA, E_TRUNCATED = 0, -1, -2, -3, -4, -5
ALGO_AUTO, ALGO_CANDIDATE, ALGO_BLOCK, ALGO_SLICE = 0, 1, 2, 3
MAX_L = 16     # uint32 codes (pms_find, pms_find_ex, pms_plan_execute)
MAX_L64 = 31   # uint64 codes (pms_find64, pms_find64_ex, pms_plan_execute64)

__all__ = ["find", "find_ex", "find64", "find64_ex", "Plan", "Launch", "Stats", "roofline", "device_info", "strerror",
           "PmsError", "load", "build", "decode_code", "LIB"]


class PmsError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        detail = f" [{last_error()}]" if status == E_CUDA else ""
        super().__init__(f"{what}: {strerror(status)} (status {status}){detail}" if what else
                         f"{strerror(status)} (status {status}){detail}")


class Launch(ctypes.Structure):
    _fields_ = [("ctas_per_sm", ctypes.c_int32), ("warps_per_cta", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("lanes_per_cand", ctypes.c_int32),
                ("force_generic", ctypes.c_int32), ("grid_ctas", ctypes.c_int32),
                ("no_skip", ctypes.c_int32), ("algo", ctypes.c_int32),
                ("block_digits", ctypes.c_int32), ("table_global", ctypes.c_int32),
                ("handoff", ctypes.c_int32), ("wide_words", ctypes.c_int32),
                ("seq_parallel", ctypes.c_int32), ("overlap_prepass", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("pack_ms", ctypes.c_double), ("search_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("candidates", ctypes.c_uint64),
                ("issued_compares", ctypes.c_uint64), ("motifs", ctypes.c_uint64),
                ("grid", ctypes.c_int32), ("block", ctypes.c_int32),
                ("lanes_per_cand", ctypes.c_int32), ("windows_per_lane", ctypes.c_int32),
                ("generic", ctypes.c_int32), ("table_in_smem", ctypes.c_int32),
                ("smem_bytes", ctypes.c_uint32), ("algo", ctypes.c_int32),
                ("block_scans", ctypes.c_uint64), ("block_digits", ctypes.c_int32),
                ("mode_flags", ctypes.c_int32), ("sparse_steps", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def load() -> ctypes.CDLL:
    """Load libpms_b200.so (built in-tree by build()); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} not built: run paper_1403_1313_b200.build() "
                              "(nvcc, sm_100a); there is no CPU fallback")
        lib = ctypes.CDLL(LIB)
        vp, u8p, u32p, u64p = (ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint8),
                               ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint64))
        i32, u64 = ctypes.c_int32, ctypes.c_uint64
        lib.pms_find.argtypes = [u8p, i32, i32, i32, i32, u32p, u64, u64p]
        lib.pms_find.restype = ctypes.c_int
        # (void* for the byte and code buffers: _find_ex passes raw addresses,
        # which skips a ctypes pointer object per call)
        lib.pms_find_ex.argtypes = [vp, i32, i32, i32, i32, u64, u64, ctypes.POINTER(Launch),
                                    vp, u64, u64p, ctypes.POINTER(Stats)]
        lib.pms_find_ex.restype = ctypes.c_int
        lib.pms_find64.argtypes = [u8p, i32, i32, i32, i32, u64p, u64, u64p]
        lib.pms_find64.restype = ctypes.c_int
        lib.pms_find64_ex.argtypes = [vp, i32, i32, i32, i32, u64, u64, ctypes.POINTER(Launch),
                                      vp, u64, u64p, ctypes.POINTER(Stats)]
        lib.pms_find64_ex.restype = ctypes.c_int
        lib.pms_plan_create.argtypes = [i32, i32, i32, i32, ctypes.POINTER(Launch),
                                        ctypes.POINTER(vp)]
        lib.pms_plan_create.restype = ctypes.c_int
        lib.pms_plan_execute.argtypes = [vp, vp, u64, u64, vp, u64, vp, vp]
        lib.pms_plan_execute.restype = ctypes.c_int
        lib.pms_plan_execute64.argtypes = [vp, vp, u64, u64, vp, u64, vp, vp]
        lib.pms_plan_execute64.restype = ctypes.c_int
        lib.pms_plan_wait.argtypes = [vp, ctypes.POINTER(Stats)]
        lib.pms_plan_wait.restype = ctypes.c_int
        lib.pms_plan_destroy.argtypes = [vp]
        lib.pms_plan_destroy.restype = None
        lib.pms_roofline.argtypes = [i32, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)]
        lib.pms_roofline.restype = ctypes.c_int
        lib.pms_plan_roofline.argtypes = [vp, i32, i32, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double)]
        lib.pms_plan_roofline.restype = ctypes.c_int
        lib.pms_strerror.argtypes = [ctypes.c_int]
        lib.pms_strerror.restype = ctypes.c_char_p
        lib.pms_debug_violations.argtypes = [ctypes.c_int32]
        lib.pms_debug_violations.restype = ctypes.c_int64
        lib.pms_last_error.argtypes = []
        lib.pms_last_error.restype = ctypes.c_char_p
        lib.pms_device_info.argtypes = [ctypes.POINTER(i32)] * 3
        lib.pms_device_info.restype = ctypes.c_int
        _lib = lib
    return _lib


def strerror(status: int) -> str:
    return load().pms_strerror(int(status)).decode()


def debug_violations(reset: bool = False) -> int:
    """Out-of-range device indices counted by the debug build (-1: release)."""
    return int(load().pms_debug_violations(1 if reset else 0))


def last_error() -> str:
    """Source line + CUDA error string of this thread's last PMS_E_CUDA."""
    return load().pms_last_error().decode()


def _rows(seqs) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(seqs, dtype=np.uint8))
    if a.ndim != 2:
        raise ValueError("seqs must be a 2-D uint8 array [n, t]")
    return a


@dataclass
class FindResult:
    status: int
    codes: np.ndarray   # ascending codes when status == OK, else empty
    count: int          # exact number of motifs
    stats: Stats | None = None


def _find_ex(fname, ctype, seqs, l, d, lo, hi, launch, max_out, want_stats) -> FindResult:
    lib = load()
    a = _rows(seqs)
    n, t = a.shape
    if hi is None:
        hi = (1 << 64) - 1
    out = _scratch(max(int(max_out), 1), np.uint32 if ctype is ctypes.c_uint32 else np.uint64)
    cnt = ctypes.c_uint64(0)
    st = Stats() if want_stats else None
    status = getattr(lib, fname)(a.ctypes.data, n, t, l, d, int(lo), int(hi),
                                 ctypes.byref(launch) if launch else None, out.ctypes.data,
                                 int(max_out), ctypes.byref(cnt),
                                 ctypes.byref(st) if st is not None else None)
    # codes are defined only on OK (include/pms.h: on PMS_E_TRUNCATED the
    # caller's buffer is unspecified, so nothing of it is returned)
    k = int(cnt.value) if status == OK else 0
    return FindResult(status, out[:k].copy(), int(cnt.value), st)


_tls = threading.local()


def _scratch(size: int, dtype) -> np.ndarray:
    """Per-thread code buffer reused across calls (results are copied out)."""
    key = np.dtype(dtype).char
    buf = getattr(_tls, key, None)
    if buf is None or buf.size < size:
        buf = np.empty(size, dtype=dtype)
        setattr(_tls, key, buf)
    return buf[:size]


def find_ex(seqs, l: int, d: int, lo: int = 0, hi: int | None = None,
            launch: Launch | None = None, max_out: int = 1 << 20,
            want_stats: bool = True) -> FindResult:
    """One call of pms_find_ex (uint32 codes, l <= 16) from host buffers;
    returns the raw status."""
    return _find_ex("pms_find_ex", ctypes.c_uint32, seqs, l, d, lo, hi, launch, max_out,
                    want_stats)


def find64_ex(seqs, l: int, d: int, lo: int = 0, hi: int | None = None,
              launch: Launch | None = None, max_out: int = 1 << 20,
              want_stats: bool = True) -> FindResult:
    """One call of pms_find64_ex (uint64 codes, l <= 31) from host buffers."""
    return _find_ex("pms_find64_ex", ctypes.c_uint64, seqs, l, d, lo, hi, launch, max_out,
                    want_stats)


def _find_all(fx, name, seqs, l, d, lo, hi, launch) -> np.ndarray:
    cap = 1 << 16
    while True:
        r = fx(seqs, l, d, lo, hi, launch, max_out=cap, want_stats=False)
        if r.status == E_TRUNCATED and r.count > cap:
            cap = r.count
            continue
        if r.status != OK:
            raise PmsError(r.status, name)
        return r.codes


def find(seqs, l: int, d: int, lo: int = 0, hi: int | None = None,
         launch: Launch | None = None) -> np.ndarray:
    """All motif codes (ascending uint32) of seqs for (l, d); raises PmsError."""
    return _find_all(find_ex, "pms_find_ex", seqs, l, d, lo, hi, launch)


def find64(seqs, l: int, d: int, lo: int = 0, hi: int | None = None,
           launch: Launch | None = None) -> np.ndarray:
    """All motif codes (ascending uint64) for l <= 31 over [lo, hi); raises PmsError."""
    return _find_all(find64_ex, "pms_find64_ex", seqs, l, d, lo, hi, launch)


def decode_code(code: int, l: int) -> str:
    """Code -> l-mer string (big-endian base 4, A0 C1 G2 T3) for display."""
    return "".join("ACGT"[(int(code) >> (2 * (l - 1 - j))) & 3] for j in range(l))


class Plan:
    """Device-resident plan (pms_plan_*): enqueue on a torch/CUDA stream."""

    def __init__(self, n: int, t: int, l: int, d: int, launch: Launch | None = None):
        self._lib = load()
        self._h = ctypes.c_void_p()
        self.n, self.t, self.l, self.d = n, t, l, d
        s = self._lib.pms_plan_create(n, t, l, d, ctypes.byref(launch) if launch else None,
                                      ctypes.byref(self._h))
        if s != OK:
            raise PmsError(s, "pms_plan_create")

    def execute(self, d_seqs_ptr: int, lo: int, hi: int, d_out_ptr: int, cap: int,
                d_count_ptr: int, stream: int = 0, wide: bool = False) -> None:
        """pms_plan_execute (uint32 codes), or pms_plan_execute64 with wide=True."""
        fname = "pms_plan_execute64" if wide else "pms_plan_execute"
        s = getattr(self._lib, fname)(self._h, ctypes.c_void_p(d_seqs_ptr), int(lo), int(hi),
                                      ctypes.c_void_p(d_out_ptr) if d_out_ptr else None,
                                      int(cap), ctypes.c_void_p(d_count_ptr),
                                      ctypes.c_void_p(stream) if stream else None)
        if s != OK:
            raise PmsError(s, fname)

    def execute_tensors(self, seqs, out, count, lo: int = 0, hi: int | None = None,
                        stream=None) -> None:
        """torch tensors on the current device: seqs uint8 [n,t], out int32/uint32
        [cap] (or int64/uint64 [cap]: 64-bit codes, required for l > 16), count
        int64 [1]; stream defaults to torch's current stream."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        assert seqs.is_cuda and seqs.dtype == torch.uint8 and seqs.is_contiguous()
        assert tuple(seqs.shape) == (self.n, self.t)
        assert count.dtype == torch.int64 and count.numel() >= 1 and count.is_cuda
        hi = 4 ** self.l if hi is None else hi
        wide = out.element_size() == 8
        assert out.is_cuda and out.element_size() in (4, 8)
        self.execute(seqs.data_ptr(), lo, hi, out.data_ptr() if out.numel() else 0, out.numel(),
                     count.data_ptr(), stream.cuda_stream, wide=wide)

    def roofline(self, mode: int, scans_per_warp: int = 64) -> dict:
        """pms_plan_roofline: the plan's per-unit code without its dynamic
        parts (mode 0: pass 1 only, R_pass1; mode 1: the whole scan, R_scan;
        mode 2: sparse-mode steps, R_sparse; mode 3: both interleaved at the
        last execution's ratio, R_mix) on the tables of its last execution."""
        a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        s = self._lib.pms_plan_roofline(self._h, int(mode), int(scans_per_warp), ctypes.byref(a),
                                        ctypes.byref(b), ctypes.byref(c))
        if s != OK:
            raise PmsError(s, "pms_plan_roofline")
        return dict(tests_per_s=a.value, scans_per_s=b.value, ms=c.value)

    def wait(self) -> tuple[int, Stats]:
        st = Stats()
        s = self._lib.pms_plan_wait(self._h, ctypes.byref(st))
        return s, st

    def close(self) -> None:
        if self._h:
            self._lib.pms_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def roofline(iters: int = 1 << 14) -> dict:
    """R_mix microbenchmark: the search kernel's per-compare sequence at full
    occupancy with no early exit (pms_roofline)."""
    a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    s = load().pms_roofline(int(iters), ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    if s != OK:
        raise PmsError(s, "pms_roofline")
    return dict(compares_per_s=a.value, compares_per_clk_sm_at_max=b.value, ms=c.value)


def device_info() -> dict:
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    s = load().pms_device_info(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
    if s != OK:
        raise PmsError(s, "pms_device_info")
    return dict(sms=a.value, smem_optin=b.value, clock_khz=c.value)
