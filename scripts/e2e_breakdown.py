#!/usr/bin/env python
"""Where the end-to-end time of pms_find_ex goes at (15,4) n=20 t=600 (GPU box):
wall time per call through the Python binding, through a bare ctypes call
with preallocated buffers, and the device-resident plan step (no L2 flush)."""
from __future__ import annotations

import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1403_1313_b200 as pms  # noqa: E402
import fmgen  # noqa: E402


def wall(f, k=200, w=20):
    for _ in range(w):
        f()
    t0 = time.perf_counter()
    for _ in range(k):
        f()
    return 1e6 * (time.perf_counter() - t0) / k


def main() -> None:
    l, d, n, t = 15, 4, 20, 600
    s, _ = fmgen.generate_fm(n, t, l, d, 1)
    lib = pms.load()
    res = {}
    res["find_ex_us"] = wall(lambda: pms.find_ex(s, l, d, want_stats=False))
    a = np.ascontiguousarray(s)
    out = np.empty(1 << 20, dtype=np.uint32)
    cnt = ctypes.c_uint64(0)
    pa = a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    po = out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    res["ctypes_us"] = wall(lambda: lib.pms_find_ex(pa, n, t, l, d, 0, 4 ** l, None, po, 1 << 20,
                                                     ctypes.byref(cnt), None))
    dev = torch.device("cuda", 0)
    seqs = torch.from_numpy(a).to(dev)
    o = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
    c = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream()
    plan = pms.Plan(n, t, l, d)

    def step():
        plan.execute_tensors(seqs, o, c, stream=stream)
        plan.wait()
    res["plan_step_wall_us"] = wall(step)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(stream):
        ev[0].record(stream)
        for _ in range(200):
            plan.execute_tensors(seqs, o, c, stream=stream)
        ev[1].record(stream)
    torch.cuda.synchronize()
    res["plan_step_device_us_back_to_back"] = 1e3 * ev[0].elapsed_time(ev[1]) / 200
    print(json.dumps(res))


if __name__ == "__main__":
    main()
