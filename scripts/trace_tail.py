"""Tail analysis of the slice search kernel (GPU box, tuning only): builds a
-DPMS_TRACE variant library, runs BASELINE configs through the plan API and
prints, per config, where the kernel's time goes -- launch to ready
(prologue), the per-warp end-time distribution, the longest blocks.

    python scripts/trace_tail.py [--configs 1,2,3] [--variants "handoff=1;handoff=4"]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="1,2,3")
ap.add_argument("--variants", default="")
ap.add_argument("--defs", default="")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--lib", default="", help="a prebuilt -DPMS_TRACE library (skip the build)")
args = ap.parse_args()

lib = args.lib or subprocess.check_output([sys.executable, os.path.join(ROOT, "scripts", "variants.py"), "build",
                               "trace", "-DPMS_TRACE"] + args.defs.split()).decode().split()[-1]
os.environ["PMS_LIB_OVERRIDE"] = lib

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fmgen  # noqa: E402
import paper_1403_1313_b200 as pms  # noqa: E402

L = pms.load()
L.pms_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.pms_trace_read_ht.argtypes = [ctypes.c_void_p, ctypes.c_int]
dev = torch.device("cuda", 0)
out = torch.zeros(1 << 20, dtype=torch.int32, device=dev)
cnt = torch.zeros(1, dtype=torch.int64, device=dev)
stream = torch.cuda.Stream()
for ci in [int(x) for x in args.configs.split(",")]:
    c = fmgen.BASELINE_CONFIGS[ci]
    s_np, _ = fmgen.generate_fm(c["n"], c["t"], c["l"], c["d"], 1)
    s = torch.from_numpy(s_np).to(dev)
    for v in (args.variants.split(";") if args.variants else [""]):
        kw = {k: int(x) for k, x in (p.split("=") for p in v.split(",") if p)}
        with pms.Plan(c["n"], c["t"], c["l"], c["d"], pms.Launch(**kw)) as plan:
            ms = []
            with torch.cuda.stream(stream):
                for r in range(args.reps + 2):
                    plan.execute_tensors(s, out, cnt, stream=stream)
                    st_, st = plan.wait()
                    assert st_ == 0
                    ms.append(st.search_ms)
            nw = st.grid * st.block // 32
            buf = np.zeros((8192, 8), dtype=np.uint64)
            # the instance that ran (mode_flags bit 1: the hand-off-on-tables
            # one, its own translation unit and trace buffer)
            rd = L.pms_trace_read_ht if (st.mode_flags >> 1) & 1 else L.pms_trace_read
            assert rd(buf.ctypes.data, nw) == 0
            tr = buf[:nw].astype(np.int64)
            t0 = tr[:, 0].min()
            enter, ready, end = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
            blocks, scans, hand, maxs, maxt = tr[:, 3], tr[:, 4], tr[:, 5], tr[:, 6], tr[:, 7] / 1e3
            q = lambda x: " ".join(f"{np.percentile(x, p):7.2f}" for p in (0, 50, 90, 99, 100))
            res = {
                "config": c["name"], "variant": v, "S": st.block_digits, "grid": st.grid,
                "block": st.block, "search_us_med": float(np.median(ms[2:]) * 1e3),
                "scans": int(st.block_scans), "warps_with_work": int((blocks > 0).sum()),
                "enter_us(p0 50 90 99 100)": q(enter), "ready_us": q(ready), "end_us": q(end),
                "blocks_per_warp": q(blocks), "scans_per_warp": q(scans),
                "handoff_checks_per_warp": q(hand), "max_scans_one_block": q(maxs),
                "longest_block_us": q(maxt),
            }
            ix = np.argsort(-end)[:5]
            res["slowest_warps"] = [
                {"end": round(float(end[k]), 2), "ready": round(float(ready[k]), 2), "blocks": int(blocks[k]),
                 "scans": int(scans[k]), "hand": int(hand[k]), "maxs": int(maxs[k]),
                 "maxt": round(float(maxt[k]), 2)} for k in ix]
            print(json.dumps(res, indent=1), flush=True)
