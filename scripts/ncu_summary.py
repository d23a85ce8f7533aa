#!/usr/bin/env python
"""Summaries of ncu output for profiles/ (run here, after gpurun brought the
files back):

    python scripts/ncu_summary.py full REPORT.ncu-rep [--title ...]   # --set full capture
    python scripts/ncu_summary.py launches LAUNCHES.csv                 # gpu__time_duration list
    python scripts/ncu_summary.py json REPORT.ncu-rep --scans N --out F  # bench.py's issue roofline

`full` prints the pipe utilisations, issue rate, stall reasons and DRAM
traffic of the captured kernel; `launches` groups the launch list by kernel
and prints each kernel's share of the device time (cold-cache, serialised
under ncu: compare SHARES with the live bench, not absolute times).
"""
from __future__ import annotations

import collections
import csv
import io
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    # the L1 data pipe (shared-memory wavefronts: one per cycle per SM)
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "smsp__inst_executed_op_shared_atom.sum",
    "memory_l1_wavefronts_shared", "memory_l1_wavefronts_shared_ideal",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
]


def full(rep: str, title: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"# {title}\n# kernel: {name}\n# report: {rep}\n")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"{k:<84} {vals[i]:>14} {units[i]}")
        print()


def to_json(rep: str, scans: int, out: str, kernel_note: str, config: str = "") -> None:
    """The numbers bench.py's roofline object reads (profiles/slice_kernel_ncu.json):
    warp instructions per block scan (smsp__inst_executed.sum / the launch's
    block scans, from the same bench command's stats) and DRAM bytes per launch."""
    import json
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, vals = rows[0], rows[2]

    units = rows[1]

    def num(k):
        i = hdr.index(k)
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[i], 1.0)
        return float(vals[i].replace(",", "")) * scale
    inst = num("smsp__inst_executed.sum")
    doc = {"kernel": vals[hdr.index("Kernel Name")], "note": kernel_note,
           "config": json.loads(config) if config else None,
           "source": os.path.relpath(rep) + " (ncu --set full --clock-control none)",
           "warp_instructions_per_launch": inst, "block_scans_per_launch": scans,
           "warp_instructions_per_scan": inst / scans,
           "dram_bytes_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
           "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
           "ipc_per_sm": num("sm__inst_executed.avg.per_cycle_active"),
           "alu_pipe_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
           "lsu_pipe_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
           "xu_pipe_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
           "kernel_us": num("gpu__time_duration.sum") / (1e3 if "nsecond" in units[hdr.index(
               "gpu__time_duration.sum")] else 1.0),
           "shared_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
           "l1_data_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
           "shared_wavefronts_per_scan": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / scans,
           "shared_atom_wavefronts_per_scan":
               num("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum") / scans}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
        f.write("\n")
    print(json.dumps(doc, indent=1))


def launches(path: str) -> None:
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "nsecond": 1e-3}.get(r["Metric Unit"], 1.0)
        tot[r["Kernel Name"]] += v * scale
        cnt[r["Kernel Name"]] += 1
    allt = sum(tot.values())
    print(f"# launch list: {path} ({sum(cnt.values())} launches, {allt:.1f} us total)")
    print(f"{'kernel':<90} {'launches':>8} {'total_us':>10} {'mean_us':>10} {'share':>7}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k[:90]:<90} {cnt[k]:>8} {v:>10.1f} {v / cnt[k]:>10.2f} {100 * v / allt:>6.1f}%")


if __name__ == "__main__":
    if len(sys.argv) >= 3 and sys.argv[1] == "full":
        title = sys.argv[sys.argv.index("--title") + 1] if "--title" in sys.argv else ""
        full(sys.argv[2], title)
    elif len(sys.argv) >= 3 and sys.argv[1] == "launches":
        launches(sys.argv[2])
    elif len(sys.argv) >= 3 and sys.argv[1] == "json":
        a = sys.argv
        to_json(a[2], int(a[a.index("--scans") + 1]), a[a.index("--out") + 1],
                a[a.index("--note") + 1] if "--note" in a else "",
                a[a.index("--config") + 1] if "--config" in a else "")
    else:
        raise SystemExit(__doc__)
