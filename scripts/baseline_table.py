"""Render BASELINE.md's results table from a bench.py --all-configs document
(profiles/r02_configs.json): every config x seed, search time, rates, the
roofline fraction (vs the measured R_mix microbenchmark: the kernel's dense
scans with its sparse-mode steps interleaved at the run's own ratio) and the
oracle timings.
    python scripts/baseline_table.py profiles/r02_configs.json"""
import json
import sys

d = json.load(open(sys.argv[1]))
orc = {o["config"]: o for o in d["oracle"]["rows"]}
cores = d["oracle"]["cores"]
print("| Config | seed | GPU search ms (median / mean of 9) | candidates/s | skip-BF-equivalent compares/s (C_alg / t) | executed window tests/s | frac of R_mix | frac of R_pass1 | SM MHz | oracle s (%d cores) | oracle candidates/s | parity |" % cores)
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in d["rows"]:
    o = orc.get(r["config"]) if r["seed"] == 1 else None
    ms = r["search_ms_median"]
    calg = r["skipbf_c_alg"] / (ms * 1e-3) if r["skipbf_c_alg"] else None
    name = r["workload"].split(" FM")[0]
    if r["config"] == 3:
        name = "**" + name + "**"
    fr = r["roofline_frac"]
    fp = r["frac_vs_pass1"]
    print(f"| {name} | {r['seed']} | {ms:.4f} / {r['search_ms_mean']:.4f} | {r['candidates_per_s']:.3e} | "
          f"{calg:.3e} | {r['executed_tests_per_s']:.3e} | {fr:.2f} | {fp:.3f} | {r['sm_mhz']:.0f} | "
          + (f"{o['seconds_median']:.3f} / {o['seconds_mean']:.3f} ({o['range']}) | {o['candidates_per_s']:.3e} |"
             if o else " | |")
          + f" {'yes' if r['parity_vs_golden'] else 'NO'} |")
print()
print("f3 (PAPER.md:63 'enhanced version'): work without vs with the skip rule, exact counters")
print()
print("| Config | seed | naive per-candidate BF compares 4^l·n·W / skip-BF C_alg | block-family scans without / with the skip rule |")
print("|---|---|---|---|")
for r in d["rows"]:
    print(f"| {r['workload'].split(' FM')[0]} | {r['seed']} | {r['naive_bf_over_c_alg']:.1f} | "
          f"{r['naive_over_skip_issued']:.2f}{' (sequence-parallel: every pair is scanned either way)' if r['config'] == 0 else ''} |")
