"""Paper-experiment analogues on B200.  Run on the GPU box:

    python tests/tools/experiments.py [--out profiles/r01_experiments]

1. l-sweep (Fig. 2 "exponential run time with the increase of
   the motif length"): search-kernel time for l = 9..16 at d = 3, n=20, t=600,
   and for the paper's instances (11,3) (12,3) (13,3) (14,4) (15,4); the
   consecutive time ratios are expected near 4 (candidate space x4 per l).
2. Worker sweep (Fig. 3/4 speedup vs threads): the GPU's
   workers are persistent CTAs; speedup(W) = time(1 CTA) / time(W CTAs).
3. Table II layout: speedup per (l,d) at 32 workers and at
   the full grid, next to the paper's 32-core multicore and 32-node grid values
   (quoted, other hardware) and the CPU oracle's own thread sweep on this host
   (the paper's experiment itself, with its static partition).
Every GPU result is checked against the golden/oracle motif set where one is
available (the motif set must not depend on the number of workers).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import fmgen  # noqa: E402
import paper_1403_1313_b200 as pms  # noqa: E402

PAPER_TABLE2 = {  # PAPER.md:130-134 (speedup over 1 thread; other hardware, context only)
    (11, 3): (13.258, 32.390), (12, 3): (19.418, 32.308), (13, 3): (22.133, 33.152),
    (14, 4): (23.156, 33.537), (15, 4): (23.608, 38.348)}


ALGO = pms.ALGO_AUTO


def kernel_ms(seqs, l, d, launch=None, reps=3):
    if launch is None:
        launch = pms.Launch(algo=ALGO)
    best, codes = None, None
    for _ in range(reps):
        r = pms.find_ex(seqs, l, d, launch=launch, max_out=1 << 22)
        assert r.status == 0, pms.strerror(r.status)
        ms = r.stats.search_ms
        best = ms if best is None else min(best, ms)
        if codes is None:
            codes = r.codes.tolist()
        assert r.codes.tolist() == codes
    return best, codes, r.stats


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--algo", choices=["auto", "candidate", "block", "slice"], default="auto")
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    global ALGO
    ALGO = {"auto": pms.ALGO_AUTO, "candidate": pms.ALGO_CANDIDATE, "block": pms.ALGO_BLOCK,
            "slice": pms.ALGO_SLICE}[args.algo]
    if args.out is None:
        args.out = os.path.join(ROOT, "profiles", f"r02_experiments_{args.algo}")
    pms.build()
    res = {"device": pms.device_info(), "algo": args.algo, "lsweep": [], "paper_instances": [],
           "workers": {}, "cpu_threads": {}}

    # 1. l-sweep at d = 3 and the paper's instances
    for l in range(9, 17):
        s, _ = fmgen.generate_fm(20, 600, l, 3, 1)
        ms, codes, st = kernel_ms(s, l, 3, reps=2 if l >= 15 else 3)
        res["lsweep"].append({"l": l, "d": 3, "search_ms": ms, "motifs": len(codes),
                              "candidates_per_s": 4 ** l / (ms * 1e-3),
                              "issued_compares_per_s": st.issued_compares / (ms * 1e-3)})
        print("lsweep", res["lsweep"][-1], flush=True)
    for a, b in zip(res["lsweep"], res["lsweep"][1:]):
        b["ratio_to_prev"] = b["search_ms"] / a["search_ms"]

    inst = [(11, 3), (12, 3), (13, 3), (14, 4), (15, 4)]
    base = {}
    for l, d in inst:
        s, _ = fmgen.generate_fm(20, 600, l, d, 1)
        ms, codes, st = kernel_ms(s, l, d)
        base[(l, d)] = (s, codes, st.grid)
        res["paper_instances"].append({"l": l, "d": d, "search_ms": ms, "motifs": len(codes),
                                       "candidates_per_s": 4 ** l / (ms * 1e-3)})
        print("inst", res["paper_instances"][-1], flush=True)

    # 2. worker sweep (persistent CTAs)
    for l, d in inst:
        s, codes, full_grid = base[(l, d)]
        workers = [w for w in (1, 2, 4, 8, 16, 32, 64, 148, full_grid)
                   if not (l == 15 and w < 8 and ALGO == pms.ALGO_CANDIDATE)]
        rows = []
        for w in sorted(set(workers)):
            ms, c, st = kernel_ms(s, l, d, launch=pms.Launch(grid_ctas=w, algo=ALGO),
                                  reps=1 if w < 8 else 2)
            assert c == codes, "motif set depends on the number of workers"
            rows.append({"ctas": st.grid, "search_ms": ms})
        t1 = rows[0]["search_ms"] * rows[0]["ctas"]  # normalise to 1 CTA if 1 was skipped
        for r in rows:
            r["speedup_vs_1cta"] = t1 / r["search_ms"]
        res["workers"][f"({l},{d})"] = rows
        print("workers", l, d, rows, flush=True)

    # 3. CPU oracle thread sweep (the paper's own experiment, this host)
    if not args.skip_cpu:
        import oracle
        oracle.build()
        cores = oracle.default_threads()
        s, codes, _ = base[(11, 3)]
        rows = []
        for th in sorted({1, 2, 4, 8, cores, 2 * cores}):
            t0 = time.perf_counter()
            r = oracle.find(s, 11, 3, threads=th)
            dt = time.perf_counter() - t0
            assert r.codes.tolist() == codes
            rows.append({"threads": th, "seconds": dt})
        for r in rows:
            r["speedup"] = rows[0]["seconds"] / r["seconds"]
        res["cpu_threads"] = {"instance": "(11,3) n=20 t=600 seed 1", "cores": cores,
                              "rows": rows}
        print("cpu", rows, flush=True)

    json.dump(res, open(args.out + ".json", "w"), indent=1)
    # Table II layout
    lines = [f"# Paper-experiment analogues on B200 (tests/tools/experiments.py --algo {args.algo})", "",
             "## Fig. 2 analogue: search-kernel time vs l (d = 3, n=20, t=600, seed 1)", "",
             "| l | kernel ms | ratio to l-1 | candidates/s | motifs |", "|---|---|---|---|---|"]
    for r in res["lsweep"]:
        lines.append(f"| {r['l']} | {r['search_ms']:.3f} | {r.get('ratio_to_prev', float('nan')):.2f}"
                     f" | {r['candidates_per_s']:.3e} | {r['motifs']} |")
    lines += ["", "## Table II layout: speedup over one worker", "",
              "| (l,d) | grid 32 nodes (paper) | multicore 32 cores (paper) | B200 32 CTAs | "
              "B200 full grid | full-grid CTAs | kernel ms (full) |", "|---|---|---|---|---|---|---|"]
    for l, d in inst:
        rows = res["workers"][f"({l},{d})"]
        r32 = next(r for r in rows if r["ctas"] == 32)
        rf = rows[-1]
        g, m = PAPER_TABLE2[(l, d)]
        lines.append(f"| ({l},{d}) | {g} | {m} | {r32['speedup_vs_1cta']:.1f} | "
                     f"{rf['speedup_vs_1cta']:.1f} | {rf['ctas']} | {rf['search_ms']:.3f} |")
    if res["cpu_threads"]:
        lines += ["", f"## Fig. 3/4 analogue on this host's CPU: oracle (paper's static partition), "
                  f"{res['cpu_threads']['instance']}, {res['cpu_threads']['cores']} cores", "",
                  "| threads | seconds | speedup |", "|---|---|---|"]
        for r in res["cpu_threads"]["rows"]:
            lines.append(f"| {r['threads']} | {r['seconds']:.2f} | {r['speedup']:.2f} |")
    open(args.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
