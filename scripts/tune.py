"""Launch-configuration sweep for one config (GPU box):

    python scripts/tune.py --cfg 3 --algo block --warps 8 12 16 --ctas 0 1 2
Prints the best search-kernel time per setting and checks every motif set
against the first one (launch settings must not change the result)."""
from __future__ import annotations

import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import fmgen  # noqa: E402
import paper_1403_1313_b200 as pms  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--algo", choices=["candidate", "block"], default="block")
    ap.add_argument("--warps", type=int, nargs="+", default=[0])
    ap.add_argument("--ctas", type=int, nargs="+", default=[0])
    ap.add_argument("--batch", type=int, nargs="+", default=[0])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--S", type=int, nargs="+", default=[0])
    ap.add_argument("--tglobal", type=int, nargs="+", default=[0])
    ap.add_argument("--handoff", type=int, nargs="+", default=[0])
    args = ap.parse_args()
    c = fmgen.BASELINE_CONFIGS[args.cfg]
    s, _ = fmgen.generate_fm(c["n"], c["t"], c["l"], c["d"], args.seed)
    algo = pms.ALGO_BLOCK if args.algo == "block" else pms.ALGO_CANDIDATE
    ref = None
    rows = []
    for w, ct, b, S, tg, ho in itertools.product(args.warps, args.ctas, args.batch, args.S,
                                                 args.tglobal, args.handoff):
        L = pms.Launch(algo=algo, warps_per_cta=w, ctas_per_sm=ct, batch=b, block_digits=S,
                       table_global=tg, handoff=ho)
        best = None
        for _ in range(args.reps):
            r = pms.find_ex(s, c["l"], c["d"], launch=L, max_out=1 << 22)
            assert r.status == 0, pms.strerror(r.status)
            if ref is None:
                ref = r.codes.tolist()
            assert r.codes.tolist() == ref
            best = r.stats.search_ms if best is None else min(best, r.stats.search_ms)
        row = dict(warps=w, ctas_per_sm=ct, batch=b, S=r.stats.block_digits, tglobal=tg, handoff=ho,
                   grid=r.stats.grid, block=r.stats.block,
                   nw=r.stats.windows_per_lane, search_ms=best,
                   cands_per_s=(4 ** c["l"]) / (best * 1e-3),
                   issued_per_s=r.stats.issued_compares / (best * 1e-3),
                   block_scans=r.stats.block_scans, motifs=r.count)
        rows.append(row)
        print(json.dumps(row), flush=True)
    best = min(rows, key=lambda x: x["search_ms"])
    print("BEST", json.dumps(best))


if __name__ == "__main__":
    main()
