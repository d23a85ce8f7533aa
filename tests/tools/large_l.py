#!/usr/bin/env python
"""Time the 64-bit path (l > 16) on FM instances shaped
like the paper's challenge problem (n=20, t=600) at larger (l, d):
exhaustive 4^l enumeration on one B200, planted-consensus recovery, and an
oracle spot check on a code range around the consensus (oracle_find64).

    python tests/tools/large_l.py [--configs 17,6 18,6 19,7] [--budget-s 60]
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


def rank_of(s: str) -> int:
    r = 0
    for ch in s:
        r = r * 4 + "ACGT".index(ch)
    return r


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["17,6", "18,6", "19,7"])
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--t", type=int, default=600)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--lo-frac", type=float, default=0.0,
                    help="time only [lo_frac, hi_frac) of the code space (1.0 = all)")
    ap.add_argument("--hi-frac", type=float, default=1.0)
    ap.add_argument("--block-digits", type=int, default=0)
    ap.add_argument("--algo", type=int, default=0, help="pms_launch.algo (0: AUTO)")
    ap.add_argument("--oracle-range", type=int, default=200000)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import oracle  # test infrastructure: spot check only
    oracle.build()
    rows = []
    for cfg in args.configs:
        l, d = (int(x) for x in cfg.split(","))
        s, rec = fmgen.generate_fm(args.n, args.t, l, d, args.seed)
        c = rank_of(rec.consensus)
        top = 4 ** l
        lo, hi = int(top * args.lo_frac), int(top * args.hi_frac)
        L = pms.Launch(block_digits=args.block_digits, algo=args.algo)
        pms.find64_ex(s, l, d, lo=c - 4096, hi=c + 4096, launch=L)  # warm-up (plan, module)
        t0 = time.time()
        r = pms.find64_ex(s, l, d, lo=lo, hi=hi, launch=L, max_out=1 << 24)
        wall = time.time() - t0
        assert r.status == 0, (r.status, pms.last_error())
        st = r.stats
        olo, ohi = max(c - args.oracle_range // 2, 0), min(c + args.oracle_range // 2, top)
        want = oracle.find64(s, l, d, lo=olo, hi=ohi).codes.tolist()
        got_rng = pms.find64_ex(s, l, d, lo=olo, hi=ohi, launch=L).codes.tolist()
        row = dict(l=l, d=d, n=args.n, t=args.t, seed=args.seed, lo=lo, hi=hi,
                   candidates=hi - lo, motifs=r.count, search_ms=st.search_ms, wall_s=wall,
                   candidates_per_s=(hi - lo) / (st.search_ms * 1e-3),
                   algo=st.algo, block_scans=st.block_scans, block_digits=st.block_digits,
                   grid=st.grid, block=st.block, table_in_smem=st.table_in_smem,
                   consensus_found=(c in set(r.codes.tolist())) if lo <= c < hi else None,
                   oracle_range=[olo, ohi], oracle_range_parity=(got_rng == want),
                   oracle_range_motifs=len(want))
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
