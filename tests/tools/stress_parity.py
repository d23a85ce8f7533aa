#!/usr/bin/env python
"""Randomised parity stress (GPU box): random shapes, (l, d), families, block
sizes, launch knobs and code ranges against the CPU oracle, bit for bit.

    python tests/tools/stress_parity.py [--seconds 240] [--seed 1]

Covers corners the fixed tests sample sparsely: W not a multiple of 32, the
streaming (NW = 0) path for W > 1536, many sequences, d near l, l > 16 on
ranges, unaligned range ends, the slice family at S = 5 / 6 / 7 (incl. its
queue-overflow path and tables read through L1/L2).  Prints one line per failure and a summary;
exit status 1 on any mismatch.
"""
from __future__ import annotations

import argparse
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import fmgen  # noqa: E402
import oracle  # noqa: E402
import paper_1403_1313_b200 as pms  # noqa: E402


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=240.0)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    oracle.build()
    rng = random.Random(args.seed)
    t_end = time.time() + args.seconds
    runs = fails = 0
    while time.time() < t_end:
        wide = rng.random() < 0.25
        l = rng.randint(17, 31) if wide else rng.randint(5, 16)
        d = rng.randint(0, min(l, 8))
        n = rng.randint(1, 40)
        t = rng.randint(l, 2600 if rng.random() < 0.2 else 700)
        seed = rng.randrange(1 << 30)
        s = fmgen.generate_fm(n, t, l, min(d, l), seed)[0] if rng.random() < 0.7 else \
            fmgen.random_sequences(n, t, seed)
        top = 4 ** l
        span = rng.choice([1, 37, 4096, 4097, 65536, 200003])
        lo = rng.randrange(0, max(1, top - span))
        hi = min(top, lo + span)
        launch = pms.Launch(algo=rng.choice([0, 0, 0, 1, 2, 3, 3]),
                            block_digits=rng.choice([0, 5, 6, 7]),
                            handoff=rng.choice([0, 0, 1, 3, 17]),
                            table_global=rng.choice([0, 0, 1]), wide_words=int(rng.random() < 0.1))
        want = oracle.find64(s, l, d, lo=lo, hi=hi)
        got = pms.find64_ex(s, l, d, lo=lo, hi=hi, launch=launch, max_out=1 << 22)
        runs += 1
        # (codes are defined only on OK; a truncated result compares counts)
        if got.status != want.status or got.count != want.count or \
                (want.status == 0 and got.codes.tolist() != want.codes.tolist()):
            fails += 1
            print(f"FAIL n={n} t={t} l={l} d={d} seed={seed} lo={lo} hi={hi} "
                  f"launch=({launch.algo},{launch.block_digits},{launch.handoff},"
                  f"{launch.table_global},{launch.wide_words}) status {got.status}/{want.status} "
                  f"count {got.count}/{want.count}", flush=True)
        if not wide and got.status == 0 and rng.random() < 0.5:  # the uint32 entry point too
            g32 = pms.find_ex(s, l, d, lo=lo, hi=hi, launch=launch, max_out=1 << 22)
            if g32.codes.astype("uint64").tolist() != want.codes.tolist():
                fails += 1
                print(f"FAIL32 n={n} t={t} l={l} d={d} seed={seed} lo={lo} hi={hi}", flush=True)
    print(f"stress: {runs} runs, {fails} failures")
    if os.environ.get("PMS_DEBUG_LIB") == "1":
        # the bounds / protocol-checked library: failed device checks over the whole run
        v = pms.debug_violations()
        print(f"stress: {v} debug-check violations")
        fails += int(v != 0)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
