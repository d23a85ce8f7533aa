"""Write golden motif sets for BASELINE.json configs with the CPU ORACLE ONLY.

Every expected value under tests/golden/bj*_seed*.json is produced here by
oracle.find() (plain character-compare skip-BF, oracle/pms_oracle.c) on the
inputs of fmgen.generate_fm(n, t, l, d, seed).  Nothing here touches the CUDA
path.  Usage:

    python scripts/make_golden.py --configs 0 1 2 3 --seeds 1 2 3 [--threads 8]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import fmgen  # noqa: E402
import oracle  # noqa: E402


def golden_path(idx: int, seed: int) -> str:
    return os.path.join(ROOT, "tests", "golden", f"bj{idx}_seed{seed}.json")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[0, 1, 2, 3])
    ap.add_argument("--seeds", type=int, nargs="+", default=list(fmgen.SEEDS))
    ap.add_argument("--threads", type=int, default=oracle.default_threads())
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args()
    oracle.build()
    for idx in args.configs:
        cfg = fmgen.BASELINE_CONFIGS[idx]
        for seed in args.seeds:
            path = golden_path(idx, seed)
            if os.path.exists(path) and not args.force:
                print("exists", path)
                continue
            s, rec = fmgen.generate_fm(cfg["n"], cfg["t"], cfg["l"], cfg["d"], seed)
            t0 = time.time()
            r = oracle.find(s, cfg["l"], cfg["d"], threads=args.threads)
            dt = time.time() - t0
            assert r.status == 0, r.status
            doc = dict(config=cfg["name"], baseline_index=idx, n=cfg["n"], t=cfg["t"],
                       l=cfg["l"], d=cfg["d"], seed=seed,
                       generator="fmgen.generate_fm(n, t, l, d, seed)",
                       producer="oracle.find (oracle/pms_oracle.c), scripts/make_golden.py",
                       count=r.count, codes=r.codes.tolist(),
                       motifs=[oracle.decode(c, cfg["l"]) for c in r.codes.tolist()],
                       consensus=rec.consensus, c_alg=r.c_alg,
                       oracle_threads=args.threads, oracle_seconds=round(dt, 2))
            with open(path + ".tmp", "w") as f:
                json.dump(doc, f, indent=1)
            os.replace(path + ".tmp", path)
            print(f"{cfg['name']} seed {seed}: {r.count} motifs, C_alg {r.c_alg:.3e}, "
                  f"{dt:.1f}s on {args.threads} threads", flush=True)


if __name__ == "__main__":
    main()
