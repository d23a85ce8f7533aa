"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
both kernel families, shared-memory and global tables, ranges, both block
sizes, the no-skip variants and an invalid byte -- each result checked against
the oracle.  Usage on the GPU box (one tool per call):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tests/tools/sanitize_case.py
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import fmgen  # noqa: E402
import oracle  # noqa: E402
import paper_1403_1313_b200 as pms  # noqa: E402


def check(seqs, l, d, launch, lo=0, hi=None):
    want = oracle.find(seqs, l, d, lo=lo, hi=hi)
    got = pms.find_ex(seqs, l, d, lo=lo, hi=hi, launch=launch, max_out=1 << 20)
    assert got.status == want.status, (got.status, want.status, pms.last_error())
    assert got.codes.tolist() == want.codes.tolist()


def main():
    oracle.build()
    s9, _ = fmgen.generate_fm(8, 120, 9, 2, 1)
    big, _ = fmgen.generate_fm(100, 600, 8, 1, 2)  # table > smem -> global
    s13, _ = fmgen.generate_fm(4, 60, 13, 3, 3)
    launches = [pms.Launch(algo=pms.ALGO_CANDIDATE), pms.Launch(algo=pms.ALGO_CANDIDATE, lanes_per_cand=32),
                pms.Launch(algo=pms.ALGO_CANDIDATE, force_generic=1),
                pms.Launch(algo=pms.ALGO_CANDIDATE, no_skip=1),
                pms.Launch(algo=pms.ALGO_BLOCK, block_digits=5),
                pms.Launch(algo=pms.ALGO_BLOCK, block_digits=6),
                pms.Launch(algo=pms.ALGO_BLOCK, block_digits=6, table_global=1),
                pms.Launch(algo=pms.ALGO_BLOCK, block_digits=5, no_skip=1)]
    for L in launches:
        check(s9, 9, 2, L)
        check(s9, 9, 2, L, lo=1000, hi=70001)
        check(s13, 13, 3, L, lo=5_000_000, hi=5_200_000)
    for L in launches[:1] + launches[4:6]:
        check(big, 8, 1, L)
    bad = s9.copy()
    bad[3, 7] = ord("N")
    for L in launches:
        assert pms.find_ex(bad, 9, 2, launch=L).status == pms.E_CHAR
    print("sanitize case ok")


if __name__ == "__main__":
    main()
