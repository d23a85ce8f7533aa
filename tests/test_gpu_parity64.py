"""GPU parity of the 64-bit path (l = 17..31, uint64 codes,
SPEC.md:117) against the CPU oracle's oracle_find64.

Bit-exact: identical sorted uint64 code sets, counts and statuses.  At l > 16
the oracle cannot enumerate 4^l candidates, so parity runs on code ranges
[lo, hi) (range additivity) -- around planted consensuses, at random
offsets, at both ends of the code space, with unaligned ends -- plus full
exhaustive GPU runs checked by properties that hold at any size: the planted
consensus is in the set (FM model), every reported code re-verifies
with the oracle's independent verify_motif, and the oracle agrees on
ranges around every reported code.
"""
from __future__ import annotations

import random

import numpy as np
import pytest

import fmgen
import paper_1403_1313_b200 as pms

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")
    pms.build()
    pms.load()


ACGT = "ACGT"
WIDE = pms.Launch(wide_words=1)
FAMILIES64 = [pms.Launch(), pms.Launch(algo=pms.ALGO_SLICE),
              pms.Launch(algo=pms.ALGO_SLICE, table_global=1),
              pms.Launch(algo=pms.ALGO_BLOCK, block_digits=5),
              pms.Launch(algo=pms.ALGO_BLOCK, block_digits=6),
              pms.Launch(algo=pms.ALGO_CANDIDATE)]


def rank_of(s: str) -> int:
    r = 0
    for ch in s:
        r = r * 4 + ACGT.index(ch)
    return r


def gpu64(seqs, l, d, **kw):
    return pms.find64_ex(seqs, l, d, max_out=kw.pop("max_out", 1 << 22), **kw)


def assert_same64(seqs, l, d, orc, lo=0, hi=None, launch=None):
    want = orc.find64(seqs, l, d, lo=lo, hi=hi)
    got = gpu64(seqs, l, d, lo=lo, hi=hi, launch=launch)
    assert got.status == want.status, (got.status, want.status, pms.last_error())
    assert got.count == want.count, (l, d, lo, hi, got.count, want.count)
    assert got.codes.dtype == np.uint64
    assert got.codes.tolist() == want.codes.tolist()
    return got, want


# ----------------------------------------- 64-bit words at small l (full sets)

def test_wide_words_small_l_tiny_random(orc):
    """wide_words=1 runs the 64-bit-word kernels at l <= 16, where the oracle
    enumerates everything: both kernel families, both block sizes."""
    rng = random.Random(6464)
    for trial in range(60):
        l = rng.randint(1, 9)
        n = rng.randint(1, 5)
        t = rng.randint(l, 90)
        d = rng.randint(0, min(5, l))
        s = fmgen.random_sequences(n, t, 9100 + trial)
        for fam in FAMILIES64:
            L = pms.Launch(algo=fam.algo, block_digits=fam.block_digits, wide_words=1)
            got, _ = assert_same64(s, l, d, orc, launch=L)
            assert got.stats.algo == (pms.ALGO_BLOCK if l >= 5 and fam.algo != pms.ALGO_CANDIDATE
                                      else pms.ALGO_CANDIDATE)


def test_wide_words_planted_and_window_counts(orc):
    for seed in range(4):
        s, _ = fmgen.generate_fm(10, 200, 9, 2, seed)
        assert_same64(s, 9, 2, orc, launch=WIDE)
    for W in (1, 31, 33, 586, 985, 1100):  # register tiles, padding, the NW = 0 kernel
        s, _ = fmgen.generate_fm(3, W + 7, 8, 2, W)
        for S in (5, 6):
            assert_same64(s, 8, 2, orc,
                          launch=pms.Launch(algo=pms.ALGO_BLOCK, block_digits=S, wide_words=1))


def test_find64_equals_find_for_l_up_to_16(orc):
    s, _ = fmgen.generate_fm(20, 600, 11, 3, 1)
    a = pms.find_ex(s, 11, 3)
    b = gpu64(s, 11, 3)
    assert a.status == b.status == 0
    assert b.codes.astype(np.uint64).tolist() == a.codes.astype(np.uint64).tolist()
    s, _ = fmgen.generate_fm(3, 20, 16, 5, 16)
    lo, hi = (1 << 32) - (1 << 20), 1 << 32  # top of the 32-bit code space
    assert_same64(s, 16, 5, orc, lo=lo, hi=hi)
    assert_same64(s, 16, 5, orc, lo=lo, hi=hi, launch=WIDE)


# ------------------------------------------------------ l = 17..31 on ranges

@pytest.mark.parametrize("l,d", [(17, 5), (18, 5), (20, 6), (24, 7), (31, 9)])
def test_large_l_planted_ranges(orc, l, d):
    """FM instances at l > 16: ranges around the planted consensus (which
    must be found), random ranges with unaligned ends, and the last codes of
    the 4^l space; every kernel family."""
    rng = random.Random(l * 100 + d)
    s, rec = fmgen.generate_fm(6, 80, l, d, l + d)
    c = rank_of(rec.consensus)
    top = 4 ** l
    ranges = [(max(c - 5000, 0), min(c + 7001, top)), (c, c + 1),
              (top - 9000, top), (0, 4097)]
    for _ in range(3):
        lo = rng.randrange(0, top - 20000)
        ranges.append((lo, lo + rng.randrange(1, 20000)))
    for fam in FAMILIES64:
        for lo, hi in ranges:
            got, _ = assert_same64(s, l, d, orc, lo=lo, hi=hi, launch=fam)
            if lo <= c < hi:
                assert c in set(got.codes.tolist())
            assert got.stats.candidates == hi - lo


@pytest.mark.parametrize("l,d", [(17, 2), (20, 1), (24, 2), (31, 1)])
def test_large_l_hamming_ball_ranges(orc, l, d):
    """n = 1, t = l: the result is the Hamming ball of the string (closed form
    sum_i C(l,i) 3^i); on ranges around ball members the GPU returns exactly
    the ball members in the range (ball enumerated here by mutation)."""
    rng = random.Random(l * 7 + d)
    x = "".join(rng.choice(ACGT) for _ in range(l))
    ball, frontier = {x}, {x}
    for _ in range(d):
        nxt = set()
        for y in frontier:
            for p in range(l):
                for ch in ACGT:
                    if ch != y[p]:
                        nxt.add(y[:p] + ch + y[p + 1:])
        ball |= nxt
        frontier = nxt
    codes = sorted(rank_of(y) for y in ball)
    s = fmgen.from_strings([x])
    for c in rng.sample(codes, 12):
        lo, hi = max(c - 4100, 0), min(c + 4100, 4 ** l)
        got = gpu64(s, l, d, lo=lo, hi=hi)
        assert got.status == 0
        assert got.codes.tolist() == [v for v in codes if lo <= v < hi]


def test_large_l_d_at_least_l_and_empty(orc):
    s = fmgen.random_sequences(3, 40, 5)
    lo = 4 ** 19 // 3
    r = gpu64(s, 19, 19, lo=lo, hi=lo + 5000)
    assert r.status == 0 and r.codes.tolist() == list(range(lo, lo + 5000))
    r = gpu64(s, 19, 25, lo=lo, hi=lo + 3)
    assert r.codes.tolist() == [lo, lo + 1, lo + 2]
    assert gpu64(s, 19, 2, lo=lo, hi=lo).count == 0
    assert_same64(s, 19, 0, orc, lo=0, hi=1 << 20)


def test_large_l_truncation_and_errors(orc):
    s = fmgen.random_sequences(2, 30, 9)
    lo = 12345678
    r = gpu64(s, 18, 18, lo=lo, hi=lo + 1000, max_out=10)
    assert r.status == pms.E_TRUNCATED and r.count == 1000
    r = gpu64(s, 18, 18, lo=lo, hi=lo + 1000, max_out=0)
    assert r.status == pms.E_TRUNCATED and r.count == 1000
    assert gpu64(s, 32, 1).status == pms.E_ARG
    assert gpu64(s, 31, 1, lo=10, hi=5).status == pms.E_ARG
    assert pms.find_ex(s, 17, 1).status == pms.E_ARG  # uint32 codes stop at l = 16
    bad = s.copy()
    bad[1, 7] = ord("N")
    assert gpu64(bad, 18, 3, lo=0, hi=100).status == pms.E_CHAR


def test_large_l_launch_invariance(orc):
    s, rec = fmgen.generate_fm(8, 120, 18, 5, 3)
    c = rank_of(rec.consensus)
    lo, hi = c - 300000, c + 300000
    want = orc.find64(s, 18, 5, lo=lo, hi=hi).codes.tolist()
    assert c in want
    for kw in [dict(), dict(grid_ctas=1), dict(grid_ctas=5), dict(warps_per_cta=3),
               dict(batch=4096), dict(batch=12288), dict(force_generic=1), dict(table_global=1),
               dict(handoff=40), dict(block_digits=5), dict(algo=pms.ALGO_BLOCK, no_skip=1)]:
        r = gpu64(s, 18, 5, lo=lo, hi=hi, launch=pms.Launch(**kw))
        assert r.status == 0 and r.codes.tolist() == want, kw


def test_large_l_exhaustive_properties(orc):
    """A full 4^17 enumeration (1.7e10 candidates) on the GPU: the planted
    consensus is found, every reported code re-verifies with the oracle's
    independent check, and the oracle agrees on a range around every
    reported code and on random ranges."""
    l, d = 17, 5
    s, rec = fmgen.generate_fm(12, 150, l, d, 77)
    r = gpu64(s, l, d)
    assert r.status == 0 and r.stats.candidates == 4 ** l
    got = r.codes.tolist()
    assert got == sorted(set(got))
    c = rank_of(rec.consensus)
    assert c in got
    for m in got[:200]:
        assert orc.verify_motif(s, l, d, m)
    rng = random.Random(5)
    for m in rng.sample(got, min(len(got), 8)):
        lo, hi = max(m - 3000, 0), min(m + 3000, 4 ** l)
        assert [v for v in got if lo <= v < hi] == orc.find64(s, l, d, lo=lo, hi=hi).codes.tolist()
    for _ in range(4):
        lo = rng.randrange(0, 4 ** l - 100000)
        assert [v for v in got if lo <= v < lo + 100000] == \
            orc.find64(s, l, d, lo=lo, hi=lo + 100000).codes.tolist()


def test_plan_execute64_with_torch_tensors(orc):
    import torch
    l, d = 18, 5
    s, rec = fmgen.generate_fm(10, 100, l, d, 8)
    c = rank_of(rec.consensus)
    dev = torch.device("cuda:0")
    seqs = torch.from_numpy(s).to(dev)
    out = torch.zeros(1 << 12, dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    lo, hi = c - 100000, c + 100000
    with pms.Plan(10, 100, l, d) as plan:
        plan.execute_tensors(seqs, out, cnt, lo=lo, hi=hi)
        status, st = plan.wait()
        assert status == 0
        n = int(cnt.item())
        got = sorted(out[:n].cpu().numpy().astype(np.uint64).tolist())
        assert got == orc.find64(s, l, d, lo=lo, hi=hi).codes.tolist()
        assert c in got
        # uint32 output from a plan with l > 16 is an argument error
        out32 = torch.zeros(16, dtype=torch.int32, device=dev)
        with pytest.raises(pms.PmsError):
            plan.execute_tensors(seqs, out32, cnt, lo=lo, hi=hi)


@pytest.mark.parametrize("l,d", [(17, 5), (19, 7), (21, 8), (23, 9), (25, 10), (28, 12)])
def test_large_l_slice_family_default(orc, l, d):
    """l = 17..31 runs the slice family by default (S = 7, LP = l - 7 prefix
    digits; pms_slice_wide.cu) wherever the prefix counter holds it (d <= 15,
    LP - d <= 16); with d + S >= 16 the sparse test's sum can pass 31 (its
    carry out of bit 4 counts: (23,9), (25,10), (28,12)).
    FM instances at n = 20, t = 600 (the paper's shape at larger (l, d)): the
    planted consensus is found on a range around it and the set equals the
    oracle's there and on a random range, every hand-off threshold."""
    s, rec = fmgen.generate_fm(20, 600, l, d, 2)
    c = rank_of(rec.consensus)
    rng = random.Random(l)
    lo = rng.randrange(0, 4 ** l - 70000)
    for a, b in ((c - 40000, c + 30001), (lo, lo + 65536)):
        want = orc.find64(s, l, d, lo=a, hi=b).codes.tolist()
        for h in (0, 1, 3):
            got = gpu64(s, l, d, lo=a, hi=b, launch=pms.Launch(handoff=h))
            assert got.status == 0 and got.codes.tolist() == want, (l, d, a, b, h)
            assert got.stats.algo == pms.ALGO_SLICE and got.stats.block_digits == 7
        if a <= c < b:
            assert c in set(want)
    # outside the counter's range: the block family
    r = gpu64(s, 27, 3, lo=c % 4 ** 27, hi=c % 4 ** 27 + 100)  # LP - d = 17
    assert r.status == 0 and r.stats.algo == pms.ALGO_BLOCK
