"""Pins for the CPU oracle (oracle/), all CPU-only (-m "not gpu").

Each test pins the oracle to something other than itself: SPEC.md worked
examples (tests/golden/spec_examples.json), closed forms, brute force on tiny
inputs, an independent algorithm (Hamming-ball intersection, in C and again
in pure Python below), planted recovery under the FM model, per-motif
re-verification and metamorphic relations.  A plausible slip in the oracle (a
dropped window, an off-by-one in t-l+1, `<` for `<=`, a reversed digit order,
a skipped sequence) fails at least one of these.
"""
from __future__ import annotations

import itertools
import json
import math
import os
import random

import numpy as np
import pytest

import fmgen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ACGT = "ACGT"


def spec():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        return json.load(f)


def rank_of(s: str) -> int:
    """Big-endian base 4 with A0 C1 G2 T3 -- the test's
    own encoder, independent of the oracle's decoder."""
    r = 0
    for ch in s:
        r = 4 * r + ACGT.index(ch)
    return r


def ball_volume(l: int, d: int) -> int:
    """|{x : Hamming(x, y) <= d}| over a 4-letter alphabet."""
    return sum(math.comb(l, i) * 3 ** i for i in range(min(d, l) + 1))


def pair_count(l: int, h: int, d: int) -> int:
    """Number of l-mers within distance d of both x and y, Hamming(x,y)=h.
    Agreeing positions: a of them changed (3 letters each).  Disagreeing
    positions: i equal x, j equal y, h-i-j equal neither (2 letters each)."""
    tot = 0
    for a in range(l - h + 1):
        for i in range(h + 1):
            for j in range(h - i + 1):
                if a + h - i <= d and a + h - j <= d:
                    tot += (math.comb(l - h, a) * 3 ** a * math.factorial(h)
                            // (math.factorial(i) * math.factorial(j) * math.factorial(h - i - j))
                            * 2 ** (h - i - j))
    return tot


def py_ball_set(strings: list[str], l: int, d: int) -> set[int]:
    """Pure-Python neighbourhood intersection (itertools), a third algorithm."""
    acc = None
    for s in strings:
        cur = set()
        for k in range(len(s) - l + 1):
            w = s[k:k + l]
            for pos in itertools.chain.from_iterable(
                    itertools.combinations(range(l), r) for r in range(min(d, l) + 1)):
                for subs in itertools.product(*[[c for c in ACGT if c != w[p]] for p in pos]):
                    x = list(w)
                    for p, c in zip(pos, subs):
                        x[p] = c
                    cur.add(rank_of("".join(x)))
        acc = cur if acc is None else acc & cur
    return acc


# ---------------------------------------------------------------- SPEC pins

def test_decode_spec_examples(orc):
    for e in spec()["decode"]:
        assert orc.decode(e["rank"], e["l"]) == e["lmer"], e["cite"]


def test_rank_order_is_lex_order(orc):
    for l in range(1, 7):
        strs = [orc.decode(r, l) for r in range(4 ** l)]
        assert strs == sorted(strs)
        assert strs == ["".join(p) for p in itertools.product(ACGT, repeat=l)]
        assert all(rank_of(s) == r for r, s in enumerate(strs))


def test_hamming_spec_examples(orc):
    for e in spec()["hamming"]:
        assert orc.hamming(e["a"], e["b"]) == e["h"], e["cite"]
    rng = random.Random(7)
    for _ in range(200):  # metric axioms
        l = rng.randint(1, 12)
        x, y, z = ("".join(rng.choice(ACGT) for _ in range(l)) for _ in range(3))
        assert orc.hamming(x, x) == 0
        assert orc.hamming(x, y) == orc.hamming(y, x)
        assert orc.hamming(x, z) <= orc.hamming(x, y) + orc.hamming(y, z)


def test_matches_within_examples(orc):
    for e in spec()["matches_within"]:
        l = len(e["a"])
        res = orc.find(fmgen.from_strings([e["b"]]), l, e["d"])
        assert (rank_of(e["a"]) in set(res.codes.tolist())) == e["match"], e["cite"]


def test_window_count(orc):
    # W = t - l + 1: naive BF compares every window of every
    # sequence once per candidate, so its work counter is 4^l * n * W.
    for t, l in [(600, 3), (20, 4), (4, 4), (9, 1)]:
        s = fmgen.random_sequences(2, t, t + l)
        r = orc.naive_find(s, l, 1, threads=4)
        assert r.c_alg == 4 ** l * 2 * (t - l + 1)
    e = spec()["windows"][1]
    s = fmgen.from_strings([e["seq"]])
    r = orc.find(s, e["l"], 0)
    assert [orc.decode(c, e["l"]) for c in r.codes] == sorted(set(e["windows"]))


def test_partition_examples(orc):
    p = orc.partition(0, 4 ** 11, 64)
    assert len(p) == 64 and all(b - a == 65536 for a, b in p)
    assert orc.partition(0, 64, 1) == [(0, 64)]
    assert [b - a for a, b in orc.partition(0, 64, 5)] == [13, 13, 13, 13, 12]
    for l in (1, 3, 6):
        for w in (1, 2, 7, 64, 100):
            p = orc.partition(0, 4 ** l, w)
            assert p[0][0] == 0 and p[-1][1] == 4 ** l
            assert all(p[i][1] == p[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in p]
            assert max(sizes) - min(sizes) <= 1


def test_hand_derived_work_count(orc):
    e = spec()["search"][0]
    r = orc.find(fmgen.from_strings(e["seqs"]), e["l"], e["d"], threads=1)
    assert r.count == 0 and r.c_alg == e["c_alg"], e["cite"]
    e = spec()["search"][1]
    r = orc.find(fmgen.from_strings(e["seqs"]), e["l"], e["d"])
    assert [orc.decode(c, e["l"]) for c in r.codes] == e["motifs"], e["cite"]


# ---------------------------------------------------------------- closed forms

@pytest.mark.parametrize("l,d", [(1, 0), (4, 1), (5, 1), (6, 2), (4, 4), (6, 0), (8, 2), (9, 3)])
def test_single_window_is_hamming_ball(orc, l, d):
    """n=1, t=l: result = Ball(s, d), |Ball| = sum_{i<=d} C(l,i) 3^i."""
    s = "".join(random.Random(l * 31 + d).choice(ACGT) for _ in range(l))
    r = orc.find(fmgen.from_strings([s]), l, d)
    assert r.count == ball_volume(l, d)
    assert set(r.codes.tolist()) == {c for c in range(4 ** l)
                                     if sum(a != b for a, b in zip(orc.decode(c, l), s)) <= d}


def test_homopolymer_ball(orc):
    r = orc.find(fmgen.from_strings(["AAAAAAAA"]), 8, 2)
    assert r.count == 277  # V(8,2) = 1 + 8*3 + 28*9


@pytest.mark.parametrize("l,d", [(5, 2), (6, 2), (6, 3), (7, 3)])
def test_two_strings_closed_form(orc, l, d):
    rng = random.Random(l * 100 + d)
    for h in range(l + 1):
        x = [rng.choice(ACGT) for _ in range(l)]
        y = list(x)
        for p in rng.sample(range(l), h):
            y[p] = rng.choice([c for c in ACGT if c != x[p]])
        r = orc.find(fmgen.from_strings(["".join(x), "".join(y)]), l, d)
        assert r.count == pair_count(l, h, d), (l, d, h)


def test_d_zero_is_window_intersection(orc):
    rng = random.Random(3)
    for _ in range(20):
        n, t, l = rng.randint(1, 4), rng.randint(5, 30), rng.randint(1, 4)
        strs = ["".join(rng.choice("AC" if rng.random() < 0.5 else ACGT) for _ in range(t))
                for _ in range(n)]
        want = set.intersection(*[{rank_of(s[k:k + l]) for k in range(t - l + 1)} for s in strs])
        r = orc.find(fmgen.from_strings(strs), l, 0)
        assert r.codes.tolist() == sorted(want)


def test_d_at_least_l_is_everything(orc):
    s = fmgen.random_sequences(3, 12, 1)
    for l, d in [(3, 3), (4, 7), (5, 5)]:
        r = orc.find(s, l, d)
        assert r.count == 4 ** l and r.codes.tolist() == list(range(4 ** l))


# ------------------------------------------------------- brute force, tiny

def test_tiny_random_equivalence(orc):
    """S:449 acceptance 1: >= 50 random instances; skip-BF == naive BF ==
    Hamming-ball intersection (C) ; a subset also == pure-Python balls."""
    rng = random.Random(1234)
    for trial in range(60):
        l, n, t, d = rng.randint(3, 7), rng.randint(2, 5), rng.randint(10, 40), rng.randint(0, 2)
        s = fmgen.random_sequences(n, t, 1000 + trial)
        a = orc.find(s, l, d, threads=3)
        b = orc.naive_find(s, l, d, threads=2)
        c = orc.ball_find(s, l, d)
        assert a.status == b.status == c.status == 0
        assert a.codes.tolist() == b.codes.tolist() == c.codes.tolist(), (l, n, t, d)
        assert a.c_alg <= b.c_alg
        if l <= 5 and trial % 4 == 0:
            strs = [bytes(row).decode() for row in s]
            assert set(a.codes.tolist()) == py_ball_set(strs, l, d)


def test_planted_small_l_brute_force(orc):
    rng = random.Random(99)
    for trial in range(15):
        l = rng.randint(4, 6)
        d = rng.randint(0, 2)
        s, rec = fmgen.generate_fm(rng.randint(2, 6), rng.randint(l, 30), l, d, trial)
        a = orc.find(s, l, d)
        assert a.codes.tolist() == orc.ball_find(s, l, d).codes.tolist()
        assert rank_of(rec.consensus) in set(a.codes.tolist())


# ------------------------------------------------------------ planted recovery

def test_fm_generator_invariants():
    for seed in range(30):
        s, rec = fmgen.generate_fm(20, 200, 9, 2, seed)
        assert s.shape == (20, 200)
        for p in rec.plants:
            inst = bytes(s[p.seq, p.offset:p.offset + 9]).decode()
            assert inst == p.instance
            assert sum(a != b for a, b in zip(inst, rec.consensus)) == 2
            assert len(set(p.mutated_positions)) == 2
    s1, _ = fmgen.generate_fm(5, 50, 8, 2, 42)
    s2, _ = fmgen.generate_fm(5, 50, 8, 2, 42)
    assert np.array_equal(s1, s2)
    big = fmgen.random_sequences(100, 1000, 5)
    for b in b"ACGT":  # within 3 sigma of 0.25
        f = (big == b).mean()
        assert abs(f - 0.25) < 3 * math.sqrt(0.25 * 0.75 / big.size)


def test_planted_recovery_100_datasets(orc):
    """100 FM datasets at (9,2), n=20, t=200: consensus always found,
    and every reported motif re-verified."""
    for seed in range(100):
        s, rec = fmgen.generate_fm(20, 200, 9, 2, 10_000 + seed)
        r = orc.find(s, 9, 2)
        codes = set(r.codes.tolist())
        assert rank_of(rec.consensus) in codes
        if seed % 10 == 0:
            for c in codes:
                assert orc.verify_motif(s, 9, 2, c)


# ---------------------------------------------------------------- metamorphic

def test_metamorphic_relations(orc):
    s, rec = fmgen.generate_fm(6, 40, 6, 1, 77)
    l, d = 6, 1
    base = orc.find(s, l, d).codes.tolist()
    assert rank_of(rec.consensus) in base
    # (i) permuting sequences
    assert orc.find(s[::-1].copy(), l, d).codes.tolist() == base
    # (ii) duplicating a sequence
    assert orc.find(np.vstack([s, s[2:3]]), l, d).codes.tolist() == base
    # (iii) adding a sequence -> subset
    extra = fmgen.random_sequences(1, 40, 5)
    assert set(orc.find(np.vstack([s, extra]), l, d).codes.tolist()) <= set(base)
    # (iv) monotone in d
    prev = set()
    for dd in range(0, 4):
        cur = set(orc.find(s, l, dd).codes.tolist())
        assert prev <= cur
        prev = cur
    # (v) range additivity
    for cut in (0, 1, 1000, 2048, 4095, 4096):
        a = orc.find(s, l, d, lo=0, hi=cut).codes.tolist()
        b = orc.find(s, l, d, lo=cut, hi=4 ** l).codes.tolist()
        assert a + b == base
    # (vi) complement b -> 3-b maps code c -> c ^ (4^l - 1)
    comp = np.vectorize(lambda x: b"TGCA"[b"ACGT".index(x)])(s).astype(np.uint8)
    assert sorted(c ^ (4 ** l - 1) for c in base) == orc.find(comp, l, d).codes.tolist()
    # (vi') arbitrary base permutation maps each digit
    perm = [2, 0, 3, 1]
    ps = np.vectorize(lambda x: b"ACGT"[perm[b"ACGT".index(x)]])(s).astype(np.uint8)
    mapped = sorted(rank_of("".join(ACGT[perm[ACGT.index(ch)]] for ch in orc.decode(c, l)))
                    for c in base)
    assert orc.find(ps, l, d).codes.tolist() == mapped
    # (vii) reversing every sequence -> digit-reversed codes
    rev = s[:, ::-1].copy()
    assert orc.find(rev, l, d).codes.tolist() == sorted(rank_of(orc.decode(c, l)[::-1])
                                                         for c in base)
    # worker-count invariance
    for w in (1, 2, 5, 16):
        assert orc.find(s, l, d, threads=w).codes.tolist() == base


# ---------------------------------------------------------- statuses & edges

def test_status_codes(orc):
    s = fmgen.random_sequences(2, 10, 1)
    assert orc.find(s, 0, 0).status == orc.E_ARG
    assert orc.find(s, 17, 0).status == orc.E_ARG
    assert orc.find(s, 11, 0).status == orc.E_ARG      # l > t
    assert orc.find(s, 3, -1).status == orc.E_ARG
    bad = s.copy()
    bad[1, 4] = ord("N")
    assert orc.find(bad, 3, 1).status == orc.E_CHAR
    bad = s.copy()
    bad[0, 0] = 0
    assert orc.find(bad, 3, 1).status == orc.E_CHAR
    assert orc.find(bad, 0, 1).status == orc.E_ARG    # ARG checked before CHAR
    low = np.frombuffer(bytes(s).lower(), dtype=np.uint8).reshape(s.shape)
    assert orc.find(low, 3, 1).codes.tolist() == orc.find(s, 3, 1).codes.tolist()


def test_truncation_and_size_query(orc):
    s = fmgen.random_sequences(1, 10, 3)
    full = orc.find(s, 4, 2)
    assert full.status == 0 and full.count > 10
    q = orc.find(s, 4, 2, max_out=0)
    assert q.status == orc.E_TRUNCATED and q.count == full.count
    tr = orc.find(s, 4, 2, max_out=5)
    assert tr.status == orc.E_TRUNCATED and tr.count == full.count
    ok = orc.find(s, 4, 2, max_out=full.count)
    assert ok.status == 0 and ok.codes.tolist() == full.codes.tolist()


def test_edge_shapes(orc):
    # n = 1; t = l (W = 1); l = 1; empty range
    s = fmgen.from_strings(["G"])
    assert orc.find(s, 1, 0).codes.tolist() == [2]
    s = fmgen.random_sequences(3, 8, 4)
    assert orc.find(s, 5, 1, lo=100, hi=100).count == 0
    # verify_motif agrees with membership on a small instance
    s, _ = fmgen.generate_fm(4, 25, 5, 1, 8)
    got = set(orc.find(s, 5, 1).codes.tolist())
    for c in range(4 ** 5):
        assert orc.verify_motif(s, 5, 1, c) == (c in got)


# ----------------------------------------------------- l = 17..31 (u64 codes)

def test_find64_matches_find_for_small_l(orc):
    s, _ = fmgen.generate_fm(5, 60, 8, 2, 12)
    for l, d in [(6, 1), (8, 2), (9, 2)]:
        a = orc.find(s, l, d)
        b = orc.find64(s, l, d)
        assert b.status == 0 and b.codes.tolist() == a.codes.tolist() and b.c_alg == a.c_alg
    assert orc.find64(s, 32, 1).status == orc.E_ARG  # l <= 31
    assert orc.find(s, 17, 1).status == orc.E_ARG    # the u32 API keeps l <= 16


def test_decode_l31(orc):
    rng = random.Random(31)
    for _ in range(200):
        l = rng.randint(17, 31)
        x = "".join(rng.choice(ACGT) for _ in range(l))
        assert orc.decode(rank_of(x), l) == x


@pytest.mark.parametrize("l,d", [(20, 1), (24, 2), (31, 1)])
def test_large_l_hamming_ball_on_ranges(orc, l, d):
    """n=1, t=l: the result is the Hamming ball of the string.  For every ball
    member c (enumerated here by mutating the string), the oracle over the
    range [c-3, c+4) returns exactly the ball members in that range."""
    rng = random.Random(l * 7 + d)
    x = "".join(rng.choice(ACGT) for _ in range(l))
    ball = {x}
    frontier = {x}
    for _ in range(d):
        nxt = set()
        for y in frontier:
            for p in range(l):
                for ch in ACGT:
                    if ch != y[p]:
                        nxt.add(y[:p] + ch + y[p + 1:])
        ball |= nxt
        frontier = nxt
    ball_codes = {rank_of(y) for y in ball}
    assert len(ball_codes) == ball_volume(l, d)
    s = fmgen.from_strings([x])
    for c in rng.sample(sorted(ball_codes), 25):
        lo, hi = max(c - 3, 0), min(c + 4, 4 ** l)
        got = orc.find64(s, l, d, lo=lo, hi=hi).codes.tolist()
        assert got == sorted(v for v in ball_codes if lo <= v < hi)


def test_large_l_planted_recovery_on_ranges(orc):
    for seed in range(3):
        s, rec = fmgen.generate_fm(8, 100, 18, 3, 40 + seed)
        c = rank_of(rec.consensus)
        r = orc.find64(s, 18, 3, lo=c - 2000, hi=c + 2000)
        assert c in set(r.codes.tolist())
        for m in r.codes.tolist():
            assert orc.verify_motif(s, 18, 3, m)
