"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

All integer work, so the bar is bit-exact: identical sorted uint32 code sets,
identical counts and statuses.  Full BASELINE.json sizes compare against
golden sets written by scripts/make_golden.py (oracle only); the rest run
the oracle live on the same seeded inputs.
"""
from __future__ import annotations

import glob
import json
import os
import random

import numpy as np
import pytest

import fmgen
import paper_1403_1313_b200 as pms

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")
    pms.build()
    pms.load()
    debug = os.environ.get("PMS_DEBUG_LIB") == "1"
    if debug:
        pms.debug_violations(reset=True)
    yield
    if debug:  # bounds-checked build: no out-of-range device index anywhere
        assert pms.debug_violations() == 0


CAND = pms.Launch(algo=pms.ALGO_CANDIDATE)


def auto_algo(t, l, d):
    """The family PMS_ALGO_AUTO runs (include/pms.h): SLICE where it applies
    (l <= 16, W <= 1024, 1 <= d + 1 <= l - S), else BLOCK for l >= 5, else
    CANDIDATE."""
    if l < 5:
        return pms.ALGO_CANDIDATE
    S = 7 if l >= 13 else 5
    lp = l - S
    if l <= 16 and t - l + 1 <= 1024 and lp >= 1 and d < lp:
        return pms.ALGO_SLICE
    return pms.ALGO_BLOCK


def gpu(seqs, l, d, **kw):
    r = pms.find_ex(seqs, l, d, max_out=kw.pop("max_out", 1 << 22), **kw)
    return r


def assert_same(seqs, l, d, orc, lo=0, hi=None, launch=None):
    want = orc.find(seqs, l, d, lo=lo, hi=hi)
    got = gpu(seqs, l, d, lo=lo, hi=hi, launch=launch)
    assert got.status == want.status, (got.status, want.status)
    assert got.count == want.count
    assert got.codes.tolist() == want.codes.tolist()
    return got, want


# ------------------------------------------------------------- tiny / random

def test_tiny_random_instances(orc):
    rng = random.Random(2024)
    for trial in range(80):
        l = rng.randint(1, 8)
        n = rng.randint(1, 5)
        t = rng.randint(l, 70)
        d = rng.randint(0, min(3, l))
        s = fmgen.random_sequences(n, t, 500 + trial)
        got, _ = assert_same(s, l, d, orc)  # default family (AUTO)
        assert got.stats.algo == auto_algo(t, l, d)
        assert_same(s, l, d, orc, launch=CAND)


def test_planted_small_configs(orc):
    for seed in range(10):
        s, rec = fmgen.generate_fm(8, 120, 8, 2, seed)
        got, _ = assert_same(s, 8, 2, orc)
        code = int("".join(str("ACGT".index(c)) for c in rec.consensus), 4)
        assert code in set(got.codes.tolist())


@pytest.mark.parametrize("W", [1, 2, 15, 16, 17, 31, 32, 33, 63, 64, 65, 97, 255, 586, 600, 769,
                               985, 1537, 2100])
def test_window_counts_and_padding(orc, W):
    """Ragged W around the 16/32-lane tiles, the register-resident limits
    (16*48, 32*48) and the generic kernel beyond them."""
    l, d = 7, 2
    t = W + l - 1
    n = 3 if W < 1000 else 2
    s, _ = fmgen.generate_fm(n, t, l, d, W)
    assert_same(s, l, d, orc, launch=CAND)


@pytest.mark.parametrize("l,d", [(1, 0), (1, 1), (2, 0), (2, 1), (3, 1), (4, 0), (5, 2), (8, 8),
                                 (8, 20), (12, 4)])
def test_l_and_d_edges(orc, l, d):
    s = fmgen.random_sequences(4, 40, l * 10 + d)
    assert_same(s, l, d, orc)


def test_d_at_least_l_all_codes():
    s = fmgen.random_sequences(3, 30, 1)
    for l, d in [(6, 6), (7, 9)]:
        r = gpu(s, l, d)
        assert r.status == 0 and r.codes.tolist() == list(range(4 ** l))


def test_t_equals_l_closed_form():
    # n=1, t=l: the Hamming ball, |Ball(15,4)| = 123,841; (16,5) = 1,225,093
    for l, d, want in [(8, 2, 277), (15, 4, 123841), (16, 5, 1225093)]:
        s = fmgen.random_sequences(1, l, l)
        r = gpu(s, l, d)
        assert r.status == 0 and r.count == want


def test_identical_and_homopolymer_sequences(orc):
    s = np.tile(fmgen.random_sequences(1, 50, 3), (4, 1))
    assert_same(s, 6, 0, orc)
    assert_same(s, 6, 1, orc)
    h = np.full((3, 30), ord("G"), np.uint8)
    assert_same(h, 5, 1, orc)


def test_lowercase_and_invalid_bytes(orc):
    s = fmgen.random_sequences(3, 40, 9)
    low = np.frombuffer(bytes(s).lower(), dtype=np.uint8).reshape(s.shape).copy()
    a = gpu(s, 6, 1)
    b = gpu(low, 6, 1)
    assert a.codes.tolist() == b.codes.tolist() == orc.find(s, 6, 1).codes.tolist()
    for bad_byte in (ord("N"), 0, ord("U"), 0xC1):
        bad = s.copy()
        bad[2, 39] = bad_byte
        assert gpu(bad, 6, 1).status == pms.E_CHAR == orc.find(bad, 6, 1).status
    bad = s.copy()
    bad[0, 0] = ord("x")
    assert gpu(bad, 6, 1).status == pms.E_CHAR


@pytest.mark.parametrize("l", [7, 16, 23])
def test_invalid_byte_in_every_prepass_tile(l):
    """The pre-pass checks each byte once, in the 256-window tile of its row
    that stages it (tiles overlap by l-1 bytes): an invalid byte at a tile
    edge, in the overlap, in the last window's tail or in the last row must
    still be reported, in both word widths; the clean input searches normally."""
    n, t = 3, 256 * 3 + l + 5
    s = fmgen.random_sequences(n, t, 40 + l)
    find = pms.find_ex if l <= 16 else pms.find64_ex
    assert find(s, l, 1, lo=0, hi=5000, want_stats=False).status == 0
    for i, j in [(0, 0), (1, 255), (1, 256), (0, 255 + l - 1), (2, 511 + l - 1), (2, 512),
                 (2, t - 1), (0, t - l)]:
        bad = s.copy()
        bad[i, j] = ord("N")
        r = find(bad, l, 1, lo=0, hi=5000, want_stats=False)
        assert r.status == pms.E_CHAR and r.count == 0, (i, j)
        assert find(s, l, 1, lo=0, hi=5000, want_stats=False).status == 0


def test_truncation_and_size_query(orc):
    s = fmgen.random_sequences(1, 12, 3)
    full = gpu(s, 5, 2)
    assert full.status == 0 and full.count > 20
    q = gpu(s, 5, 2, max_out=0)
    assert q.status == pms.E_TRUNCATED and q.count == full.count
    tr = gpu(s, 5, 2, max_out=7)
    assert tr.status == pms.E_TRUNCATED and tr.count == full.count
    ok = gpu(s, 5, 2, max_out=full.count)
    assert ok.status == 0 and ok.codes.tolist() == full.codes.tolist()
    assert full.codes.tolist() == orc.find(s, 5, 2).codes.tolist()


def test_ranges_and_additivity(orc):
    s, _ = fmgen.generate_fm(5, 60, 7, 1, 4)
    full = gpu(s, 7, 1, launch=CAND).codes.tolist()
    for lo, hi in [(0, 0), (0, 1), (1, 255), (255, 257), (300, 5000), (4095, 4 ** 7),
                   (16383, 16384)]:
        assert_same(s, 7, 1, orc, lo=lo, hi=hi, launch=CAND)
    for cut in (0, 1, 777, 8192, 16384):
        a = gpu(s, 7, 1, lo=0, hi=cut, launch=CAND).codes.tolist()
        b = gpu(s, 7, 1, lo=cut, hi=4 ** 7, launch=CAND).codes.tolist()
        assert a + b == full


def test_launch_configuration_invariance():
    s, _ = fmgen.generate_fm(20, 600, 11, 3, 1)
    base = gpu(s, 11, 3).codes.tolist()
    for kw in [dict(lanes_per_cand=16), dict(lanes_per_cand=32), dict(force_generic=1),
               dict(ctas_per_sm=1, warps_per_cta=1), dict(batch=256), dict(batch=4096),
               dict(warps_per_cta=3, batch=512)]:
        L = pms.Launch(algo=pms.ALGO_CANDIDATE, **kw)
        for _ in range(2):  # determinism across repeated runs
            assert gpu(s, 11, 3, launch=L).codes.tolist() == base, kw


def test_table_in_global_memory(orc):
    # n * Wp * 4 = 100 * 608 * 4 = 243,200 B > 227 KB opt-in smem -> global table
    s, _ = fmgen.generate_fm(100, 600, 9, 2, 5)
    got, _ = assert_same(s, 9, 2, orc, launch=CAND)
    assert got.stats.table_in_smem == 0
    got = gpu(s, 9, 2, launch=pms.Launch(algo=pms.ALGO_CANDIDATE, force_generic=1))
    assert got.codes.tolist() == orc.find(s, 9, 2).codes.tolist()


def test_l16_subranges(orc):
    """l = 16 fills the uint32 code space: u64 counters and loop bounds."""
    s, rec = fmgen.generate_fm(3, 20, 16, 5, 16)
    cons = int("".join(str("ACGT".index(c)) for c in rec.consensus), 4)
    for lo, hi in [(0, 1 << 20), (cons - (1 << 19), cons + (1 << 19)),
                   ((1 << 32) - (1 << 20), 1 << 32)]:
        lo, hi = max(lo, 0), min(hi, 1 << 32)
        assert_same(s, 16, 5, orc, lo=lo, hi=hi)
    full = gpu(s, 16, 5, max_out=1 << 26)
    assert full.status == 0 and cons in set(full.codes.tolist())
    codes = full.codes.tolist()
    pick = random.Random(0).sample(codes, min(50, len(codes)))
    for c in pick:
        assert orc.verify_motif(s, 16, 5, c)


def test_plan_api_with_torch_tensors(orc):
    import torch
    s, _ = fmgen.generate_fm(20, 600, 9, 2, 2)
    dev = torch.device("cuda:0")
    seqs = torch.from_numpy(s).to(dev)
    out = torch.zeros(1 << 16, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream()
    with pms.Plan(20, 600, 9, 2) as plan:
        with torch.cuda.stream(stream):
            plan.execute_tensors(seqs, out, cnt)
        status, st = plan.wait()
        assert status == 0
        n = int(cnt.item())
        got = sorted(out[:n].cpu().numpy().astype(np.uint32).tolist())
        assert got == orc.find(s, 9, 2).codes.tolist()
        # re-execute the same plan on a range
        with torch.cuda.stream(stream):
            plan.execute_tensors(seqs, out, cnt, lo=1000, hi=200000)
        status, st = plan.wait()
        n = int(cnt.item())
        got = sorted(out[:n].cpu().numpy().astype(np.uint32).tolist())
        assert got == orc.find(s, 9, 2, lo=1000, hi=200000).codes.tolist()
        assert st.candidates == 199000
        bad = seqs.clone()
        bad[3, 3] = ord("N")
        with torch.cuda.stream(stream):
            plan.execute_tensors(bad, out, cnt)
        status, _ = plan.wait()
        assert status == pms.E_CHAR and int(cnt.item()) == 0
        # the invalid-input flag of a step never leaks into the next one, even
        # when that step is enqueued right behind it with no wait in between
        with torch.cuda.stream(stream):
            plan.execute_tensors(bad, out, cnt)
            plan.execute_tensors(seqs, out, cnt)
        status, _ = plan.wait()
        assert status == 0
        n = int(cnt.item())
        assert sorted(out[:n].cpu().numpy().astype(np.uint32).tolist()) == \
            orc.find(s, 9, 2).codes.tolist()


# ------------------------------------------------- BASELINE.json full sizes

GOLDEN_FILES = sorted(glob.glob(os.path.join(GOLDEN, "bj*_seed*.json")))


@pytest.mark.parametrize("path", GOLDEN_FILES, ids=[os.path.basename(p) for p in GOLDEN_FILES])
def test_baseline_configs_against_golden(orc, path):
    g = json.load(open(path))
    s, rec = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
    assert rec.consensus == g["consensus"]  # the generator reproduces the golden input
    r = gpu(s, g["l"], g["d"], launch=CAND)
    assert r.status == 0
    assert r.count == g["count"]
    assert r.codes.tolist() == g["codes"]
    # work counters: the kernel scans whole sequences, so it issues at least C_alg
    assert r.stats.issued_compares >= g["c_alg"]
    for c in r.codes.tolist():
        assert orc.verify_motif(s, g["l"], g["d"], c)


# ------------------------------------------------ plain brute force variant

def test_naive_brute_force_variant(orc):
    """no_skip = 1: every candidate scans all n sequences (PAPER.md:63 before
    the skip rule).  Same result; issued compares = (hi-lo) * n * W exactly."""
    rng = random.Random(77)
    L = pms.Launch(no_skip=1)
    for trial in range(20):
        l = rng.randint(1, 7)
        n = rng.randint(1, 4)
        t = rng.randint(l, 50)
        d = rng.randint(0, 2)
        s = fmgen.random_sequences(n, t, 900 + trial)
        got, _ = assert_same(s, l, d, orc, launch=L)
        assert got.stats.issued_compares == 4 ** l * n * (t - l + 1)
    s, _ = fmgen.generate_fm(20, 600, 9, 2, 1)
    got = gpu(s, 9, 2, launch=L)
    skip = gpu(s, 9, 2)
    assert got.codes.tolist() == skip.codes.tolist() == orc.find(s, 9, 2).codes.tolist()
    assert got.stats.issued_compares == 4 ** 9 * 20 * 592
    assert skip.stats.issued_compares < got.stats.issued_compares


def test_grid_size_override():
    s, _ = fmgen.generate_fm(20, 600, 10, 2, 3)
    base = gpu(s, 10, 2).codes.tolist()
    for algo in (pms.ALGO_CANDIDATE, pms.ALGO_BLOCK):
        for g in (1, 2, 7, 148):
            r = gpu(s, 10, 2, launch=pms.Launch(grid_ctas=g, algo=algo))
            assert r.stats.grid == g and r.codes.tolist() == base


# ------------------------------------------------ PMS_ALGO_BLOCK family

BLOCK = pms.Launch(algo=pms.ALGO_BLOCK)
BLOCKS = [pms.Launch(algo=pms.ALGO_BLOCK, block_digits=5),
          pms.Launch(algo=pms.ALGO_BLOCK, block_digits=6)]


@pytest.mark.parametrize("S", [5, 6])
def test_block_algo_tiny_random(orc, S):
    rng = random.Random(4242 + S)
    L = pms.Launch(algo=pms.ALGO_BLOCK, block_digits=S)
    for trial in range(80):
        l = rng.randint(1, 9)
        n = rng.randint(1, 5)
        t = rng.randint(l, 90)
        d = rng.randint(0, min(5, l))
        s = fmgen.random_sequences(n, t, 7000 + trial)
        got, _ = assert_same(s, l, d, orc, launch=L)
        assert got.stats.algo == (pms.ALGO_BLOCK if l >= 5 else pms.ALGO_CANDIDATE)
        if l >= 5:
            assert got.stats.block_digits == (S if l >= S else 5)
    # 1024-candidate blocks: l = 5 is a single block with an empty prefix
    for seed in range(5):
        s = fmgen.random_sequences(3, 30, 60 + seed)
        for d in range(0, 6):
            assert_same(s, 5, d, orc, launch=BLOCK)


def test_block_algo_planted_and_edges(orc):
    for seed in range(6):
        s, _ = fmgen.generate_fm(10, 200, 9, 2, seed)
        assert_same(s, 9, 2, orc, launch=BLOCK)
    for l, d in [(5, 0), (5, 5), (6, 6), (7, 9), (8, 3), (10, 4), (12, 5)]:
        s = fmgen.random_sequences(4, 40, l * 3 + d)
        assert_same(s, l, d, orc, launch=BLOCK)
    h = np.full((3, 30), ord("T"), np.uint8)
    assert_same(h, 6, 1, orc, launch=BLOCK)
    s = np.tile(fmgen.random_sequences(1, 50, 3), (4, 1))
    assert_same(s, 7, 0, orc, launch=BLOCK)
    assert_same(s, 7, 2, orc, launch=BLOCK)


@pytest.mark.parametrize("S", [5, 6])
def test_block_algo_ranges(orc, S):
    L = pms.Launch(algo=pms.ALGO_BLOCK, block_digits=S)
    s, _ = fmgen.generate_fm(5, 60, 7, 1, 4)
    full = gpu(s, 7, 1, launch=L).codes.tolist()
    assert full == orc.find(s, 7, 1).codes.tolist()
    for lo, hi in [(0, 1), (1, 255), (3, 9), (255, 257), (300, 5000), (4095, 4 ** 7),
                   (16383, 16384), (100, 100), (1023, 1025), (1000, 3100), (31, 33),
                   (4095, 4097), (4000, 12300)]:
        assert_same(s, 7, 1, orc, lo=lo, hi=hi, launch=L)
    for cut in (1, 777, 8192):
        a = gpu(s, 7, 1, lo=0, hi=cut, launch=L).codes.tolist()
        b = gpu(s, 7, 1, lo=cut, hi=4 ** 7, launch=L).codes.tolist()
        assert a + b == full


def test_block_algo_window_counts(orc):
    for W in (1, 31, 33, 586, 985, 2100):
        l, d = 8, 2
        s, _ = fmgen.generate_fm(3, W + l - 1, l, d, W)
        for L in BLOCKS:
            assert_same(s, l, d, orc, launch=L)


def test_block_algo_global_table_and_l16(orc):
    s, _ = fmgen.generate_fm(100, 600, 9, 2, 5)
    got, _ = assert_same(s, 9, 2, orc, launch=BLOCK)
    assert got.stats.table_in_smem == 0
    s, rec = fmgen.generate_fm(3, 20, 16, 5, 16)
    cons = int("".join(str("ACGT".index(c)) for c in rec.consensus), 4)
    for lo, hi in [(0, 1 << 20), (cons - (1 << 19), cons + (1 << 19)),
                   ((1 << 32) - (1 << 20), 1 << 32)]:
        for L in BLOCKS:
            assert_same(s, 16, 5, orc, lo=max(lo, 0), hi=min(hi, 1 << 32), launch=L)
    a = gpu(s, 16, 5, max_out=1 << 26, launch=BLOCK)
    b = gpu(s, 16, 5, max_out=1 << 26)
    assert a.status == b.status == 0 and a.codes.tolist() == b.codes.tolist()


def test_block_algo_launch_invariance():
    s, _ = fmgen.generate_fm(20, 600, 11, 3, 1)
    base = gpu(s, 11, 3, launch=CAND).codes.tolist()
    for S in (5, 6):
        for kw in [dict(), dict(grid_ctas=1), dict(grid_ctas=7), dict(warps_per_cta=3),
                   dict(batch=4096), dict(batch=256), dict(batch=12288), dict(force_generic=1)]:
            L = pms.Launch(algo=pms.ALGO_BLOCK, block_digits=S, **kw)
            assert gpu(s, 11, 3, launch=L).codes.tolist() == base, (S, kw)


@pytest.mark.parametrize("path", GOLDEN_FILES, ids=[os.path.basename(p) for p in GOLDEN_FILES])
def test_block_algo_baseline_configs(orc, path):
    g = json.load(open(path))
    s, _ = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
    for launch in BLOCKS + [None]:  # both block sizes and the default (AUTO) family
        r = gpu(s, g["l"], g["d"], launch=launch)
        assert r.status == 0
        assert r.stats.algo == (pms.ALGO_BLOCK if launch is not None else pms.ALGO_SLICE)
        assert r.count == g["count"] and r.codes.tolist() == g["codes"]


def test_concurrent_host_calls_and_context_reuse(orc):
    """pms_find_ex from several host threads at once (ctypes drops the GIL):
    each call takes its own pooled context; results stay exact."""
    import threading
    inputs = [fmgen.generate_fm(8, 150, 8, 2, 300 + k)[0] for k in range(6)]
    want = [orc.find(s, 8, 2).codes.tolist() for s in inputs]
    got = [None] * len(inputs)

    def work(k):
        for _ in range(3):
            got[k] = gpu(inputs[k], 8, 2).codes.tolist()

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(inputs))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert got == want
    # a pooled context must not leak state between shapes / ranges / bad inputs
    bad = inputs[0].copy()
    bad[1, 1] = ord("N")
    assert gpu(bad, 8, 2).status == pms.E_CHAR
    assert gpu(inputs[0], 8, 2).codes.tolist() == want[0]
    assert gpu(inputs[0], 8, 2, lo=5000, hi=9000).codes.tolist() == \
        orc.find(inputs[0], 8, 2, lo=5000, hi=9000).codes.tolist()


def test_pooled_plans_sharing_a_kernel(orc):
    """Regression: two shapes that launch the same kernel instance with
    different dynamic shared memory; the larger one is reused after the
    smaller one was created (the per-kernel smem attribute must not shrink)."""
    big = fmgen.random_sequences(9, 48, 1)    # l=7: W=42 -> same block kernel, 9 rows
    small = fmgen.random_sequences(2, 48, 2)  # 2 rows
    for algo in (pms.ALGO_BLOCK, pms.ALGO_CANDIDATE):
        L = pms.Launch(algo=algo)
        r1 = gpu(big, 7, 2, launch=L)
        r2 = gpu(small, 7, 2, launch=L)
        r3 = gpu(big, 7, 2, launch=L)
        assert r1.status == r2.status == r3.status == 0, pms.last_error()
        assert r1.codes.tolist() == r3.codes.tolist() == orc.find(big, 7, 2).codes.tolist()
        assert r2.codes.tolist() == orc.find(small, 7, 2).codes.tolist()


def test_block_algo_without_skip_rule(orc):
    """algo = BLOCK + no_skip: every block scans all n sequences (plain brute
    force, bit-parallel over 4^S candidates); same set; (block, sequence)
    scans = blocks * n exactly."""
    for S in (5, 6):
        L = pms.Launch(algo=pms.ALGO_BLOCK, block_digits=S, no_skip=1)
        s, _ = fmgen.generate_fm(6, 100, 9, 2, S)
        got, _ = assert_same(s, 9, 2, orc, launch=L)
        assert got.stats.block_scans == (4 ** 9 // 4 ** S) * 6
        assert got.stats.issued_compares == got.stats.block_scans * 92
        for seed in range(3):
            s = fmgen.random_sequences(3, 40, 80 + seed)
            assert_same(s, 7, 2, orc, launch=L)


def test_block_algo_handoff_thresholds(orc):
    """Any hand-off threshold (block scans -> per-candidate checks) gives the
    same set, including several survivors finished one by one."""
    s, _ = fmgen.generate_fm(12, 150, 9, 2, 21)
    want = orc.find(s, 9, 2).codes.tolist()
    for S in (5, 6):
        for h in (1, 2, 5, 40, 5000):
            L = pms.Launch(algo=pms.ALGO_BLOCK, block_digits=S, handoff=h)
            assert gpu(s, 9, 2, launch=L).codes.tolist() == want, (S, h)


# --------------------------------- compaction stress (SURVEY 8(d) extra configs)

def test_compaction_stress_10_4(orc):
    """(10,4), n=20, t=600: nearly every candidate is a motif (~1e6 of 4^10):
    the atomic-append compaction writes ~1e6 codes; both families; exact
    count on truncation (max_out = 0 size query, then a too-small buffer)."""
    s, _ = fmgen.generate_fm(20, 600, 10, 4, 1)
    want = orc.find(s, 10, 4)
    assert want.status == 0 and want.count > 900_000
    for L in (None, CAND, pms.Launch(algo=pms.ALGO_BLOCK, block_digits=6)):
        got = gpu(s, 10, 4, launch=L, max_out=1 << 21)
        assert got.status == 0 and got.count == want.count
        assert np.array_equal(got.codes, want.codes)
    r = gpu(s, 10, 4, max_out=0)
    assert r.status == pms.E_TRUNCATED and r.count == want.count
    r = gpu(s, 10, 4, max_out=want.count - 1)
    assert r.status == pms.E_TRUNCATED and r.count == want.count


def test_compaction_stress_16_6(orc):
    """(16,6), n=20, t=600: ~1e5 spurious motifs over the full 4^16 space.
    Exhaustive GPU run; oracle parity on ranges; every sampled motif
    re-verifies; the planted consensus is present."""
    s, rec = fmgen.generate_fm(20, 600, 16, 6, 1)
    full = gpu(s, 16, 6, max_out=1 << 24)
    assert full.status == 0 and full.count > 10_000
    got = full.codes.tolist()
    cons = int("".join(str("ACGT".index(c)) for c in rec.consensus), 4)
    assert cons in set(got)
    rng = random.Random(166)
    for m in rng.sample(got, 50):
        assert orc.verify_motif(s, 16, 6, m)
    for lo in [cons - 20000] + [rng.randrange(0, 4 ** 16 - 60000) for _ in range(3)]:
        hi = lo + 40000
        want = orc.find(s, 16, 6, lo=lo, hi=hi).codes.tolist()
        assert [c for c in got if lo <= c < hi] == want


# ------------------------------------------ metamorphic relations on the GPU

def _digits_reversed(c: int, l: int) -> int:
    r = 0
    for _ in range(l):
        r = r * 4 + (c & 3)
        c >>= 2
    return r


def test_gpu_metamorphic_relations():
    """Relations the result set must satisfy, checked on the GPU
    path directly: permuting or duplicating sequences keeps the set; adding a
    sequence gives a subset; complementing every base (b -> 3-b) maps each code
    c to c ^ (4^l - 1); reversing every sequence reverses each code's digits;
    the set grows monotonically with d."""
    l, d = 11, 3
    s, _ = fmgen.generate_fm(20, 600, l, d, 2)
    base = set(gpu(s, l, d).codes.tolist())
    rng = np.random.default_rng(7)
    assert set(gpu(s[rng.permutation(20)], l, d).codes.tolist()) == base
    assert set(gpu(np.vstack([s, s[3:5]]), l, d).codes.tolist()) == base
    extra = fmgen.random_sequences(1, 600, 99)
    assert set(gpu(np.vstack([s, extra]), l, d).codes.tolist()) <= base
    comp = {ord("A"): ord("T"), ord("C"): ord("G"), ord("G"): ord("C"), ord("T"): ord("A")}
    sc = np.vectorize(comp.get)(s).astype(np.uint8)
    mask = 4 ** l - 1
    assert set(gpu(sc, l, d).codes.tolist()) == {c ^ mask for c in base}
    sr = np.ascontiguousarray(s[:, ::-1])
    assert set(gpu(sr, l, d).codes.tolist()) == {_digits_reversed(c, l) for c in base}
    assert base <= set(gpu(s, l, d + 1).codes.tolist())
    assert set(gpu(s, l, d - 1).codes.tolist()) <= base


def test_graph_replay_sees_new_inputs(orc):
    """Repeated calls with the same shape, range and capacity replay the
    device work as a CUDA graph (include/pms.h); each call must still search
    its own input: alternate two inputs of one shape and compare with the
    oracle every time (with and without stats, and after a range change)."""
    a, _ = fmgen.generate_fm(10, 120, 9, 2, 501)
    b, _ = fmgen.generate_fm(10, 120, 9, 2, 502)
    want = {id(a): orc.find(a, 9, 2).codes.tolist(), id(b): orc.find(b, 9, 2).codes.tolist()}
    assert want[id(a)] != want[id(b)]
    for k in range(8):
        s = a if k % 2 == 0 else b
        r = pms.find_ex(s, 9, 2, want_stats=(k == 5))
        assert r.status == 0 and r.codes.tolist() == want[id(s)], k
    r = pms.find_ex(a, 9, 2, lo=1000, hi=90000, want_stats=False)
    assert r.codes.tolist() == orc.find(a, 9, 2, lo=1000, hi=90000).codes.tolist()
    r = pms.find_ex(b, 9, 2, lo=1000, hi=90000, want_stats=False)
    assert r.codes.tolist() == orc.find(b, 9, 2, lo=1000, hi=90000).codes.tolist()
    bad = a.copy()
    bad[0, 0] = ord("N")
    for _ in range(2):  # replays of one graph reuse its step id
        assert pms.find_ex(bad, 9, 2, lo=1000, hi=90000, want_stats=False).status == pms.E_CHAR
    assert pms.find_ex(b, 9, 2, lo=1000, hi=90000, want_stats=False).codes.tolist() == \
        orc.find(b, 9, 2, lo=1000, hi=90000).codes.tolist()


@pytest.mark.parametrize("W", [992, 1024, 1025, 1100, 1300, 1536, 1537, 1600])
def test_block_algo_long_rows(orc, W):
    """Rows of 1025..1536 windows (regression: the block family once used
    register tiles of more than 32 windows per lane there, overflowing the
    per-lane 32-bit hit mask); both block sizes, the hand-off, a global table,
    and the 64-bit words."""
    l, d = 8, 1
    s, _ = fmgen.generate_fm(3, W + l - 1, l, d, W)
    for L in [pms.Launch(), pms.Launch(algo=pms.ALGO_BLOCK, block_digits=5),
              pms.Launch(algo=pms.ALGO_BLOCK, block_digits=6, handoff=17),
              pms.Launch(algo=pms.ALGO_BLOCK, table_global=1),
              pms.Launch(algo=pms.ALGO_BLOCK, wide_words=1)]:
        assert_same(s, l, d, orc, launch=L)
    s2 = fmgen.random_sequences(12, W + 13, W + 1)  # l = 14, dense hits, ranges
    for lo in (0, 4 ** 14 // 3):
        assert_same(s2, 14, 4, orc, lo=lo, hi=lo + 20000)


@pytest.mark.parametrize("env", [{"PMS_NO_PDL": "1"}, {"PMS_NO_GRAPH": "1"},
                                 {"PMS_NO_PDL": "1", "PMS_NO_GRAPH": "1"}])
def test_plain_launch_paths(env):
    """The switches read once per process (include/pms.h): plain stream order
    instead of the programmatic dependent launch, and call-by-call enqueue
    instead of graph replay, give the golden set of a BASELINE config, on
    repeated calls (a fresh process per switch)."""
    import subprocess
    import sys
    path = os.path.join(GOLDEN, "bj2_seed1.json")
    code = f"""
import json, sys
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import fmgen, paper_1403_1313_b200 as pms
g = json.load(open({path!r}))
s, _ = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
for _ in range(3):
    r = pms.find_ex(s, g["l"], g["d"], want_stats=False)
    assert r.status == 0 and r.codes.tolist() == g["codes"], r.status
print("ok")
"""
    p = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stderr[-2000:]


@pytest.mark.parametrize("force", ["0", "1"])
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_handoff_check_kinds(cfg, force):
    """The slice family's two hand-off paths -- the check on
    the staged planes and slots, one candidate at a time (chosen for ranges
    with few blocks per warp), and the sparse mode (candidate lists of up to
    32 entries tested on the planes of all l positions) -- each forced in a
    fresh process (PMS_HANDOFF_TABLES is read once), give the golden set of
    (11,3), (13,3) and (15,4), whole and on a sub-range, for hand-off
    thresholds 1..5000; mode_flags bit 1 reports the kind that ran.  With the default, (13,3) (4,096 blocks for
    4,736 warps) runs the tables check and (15,4) the packed-word one."""
    import subprocess
    import sys
    path = os.path.join(GOLDEN, f"bj{cfg}_seed1.json")
    code = f"""
import json, sys
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import fmgen, paper_1403_1313_b200 as pms
g = json.load(open({path!r}))
s, _ = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
r = pms.find_ex(s, g["l"], g["d"])
assert r.status == 0 and r.codes.tolist() == g["codes"], r.status
assert r.stats.algo == pms.ALGO_SLICE
assert (r.stats.mode_flags >> 1) & 1 == {int(force)}, r.stats.mode_flags
lo, hi = 4 ** g["l"] // 3, 4 ** g["l"] // 3 + 3 * 4 ** (g["l"] - 3) + 777
r = pms.find_ex(s, g["l"], g["d"], lo=lo, hi=hi)
want = [c for c in g["codes"] if lo <= c < hi]
assert r.status == 0 and r.codes.tolist() == want
for h in (1, 2, 8, 31, 32, 5000):  # sparse-mode / tables-check thresholds (32: one entry per lane)
    r = pms.find_ex(s, g["l"], g["d"], launch=pms.Launch(handoff=h))
    assert r.status == 0 and r.codes.tolist() == g["codes"], h
    r = pms.find_ex(s, g["l"], g["d"], lo=lo, hi=hi, launch=pms.Launch(handoff=h))
    assert r.status == 0 and r.codes.tolist() == want, h
print("ok")
"""
    p = subprocess.run([sys.executable, "-c", code],
                       env={**os.environ, "PMS_HANDOFF_TABLES": force},
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stderr[-2000:]


def test_handoff_kind_default_by_blocks_per_warp():
    """Default choice of the hand-off check: staged tables below two blocks per
    resident warp ((13,3): 4,096 blocks), packed words above ((15,4): 65,536)."""
    for cfg, want in ((2, 1), (3, 0)):
        g = json.load(open(os.path.join(GOLDEN, f"bj{cfg}_seed1.json")))
        s, _ = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
        r = pms.find_ex(s, g["l"], g["d"])
        assert r.status == 0 and r.codes.tolist() == g["codes"]
        assert (r.stats.mode_flags >> 1) & 1 == want, (cfg, r.stats.mode_flags)
