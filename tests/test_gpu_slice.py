"""GPU parity of PMS_ALGO_SLICE (bit-sliced pass 1, batched hit resolution;
DESIGN.md section 6c) against the CPU oracle and the golden sets.

Integer work only: the bar is bit-exact (identical sorted code sets, counts,
statuses).  The slice family computes the block family's per-candidate skip-BF
 with a different mapping onto the machine, so every case here
is checked against the oracle (or an oracle-written golden set), never
against another GPU family.
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
GOLDEN_FILES = sorted(glob.glob(os.path.join(GOLDEN, "bj*_seed*.json")))


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
    if debug:
        assert pms.debug_violations() == 0


def slice_launch(S=0, **kw):
    return pms.Launch(algo=pms.ALGO_SLICE, block_digits=S, **kw)


def applies(t, l, d, S):
    """pms_plan_create's eligibility rule for the slice family."""
    return 5 <= l <= 16 and t - l + 1 <= 1024 and 1 <= l - S and d < l - S


def check(seqs, l, d, orc, lo=0, hi=None, launch=None, expect_slice=None):
    want = orc.find(seqs, l, d, lo=lo, hi=hi)
    got = pms.find_ex(seqs, l, d, lo=lo, hi=hi, launch=launch, max_out=1 << 22)
    assert got.status == want.status, (got.status, want.status)
    assert got.count == want.count
    if want.status == pms.OK:  # (on PMS_E_TRUNCATED the codes are unspecified)
        assert got.codes.tolist() == want.codes.tolist()
    if expect_slice is not None and got.status == 0 and (hi is None or hi > lo):
        assert (got.stats.algo == pms.ALGO_SLICE) == expect_slice, got.stats.algo
    return got


@pytest.mark.parametrize("path", GOLDEN_FILES, ids=[os.path.basename(p) for p in GOLDEN_FILES])
@pytest.mark.parametrize("S", [0, 5, 6, 7])
def test_slice_baseline_configs_against_golden(orc, path, S):
    g = json.load(open(path))
    s, rec = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
    assert rec.consensus == g["consensus"]
    r = pms.find_ex(s, g["l"], g["d"], launch=slice_launch(S), max_out=1 << 22)
    assert r.status == 0
    S_ran = S or (7 if g["l"] >= 13 else 5)
    assert (r.stats.algo == pms.ALGO_SLICE) == applies(g["t"], g["l"], g["d"], S_ran)
    assert r.count == g["count"] and r.codes.tolist() == g["codes"]


@pytest.mark.parametrize("S", [5, 6, 7])
def test_slice_tiny_random(orc, S):
    rng = random.Random(5150 + S)
    for trial in range(120):
        l = rng.randint(S + 1, max(12, S + 4))
        n = rng.randint(1, 6)
        t = rng.randint(l, 140)
        d = rng.randint(0, min(6, l - S - 1))
        s = fmgen.random_sequences(n, t, 31000 + 97 * S + trial)
        check(s, l, d, orc, launch=slice_launch(S), expect_slice=True)


def test_slice_planted_small(orc):
    for seed in range(8):
        s, rec = fmgen.generate_fm(10, 200, 9, 2, seed)
        got = check(s, 9, 2, orc, launch=slice_launch(), expect_slice=True)
        code = int("".join(str("ACGT".index(c)) for c in rec.consensus), 4)
        assert code in set(got.codes.tolist())


@pytest.mark.parametrize("S", [5, 6, 7])
def test_slice_ranges_and_additivity(orc, S):
    L = slice_launch(S)
    s, _ = fmgen.generate_fm(5, 60, 9, 2, 4)
    full = pms.find_ex(s, 9, 2, launch=L).codes.tolist()
    assert full == orc.find(s, 9, 2).codes.tolist()
    for lo, hi in [(0, 1), (1, 255), (3, 9), (1023, 1025), (4095, 4097), (4000, 12300),
                   (100, 100), (31, 33), (65535, 70000), (4 ** 9 - 5, 4 ** 9)]:
        check(s, 9, 2, orc, lo=lo, hi=hi, launch=L)
    for cut in (1, 777, 8192, 100000):
        a = pms.find_ex(s, 9, 2, lo=0, hi=cut, launch=L).codes.tolist()
        b = pms.find_ex(s, 9, 2, lo=cut, hi=4 ** 9, launch=L).codes.tolist()
        assert a + b == full


@pytest.mark.parametrize("W", [1, 2, 31, 32, 33, 63, 64, 65, 500, 586, 608, 985, 992, 1000,
                               1023, 1024])
def test_slice_window_counts(orc, W):
    """Rows of 1..1024 windows: every padding pattern of the lane words (lane
    L owns windows L*ceil(W/32) + q)."""
    l, d = 8, 1
    s, _ = fmgen.generate_fm(3, W + l - 1, l, d, W)
    check(s, l, d, orc, launch=slice_launch(5), expect_slice=True)


def test_slice_long_rows_fall_back(orc):
    """W > 1024 is outside the slice family: a request for it runs the block
    family, with the same result."""
    s, _ = fmgen.generate_fm(2, 1100 + 7, 8, 1, 3)
    check(s, 8, 1, orc, launch=slice_launch(5), expect_slice=False)


def test_slice_dense_hits_queue_overflow(orc):
    """Small prefix, large d: most windows hit, the per-warp queues overflow
    and the per-lane resolution path runs (same updates)."""
    for (l, d, S, seed) in [(7, 1, 5, 1), (8, 2, 5, 2), (9, 3, 5, 3), (10, 4, 5, 4), (12, 5, 6, 5),
                            (11, 4, 6, 6)]:
        s = fmgen.random_sequences(4, 300, 400 + seed)
        check(s, l, d, orc, launch=slice_launch(S), expect_slice=True)


def test_slice_l16_and_prefix_lengths(orc):
    # every prefix length LP = l - S of both block sizes, d from 0 to LP - 1
    rng = random.Random(99)
    for S in (5, 6, 7):
        for l in range(S + 1, 17):
            d = rng.randint(0, l - S - 1)
            s = fmgen.random_sequences(3, 60, 1000 * S + l)
            lo = rng.randrange(0, 4 ** l - 50000) if l > 8 else 0
            hi = lo + 50000 if l > 8 else None
            check(s, l, d, orc, lo=lo, hi=hi, launch=slice_launch(S), expect_slice=True)


def test_slice_ineligible_d_and_auto(orc):
    """d >= l - S (every window a hit) runs the block family; AUTO picks the
    slice family exactly where it applies."""
    for (n, t, l, d) in [(3, 40, 7, 2), (3, 40, 7, 1), (4, 60, 9, 4), (4, 60, 9, 3),
                         (2, 30, 13, 7), (2, 30, 13, 6), (5, 80, 11, 2), (2, 30, 14, 6),
                         (2, 30, 14, 7), (3, 40, 15, 4)]:
        s = fmgen.random_sequences(n, t, l * 10 + d)
        S = 7 if l >= 13 else 5
        check(s, l, d, orc, expect_slice=applies(t, l, d, S))


def test_slice_no_skip_and_handoff(orc):
    s, _ = fmgen.generate_fm(12, 150, 10, 2, 7)
    want = orc.find(s, 10, 2).codes.tolist()
    for kw in [dict(no_skip=1), dict(handoff=0), dict(handoff=1), dict(handoff=5),
               dict(handoff=60), dict(handoff=5000)]:
        for S in (5, 6, 7):
            r = pms.find_ex(s, 10, 2, launch=slice_launch(S, **kw))
            assert r.status == 0 and r.stats.algo == pms.ALGO_SLICE
            assert r.codes.tolist() == want, (S, kw)
    full = pms.find_ex(s, 10, 2, launch=slice_launch(5, no_skip=1))
    assert full.stats.block_scans == (4 ** 10 // 1024) * 12  # every block, every sequence


def test_slice_launch_invariance_and_global_tables(orc):
    s, _ = fmgen.generate_fm(20, 600, 11, 3, 1)
    base = orc.find(s, 11, 3).codes.tolist()
    for S in (5, 6, 7):
        for kw in [dict(), dict(grid_ctas=1), dict(grid_ctas=5), dict(batch=4096),
                   dict(batch=12288), dict(table_global=1)]:
            r = pms.find_ex(s, 11, 3, launch=slice_launch(S, **kw))
            assert r.stats.algo == pms.ALGO_SLICE
            assert r.codes.tolist() == base, (S, kw)
            if kw.get("table_global"):
                assert r.stats.table_in_smem == 0
    # too many sequences for shared memory: planes and slots read through L1/L2
    s, _ = fmgen.generate_fm(120, 600, 9, 2, 5)
    r = check(s, 9, 2, orc, launch=slice_launch(), expect_slice=True)
    assert r.stats.table_in_smem == 0


def test_slice_invalid_bytes_truncation_and_plan(orc):
    s, _ = fmgen.generate_fm(6, 100, 9, 2, 11)
    bad = s.copy()
    bad[5, 99] = ord("N")
    r = pms.find_ex(bad, 9, 2, launch=slice_launch())
    assert r.status == pms.E_CHAR
    r = pms.find_ex(s, 9, 2, launch=slice_launch())  # a clean call after the bad one
    want = orc.find(s, 9, 2)
    assert r.status == 0 and r.codes.tolist() == want.codes.tolist()
    r = pms.find_ex(s, 9, 2, launch=slice_launch(), max_out=0)
    assert r.status == (pms.E_TRUNCATED if want.count else 0) and r.count == want.count
    lower = s | np.uint8(0x20)  # ASCII lower case
    assert pms.find_ex(lower, 9, 2, launch=slice_launch()).codes.tolist() == want.codes.tolist()


def test_slice_compaction_stress(orc):
    """(10,4) at n=20, t=600: ~1e6 motifs through the slice family's append."""
    s, _ = fmgen.generate_fm(20, 600, 10, 4, 1)
    # d = 4 < LP = 5 at S = 5: the slice family applies
    r = pms.find_ex(s, 10, 4, launch=slice_launch(5), max_out=1 << 21)
    want = orc.find(s, 10, 4)
    assert r.stats.algo == pms.ALGO_SLICE
    assert r.status == 0 and r.count == want.count
    assert r.codes.tolist() == want.codes.tolist()


# ------------------------------------------------- sequence-parallel mode

def test_seq_parallel_auto_for_few_blocks():
    """(9,2) has 256 blocks for 4,736 resident warps: AUTO runs every (block,
    sequence) pair in parallel (pms_stats.mode_flags bit 0); (15,4) does not."""
    g = json.load(open(os.path.join(GOLDEN, "bj0_seed1.json")))
    s, _ = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
    r = pms.find_ex(s, g["l"], g["d"], max_out=1 << 20)
    assert r.status == 0 and r.stats.algo == pms.ALGO_SLICE and r.stats.mode_flags & 1
    assert r.codes.tolist() == g["codes"]
    assert r.stats.block_scans <= 256 * 20  # dead blocks skip their remaining units
    r2 = pms.find_ex(s, g["l"], g["d"], launch=slice_launch(seq_parallel=-1), max_out=1 << 20)
    assert not (r2.stats.mode_flags & 1) and r2.codes.tolist() == g["codes"]
    s3, _ = fmgen.generate_fm(20, 600, 15, 4, 1)
    r3 = pms.find_ex(s3, 15, 4, lo=0, hi=1 << 24)
    assert not (r3.stats.mode_flags & 1)


@pytest.mark.parametrize("path", GOLDEN_FILES[:9], ids=[os.path.basename(p) for p in GOLDEN_FILES[:9]])
def test_seq_parallel_forced_against_golden(orc, path):
    g = json.load(open(path))
    s, _ = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
    for S in (5, 6):
        r = pms.find_ex(s, g["l"], g["d"], launch=slice_launch(S, seq_parallel=1), max_out=1 << 22)
        assert r.status == 0 and r.count == g["count"] and r.codes.tolist() == g["codes"]
        assert r.stats.mode_flags & 1


def test_seq_parallel_tiny_random_and_ranges(orc):
    rng = random.Random(909)
    for trial in range(60):
        S = rng.choice([5, 6])
        l = rng.randint(S + 1, 11)
        n = rng.randint(1, 8)
        t = rng.randint(l, 160)
        d = rng.randint(0, min(5, l - S - 1))
        s = fmgen.random_sequences(n, t, 81000 + trial)
        L = slice_launch(S, seq_parallel=1)
        check(s, l, d, orc, launch=L, expect_slice=True)
        lo = rng.randrange(0, 4 ** l)
        hi = min(4 ** l, lo + rng.choice([1, 7, 1023, 1025, 5000, 70000]))
        check(s, l, d, orc, lo=lo, hi=hi, launch=L)
    # planted (9,2) instances: the consensus is among the survivors
    for seed in range(4):
        s, rec = fmgen.generate_fm(12, 300, 9, 2, 60 + seed)
        got = check(s, 9, 2, orc, launch=slice_launch(5, seq_parallel=1), expect_slice=True)
        code = int("".join(str("ACGT".index(c)) for c in rec.consensus), 4)
        assert code in set(got.codes.tolist())


def test_overlap_prepass_plan_parity(orc):
    """pms_launch.overlap_prepass: no event between the pre-pass and the
    search (they overlap through the programmatic dependent launch); the set
    is unchanged and search_ms then covers both kernels."""
    import torch
    s, _ = fmgen.generate_fm(20, 600, 13, 3, 2)
    want = orc.find(s, 13, 3).codes.tolist()
    dev = torch.device("cuda", 0)
    seqs = torch.from_numpy(s).to(dev)
    out = torch.zeros(1 << 16, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    for ov in (0, 1):
        with pms.Plan(20, 600, 13, 3, pms.Launch(overlap_prepass=ov)) as plan:
            for _ in range(3):
                plan.execute_tensors(seqs, out, cnt)
                status, st = plan.wait()
                assert status == 0
                got = sorted(out[:int(cnt.item())].cpu().numpy().astype(np.uint32).tolist())
                assert got == want
                assert (st.pack_ms == 0.0) == bool(ov) and st.search_ms > 0.0


def test_slice_sparse_mode_dense_and_ranges(orc):
    """The sparse mode (packed-word instances, PMS_HANDOFF_TABLES=0, fresh
    process) on small random instances: dense hits, every block size, d from
    0 to LP - 1, unaligned ranges, thresholds 1..32 -- each set equal to the
    oracle's."""
    import subprocess
    import sys
    cases = []
    rng = random.Random(7)
    for S in (5, 6, 7):
        for l in (S + 2, S + 4, 16):
            d = rng.randint(0, l - S - 1)
            s = fmgen.random_sequences(5, 120, 77 * S + l)
            lo = rng.randrange(0, 4 ** l - 300000) if l > 9 else 0
            hi = lo + 300000 if l > 9 else 4 ** l
            want = orc.find(s, l, d, lo=lo, hi=hi).codes.tolist()
            cases.append((s.tolist(), l, d, S, lo, hi, want))
    code = f"""
import json, sys
import numpy as np
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import paper_1403_1313_b200 as pms
cases = json.loads(sys.stdin.read())
for s, l, d, S, lo, hi, want in cases:
    s = np.array(s, dtype=np.uint8)
    for h in (1, 3, 8, 32):
        r = pms.find_ex(s, l, d, lo=lo, hi=hi,
                        launch=pms.Launch(algo=pms.ALGO_SLICE, block_digits=S, handoff=h))
        assert r.status == 0 and r.stats.algo == pms.ALGO_SLICE, (l, d, S, h, r.status)
        assert (r.stats.mode_flags >> 1) & 1 == 0
        assert r.codes.tolist() == want, (l, d, S, h)
print("ok")
"""
    p = subprocess.run([sys.executable, "-c", code], input=json.dumps(cases),
                       env={**os.environ, "PMS_HANDOFF_TABLES": "0"},
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stderr[-2000:]


def test_plan_roofline_modes():
    """pms_plan_roofline: R_pass1 (mode 0), R_scan (mode 1),
    R_sparse (mode 2) and R_mix (mode 3) on the (15,4) headline instance after
    an execution;
    the prefix test alone is faster per window than the whole scan; the
    plan's next execution is unaffected; bad modes / unexecuted plans are
    PMS_E_ARG.  The sparse-mode counters are consistent: every step checks
    at least one candidate."""
    import torch
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bj3_seed1.json")))
    s_np, _ = fmgen.generate_fm(g["n"], g["t"], g["l"], g["d"], g["seed"])
    dev = torch.device("cuda", 0)
    s = torch.from_numpy(s_np).to(dev)
    out = torch.zeros(1 << 16, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    with pms.Plan(g["n"], g["t"], g["l"], g["d"]) as plan:
        with pytest.raises(pms.PmsError):
            plan.roofline(1, 4)  # not executed yet
        plan.execute_tensors(s, out, cnt)
        status, st = plan.wait()
        assert status == 0 and st.algo == pms.ALGO_SLICE
        W = g["t"] - g["l"] + 1
        checks = st.issued_compares // W - st.block_scans
        assert st.sparse_steps > 0 and checks >= st.sparse_steps
        r0, r1, r2, r3 = (plan.roofline(m, 16) for m in range(4))
        for r in (r0, r1, r2, r3):
            assert r["tests_per_s"] > 0 and r["scans_per_s"] > 0 and r["ms"] > 0
        assert r0["tests_per_s"] > r1["tests_per_s"]
        for bad in (-1, 4):
            with pytest.raises(pms.PmsError):
                plan.roofline(bad, 4)
        plan.execute_tensors(s, out, cnt)
        status, st2 = plan.wait()
        assert status == 0
        assert sorted(out[:int(cnt.item())].cpu().numpy().astype(np.uint32).tolist()) == g["codes"]
        assert (st2.block_scans, st2.sparse_steps) == (st.block_scans, st.sparse_steps)
