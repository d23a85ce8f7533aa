#!/usr/bin/env python
"""bench.py -- BASELINE.json metric on B200: candidate l-mers/s of the skip-BF
search at (15,4), n=20, t=600 (BASELINE.json configs[3]), with the executed
window-test rate, the kernel's roofline fraction, the end-to-end C-ABI number
and the CPU oracle baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--scaling weak|strong] [--all-configs]

A step = one pass of the whole hot path (device pre-pass + persistent search
over all 4^15 candidates + result compaction) on one FM instance already
resident in HBM (a1/a7 are in the e2e number).

* `--gpus N` (torchrun, one rank per GPU): `--scaling weak` (default) -- every
  rank solves its own instance (seed 1 + rank), no data-path collective;
  `--scaling strong` -- one instance, the candidate range split over the
  ranks (PAPER.md:75's contiguous partition at GPU granularity, shard.py) and
  the counts + codes all-gathered every step (the one exchange the path has).
* `--impl reference` times the CPU oracle (oracle/, the paper's static-
  partition threads) on the host cores over a bounded candidate sample.
* `--all-configs` measures every BASELINE.json config x seeds 1-3 (search
  time median/mean, candidates/s, executed tests/s, roofline fraction, SM
  clock, golden parity, naive/skip work ratio) and times the oracle on the
  host cores; one JSON document to --out (profiles/), not a bench line.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import fmgen  # noqa: E402

HEADLINE = 3  # BASELINE.json configs[3]: (15,4) n=20 t=600
METRIC = "candidate l-mers/s & window compares/s at (15,4) n=20 t=600; INT-pipe % roofline"
NCU_SUMMARY = os.path.join(ROOT, "profiles", "slice_kernel_ncu.json")  # committed capture


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload_name(ci: int, seed: int) -> str:
    """One string for both arms, so the driver sees the same config."""
    c = fmgen.BASELINE_CONFIGS[ci]
    return f"{c['name']} FM seed {seed} (BASELINE.json configs[{ci}])"


# --------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled in-process (NVML) every 5 ms
    during a region, plus one sample on entry and one on exit, so even a
    region of a few milliseconds carries its own clock record."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples: list[tuple[float, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._nv = None

    def _sample(self):
        nv = self._nv
        try:
            mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            rs = get(self._h)
        except Exception:  # pragma: no cover - driver without the query
            return
        self.samples.append((float(mhz), int(rs)))

    def _run(self):
        while not self._stop.wait(self.period):
            self._sample()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
            self._sample()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            log(f"clock sampler unavailable: {e}")
            self._nv = None
        return self

    def __exit__(self, *exc):
        if self._nv is not None:
            self._stop.set()
            self._t.join(timeout=1)
            self._sample()

    def summary(self) -> dict:
        sm = [m for m, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for bit, nm in self.REASONS.items() if r & bit})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm),
                "sm_mhz_min": min(sm) if sm else None, "source": "NVML, in-process, 5 ms"}


# --------------------------------------------------------------- helpers
def golden(ci: int, seed: int):
    p = os.path.join(ROOT, "tests", "golden", f"bj{ci}_seed{seed}.json")
    return json.load(open(p)) if os.path.exists(p) else None


def dist_setup(n_gpus: int):
    if n_gpus <= 1 and "RANK" not in os.environ:
        return 0, 1, 0
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", n_gpus))
    local = int(os.environ.get("LOCAL_RANK", rank))
    return rank, world, local


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def oracle_sample(l: int, d: int, seqs, seconds: float, lo_frac: float = 0.5):
    """A contiguous candidate range sized for about `seconds` of oracle work."""
    import oracle
    oracle.build()
    cores = oracle.default_threads()
    lo = int(4 ** l * lo_frac)
    n = 1 << 14
    oracle.find(seqs, l, d, lo=lo, hi=lo + n, threads=cores)  # warm-up / calibration
    t0 = time.perf_counter()
    oracle.find(seqs, l, d, lo=lo, hi=lo + n, threads=cores)
    dt = time.perf_counter() - t0
    n = int(min(4 ** l - lo, max(n, n * seconds / max(dt, 1e-4))))
    return lo, n, cores


def ncu_context():
    """The committed ncu capture of the default kernel (profiles/): warp
    instructions per block scan and DRAM bytes per launch."""
    if os.path.exists(NCU_SUMMARY):
        return json.load(open(NCU_SUMMARY))
    return None


# --------------------------------------------------------------- reference arm
def run_reference(args) -> int:
    rank, world, _ = dist_setup(args.gpus)
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    c = fmgen.BASELINE_CONFIGS[HEADLINE]
    l, d = c["l"], c["d"]
    seqs, _ = fmgen.generate_fm(c["n"], c["t"], l, d, args.seed)
    # each step a bounded sample: the whole warm-up + timed run takes about
    # --ref-seconds of CPU time whatever --steps is (minimum 2^14 codes a step)
    lo, n, cores = oracle_sample(l, d, seqs, args.ref_seconds / max(1, args.steps + args.warmup))
    times, work = [], 0
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = oracle.find(seqs, l, d, lo=lo, hi=lo + n, threads=cores)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            work += r.c_alg
    tot = sum(times)
    value = args.steps * n / tot
    sample = (f"codes [{lo}, {lo + n}) of 4^{l} (contiguous, from 4^{l}/2), "
              f"{args.steps} timed repetitions after {args.warmup} warm-up")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "candidates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": workload_name(HEADLINE, args.seed), "n": c["n"], "t": c["t"],
                   "l": l, "d": d, "seed": args.seed, "l2": "n/a (CPU oracle)"},
        "executed_window_compares_per_s": work / tot,
        "cpu_baseline": {"value": value, "unit": "candidates/s", "cores": cores,
                         "kind": "oracle", "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm
def roofline_object(pms, plan, st, search_ms: float, clk: dict, sms: int) -> dict:
    """Roofline of the timed kernel.

    The kernel's work per launch is two kinds of unit (PAPER.md:63's window
    test, done two ways): dense (block, sequence) scans -- W window tests
    against a block's shared prefix, hits resolved as Hamming balls -- and
    sparse-mode steps -- a short list of candidates each tested against W
    windows.  achieved = executed window tests (W per scan and per candidate
    check, pms_stats.issued_compares) / mean kernel event time.
    peak = R_mix (pms_plan_roofline mode 3): a microbenchmark of the kernel's
    own code for both units, interleaved at this launch's own ratio (sparse
    steps per scan, mean list size), on this instance's tables and hit mix,
    with the dynamic parts removed (work counter, skip rule, list
    extraction, output), every warp busy, all SMs, same run -- the north
    star's "microbenchmark of the same instruction mix".  frac = achieved /
    R_mix.  Also reported: R_scan and R_sparse (modes 1, 2: each unit alone),
    R_pass1 (mode 0, the prefix test alone) with frac_vs_pass1 = dense-scan
    tests / R_pass1, and the hardware issue roofline (ncu warp instructions of
    this launch / 4 warp-instructions/clk/SM x SMs x the sampled clock)."""
    W = plan.t - plan.l + 1
    t = search_ms * 1e-3
    tests = st.issued_compares
    obj = {"bound": "alu", "unit": "G window-tests/s", "achieved": tests / t / 1e9,
           "achieved_basis": "executed window tests per launch (W per dense (block, sequence) "
                             "scan + W per sparse-mode candidate check: pms_stats."
                             "issued_compares) / mean search-kernel event time",
           "block_scans": int(st.block_scans), "sparse_steps": int(st.sparse_steps),
           "candidate_checks": int(tests // W - st.block_scans)}
    try:
        r_mix = plan.roofline(3, 64)
        r_scan = plan.roofline(1, 64)
        r_pass1 = plan.roofline(0, 256)
        r_sparse = plan.roofline(2, 64) if st.sparse_steps else None
    except pms.PmsError as e:  # only the slice family has the microbenchmark
        obj.update(peak=None, frac=None, traffic=None, peak_basis=f"n/a ({e})")
        return obj
    t_sep = st.block_scans / r_scan["scans_per_s"] + \
        (st.sparse_steps / r_sparse["scans_per_s"] if r_sparse else 0.0)
    obj.update(peak=r_mix["tests_per_s"] / 1e9, frac=tests / t / r_mix["tests_per_s"],
               peak_basis="measured: pms_plan_roofline mode 3 (R_mix) -- this kernel's dense "
                          "scans with its sparse-mode steps interleaved at this launch's ratio "
                          "and list size, its own code on this instance's tables and hit mix, "
                          "no work counter / skip rule / list extraction / output, all SMs, "
                          "same run",
               r_scan=r_scan["tests_per_s"] / 1e9,
               r_sparse=r_sparse["tests_per_s"] / 1e9 if r_sparse else None,
               separate_units_us=t_sep * 1e6, kernel_us=t * 1e6,
               separate_units_note="scans / R_scan + steps / R_sparse: each unit measured "
                                   "alone; latency-bound sparse steps overlap dense scans of "
                                   "other warps in the kernel, so this can exceed R_mix's time",
               dense_share=st.block_scans / r_scan["scans_per_s"] / t,
               r_pass1=r_pass1["tests_per_s"] / 1e9,
               frac_vs_pass1=st.block_scans * W / t / r_pass1["tests_per_s"],
               r_pass1_basis="measured: pms_plan_roofline mode 0 -- the bit-sliced prefix "
                             "test alone (one-hot plane loads + carry-save classification); "
                             "frac_vs_pass1 = dense-scan window tests / time / R_pass1")
    ctx = ncu_context()
    cfg = (ctx or {}).get("config") or {}
    same = (cfg.get("n"), cfg.get("t"), cfg.get("l"), cfg.get("d"), cfg.get("block_digits")) == \
        (plan.n, plan.t, plan.l, plan.d, st.block_digits)
    if not same:  # the capture is of another workload: no per-launch numbers from it
        ctx = None
    obj["traffic"] = ctx.get("dram_bytes_per_launch") if ctx else None
    if ctx and ctx.get("warp_instructions_per_scan") and clk.get("sm_mhz"):
        instr = ctx["warp_instructions_per_scan"] * st.block_scans
        peak_issue = 4 * sms * clk["sm_mhz"] * 1e6
        obj["issue"] = {"warp_instructions_per_launch_est": instr,
                        "achieved_warp_inst_per_s": instr / (search_ms * 1e-3),
                        "peak_warp_inst_per_s": peak_issue,
                        "frac": instr / (search_ms * 1e-3) / peak_issue,
                        "basis": f"{ctx['warp_instructions_per_scan']:.1f} warp instructions "
                                 f"per block scan ({ctx['source']}) x this launch's scans / "
                                 f"kernel time / (4 x {sms} SMs x sampled SM clock)"}
    return obj


def run_gpu(args) -> int:
    import torch
    import paper_1403_1313_b200 as pms

    rank, world, local = dist_setup(args.gpus)
    dist = None
    one_gpu = os.environ.get("BENCH_ONE_GPU") == "1"
    if world > 1:
        import torch.distributed as dist
        # BENCH_ONE_GPU=1 (tests only): every rank on cuda:0 over gloo, so the
        # N > 1 code path can be exercised on a one-GPU box; the ranks' kernels
        # are independent (they never wait on one another), collectives go
        # through CPU tensors.  Its timings mean nothing.
        if one_gpu:
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    pms.build()
    pms.load()

    c = fmgen.BASELINE_CONFIGS[HEADLINE]
    n, t, l, d = c["n"], c["t"], c["l"], c["d"]
    strong = args.scaling == "strong"
    seed = args.seed if strong else args.seed + rank
    seqs_np, _ = fmgen.generate_fm(n, t, l, d, seed)
    seqs = torch.from_numpy(seqs_np).to(dev)
    cap = 1 << 20
    out = torch.zeros(cap, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.Stream(device=dev)
    algo = {"auto": pms.ALGO_AUTO, "candidate": pms.ALGO_CANDIDATE, "block": pms.ALGO_BLOCK,
            "slice": pms.ALGO_SLICE}[args.algo]
    launch = pms.Launch(algo=algo, block_digits=args.block_digits)
    # steps: no timing event between the pre-pass and the search kernel, so
    # the search (a programmatic dependent launch) overlaps the pre-pass's
    # tail; the kernel's own duration comes from a second timed region with
    # the boundary event (`plan`), right after
    step_plan = pms.Plan(n, t, l, d, pms.Launch(algo=algo, block_digits=args.block_digits,
                                                overlap_prepass=1))
    plan = pms.Plan(n, t, l, d, launch)
    total = 4 ** l
    from paper_1403_1313_b200.shard import shard_range
    lo, hi = shard_range(total, rank, world) if strong else (0, total)
    gcap = 64  # codes gathered per rank per step (a planted instance has ~1)
    cdev = torch.device("cpu") if one_gpu else dev  # where the collectives' tensors live
    gbuf = torch.zeros(gcap, dtype=torch.int64, device=dev)
    gcounts = [torch.zeros(1, dtype=torch.int64, device=cdev) for _ in range(world)]
    gcodes = [torch.zeros(gcap, dtype=torch.int64, device=cdev) for _ in range(world)]

    def step(ev_end=None, pl=step_plan):
        pl.execute_tensors(seqs, out, cnt, lo, hi, stream=stream)
        if strong and dist:  # the exchange step: every rank's count and codes
            dist.all_gather(gcounts, cnt.to(cdev))
            gbuf.copy_(out[:gcap].to(torch.int64))
            dist.all_gather(gcodes, gbuf.to(cdev))
        if ev_end is not None:  # end of the step's device work, before the host waits
            ev_end.record(stream)
        status, st = pl.wait()
        if status != 0:
            raise pms.PmsError(status, "step")
        return st

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
            step(pl=plan)
    torch.cuda.synchronize()

    # ---------------------------------------------------------- timed region
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    search_ms, last = [], None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.fill_(i & 0xFF)  # L2 flush between timed steps (not timed)
                evs[i][0].record(stream)
                step(evs[i][1])
        torch.cuda.synchronize()
        # the kernel's duration: the same K steps with the pre-pass/search event
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.fill_(i & 0xFF)
                last = step(pl=plan)
                search_ms.append(last.search_ms)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    tmax = sum(step_ms)
    if dist:
        x = torch.tensor([tmax], device=cdev, dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        tmax = float(x.item())
    nfound = int(cnt.item())
    codes = sorted(out[:nfound].cpu().numpy().astype(np.uint32).tolist())
    if strong and dist:  # the full set = union of the rank shards, in range order
        counts = [int(x.item()) for x in gcounts]
        codes = sorted(v for r, x in enumerate(gcodes) for v in
                       x[:min(counts[r], gcap)].cpu().numpy().tolist())
        nfound = sum(counts)
    g = golden(HEADLINE, seed)
    parity = None if g is None else (codes == g["codes"] and nfound == g["count"])
    # weak scaling: every rank checks its own instance against its golden set
    # (tests/golden holds (15,4) seeds 1-8); 1 / 0 / -1 = equal / differs / no golden
    parity_ranks = None
    if dist and not strong:
        pr = torch.zeros(world, dtype=torch.int64, device=cdev)
        pr[rank] = -1 if parity is None else int(parity)
        dist.all_reduce(pr)
        parity_ranks = [None if v < 0 else bool(v) for v in pr.cpu().tolist()]
    search_avg = float(np.mean(search_ms))
    cs = clk.summary()
    sms = pms.device_info()["sms"]
    roof = roofline_object(pms, plan, last, search_avg, cs, sms)

    # ------------------------------------------------ end to end (host buffers)
    e2e_ms = []
    for i in range(args.warmup + args.e2e_steps):
        t0 = time.perf_counter()
        r = pms.find_ex(seqs_np, l, d, lo=lo, hi=hi, launch=launch, max_out=cap, want_stats=False)
        dt = time.perf_counter() - t0
        assert r.status == 0
        if i >= args.warmup:
            e2e_ms.append(1e3 * dt)
    e2e_tot = float(sum(e2e_ms))
    if dist:
        x = torch.tensor([e2e_tot], device=cdev, dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        e2e_tot = float(x.item())

    # -------------------------- the per-candidate (north-star) kernel, same input
    cand = None
    if args.candidate_steps > 0 and world == 1:
        with pms.Plan(n, t, l, d, pms.Launch(algo=pms.ALGO_CANDIDATE)) as cplan:
            cms, cissued = [], 0
            with torch.cuda.stream(stream):
                for i in range(1 + args.candidate_steps):
                    cplan.execute_tensors(seqs, out, cnt, 0, total, stream=stream)
                    status, cst = cplan.wait()
                    assert status == 0
                    if i:
                        cms.append(cst.search_ms)
                        cissued += cst.issued_compares
            ccodes = sorted(out[:int(cnt.item())].cpu().numpy().astype(np.uint32).tolist())
        rm = pms.roofline(1 << 15)
        c_alg = g["c_alg"] if g else None
        cand = {"search_kernel_ms": float(np.mean(cms)), "steps": args.candidate_steps,
                "candidates_per_s": total / (np.mean(cms) * 1e-3),
                "same_motifs_as_headline": ccodes == codes,
                "roofline": {"bound": "alu", "unit": "G compares/s",
                             "peak": rm["compares_per_s"] / 1e9,
                             "peak_basis": "measured: pms_roofline (this kernel's per-compare "
                                           "loop, register-resident, no early exit, all SMs)",
                             "achieved": c_alg / (np.mean(cms) * 1e-3) / 1e9 if c_alg else None,
                             "frac": c_alg / (np.mean(cms) * 1e-3) / rm["compares_per_s"]
                             if c_alg else None,
                             "issued_frac": cissued / args.candidate_steps /
                             (np.mean(cms) * 1e-3) / rm["compares_per_s"],
                             "achieved_basis": "oracle C_alg / mean search-kernel event time"}}

    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return 0

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle
        lo_s, ns, cores = oracle_sample(l, d, seqs_np, args.cpu_seconds)
        t0 = time.perf_counter()
        rr = oracle.find(seqs_np, l, d, lo=lo_s, hi=lo_s + ns, threads=cores)
        dt = time.perf_counter() - t0
        cpu = {"value": ns / dt, "unit": "candidates/s", "cores": cores, "kind": "oracle",
               "sample": f"codes [{lo_s}, {lo_s + ns}) of 4^{l} (contiguous from 4^{l}/2), "
                         "one run after a calibration run",
               "cpu_model": cpu_model(),
               "executed_window_compares_per_s": rr.c_alg / dt}

    per = 1 if strong else world
    c_alg = g["c_alg"] if g else None
    line = {
        "metric": METRIC,
        "value": per * args.steps * total / (tmax * 1e-3), "unit": "candidates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tmax / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": workload_name(HEADLINE, args.seed), "n": n, "t": t, "l": l, "d": d,
                   "seeds": [args.seed] if strong else [args.seed + r for r in range(world)],
                   "sharding": ("candidate-code range split over ranks (shard_range), counts + "
                                "codes all_gather every step" if strong else
                                "one independent instance per rank, no collective"),
                   "l2": "flushed between timed steps (256 MiB write, untimed)",
                   "algo": {1: "candidate", 2: "block", 3: "slice"}.get(last.algo, str(last.algo)),
                   "kernel": {"grid": last.grid, "block": last.block,
                              "block_digits": last.block_digits,
                              "windows_per_lane": last.windows_per_lane,
                              "table_in_smem": last.table_in_smem,
                              "smem_bytes": last.smem_bytes}},
        "executed_window_tests_per_s": last.issued_compares / (search_avg * 1e-3),
        "skipbf_equivalent_compares_per_s": (per * c_alg / (tmax * 1e-3 / args.steps))
        if c_alg else None,
        "skipbf_equivalent_basis": "oracle C_alg (the candidate-window compares a first-match "
                                   "skip-BF does, tests/golden) per step / device time per step; "
                                   "NOT work the GPU performs -- one block-family test serves "
                                   "up to 4^S candidates",
        "search_kernel_ms": search_avg, "pack_kernel_ms": float(last.pack_ms),
        "kernel_timing": "steps (value): pre-pass and search overlapped (no event between, "
                         "pms_launch.overlap_prepass); search_kernel_ms / roofline: the same K "
                         "steps again with the pre-pass/search event, same input, L2 flushed",
        "block_scans_per_launch": int(last.block_scans),
        "motifs": nfound, "parity_vs_golden": parity,
        **({"parity_vs_golden_ranks": parity_ranks} if parity_ranks is not None else {}),
        "roofline": roof,
        "candidate_kernel": cand,
        "cpu_baseline": cpu,
        "e2e": {"value": per * args.e2e_steps * total / (e2e_tot * 1e-3),
                "unit": "candidates/s", "h2d_bytes_per_step": n * t,
                # one copy of the result block's 128-B head (state + count) and the
                # first min(cap, 1024) codes (include/pms.h: one round trip for
                # small sets), + the codes again when the set is larger than that
                "d2h_bytes_per_step": 128 + 4 * min(cap, 1024) + (4 * nfound if nfound > 1024 else 0),
                "path": "pms_find_ex from host buffers (pooled context, H2D, kernels, D2H, sort)"},
        # pre-pass + search per step per rank (the untimed L2 flush is torch's fill)
        "gpu_launches": 2 * args.steps * world,
        "clocks": cs,
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- all configs
def run_all_configs(args) -> int:
    """Every BASELINE.json config x seeds 1-3 on one GPU, plus the oracle on
    the host cores (full runs for configs 0-2, stated subranges for 3-4)."""
    import torch
    import oracle
    import paper_1403_1313_b200 as pms
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    pms.build()
    pms.load()
    oracle.build()
    sms = pms.device_info()["sms"]
    out = torch.zeros(1 << 21, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    rows = []
    for ci, c in enumerate(fmgen.BASELINE_CONFIGS):
        n, t, l, d = c["n"], c["t"], c["l"], c["d"]
        for seed in (1, 2, 3):
            s_np, _ = fmgen.generate_fm(n, t, l, d, seed)
            s = torch.from_numpy(s_np).to(dev)
            g = golden(ci, seed)
            plan = pms.Plan(n, t, l, d)
            ms, issued = [], []
            with ClockSampler(dev.index) as clk, torch.cuda.stream(stream):
                for r in range(args.warmup + args.reps):
                    plan.execute_tensors(s, out, cnt, stream=stream)
                    status, st = plan.wait()
                    assert status == 0
                    if r >= args.warmup:
                        ms.append(st.search_ms)
                        issued.append(st.issued_compares)
            codes = sorted(out[:int(cnt.item())].cpu().numpy().astype(np.uint32).tolist())
            med = float(np.median(ms))
            cs = clk.summary()
            roof = roofline_object(pms, plan, st, float(np.mean(ms)), cs, sms)
            plan.close()
            # f3: the same family without the skip rule (every block scans all n sequences)
            with pms.Plan(n, t, l, d, pms.Launch(algo=st.algo, block_digits=st.block_digits,
                                                 no_skip=1)) as nplan:
                with torch.cuda.stream(stream):
                    nplan.execute_tensors(s, out, cnt, stream=stream)
                    status, nst = nplan.wait()
                ncodes = sorted(out[:int(cnt.item())].cpu().numpy().astype(np.uint32).tolist())
            row = {"config": ci, "workload": workload_name(ci, seed), "seed": seed,
                   "algo": st.algo, "block_digits": st.block_digits,
                   "search_ms_median": med, "search_ms_mean": float(np.mean(ms)),
                   "reps": args.reps, "pack_ms_last": st.pack_ms,
                   "candidates_per_s": 4 ** l / (med * 1e-3),
                   "executed_tests_per_s": float(np.mean(issued)) / (med * 1e-3),
                   "block_scans": st.block_scans,
                   "roofline_frac": roof.get("frac"), "r_mix_gtests": roof.get("peak"),
                   "r_scan_gtests": roof.get("r_scan"), "r_sparse_gtests": roof.get("r_sparse"),
                   "sparse_steps": st.sparse_steps, "dense_share": roof.get("dense_share"),
                   "frac_vs_pass1": roof.get("frac_vs_pass1"),
                   "issue_frac": roof.get("issue", {}).get("frac"),
                   "sm_mhz": cs["sm_mhz"], "clock_samples": cs["samples"],
                   "throttle": cs["reasons"],
                   "motifs": len(codes),
                   "parity_vs_golden": (codes == g["codes"]) if g else None,
                   "no_skip_parity": ncodes == codes,
                   "issued_tests_skip": st.issued_compares,
                   "issued_tests_no_skip": nst.issued_compares,
                   "naive_over_skip_issued": nst.issued_compares / max(1, st.issued_compares),
                   "naive_bf_compares": 4 ** l * n * (t - l + 1),
                   "skipbf_c_alg": g["c_alg"] if g else None,
                   "naive_bf_over_c_alg": (4 ** l * n * (t - l + 1) / g["c_alg"]) if g else None}
            rows.append(row)
            log(f"{row['workload']}: {med*1e3:.1f} us, {row['candidates_per_s']:.3e} cand/s, "
                f"frac {row['roofline_frac']}, parity {row['parity_vs_golden']}")
    # the oracle on the host cores: median/mean of >= 3 runs after a warm-up
    cores = oracle.default_threads()
    orc = []
    for ci, c in enumerate(fmgen.BASELINE_CONFIGS):
        n, t, l, d = c["n"], c["t"], c["l"], c["d"]
        s_np, _ = fmgen.generate_fm(n, t, l, d, 1)
        if ci <= 2:
            lo, hi, what = 0, 4 ** l, "full 4^l"
        else:
            lo = 4 ** l // 2
            hi = lo + (1 << 22 if ci == 3 else 1 << 20)
            what = f"codes [{lo}, {hi}) (contiguous from 4^l/2)"
        oracle.find(s_np, l, d, lo=lo, hi=hi, threads=cores)  # warm-up
        ts, work = [], 0
        for _ in range(args.oracle_reps):
            t0 = time.perf_counter()
            r = oracle.find(s_np, l, d, lo=lo, hi=hi, threads=cores)
            ts.append(time.perf_counter() - t0)
            work = r.c_alg
        orc.append({"config": ci, "workload": workload_name(ci, 1), "range": what,
                    "candidates": hi - lo, "seconds_median": float(np.median(ts)),
                    "seconds_mean": float(np.mean(ts)), "reps": args.oracle_reps,
                    "candidates_per_s": (hi - lo) / float(np.median(ts)),
                    "window_compares_per_s": work / float(np.median(ts)), "motifs": r.count})
        log(f"oracle {what} {c['name']}: {np.median(ts):.2f} s")
    doc = {"gpu": torch.cuda.get_device_name(0), "sms": sms, "rows": rows,
           "oracle": {"cores": cores, "cpu_model": cpu_model(), "rows": orc},
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    text = json.dumps(doc, indent=1)
    if args.out:
        with open(args.out, "w") as f:
            f.write(text + "\n")
    print(json.dumps({"all_configs": len(rows), "out": args.out}), flush=True)
    return 0


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)  # ~0.22 s timed
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--algo", choices=["auto", "candidate", "block", "slice"], default="auto")
    ap.add_argument("--block-digits", type=int, default=0,
                    help="pms_launch.block_digits (0 = automatic)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: an instance per rank; strong: one instance sharded by candidate range")
    ap.add_argument("--candidate-steps", type=int, default=3,
                    help="also time the per-candidate kernel for this many steps")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0)  # whole --impl reference run
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--all-configs", action="store_true")
    ap.add_argument("--reps", type=int, default=9, help="--all-configs timed repetitions")
    ap.add_argument("--oracle-reps", type=int, default=3, help="--all-configs oracle runs")
    ap.add_argument("--out", default="", help="--all-configs output file")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: the contract asks for >= 3 warm-up steps")
    if args.impl == "reference":
        return run_reference(args)
    if args.all_configs:
        return run_all_configs(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
