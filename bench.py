#!/usr/bin/env python
"""bench.py -- BASELINE.json metric on B200: candidate l-mers/s and window
compares/s of the skip-BF search at (15,4), n=20, t=600, plus the integer-pipe
roofline fraction, the end-to-end C-ABI number and the CPU oracle baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

A step = one pass of the whole hot path (device pre-pass + persistent search
over all 4^15 candidates + result compaction) on one FM instance already
resident in HBM.  With --gpus N (torchrun, one rank per GPU) every rank solves
its own independent instance (seed 1 + rank): weak scaling, no data-path
collective.  `--impl reference` times the CPU oracle (oracle/, the paper's
static-partition threads) on the host cores over a bounded candidate sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import fmgen  # noqa: E402

WORKLOAD = fmgen.BASELINE_CONFIGS[3]  # (15,4) n=20 t=600 -- BASELINE.json configs[3]
METRIC = "candidate l-mers/s & window compares/s at (15,4) n=20 t=600; INT-pipe % roofline"
POPC_PER_CLK_SM = 16  # POPC issue rate per SM per clock (B200; measured ~15 by the probe)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during a region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        loaded = [x for x in sm if x > 0.5 * mx] if mx else sm
        med = float(np.median(loaded)) if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- helpers
def golden_c_alg(seed: int):
    p = os.path.join(ROOT, "tests", "golden", f"bj3_seed{seed}.json")
    if os.path.exists(p):
        g = json.load(open(p))
        return g["c_alg"], g["codes"]
    return None, None


def dist_setup(n_gpus: int):
    if n_gpus <= 1 and "RANK" not in os.environ:
        return 0, 1, 0
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", n_gpus))
    local = int(os.environ.get("LOCAL_RANK", rank))
    return rank, world, local


def oracle_sample(l: int, d: int, seqs, seconds: float, lo_frac: float = 0.5):
    """Time the CPU oracle over a contiguous candidate range sized for ~seconds."""
    import oracle
    oracle.build()
    cores = oracle.default_threads()
    lo = int(4 ** l * lo_frac)
    n = 1 << 14
    r = oracle.find(seqs, l, d, lo=lo, hi=lo + n, threads=cores)  # calibration
    t0 = time.perf_counter()
    r = oracle.find(seqs, l, d, lo=lo, hi=lo + n, threads=cores)
    dt = time.perf_counter() - t0
    n = int(min(4 ** l - lo, max(n, n * seconds / max(dt, 1e-4))))
    return lo, n, cores


def run_reference(args) -> int:
    rank, world, _ = dist_setup(args.gpus)
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    l, d = WORKLOAD["l"], WORKLOAD["d"]
    seqs, _ = fmgen.generate_fm(WORKLOAD["n"], WORKLOAD["t"], l, d, args.seed)
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
        "vs_baseline": None, "dtype": "u8 chars (oracle)", "data": "synthetic",
        "config": {"workload": WORKLOAD["name"] + f" FM seed {args.seed}", "n": WORKLOAD["n"],
                   "t": WORKLOAD["t"], "l": l, "d": d, "seed": args.seed,
                   "l2": "n/a (CPU oracle)"},
        "window_compares_per_s": work / tot,
        "cpu_baseline": {"value": value, "unit": "candidates/s", "cores": cores,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "candidates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm
def run_gpu(args) -> int:
    import torch
    import paper_1403_1313_b200 as pms

    rank, world, local = dist_setup(args.gpus)
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    pms.build()
    pms.load()

    n, t, l, d = WORKLOAD["n"], WORKLOAD["t"], WORKLOAD["l"], WORKLOAD["d"]
    strong = args.scaling == "strong"
    # weak: one independent instance per rank; strong: one instance, the candidate
    # range split over the ranks (shard.shard_range) and gathered every step
    seed = args.seed if strong else args.seed + rank
    seqs_np, rec = fmgen.generate_fm(n, t, l, d, seed)
    seqs = torch.from_numpy(seqs_np).to(dev)
    cap = 1 << 20
    out = torch.zeros(cap, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.Stream(device=dev)
    algo = {"auto": pms.ALGO_AUTO, "candidate": pms.ALGO_CANDIDATE, "block": pms.ALGO_BLOCK,
            "slice": pms.ALGO_SLICE}[args.algo]
    plan = pms.Plan(n, t, l, d, pms.Launch(algo=algo, block_digits=args.block_digits))
    total = 4 ** l
    from paper_1403_1313_b200.shard import shard_range
    lo, hi = shard_range(total, rank, world) if strong else (0, total)
    gbuf = torch.zeros(64, dtype=torch.int64, device=dev)

    def step(ev_end=None):
        plan.execute_tensors(seqs, out, cnt, lo, hi, stream=stream)
        if strong and dist:  # the exchange step: gather every rank's count and codes
            cl = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
            dist.all_gather(cl, cnt)
            gbuf[:] = -1
            gbuf[:64].copy_(out[:64].to(torch.int64))
            gl = [torch.zeros(64, dtype=torch.int64, device=dev) for _ in range(world)]
            dist.all_gather(gl, gbuf)
        if ev_end is not None:  # end of the step's device work, before the host waits
            ev_end.record(stream)
        status, st = plan.wait()
        if status != 0:
            raise pms.PmsError(status, "step")
        return st

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()

    # ---------------------------------------------------------- timed region
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    search_ms, issued, last = [], 0, None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.fill_(i & 0xFF)  # L2 flush between timed steps (not timed)
                evs[i][0].record(stream)
                last = step(evs[i][1])
                search_ms.append(last.search_ms)
                issued += last.issued_compares
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    mine = sum(step_ms)
    tmax = mine
    if dist:
        x = torch.tensor([mine], device=dev, dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        tmax = float(x.item())
    nfound = int(cnt.item())
    codes = sorted(out[:nfound].cpu().numpy().astype(np.uint32).tolist())
    if strong and dist:  # the full set = union of the rank shards (in range order)
        from paper_1403_1313_b200.shard import gather_codes
        codes = sorted(gather_codes(np.asarray(codes, dtype=np.uint32), device=dev).tolist())
        nfound = len(codes)
    c_alg, gold = golden_c_alg(seed)
    parity = None if gold is None else (codes == gold)

    # ------------------------------------------------ end to end (host buffers)
    e2e_ms = []
    for i in range(args.warmup + args.e2e_steps):
        t0 = time.perf_counter()
        r = pms.find_ex(seqs_np, l, d, lo=lo, hi=hi, launch=pms.Launch(algo=algo), max_out=cap,
                        want_stats=False)
        dt = time.perf_counter() - t0
        assert r.status == 0
        if i >= args.warmup:
            e2e_ms.append(1e3 * dt)
    e2e_tot = float(sum(e2e_ms))
    if dist:
        x = torch.tensor([e2e_tot], device=dev, dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        e2e_tot = float(x.item())

    # ---------------------------- the per-candidate (north-star) kernel, same input
    cand = None
    if args.algo != "candidate" and args.candidate_steps > 0:
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
        cand = {"search_kernel_ms": float(np.mean(cms)), "steps": args.candidate_steps,
                "candidates_per_s": total / (np.mean(cms) * 1e-3),
                "issued_compares_per_s": cissued / args.candidate_steps / (np.mean(cms) * 1e-3),
                "same_motifs_as_headline": ccodes == codes,
                "kernel": {"grid": cst.grid, "block": cst.block, "lanes_per_cand": cst.lanes_per_cand,
                           "windows_per_lane": cst.windows_per_lane}}

    # ------------- block-family R_mix: the same kernel and mix without early exits
    rmix_block = None
    if last.algo == pms.ALGO_BLOCK and args.rmix_steps > 0:
        with pms.Plan(n, t, l, d, pms.Launch(algo=pms.ALGO_BLOCK, no_skip=1,
                                             block_digits=last.block_digits)) as rplan:
            rms, rissued = [], 0
            with torch.cuda.stream(stream):
                for i in range(1 + args.rmix_steps):
                    rplan.execute_tensors(seqs, out, cnt, 0, total, stream=stream)
                    status, rst = rplan.wait()
                    assert status == 0
                    if i:
                        rms.append(rst.search_ms)
                        rissued += rst.issued_compares
        rmix_block = {"window_tests_per_s": rissued / args.rmix_steps / (np.mean(rms) * 1e-3),
                      "search_kernel_ms": float(np.mean(rms)),
                      "basis": "block kernel with the skip rule off (pms_launch.no_skip): every "
                               "block scans all n sequences -- the same scan + hit-resolution "
                               "instruction mix with no early exit, all SMs"}

    # ------------------------------------------------ roofline microbenchmark
    with ClockSampler(dev.index) as clk_rm:
        rm = pms.roofline(1 << 15)
    cs = clk.summary()
    if dist:
        dist.destroy_process_group()
    if rank != 0:
        return 0

    search_avg = float(np.mean(search_ms))
    cands_per_s = (1 if strong else world) * args.steps * total / (tmax * 1e-3)
    sm_mhz = cs["sm_mhz"] or 1965.0
    sms = pms.device_info()["sms"]
    peak_popc = POPC_PER_CLK_SM * sms * sm_mhz * 1e6
    issued_per_launch = issued / args.steps
    issued_rate = issued_per_launch / (search_avg * 1e-3)
    block_family = last.algo == pms.ALGO_BLOCK
    traffic = None
    tp = os.path.join(ROOT, "profiles",
                      "block_kernel_traffic.json" if block_family else "search_kernel_traffic.json")
    ncu_ctx = None
    if os.path.exists(tp):
        tj = json.load(open(tp))
        traffic = tj.get("dram_bytes_per_launch")
        if "issue_slots_busy_pct" in tj:  # committed ncu capture of the same kernel (context)
            ncu_ctx = {k: tj[k] for k in ("issue_slots_busy_pct", "alu_pipe_pct", "xu_pipe_pct",
                                          "lsu_pipe_pct", "warp_instructions_per_launch",
                                          "source") if k in tj}
    if block_family:
        # one POPC per window test; a block-family test resolves up to 1024 candidates
        achieved = issued_rate
        basis = ("window tests the block kernel executes per launch (W per (block, sequence) "
                 "scan + W per single-candidate sequence scan; each one XOR/fold/POPC) / mean "
                 "search-kernel event time")
    else:
        achieved = (c_alg / (search_avg * 1e-3)) if c_alg else None
        basis = ("oracle C_alg (first-match window compares) of this instance / mean "
                 "search-kernel event time")
    if rmix_block:
        r_mix = rmix_block["window_tests_per_s"]
        r_mix_basis = ("measured: " + rmix_block["basis"])
    else:
        r_mix = rm["compares_per_s"]
        r_mix_basis = ("measured: pms_roofline, the candidate kernel's per-compare loop "
                       "(register-resident, no early exit, all SMs)")
    if cand is not None:
        cand["roofline"] = {
            "bound": "alu", "unit": "Gcompares/s", "peak": rm["compares_per_s"] / 1e9,
            "peak_basis": "measured: pms_roofline (this kernel's per-compare loop, no early exit)",
            "achieved": (c_alg / (cand["search_kernel_ms"] * 1e-3)) / 1e9 if c_alg else None,
            "frac": (c_alg / (cand["search_kernel_ms"] * 1e-3)) / rm["compares_per_s"]
            if c_alg else None,
            "frac_of_popc_peak": (c_alg / (cand["search_kernel_ms"] * 1e-3)) / peak_popc
            if c_alg else None,
            "issued_frac_of_r_mix": cand["issued_compares_per_s"] / rm["compares_per_s"],
            "achieved_basis": "oracle C_alg / mean search-kernel event time"}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        import oracle
        lo, ns, cores = oracle_sample(l, d, seqs_np, args.cpu_seconds)
        t0 = time.perf_counter()
        rr = oracle.find(seqs_np, l, d, lo=lo, hi=lo + ns, threads=cores)
        dt = time.perf_counter() - t0
        cpu = {"value": ns / dt, "unit": "candidates/s", "cores": cores, "kind": "oracle",
               "sample": f"codes [{lo}, {lo + ns}) of 4^{l} (contiguous from 4^{l}/2), one run",
               "window_compares_per_s": rr.c_alg / dt}

    line = {
        "metric": METRIC, "value": cands_per_s, "unit": "candidates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmax / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOAD["name"] + " FM (BASELINE.json configs[3])",
                   "n": n, "t": t, "l": l, "d": d,
                   "seeds": [args.seed] if strong else [args.seed + r for r in range(world)],
                   "sharding": ("candidate-code range split over ranks, counts+codes "
                                "all_gather per step" if strong else
                                "one independent instance per rank, no collective"),
                   "l2": "flushed between timed steps (256 MiB write, untimed)",
                   "algo": {1: "candidate", 2: "block"}.get(last.algo, str(last.algo)),
                   "kernel": {"grid": last.grid, "block": last.block,
                              "lanes_per_cand": last.lanes_per_cand,
                              "windows_per_lane": last.windows_per_lane,
                              "table_in_smem": last.table_in_smem,
                              "smem_bytes": last.smem_bytes}},
        "window_compares_per_s": ((1 if strong else world) * c_alg / (tmax * 1e-3 / args.steps))
        if c_alg else None,
        "window_compares_basis": "oracle C_alg (candidate-window tests of skip-BF with "
                                 "first-match stop) per step / device time per step",
        "issued_window_tests_per_s": issued_rate,
        "search_kernel_ms": search_avg, "pack_kernel_ms": float(last.pack_ms),
        "block_scans_per_launch": int(last.block_scans),
        "motifs": nfound, "parity_vs_golden": parity,
        "roofline": {"bound": "alu", "unit": "G window-tests/s",
                     "achieved": achieved / 1e9 if achieved else None,
                     "peak": r_mix / 1e9,
                     "frac": (achieved / r_mix) if achieved else None,
                     "traffic": traffic,
                     "peak_basis": r_mix_basis,
                     "achieved_basis": basis,
                     "popc_peak": peak_popc / 1e9,
                     "frac_of_popc_peak": (achieved / peak_popc) if achieved else None,
                     "popc_peak_basis": f"POPC {POPC_PER_CLK_SM}/clk/SM x {sms} SMs x "
                                        f"{sm_mhz:.0f} MHz (median SM clock in the timed "
                                        "region); one POPC per window test",
                     "ncu_capture": ncu_ctx,
                     "r_mix_kernel_ms": rmix_block["search_kernel_ms"] if rmix_block else None,
                     "r_mix_candidate_loop": rm["compares_per_s"] / 1e9,
                     "r_mix_clocks": clk_rm.summary()},
        "candidate_kernel": cand,
        "cpu_baseline": cpu,
        "e2e": {"value": (1 if strong else world) * args.e2e_steps * total / (e2e_tot * 1e-3),
                "unit": "candidates/s", "h2d_bytes_per_step": n * t,
                # one copy of the result block's 128-B head (state + count) and the
                # first min(cap, 1024) codes (include/pms.h: one round trip for
                # small sets), + the codes again when the set is larger than that
                "d2h_bytes_per_step": 128 + 4 * min(cap, 1024) + (4 * nfound if nfound > 1024 else 0),
                "path": "pms_find_ex from host buffers (pooled context, H2D, kernels, D2H, sort)"},
        "gpu_launches": 2 * args.steps,
        "clocks": cs,
    }
    print(json.dumps(line), flush=True)
    return 0


def main() -> int:
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)  # ~0.45 s timed: ~20 clock samples
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
    ap.add_argument("--rmix-steps", type=int, default=3,
                    help="steps of the block kernel without early exit (block-family R_mix)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-seconds", type=float, default=60.0)  # whole --impl reference run
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warning: the contract asks for >= 3 warm-up steps")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
