"""World-size-2 gloo tests (CPU) of the multi-rank host logic: the
candidate-range shard split, the final gather, and max-over-ranks timing.
The per-rank search here is the oracle (no GPU in this container); on GPUs
the same code calls the CUDA path."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import fmgen
from paper_1403_1313_b200.shard import shard_range


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank: int, world: int, port: int, q):
    import torch.distributed as dist

    import oracle
    from paper_1403_1313_b200.shard import find_sharded, max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, rec = fmgen.generate_fm(6, 80, 7, 1, 11)
        got = find_sharded(s, 7, 1, search=lambda x, l, d, lo, hi:
                           oracle.find(x, l, d, lo=lo, hi=hi, threads=1).codes)
        t = max_over_ranks(float(rank + 1))
        q.put((rank, got.tolist(), t))
    finally:
        dist.destroy_process_group()


def test_shard_range_partition():
    for total in (0, 1, 7, 64, 4 ** 11, 4 ** 16):
        for world in (1, 2, 3, 8, 64):
            r = [shard_range(total, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == total
            assert all(r[i][1] == r[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
    assert [b - a for a, b in (shard_range(64, k, 5) for k in range(5))] == [13, 13, 13, 13, 12]
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_gloo_world2_sharded_search_and_gather(orc):
    orc.build()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s, _ = fmgen.generate_fm(6, 80, 7, 1, 11)
    want = orc.find(s, 7, 1).codes.tolist()
    for rank, got, t in res:
        assert got == want
        assert t == 2.0


def _gpu_worker(rank: int, world: int, port: int, q, cases):
    """One rank of a gloo group on cuda:0: find_sharded with its default
    search, i.e. the CUDA path (pms.find / pms.find64) on this rank's shard."""
    import torch
    import torch.distributed as dist

    from paper_1403_1313_b200.shard import find_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for (n, t, l, d, seed) in cases:
            s, _ = fmgen.generate_fm(n, t, l, d, seed)
            out.append(find_sharded(s, l, d).tolist())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_cuda_path_against_golden(orc, world):
    """the candidate range split over ranks (PAPER.md:75's
    contiguous partition), each rank's shard searched by the CUDA kernels, one
    gather; the union equals the oracle's golden set (bj2 = (13,3), bj3 =
    (15,4), seed 1) and an l = 17 case exercises the 64-bit path.  All ranks
    share cuda:0 (one GPU on this pool); their kernels never wait on each
    other, so this is a correctness test of the sharded path, not a timing."""
    import json
    gold = [json.load(open(os.path.join(os.path.dirname(__file__), "golden", f)))
            for f in ("bj2_seed1.json", "bj3_seed1.json")]
    cases = [(g["n"], g["t"], g["l"], g["d"], g["seed"]) for g in gold] + [(6, 60, 17, 4, 3)]
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, cases)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    s17, rec = fmgen.generate_fm(6, 60, 17, 4, 3)
    cons = int("".join(str("ACGT".index(c)) for c in rec.consensus), 4)
    for _, got in res:
        assert got[0] == gold[0]["codes"] and got[1] == gold[1]["codes"]
        assert cons in got[2]
        for c in got[2][:50]:
            assert orc.verify_motif(s17, 17, 4, c)
        # range additivity: the shard union over a window around the plant
        near = orc.find64(s17, 17, 4, lo=max(0, cons - 50000), hi=cons + 50000).codes.tolist()
        assert [c for c in got[2] if cons - 50000 <= c < cons + 50000] == near


@pytest.mark.gpu
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_two_ranks_one_gpu(scaling):
    """`bench.py --gpus 2` launched as the driver launches it (torch.distributed.run,
    one process per rank), with BENCH_ONE_GPU=1: both ranks on cuda:0 over gloo
    (this pool has one GPU; the ranks' kernels never wait on one another).
    Checks the N > 1 line: whole-job value over both ranks, the seeds, and
    parity -- weak: every rank's own instance against its golden set; strong:
    the gathered union of the two range shards."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "5", "--warmup", "3",
           "--e2e-steps", "2", "--scaling", scaling]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["steps"] == 5 and line["scaling"] == scaling
    assert line["parity_vs_golden"] is True
    assert line["value"] > 0 and line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
    if scaling == "weak":
        assert line["config"]["seeds"] == [1, 2]
        assert line["parity_vs_golden_ranks"] == [True, True]
        # two instances per step: the whole-job value counts both
        assert abs(line["value"] - 2 * 4 ** 15 / (line["ms_per_step"] * 1e-3)) < 1e-3 * line["value"]
    else:
        assert line["config"]["seeds"] == [1]
