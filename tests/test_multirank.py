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
