"""Multi-GPU candidate-range sharding: one process per GPU.

The candidate codes [0, 4^l) split into contiguous per-rank ranges with the
paper's floor/remainder rule (section IV.A: each worker gets "the
first and the last l-mer").  Each rank searches its range on
its own GPU with no exchange during the search (range additivity); one
gather at the end (counts, then codes) concatenates the per-rank results in
rank order, which is already ascending.  The bytes moved are a few codes per
rank, so this is a plain torch.distributed all_gather (NCCL on GPUs, gloo in
the CPU tests); nothing here overlaps with compute because nothing needs to.
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of `rank` among `world` contiguous near-equal ranges of [0, total)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_codes(local: np.ndarray, device=None, group=None) -> np.ndarray:
    """All-gather variable-length code arrays (uint64 end to end: l <= 31
    codes need 62 bits); concatenated in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = device if device is not None else torch.device("cpu")
    n = torch.tensor([int(local.size)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(max(sizes), 1)
    buf = torch.zeros(cap, dtype=torch.int64, device=dev)  # codes < 2^62 fit int64
    if local.size:
        buf[:local.size] = torch.from_numpy(local.astype(np.int64)).to(dev)
    parts = [torch.zeros(cap, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return np.concatenate([p[:s].cpu().numpy() for p, s in zip(parts, sizes)]).astype(np.uint64)


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Device-timed numbers are reported as the max over ranks."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device=device if device is not None else torch.device("cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def find_sharded(seqs, l: int, d: int, group=None,
                 search: Callable | None = None) -> np.ndarray:
    """Every rank searches its shard of [0, 4^l) and all ranks return the full
    ascending motif set (uint64 codes).  `search(seqs, l, d, lo, hi) -> codes`
    defaults to the CUDA path on this rank's current device: pms.find (uint32
    codes) for l <= 16, pms.find64 for 17 <= l <= 31."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(4 ** l, rank, world)
    if search is None:
        from . import MAX_L, find, find64
        f = find if l <= MAX_L else find64
        search = lambda s, l_, d_, a, b: f(s, l_, d_, lo=a, hi=b)  # noqa: E731
    local = np.asarray(search(seqs, l, d, lo, hi)).astype(np.uint64)
    dev = None
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    return gather_codes(local, device=dev, group=group)
