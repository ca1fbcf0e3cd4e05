"""Multi-GPU plumbing (torch.distributed).

One process per GPU. The path is sharded by *problem*: every rank solves its own
independent game (weak scaling), so there is no data-path collective. The only
collectives are the bench's max-over-ranks timing and the sum of processed
valuations. Works with the ``nccl`` backend on GPUs and ``gloo`` on CPU (tests).
"""
from __future__ import annotations

import os
from typing import Sequence, Tuple


def env_ranks() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str = "nccl", device=None):
    """Initialise the default process group when WORLD_SIZE > 1; returns the module or None."""
    rank, world, _ = env_ranks()
    if world <= 1:
        return None
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if backend == "nccl" and device is not None:
        dist.init_process_group(backend, device_id=device)
    else:
        dist.init_process_group(backend)
    return dist


def game_seed(base: int, rank: int) -> int:
    """Seed of the independent game a rank solves (weak scaling)."""
    return base + rank


def shard(items: Sequence, rank: int, world: int) -> list:
    """Round-robin shard of a batch of independent games over the ranks."""
    return list(items[rank::world])


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous balanced range [lo, hi) of n units for rank (sizes differ by <= 1)."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def reduce_time_and_units(dist, ms: float, units: float, device=None) -> Tuple[float, float]:
    """Max of the per-rank times, sum of the per-rank units (no-op on one process)."""
    if dist is None:
        return ms, units
    import torch
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    u = torch.tensor([units], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def barrier(dist) -> None:
    if dist is not None:
        dist.barrier()
