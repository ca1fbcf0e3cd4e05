"""Multi-GPU plumbing (torch.distributed).

One process per GPU, two modes:

- replicas (default bench): every rank solves its own independent game (weak
  scaling); the only collectives are the bench's max-over-ranks timing and the
  sum of processed valuations;
- sharded (the bench's default for N > 1): all ranks solve ONE
  game, the valuation is replicated and the switch steps are split by vertex range.
  With ``pg_dist_init`` the per-step switch lists travel through the library's own
  NCCL communicator (:func:`nccl_join` only ships the ncclUniqueId); with
  ``pg_dist_attach`` through a caller all-gather such as :func:`torch_allgather`.

Works with the ``nccl`` backend on GPUs and ``gloo`` on CPU (tests).
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


def nccl_join(game_handle, dist, rank: int, world: int, nccl_id: bytes | None = None) -> bytes | None:
    """Make a loaded ``Game`` one of `world` ranks of a sharded solve with the library's
    own NCCL communicator: rank 0 creates the ncclUniqueId, torch.distributed
    broadcasts its 128 bytes, every rank calls ``pg_dist_init``. Returns the id: passing
    it again for another handle of the same ranks reuses the communicator."""
    from .pg import dist_unique_id
    if world < 1 or (dist is None and world > 1):
        raise ValueError("nccl_join: world > 1 needs a torch.distributed process group")
    if nccl_id is None:
        obj = [dist_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    game_handle.dist_init(nccl_id, rank, world)
    return nccl_id


def reduce_max(dist, x: float, device=None) -> float:
    """Max over ranks (no-op on one process)."""
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


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


class _CudaBuf:
    """A raw device pointer exposed through ``__cuda_array_interface__``."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, nbytes: int, device: int):
    """uint8 torch view of nbytes of device memory at ptr (no copy)."""
    import torch
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device=f"cuda:{device}")


def host_view(ptr: int, nbytes: int):
    """uint8 torch view of nbytes of host memory at ptr (no copy)."""
    import ctypes
    import torch
    return torch.frombuffer((ctypes.c_uint8 * nbytes).from_address(ptr), dtype=torch.uint8)


def torch_allgather(dist, device: int = 0):
    """The all-gather ``Game.attach_dist`` needs, over the default process group:
    NCCL gathers device tensors, gloo host tensors; buffers on the other side are
    staged. Returns only after the data has landed (synchronises the device)."""
    import torch
    world = dist.get_world_size()
    on_gpu_backend = dist.get_backend() == "nccl"

    def allgather(send: int, recv: int, nbytes: int, on_device: bool) -> None:
        if nbytes == 0:
            return
        src = device_view(send, nbytes, device) if on_device else host_view(send, nbytes)
        dst = device_view(recv, nbytes * world, device) if on_device else host_view(recv, nbytes * world)
        s = src
        if on_gpu_backend and not on_device:
            s = src.to(f"cuda:{device}")
        elif not on_gpu_backend and on_device:
            s = src.cpu()
        parts = [torch.empty_like(s) for _ in range(world)]
        dist.all_gather(parts, s)
        dst.copy_(torch.cat(parts))
        if on_device or on_gpu_backend:
            torch.cuda.synchronize(device)

    return allgather


def barrier(dist) -> None:
    if dist is not None:
        dist.barrier()
