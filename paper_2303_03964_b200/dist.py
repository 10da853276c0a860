"""Multi-process plumbing over torch.distributed (one process per GPU).

The library creates its own NCCL communicator (include/tfdp.h tfdp_dist); torch.distributed
is only used to broadcast the 128-byte NCCL unique id from rank 0 and to take the max of
per-rank timings.  Works with any backend (nccl on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import os

from .tfdp import Dist, nccl_unique_id, shard_range


def _device_for_backend():
    import torch
    import torch.distributed as dist

    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def env_rank_world():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def broadcast_bytes(payload: bytes | None, nbytes: int, src: int = 0) -> bytes:
    """Broadcast `nbytes` bytes from rank `src` (payload ignored on other ranks)."""
    import torch
    import torch.distributed as dist

    dev = _device_for_backend()
    if dist.get_rank() == src:
        assert payload is not None and len(payload) == nbytes
        t = torch.tensor(list(payload), dtype=torch.uint8, device=dev)
    else:
        t = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    dist.broadcast(t, src=src)
    return bytes(t.cpu().tolist())


def bootstrap(device: int | None = None, uid_fn=nccl_unique_id) -> Dist | None:
    """Dist descriptor for this rank: rank 0 draws the NCCL unique id, every rank receives
    it over torch.distributed.  Returns None when WORLD_SIZE == 1 (single GPU)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    rank, world = dist.get_rank(), dist.get_world_size()
    uid = broadcast_bytes(uid_fn() if rank == 0 else None, 128)
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", rank))
    return Dist(rank, world, device, uid)


def max_over_ranks(x: float) -> float:
    """Maximum of a per-rank scalar (timings are max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def my_shard(n: int):
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return 0, n
    return shard_range(n, dist.get_world_size(), dist.get_rank())
