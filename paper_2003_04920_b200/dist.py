"""Multi-GPU plumbing: one process per GPU, SPMD.

``torch.distributed`` is used only to ship the 128-byte ncclUniqueId from rank
0 to the other ranks and for the benchmark's barriers / max-over-ranks timing;
the per-iteration exchange of the sharded exploit is NCCL inside libpirrt.
"""
from __future__ import annotations

import os


def env_rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def broadcast_unique_id(make_id, group=None) -> bytes:
    """Rank 0 creates the id with ``make_id()``; every rank returns the same bytes."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def owner(v: int, nranks: int) -> int:
    """Rank whose Improve handles vertex v (vertex-cyclic split; stable as the graph grows)."""
    return v % nranks


def max_over_ranks(x: float, group=None) -> float:
    """Max of a float over all ranks (the bench's timing rule)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(x: float, group=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
