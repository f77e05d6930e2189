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


def _reduce(xs, op, group=None):
    import torch
    import torch.distributed as dist
    xs = [float(x) for x in xs]
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return xs
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(xs, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op, group=group)
    return [float(v) for v in t.tolist()]


def max_over_ranks(xs, group=None) -> list:
    """Element-wise max over all ranks (the bench's timing rule: the slowest
    rank's device time)."""
    import torch.distributed as dist
    return _reduce(xs, dist.ReduceOp.MAX, group)


def sum_over_ranks(xs, group=None) -> list:
    """Element-wise sum over all ranks (per-rank shares of the relaxation
    counts -> the job's total)."""
    import torch.distributed as dist
    return _reduce(xs, dist.ReduceOp.SUM, group)
