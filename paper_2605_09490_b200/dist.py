"""Multi-GPU plumbing for request sharding: one process per GPU,
each rank owns its own batch of B requests (global request ids rank*B + b, seeds offset
per rank), no collective inside the decode step; timing is the max over ranks."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_plan(world, rank, B):
    """Weak scaling: every rank runs B requests; returns (seed_offset, global request ids)."""
    if not (0 <= rank < world) or B < 1:
        raise ValueError("bad shard")
    return 1000 * rank, list(range(rank * B, (rank + 1) * B))


def _dev():
    return torch.device("cuda") if dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float) -> float:
    """Max of a per-rank float across the process group (identity without one)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier_sync():
    """synchronize + barrier + synchronize (bench timing contract)."""
    if torch.cuda.is_available():
        torch.cuda.synchronize()
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()
