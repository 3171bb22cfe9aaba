"""Multi-process plumbing (one process per GPU, torch.distributed).

The hot path has no data-path collective: scenarios (config 5) and bench
replicas are independent, so ranks only meet for the timing barrier and the
max-over-ranks reduction.  ``torch.distributed`` is used with NCCL on GPUs and
gloo for the CPU tests.
"""

from __future__ import annotations

import os


def world_from_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (single process default)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def max_over_ranks(value: float, device: str = "cpu") -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device: str = "cpu") -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
