"""Multi-GPU plumbing for bench.py ("replicas only").

One process per GPU (torchrun), each running an independent replica of the
configuration: no data-path collective.  Timings are reduced as the max over
ranks (the slowest rank bounds the job) and the whole-job rate counts every
rank's units.  Works on NCCL (GPU) and gloo (CPU tests).
"""
from __future__ import annotations

import os


def dist_env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str) -> bool:
    """Initialise torch.distributed when launched with WORLD_SIZE > 1."""
    _, world, _ = dist_env()
    if world <= 1:
        return False
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group(backend)
    return True


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (a timing) over all ranks; identity when alone."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def whole_job_rate(units_per_rank: float, world: int, seconds_max: float) -> float:
    """Aggregate throughput: all ranks' units over the slowest rank's time."""
    return world * units_per_rank / seconds_max


def finalize():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()
