"""Env sharding across GPUs (one process per GPU).

Environments are independent, so the step has no data-path collective: GPU
``rank`` owns the contiguous global env range returned by ``shard_range`` and
runs its own kernel launches.  The only cross-rank traffic is plumbing:
barriers and a max-reduce of the per-rank device time (the job is as slow as
its slowest rank).
"""

from __future__ import annotations


def shard_range(total_envs: int, rank: int, world: int):
    """[first, last) global env ids of ``rank`` for a strong-scaling split of ``total_envs``
    (the first ``total_envs % world`` ranks take one extra env)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(int(total_envs), world)
    first = rank * base + min(rank, extra)
    return first, first + base + (1 if rank < extra else 0)


def weak_range(envs_per_rank: int, rank: int):
    """Global env ids of ``rank`` when every rank runs ``envs_per_rank`` envs (weak scaling)."""
    return rank * envs_per_rank, (rank + 1) * envs_per_rank


def job_time(local_seconds: float, group=None, device=None):
    """Max over ranks of a per-rank time (identity when torch.distributed is not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(local_seconds)
    t = torch.tensor([float(local_seconds)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def job_throughput(env_steps_local: int, local_seconds: float, group=None, device=None):
    """Whole-job env-steps/s: sum of env-steps over ranks / max time over ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return env_steps_local / local_seconds
    n = torch.tensor([float(env_steps_local)], dtype=torch.float64, device=device)
    dist.all_reduce(n, op=dist.ReduceOp.SUM, group=group)
    return float(n.item()) / job_time(local_seconds, group, device)
