"""Multi-GPU env sharding: one process per GPU, contiguous env ranges, no
collective in the step path, one integer all-reduce of the episode
statistics per rollout.

The partition is the reference ThreadPool's static chunking
(proj/core/src/parallel.cpp:61-65: worker k of T owns [n*k/T, n*(k+1)/T)),
applied to GPUs instead of threads.  Every per-env key is a pure function of
the env's GLOBAL index (vector_env.cpp:52,55,171 -> split children are O(1) in
the index), so any sharding reproduces the single-device trajectories bit for
bit -- the analogue of the reference's thread-count invariance test
(test_vector_env.cpp:117-154).

Episode statistics are exact 64-bit integers (episodes, sum of lengths, sum
of returns in 2^-24 fixed point, see marl_venv_episode_stats), so a SUM
all-reduce gives identical totals for any GPU count and any reduction order.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

FIXED_POINT = float(1 << 24)


def shard_range(global_n: int, rank: int, world: int) -> Tuple[int, int]:
    """(global_offset, n_local) of `rank` -- parallel.cpp:61-65's chunk rule."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if global_n < world:
        raise ValueError(f"{global_n} envs cannot be split over {world} ranks")
    lo = global_n * rank // world
    hi = global_n * (rank + 1) // world
    return lo, hi - lo


def make_sharded(env, global_n: int, rank: int, world: int, device: int = 0):
    """The rank's VectorEnv shard of a global_n-env batch on cuda:`device`."""
    from .venv import VectorEnv
    off, n = shard_range(global_n, rank, world)
    return VectorEnv(env, n, device=device, global_offset=off, global_n=global_n)


def all_reduce_episode_stats(raw, group=None, device=None):
    """SUM all-reduce of the exact integer episode statistics
    [episodes, sum(final_lengths), sum(final_returns) * 2^24]: the one
    collective per rollout (the counterpart of ppo.cpp:275-276,634-638).
    Works over NCCL (device tensors) and gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(np.asarray(raw, dtype=np.int64).copy(), dtype=torch.int64)
    if device is not None:
        t = t.to(device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [int(v) for v in t.cpu().tolist()]


def summarize(raw) -> dict:
    """Mean episode length / return from the reduced integer totals."""
    eps, lens, rets = int(raw[0]), int(raw[1]), int(raw[2])
    return {"episodes": eps, "mean_length": lens / max(eps, 1),
            "mean_return": rets / FIXED_POINT / max(eps, 1)}


def fixed_point_return(ret: float) -> int:
    """One finished episode's return as the device accumulates it
    (__double2ll_rn(ret * 2^24), common.cuh stats_add)."""
    return int(np.rint(np.float64(ret) * FIXED_POINT))


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Device-timed durations are reported as the MAX over ranks."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
