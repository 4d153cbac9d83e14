"""Env sharding across GPUs (one process per GPU).

Rank r owns the contiguous global env range [base, base + n_local).  Every
random stream is keyed by the *global* env index (env.hpp:176, 213;
bench.hpp:57) and auto-reset picks episodes with the *global* env count
(rollout.hpp:286-288), so a sharded run reproduces the single-GPU run env for
env.  The step has no collective; episode statistics are the only cross-GPU
data (K4 device sums + one all-reduce).
"""
from __future__ import annotations


def shard_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(env_index_base, n_local) of `rank`; the last rank takes the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    per = n_total // world
    base = rank * per
    n_local = per if rank < world - 1 else n_total - base
    if n_local < 1:
        raise ValueError("fewer envs than ranks")
    return base, n_local


def episode_for(env_global: int, k: int, n_envs_global: int, pool_len: int, pool=None) -> int:
    """MarketVecEnv::episode_for (rollout.hpp:286-288) over the global env set."""
    i = (env_global + k * n_envs_global) % pool_len
    return int(pool[i]) if pool is not None else i


def sharded_vec_env(store, cfg, n_total: int, rank: int, world: int, seed: int = 0, **kw):
    """MarketVecEnv holding this rank's shard of an n_total-env batch."""
    from .env import MarketVecEnv
    base, n_local = shard_range(n_total, world, rank)
    return MarketVecEnv(store, cfg, seed=seed, n_envs=n_local, n_envs_global=n_total,
                        env_index_base=base, **kw)


def reduce_episode_stats(venv, group=None):
    """K4 per-type sums on this GPU, all-reduced (sum) over the process group:
    returns a float64 CUDA tensor [n_types, STAT_WORDS] = (pv, slippage,
    completion, inventory², episodes, Σ remaining).  Only the completion
    column depends on the summation order; exact_completion() rebuilds it
    from the exact columns."""
    import torch
    import torch.distributed as dist
    from .abi import STAT_WORDS
    n_types = venv.n_types()
    out = torch.zeros(STAT_WORDS * n_types, dtype=torch.float64, device="cuda")
    venv.episode_stats_device(out.data_ptr())
    venv.synchronize()
    if dist.is_available() and dist.is_initialized():
        x = out if dist.get_backend(group) == "nccl" else out.cpu()
        dist.all_reduce(x, group=group)
        out.copy_(x)
    return out.view(n_types, STAT_WORDS)


def exact_completion(row, spec) -> float:
    """completion_sum of one type from its exact K4 columns:
    Σ_episodes (1 − remaining / task_size) = episodes·count − Σremaining / task_size."""
    from .abi import EXECUTOR
    if spec.type != EXECUTOR:
        return 0.0
    return float(row[4]) * spec.count - float(row[5]) / float(spec.params.task_size)
