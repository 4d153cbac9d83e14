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
    returns a float64 CUDA tensor [n_types, 5] = (pv, slippage, completion,
    inventory², episodes)."""
    import torch
    import torch.distributed as dist
    n_types = venv.n_types()
    out = torch.zeros(5 * n_types, dtype=torch.float64, device="cuda")
    venv.episode_stats_device(out.data_ptr())
    venv.synchronize()
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(out, group=group)
    return out.view(n_types, 5)
