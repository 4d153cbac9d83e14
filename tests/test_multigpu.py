"""Multi-GPU sharding semantics on CPU (gloo, world_size 2): shards keyed by
the global env index + an all-reduce of episode statistics reproduce the
single-process MarketVecEnv (rollout.hpp:151-336) — the contract the GPU
shards implement (env_index_base / n_envs_global in mlob_venv_desc)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_02136_b200 import abi
from paper_2511_02136_b200.sharding import episode_for, shard_range
from tests import kat

N_ENVS, STEPS = 6, 20


def _cfg():
    return abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR, task_size=90)],
                          steps_per_episode=6, messages_per_step=20, start_stride_steps=2)


def _run_shard(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import OEnv, Oracle
    from tests.common import small_store
    o = Oracle("orc")
    cfg = _cfg()
    st = small_store(o, {"state_sample_every": 40})
    base, n_local = shard_range(N_ENVS, world, rank)
    envs = [OEnv(o, st, cfg, 9, base + i) for i in range(n_local)]
    n_ep = envs[0].n_episodes
    cursor = [1] * n_local
    for i, e in enumerate(envs):
        e.reset(episode_for(base + i, 0, N_ENVS, n_ep))
    stats = np.zeros((cfg.n_specs, 5))
    flat = abi.flat_specs(cfg)
    ar = [abi.action_arity(cfg.specs[s]) for s in flat]
    for t in range(STEPS):
        for i, e in enumerate(envs):
            e.step_ids(kat.bench_actions(0, base + i, t, ar))
            if e.scalars().terminal:
                for a in range(len(flat)):  # rollout.hpp:300-313
                    info = e.info(a)
                    sp = cfg.specs[flat[a]]
                    comp = (1.0 - info.task_remaining / sp.params.task_size) if sp.type == abi.EXECUTOR else 0.0
                    stats[flat[a]] += [info.portfolio_value, info.slippage_total, comp,
                                       float(info.inventory) ** 2, 0]
                stats[:, 4] += 1
                e.reset(episode_for(base + i, cursor[i], N_ENVS, n_ep))
                cursor[i] += 1
    t = torch.tensor(stats, dtype=torch.float64)
    dist.all_reduce(t)
    if rank == 0:
        q.put(t.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition():
    for n, w in [(10, 1), (10, 2), (10, 3), (1 << 20, 8), (7, 7)]:
        got = [shard_range(n, w, r) for r in range(w)]
        assert got[0][0] == 0 and sum(x[1] for x in got) == n
        assert all(got[r][0] + got[r][1] == got[r + 1][0] for r in range(w - 1))
    with pytest.raises(ValueError):
        shard_range(1, 2, 0)


def test_two_rank_gloo_matches_single_process(orc):
    from oracle.oracle import OVecEnv
    from tests.common import small_store
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_shard, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = _cfg()
    v = OVecEnv(orc, small_store(orc, {"state_sample_every": 40}), cfg, 9, N_ENVS)
    v.reset_all()
    ar = [abi.action_arity(cfg.specs[s]) for s in abi.flat_specs(cfg)]
    for t in range(STEPS):
        for e in range(N_ENVS):
            ids = kat.bench_actions(0, e, t, ar)
            for ty in range(cfg.n_specs):
                v.set_action(ty, e, ids[ty])
        v.step_all()
    for ty in range(cfg.n_specs):
        s = v.episode_stats(ty)
        assert got[ty][0] == s.pv_sum and got[ty][1] == s.slippage_sum
        assert got[ty][3] == s.inventory_sq_sum and got[ty][4] == s.episodes
        assert abs(got[ty][2] - s.completion_sum) <= 1e-12 * max(1.0, abs(s.completion_sum))
