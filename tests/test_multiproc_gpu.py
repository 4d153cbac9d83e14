"""The sharded CUDA product in two processes: each rank holds its
own libmlob handle over its shard of the global env range
(sharding.sharded_vec_env), steps through several episode boundaries with
both device-drawn actions (mlob_venv_step_random, bench.hpp:53-70) and host
actions through the fused I/O call (mlob_venv_step_io, rollout.hpp:72-98),
and all-reduces the K4 episode statistics over gloo.  Every env's book,
observations, rewards and dones must equal the single-process run, and the
reduced statistics must equal MarketVecEnv::episode_stats
(rollout.hpp:255-270) of that run.

Both ranks share cuda:0 (one GPU per gpurun box); their kernels never wait
on each other — only the host-side gloo collective joins them."""
import os
import socket

import numpy as np
import pytest

from paper_2511_02136_b200 import abi
from tests import kat

pytestmark = pytest.mark.gpu

N_ENVS, STEPS, WORLD = 10, 21, 2


def _cfg():
    return abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR, task_size=60)],
                          steps_per_episode=6, messages_per_step=40, start_stride_steps=2)


def _store():
    from paper_2511_02136_b200.env import DeviceStore, HostStore
    return DeviceStore(HostStore.synth(abi.synth_config(n_messages=20000, state_sample_every=80), 3), 0)


def _actions(genv0, n, t, ar):
    return np.array([kat.bench_actions(0, genv0 + e, t, ar) for e in range(n)], dtype=np.int32)


def _trace(venv, cfg, genv0, steps, use_io):
    """Per-step observations / resets / rewards / dones and the final books."""
    ar = [abi.action_arity(cfg.specs[s]) for s in abi.flat_specs(cfg)]
    n, A = venv.n_envs, venv.n_agents
    rew = np.zeros((n, A), dtype=np.float64)
    dn = np.zeros((n, A), dtype=np.uint8)
    rec = []
    for t in range(steps):
        if use_io and t % 2 == 1:  # host actions through the fused I/O call
            obs = [np.zeros((venv.n_streams(k), venv.obs_dim(k))) for k in range(cfg.n_specs)]
            rs = [np.zeros(venv.n_streams(k), dtype=np.uint8) for k in range(cfg.n_specs)]
            venv.step_io(actions=_actions(genv0, n, t, ar), rewards=rew, dones=dn, obs=obs, resets=rs)
            r, d = rew.copy(), dn.copy()
        else:  # device-drawn bench actions keyed (0, BenchAction, global env, t)
            venv.step_random(0, t)
            r, d = venv.rewards(), venv.dones()
            obs, rs = zip(*[venv.gather(k) for k in range(cfg.n_specs)])
        rec.append((r, d, [o.copy() for o in obs], [x.copy() for x in rs]))
    books = [(venv.view(e).book(0).tobytes(), venv.view(e).book(1).tobytes()) for e in range(n)]
    return rec, books


def _rank(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_2511_02136_b200.sharding import reduce_episode_stats, shard_range, sharded_vec_env
        cfg = _cfg()
        store = _store()
        venv = sharded_vec_env(store, cfg, N_ENVS, rank, WORLD, seed=9, device=0)
        venv.reset_all()
        base, _ = shard_range(N_ENVS, WORLD, rank)
        rec, books = _trace(venv, cfg, base, STEPS, use_io=True)
        red = reduce_episode_stats(venv).cpu().numpy()
        q.put((rank, rec, books, red))
    except BaseException as e:  # surfaced by the parent
        q.put((rank, repr(e), None, None))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_process_shards_match_single_process():
    import torch.multiprocessing as mp
    from paper_2511_02136_b200.env import MarketVecEnv
    from paper_2511_02136_b200.sharding import exact_completion, shard_range

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(WORLD):
        r, rec, books, red = q.get(timeout=600)
        assert books is not None, f"rank {r} failed: {rec}"
        got[r] = (rec, books, red)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    cfg = _cfg()
    store = _store()
    one = MarketVecEnv(store, cfg, seed=9, n_envs=N_ENVS)
    one.reset_all()
    rec1, books1 = _trace(one, cfg, 0, STEPS, use_io=False)
    counts = [cfg.specs[k].count for k in range(cfg.n_specs)]
    for t in range(STEPS):
        r1, d1, o1, s1 = rec1[t]
        for rank in range(WORLD):
            base, n = shard_range(N_ENVS, WORLD, rank)
            r, d, o, s = got[rank][0][t]
            assert np.array_equal(r, r1[base:base + n]), (t, rank)
            assert np.array_equal(d, d1[base:base + n]), (t, rank)
            for k in range(cfg.n_specs):
                c = counts[k]
                assert np.array_equal(o[k], o1[k][base * c:(base + n) * c]), (t, rank, k)
                assert np.array_equal(s[k], s1[k][base * c:(base + n) * c]), (t, rank, k)
    for rank in range(WORLD):
        base, n = shard_range(N_ENVS, WORLD, rank)
        assert got[rank][1] == books1[base:base + n]

    # K4 all-reduced over the two processes == the single process's env-ordered stats
    red = got[0][2]
    assert np.array_equal(red, got[1][2])
    for k in range(cfg.n_specs):
        s = one.episode_stats(k)
        assert s.episodes >= 2 * N_ENVS  # >= 2 episode boundaries crossed by every env
        assert (red[k][0], red[k][1], red[k][3], red[k][4]) == \
            (s.pv_sum, s.slippage_sum, s.inventory_sq_sum, float(s.episodes))
        assert abs(red[k][2] - s.completion_sum) <= 1e-12 * max(1.0, abs(s.completion_sum))
        assert abs(exact_completion(red[k], cfg.specs[k]) - s.completion_sum) <= \
            1e-12 * max(1.0, abs(s.completion_sum))
    # the C-ABI collective entry without a communicator = this handle's K4
    loc = one.allreduce_episode_stats(0)
    for k in range(cfg.n_specs):
        s = one.episode_stats(k)
        assert (loc[k].pv_sum, loc[k].slippage_sum, loc[k].inventory_sq_sum, loc[k].episodes) == \
            (s.pv_sum, s.slippage_sum, s.inventory_sq_sum, s.episodes)
        assert loc[k].completion_sum == exact_completion(red[k], cfg.specs[k])


def test_bench_two_ranks_one_line():
    """bench.py's multi-rank path (the driver's N > 1 runs): two ranks
    (gloo, both on cuda:0 — diagnostics mode), the store synthesised once per
    node and loaded by the other rank, max-over-ranks timing, the stats
    all-reduce, one JSON line from rank 0 with the whole-job figures."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MLOB_BENCH_BACKEND="gloo", MLOB_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--workload", "C", "--envs", "8192", "--steps", "4", "--warmup", "3", "--e2e-steps", "3",
           "--no-extra"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=root, env=env)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["envs_per_gpu"] == 4096 and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["roofline"]["kernel"] == "book_kernel<4, false, false>"
