"""GPU parity: the CUDA product (through the C ABI) against the oracle — the C
restatement (orc), pinned to the compiled reference — on identical synthetic
streams and actions.  Books, trades, integer state: bit-exact.  Observations,
rewards, infos: compared bit-for-bit (the north-star bar is 1e-5 relative; the
build reproduces the reference's double rounding exactly, --fmad=false)."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import OEnv, OVecEnv, Oracle, bench_run
from paper_2511_02136_b200 import abi
from paper_2511_02136_b200.sharding import exact_completion
from paper_2511_02136_b200.env import (DeviceStore, HostStore, LogicError, MarketEnvBatch,
                                       MarketVecEnv)
from tests import kat
from tests.common import (compare_env_state, random_direct_action, scenario_configs,
                          small_store)

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RTOL = 1e-5  # north_star float tolerance (we additionally hold bit equality)


def dev_store(synth_kw, seed=0):
    kw = {"n_messages": 20000, "state_sample_every": 100}
    kw.update(synth_kw)
    return DeviceStore(HostStore.synth(abi.synth_config(**kw), seed), 0)


@pytest.mark.parametrize("name", ["exec_only", "mm_exec"])
def test_config_a_golden_digest(name):
    golden = json.load(open(os.path.join(GOLDEN, "kat_config_a.json")))[name]
    synth, cfg = kat.config_a(name)
    dev = DeviceStore(HostStore.synth(synth, 0), 0)
    b = MarketEnvBatch(dev, cfg, n_envs=1, seed=0)
    b.reset([0])
    ar = [abi.action_arity(cfg.specs[s]) for s in abi.flat_specs(cfg)]

    class One:
        def step_ids(self, ids):
            b.step_ids([ids])

        def __getattr__(self, k):
            return getattr(b.view(0), k)

    got = kat.env_digest(One(), 100, ar)
    for k in ("messages", "trades", "trade_fnv", "book_fnv", "live_bid", "live_ask", "next_seq",
              "mid_half"):
        assert got[k] == golden[k], k
    assert abs(got["sum_reward"] - golden["sum_reward"]) <= RTOL * abs(golden["sum_reward"])
    assert got["sum_obs"] == golden["sum_obs"]
    assert got["sum_reward"] == golden["sum_reward"]


@pytest.mark.parametrize("scenario", list(scenario_configs().keys()))
def test_scenario_parity(orc, scenario):
    cfg, synth_kw, n_steps = scenario_configs()[scenario]
    if cfg.book_capacity > 1024:
        pytest.skip("capacity above the device limit")
    host_kw = {"n_messages": 20000, "state_sample_every": 100}
    host_kw.update(synth_kw)
    dev = dev_store(synth_kw)
    ost = small_store(orc, synth_kw)
    n_envs = 6
    env_idx = [0, 1, 3, 7, 11, 1000]
    seeds = [5, 5, 6, 7, 8, 9]
    b = MarketEnvBatch(dev, cfg, n_envs=n_envs, seed=0, env_seeds=seeds, env_indices=env_idx)
    refs = [OEnv(orc, ost, cfg, seeds[i], env_idx[i]) for i in range(n_envs)]
    n_ep = refs[0].n_episodes
    rng = kat.CounterRng(kat.make_key(31, len(scenario)))
    for rep in range(2):
        eps = [(i + rep) % n_ep for i in range(n_envs)]
        b.reset(eps)
        for i, r in enumerate(refs):
            r.reset(eps[i])
            compare_env_state(b.view(i), r)
        for t in range(n_steps):
            if rng.below(4) == 0 and b.n_agents:
                acts = [random_direct_action(rng) for _ in range(n_envs * b.n_agents)]
                b.step_actions(acts)
                for i, r in enumerate(refs):
                    r.step(acts[i * b.n_agents:(i + 1) * b.n_agents])
            else:
                ids = [[rng.below(abi.action_arity(cfg.specs[s])) for s in b.flat]
                       for _ in range(n_envs)]
                b.step_ids(np.array(ids, dtype=np.int32).reshape(n_envs, -1))
                for i, r in enumerate(refs):
                    r.step_ids(ids[i])
            for i, r in enumerate(refs):
                compare_env_state(b.view(i), r)


def _sweep(side, price, qty):
    a = abi.AgentAction()
    a.direct = 1
    a.n_quotes = 1
    a.quotes[0].side = side
    a.quotes[0].price = price
    a.quotes[0].quantity = qty
    return a


def test_fill_log_beyond_inline_and_chunks_exact(orc):
    """Agent orders that sweep a whole side: more agent fills in one env-step
    than the inline log (16) and several overflow chunks (31 each) hold.  The
    MM rewards (Ψ sums in fill order against M̄, rewards.hpp:22-36), the
    executor slippage and the agent accounting must stay bit-exact."""
    A = abi
    cfg = A.env_config([A.agent_spec(A.MARKET_MAKER, reward=A.REWARD_SPOONER),
                        A.agent_spec(A.MARKET_MAKER, reward=A.REWARD_BUYSELL, inventory_cap=5000),
                        A.agent_spec(A.EXECUTOR, task_size=100000)],
                       steps_per_episode=12, messages_per_step=100, start_stride_steps=12)
    dev = dev_store({})
    ost = small_store(orc, {})
    n_envs = 4
    b = MarketEnvBatch(dev, cfg, n_envs=n_envs, seed=2)
    refs = [OEnv(orc, ost, cfg, 2, i) for i in range(n_envs)]
    b.reset(list(range(n_envs)))
    for i, r in enumerate(refs):
        r.reset(i)
    rng = kat.CounterRng(77)
    most = 0
    for t in range(12):
        acts = []
        for e in range(n_envs):
            for a in range(b.n_agents):
                k = (t + a + e) % 3
                if k == 0:   # buy through every ask level
                    acts.append(_sweep(A.BID, 2000, 4000 + rng.below(100)))
                elif k == 1:  # sell through every bid level
                    acts.append(_sweep(A.ASK, 1, 4000 + rng.below(100)))
                else:
                    acts.append(random_direct_action(rng))
        b.step_actions(acts)
        for i, r in enumerate(refs):
            r.step(acts[i * b.n_agents:(i + 1) * b.n_agents])
        for i, r in enumerate(refs):
            compare_env_state(b.view(i), r)
            most = max(most, sum(b.view(i).info(a).step_fill_count for a in range(b.n_agents)))
    # the sweeps overflowed the inline log and at least two overflow chunks
    assert most > 16 + 2 * 31, most


def test_vec_env_auto_reset_and_episode_stats(orc):
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER, count=2), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=8, messages_per_step=20, start_stride_steps=3)
    dev = dev_store({"state_sample_every": 20})
    ost = small_store(orc, {"state_sample_every": 20})
    pool = [3, 1, 4, 1, 5, 9, 2, 6]
    g = MarketVecEnv(dev, cfg, episode_pool=pool, seed=3, n_envs=5)
    o = OVecEnv(orc, ost, cfg, 3, 5, pool=pool)
    g.reset_all()
    o.reset_all()
    rng = kat.CounterRng(123)
    for t in range(30):
        for ty in range(cfg.n_specs):
            go, gr = g.gather(ty)
            oo, orr = o.gather(ty)
            assert go.tobytes() == oo.tobytes() and gr.tobytes() == orr.tobytes()
            for s in range(g.n_streams(ty)):
                a = rng.below(g.n_actions(ty))
                g.set_action(ty, s, a)
                o.set_action(ty, s, a)
        g.step_all()
        o.step_all()
        rw, dn = g.rewards(), g.dones()
        for ty in range(cfg.n_specs):
            for s in range(g.n_streams(ty)):
                e, a = g._locate(ty, s)
                assert rw[e, a] == o.reward(ty, s)
                assert bool(dn[e, a]) == bool(o.done(ty, s))
    for ty in range(cfg.n_specs):
        a, b = g.episode_stats(ty), o.episode_stats(ty)
        assert bytes(a) == bytes(b)
    import torch
    W = abi.STAT_WORDS
    out = torch.zeros(W * cfg.n_specs, dtype=torch.float64, device="cuda")
    g.episode_stats_device(out.data_ptr())
    g.synchronize()
    red = g.allreduce_episode_stats(0)  # K4 + the host-side exact completion, no communicator
    for ty in range(cfg.n_specs):
        s = o.episode_stats(ty)
        d = out[W * ty: W * ty + W].cpu().numpy()
        assert d[0] == s.pv_sum and d[1] == s.slippage_sum and d[3] == s.inventory_sq_sum
        assert abs(d[2] - s.completion_sum) <= 1e-12 * max(1.0, abs(s.completion_sum))
        assert d[4] == s.episodes
        assert exact_completion(d, cfg.specs[ty]) == red[ty].completion_sum
        assert abs(red[ty].completion_sum - s.completion_sum) <= 1e-12 * max(1.0, abs(s.completion_sum))
        assert (red[ty].pv_sum, red[ty].slippage_sum, red[ty].inventory_sq_sum, red[ty].episodes) == \
            (s.pv_sum, s.slippage_sum, s.inventory_sq_sum, s.episodes)
    g.clear_episode_stats()
    assert g.episode_stats(0).episodes == 0


def test_bench_harness_random_actions_match_oracle(orc):
    """RandomStepHarness (bench.hpp:53-70): device-drawn actions + auto-reset."""
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=16, messages_per_step=20, start_stride_steps=16)
    dev = dev_store({"state_sample_every": 16, "n_messages": 3000})
    ost = small_store(orc, {"state_sample_every": 16, "n_messages": 3000})
    g = MarketVecEnv(dev, cfg, seed=0, n_envs=8)
    g.reset_all()
    for s in range(2 + 32):
        g.step_random(0, s)
    row = bench_run(orc, ost, cfg, 8, 32, 2, 1, 0, 20, 1)
    # total messages over all 34 steps = oracle warm-up + timed (recount on oracle)
    o = OVecEnv(orc, ost, cfg, 0, 8)
    o.reset_all()
    for s in range(34):
        for e in range(8):
            ids = kat.bench_actions(0, e, s, [8, 12])
            for ty in range(2):
                o.set_action(ty, e, ids[ty])
        o.step_all()
    tot = sum(o.instance(e).scalars().messages_processed for e in range(8))
    assert g.messages_processed() == tot
    assert row.messages > 0
    for e in range(8):
        for side in (0, 1):
            assert g.view(e).book(side).tobytes() == o.instance(e).book(side).tobytes()


def test_random_streams_zero_agents(orc):
    """test_lob.cpp:258-281 streams replayed as zero-agent episodes (capacity 256)."""
    from oracle.oracle import random_stream
    streams = [random_stream(orc, seed, n_messages=4000) for seed in range(8)]
    msgs = np.concatenate(streams)
    states = [(i * 4000, [], []) for i in range(8)]
    hs = HostStore.from_messages(msgs, states)
    dev = DeviceStore(hs, 0)
    ost = orc.store_from(msgs, states)
    cfg = abi.env_config([], steps_per_episode=40, messages_per_step=100, start_stride_steps=40,
                         book_capacity=256)
    b = MarketEnvBatch(dev, cfg, n_envs=8, seed=0)
    b.reset(list(range(8)))
    refs = [OEnv(orc, ost, cfg, 0, i) for i in range(8)]
    for i, r in enumerate(refs):
        r.reset(i)
    for t in range(40):
        b.step_ids(np.zeros((8, 0), dtype=np.int32))
        for i, r in enumerate(refs):
            r.step_ids([])
            compare_env_state(b.view(i), r)


@pytest.mark.parametrize("capacity", [64, 100, 256, 600])
def test_duplicate_live_ids_zero_agents(orc, capacity):
    """Replay streams whose resting orders share ids (oracle.dup_id_stream): the
    device's duplicate-id path (first match in storage order, book.hpp:191-206)
    for register books (SPL 2 / 4 / 8) and a shared-memory book (SPL 32),
    every step vs the oracle (books in storage order, trades, mids)."""
    from oracle.oracle import dup_id_stream
    streams = [dup_id_stream(orc, seed, n_messages=4000) for seed in range(6)]
    msgs = np.concatenate(streams)
    states = [(i * 4000, [], []) for i in range(6)]
    dev = DeviceStore(HostStore.from_messages(msgs, states), 0)
    ost = orc.store_from(msgs, states)
    cfg = abi.env_config([], steps_per_episode=40, messages_per_step=100, start_stride_steps=40,
                         book_capacity=capacity)
    b = MarketEnvBatch(dev, cfg, n_envs=6, seed=0)
    b.reset(list(range(6)))
    refs = [OEnv(orc, ost, cfg, 0, i) for i in range(6)]
    for i, r in enumerate(refs):
        r.reset(i)
    for t in range(40):
        b.step_ids(np.zeros((6, 0), dtype=np.int32))
        for i, r in enumerate(refs):
            r.step_ids([])
            compare_env_state(b.view(i), r)


def test_errors_match_reference_exceptions():
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER)], steps_per_episode=4,
                         messages_per_step=10, start_stride_steps=4)
    dev = dev_store({"state_sample_every": 40})
    b = MarketEnvBatch(dev, cfg, n_envs=2, seed=1)
    with pytest.raises(LogicError):      # step before reset (env.hpp:195)
        b.step_ids([[0], [0]])
    with pytest.raises(IndexError):      # env.hpp:144-147
        b.reset([0, b.n_episodes])
    b.reset([0, 1])
    with pytest.raises(IndexError):      # actions.hpp:69-70
        b.step_ids([[8], [0]])
    with pytest.raises(ValueError):      # env.hpp:196-199
        b.step_ids([[0, 0], [0, 0]])
    for _ in range(4):
        b.step_ids([[0], [0]])
    with pytest.raises(LogicError):
        b.step_ids([[0], [0]])
    # missing book state -> runtime_error (env.hpp:149-153)
    dev2 = dev_store({"state_sample_every": 1000, "n_messages": 5000})
    b2 = MarketEnvBatch(dev2, cfg, n_envs=1, seed=0)
    with pytest.raises(RuntimeError):
        b2.reset([1])
    with pytest.raises(ValueError):      # executor + mm_basic is UB in the reference
        MarketEnvBatch(dev, abi.env_config([abi.agent_spec(abi.EXECUTOR, obs_space=abi.OBS_MM_BASIC)]))


def test_reset_determinism_and_executor_direction():  # test_env.cpp:70-111
    cfg = abi.env_config([abi.agent_spec(abi.EXECUTOR)], steps_per_episode=4, messages_per_step=0,
                         start_stride_steps=4)
    from paper_2511_02136_b200.env import MESSAGE_DTYPE
    msgs = np.zeros(1, dtype=MESSAGE_DTYPE)
    msgs["kind"] = abi.HALT
    dev = DeviceStore(HostStore.from_messages(msgs, [(0, [], [])]), 0)
    n = 10000
    b = MarketEnvBatch(dev, cfg, n_envs=n, seed=0, env_seeds=np.arange(n), env_indices=np.zeros(n))
    b.reset(np.zeros(n))
    direction = b.obs_type(0)[:, 2]          # exec obs feature 2 = +1 buy / -1 sell
    frac = float((direction > 0).mean())
    assert 0.48 < frac < 0.52
    orc = Oracle("orc")
    ost = orc.store_from(msgs, [(0, [], [])])
    for seed in range(0, n, 997):             # per-seed agreement with the oracle
        r = OEnv(orc, ost, cfg, seed, 0)
        r.reset(0)
        assert r.agent(0).task_dir == (0 if direction[seed] > 0 else 1)
    b2 = MarketEnvBatch(dev, cfg, n_envs=n, seed=0, env_seeds=np.arange(n), env_indices=np.zeros(n))
    b2.reset(np.zeros(n))
    assert b2.obs_type(0).tobytes() == b.obs_type(0).tobytes()


def test_two_shards_equal_one_batch():
    """Sharded handles (env_index_base / n_envs_global) reproduce the unsharded
    batch env for env (what each GPU rank runs under torchrun)."""
    import torch
    from paper_2511_02136_b200.sharding import reduce_episode_stats, sharded_vec_env
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=8, messages_per_step=50, start_stride_steps=1)
    dev = dev_store({"state_sample_every": 50, "n_messages": 60000})
    n = 1000
    full = MarketVecEnv(dev, cfg, seed=4, n_envs=n)
    shards = [sharded_vec_env(dev, cfg, n, r, 3, seed=4) for r in range(3)]
    for v in [full] + shards:
        v.reset_all()
    for t in range(20):
        for v in [full] + shards:
            v.step_random(11, t)
    for ty in range(cfg.n_specs):
        a = full.gather(ty)
        b = [s.gather(ty) for s in shards]
        assert a[0].tobytes() == np.concatenate([x[0] for x in b]).tobytes()
        assert a[1].tobytes() == np.concatenate([x[1] for x in b]).tobytes()
    assert full.rewards().tobytes() == np.concatenate([s.rewards() for s in shards]).tobytes()
    tot = sum(reduce_episode_stats(s) for s in shards)
    ref = reduce_episode_stats(full)
    assert torch.equal(tot[:, [0, 1, 3, 4]], ref[:, [0, 1, 3, 4]])
    assert float(tot[:, 4].sum()) > 0


@pytest.mark.parametrize("n", [7105, 3553])
def test_rounds_cover_every_env(n):
    """The step kernel's rounds (one block per SM walking env rounds, the
    launcher's balanced block width, a partial last round) step every env
    exactly once: a batch of n envs equals the same envs run as 8 small shards
    (one round each), env for env."""
    from paper_2511_02136_b200.sharding import sharded_vec_env
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=6, messages_per_step=40, start_stride_steps=1)
    dev = dev_store({"state_sample_every": 40, "n_messages": 80000})
    full = MarketVecEnv(dev, cfg, seed=9, n_envs=n)
    shards = [sharded_vec_env(dev, cfg, n, r, 8, seed=9) for r in range(8)]
    for v in [full] + shards:
        v.reset_all()
    for t in range(14):  # crosses two auto-resets
        for v in [full] + shards:
            v.step_random(5, t)
    assert full.messages_processed() == sum(s.messages_processed() for s in shards)
    for ty in range(cfg.n_specs):
        a = full.gather(ty)
        b = [s.gather(ty) for s in shards]
        assert a[0].tobytes() == np.concatenate([x[0] for x in b]).tobytes()
        assert a[1].tobytes() == np.concatenate([x[1] for x in b]).tobytes()
    assert full.rewards().tobytes() == np.concatenate([s.rewards() for s in shards]).tobytes()


@pytest.mark.parametrize("chunks", ["1", "3"])
def test_step_io_matches_separate_calls(monkeypatch, chunks):
    """mlob_venv_step_io (chunked step on two streams + overlapped copies) gives
    the same outputs and state as set_actions + step + rewards/dones/infos/gather,
    across auto-resets; a bad action id is rejected before any env steps."""
    import torch
    monkeypatch.setenv("MLOB_IO_CHUNKS", chunks)
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER, count=2), abi.agent_spec(abi.EXECUTOR),
                          abi.agent_spec(abi.DIRECTIONAL)],
                         steps_per_episode=6, messages_per_step=30, start_stride_steps=2)
    dev = dev_store({"state_sample_every": 30})
    n = 7
    a, b = (MarketVecEnv(dev, cfg, seed=9, n_envs=n) for _ in range(2))
    a.reset_all()
    b.reset_all()
    A, T = a.n_agents, a.n_types()
    ar = np.array([abi.action_arity(cfg.specs[s]) for s in abi.flat_specs(cfg)])
    rng = np.random.default_rng(5)
    pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()  # noqa: E731
    obs = [pin((b.n_streams(t), b.obs_dim(t)), torch.float64) for t in range(T)]
    rst = [pin(b.n_streams(t), torch.uint8) for t in range(T)]
    rew, dn = pin((n, A), torch.float64), pin((n, A), torch.uint8)
    infos = np.zeros((n, A), dtype=a.infos().dtype)
    acts = pin((n, A), torch.int32)
    for step in range(15):
        if step == 4:  # rejected batch: nothing changes
            before = [(a.view(e).book(0).tobytes(), a.view(e).book(1).tobytes()) for e in range(n)]
            bad = acts.clone()
            bad[n - 1, A - 1] = int(ar[A - 1])
            with pytest.raises(IndexError):
                b.step_io(actions=bad)
            assert [(b.view(e).book(0).tobytes(), b.view(e).book(1).tobytes()) for e in range(n)] == before
        acts.copy_(torch.from_numpy((rng.integers(0, 1 << 20, size=(n, A)) % ar).astype(np.int32)))
        a.set_actions(acts.numpy())
        a.step()
        b.step_io(actions=acts, rewards=rew, dones=dn, infos=infos, obs=obs, resets=rst)
        assert rew.numpy().tobytes() == a.rewards().tobytes()
        assert dn.numpy().tobytes() == a.dones().tobytes()
        assert infos.tobytes() == a.infos().tobytes()
        for t in range(T):
            go, gr = a.gather(t)
            assert obs[t].numpy().tobytes() == go.tobytes()
            assert rst[t].numpy().tobytes() == gr.tobytes()
        for e in range(n):
            assert b.view(e).scalars().step == a.view(e).scalars().step
            assert b.view(e).book(0).tobytes() == a.view(e).book(0).tobytes()
            assert b.view(e).book(1).tobytes() == a.view(e).book(1).tobytes()
    for t in range(T):
        assert bytes(a.episode_stats(t)) == bytes(b.episode_stats(t))


def test_evaluate_matrix_matches_oracle(orc):
    """Cross-play grid on the GPU (one env per cell x episode, policies
    evaluated in the step kernel) against the oracle's evaluate_matrix."""
    from paper_2511_02136_b200.env import evaluate_matrix
    from tests.common import crossplay_case
    cfg, synth_kw, eps, t0, t1 = crossplay_case()
    got = evaluate_matrix(dev_store(synth_kw), cfg, eps, t0, t1, 7)
    want = orc.evaluate(small_store(orc, synth_kw), cfg, eps, t0, t1, 7)
    assert [bytes(x) for x in got] == [bytes(x) for x in want]
    with pytest.raises(ValueError):
        evaluate_matrix(dev_store(synth_kw), cfg, eps, [abi.policy(abi.POLICY_LEARNED)], t1, 7)
    with pytest.raises(IndexError):
        evaluate_matrix(dev_store(synth_kw), cfg, eps, [abi.policy(abi.POLICY_AVST, gamma_index=9)],
                        t1, 7)


def test_scripted_policies_per_step(orc):
    """set_policies: every env-step of scripted agents equals the oracle env
    driven by the same policies (twap.hpp:37-58, avst.hpp:19-32, evaluate.hpp:74-79)."""
    from oracle.oracle import OEnv
    from tests.common import crossplay_case
    cfg, synth_kw, eps, t0, t1 = crossplay_case()
    dev, ost = dev_store(synth_kw), small_store(orc, synth_kw)
    pols = t0 + t1
    n = len(t0) * len(t1)
    env_policy = np.array([[i // len(t1), len(t0) + i % len(t1)] for i in range(n)], dtype=np.uint8)
    cells = np.array([(i // len(t1)) * 1000 + i % len(t1) for i in range(n)], dtype=np.uint64)
    b = MarketEnvBatch(dev, cfg, n_envs=n, seed=7, env_indices=np.zeros(n))
    b.reset([eps[i % len(eps)] for i in range(n)])
    b.set_policies(pols, env_policy, cells)
    refs = [OEnv(orc, ost, cfg, 7, 0) for _ in range(n)]
    for i, r in enumerate(refs):
        r.reset(eps[i % len(eps)])
    for t in range(cfg.steps_per_episode):
        b.step()
        for i, r in enumerate(refs):
            acts = [r.policy_action(a, pols[env_policy[i, r.flat[a]]], t, 7, int(cells[i]),
                                    eps[i % len(eps)]) for a in range(len(r.flat))]
            r.step(acts)
            compare_env_state(b.view(i), r)


def test_collect_rollout_matches_oracle(orc):
    """On-device collect_rollout against the oracle's (pinned to the reference):
    actions, rewards, dones, resets and observations exact; values, log-probs,
    advantages, returns and hidden states within 1e-10 relative + 1e-12 absolute (device exp /
    tanh / log vs glibc; sums in the reference's order, no FMA)."""
    from tests.common import rollout_case
    cfg, synth_kw, nets = rollout_case(orc)
    g = MarketVecEnv(dev_store(synth_kw), cfg, seed=3, n_envs=5)
    o = OVecEnv(orc, small_store(orc, synth_kw), cfg, 3, 5)
    g.reset_all()
    o.reset_all()
    with pytest.raises(RuntimeError):        # no nets yet
        g.collect_rollout(12)
    g.set_nets(nets)
    exact = (abi.RB_OBS, abi.RB_ACTIONS, abi.RB_REWARDS, abi.RB_DONES, abi.RB_RESETS)
    for upd in (1, 2, 3):
        g.collect_rollout(12, 0.99, 0.95, seed=77, update_index=upd)
        o.collect_rollout(nets, 12, 0.99, 0.95, 77, upd)
        for t in range(cfg.n_specs):
            for f in range(11):
                a, b = g.rollout(t, f), o.rollout(t, f)
                assert a.shape == b.shape, (t, f)
                if f in exact:
                    assert a.tobytes() == b.tobytes(), (upd, t, f)
                else:
                    np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-12, err_msg=f"{upd} {t} {f}")
    bad = [nets[1], nets[0]]                 # shapes swapped
    with pytest.raises(ValueError):
        g.set_nets(bad)


def test_evaluate_matrix_learned_matches_oracle(orc):
    """Learned cross-play options on the device (policy kernel in argmax mode per
    option, then the scripted step) against the oracle's evaluate_matrix."""
    from paper_2511_02136_b200.env import evaluate_matrix
    from tests.common import crossplay_learned_case
    cfg, synth_kw, eps, t0, t1 = crossplay_learned_case(orc)
    got = evaluate_matrix(dev_store(synth_kw), cfg, eps, t0, t1, 5)
    want = orc.evaluate(small_store(orc, synth_kw), cfg, eps, t0, t1, 5)
    assert [bytes(x) for x in got] == [bytes(x) for x in want]
    wrong = abi.policy(abi.POLICY_LEARNED, net=orc.make_policy_net(3, 8, 4, 0))
    with pytest.raises(ValueError):
        evaluate_matrix(dev_store(synth_kw), cfg, eps, [wrong], t1, 5)


def test_lobster_device_loader(orc, tmp_path):
    """mlob_store_load_lobster (GPU parse) against the oracle's load_lobster
    (pinned to the reference): the device store equals the upload of the
    oracle's store, malformed inputs raise the same class and text, and an env
    replaying the loaded store matches the oracle env on the oracle store."""
    from paper_2511_02136_b200.env import DeviceStore as DS
    from tests.lobster_util import ACCEPTED, MALFORMED, write_lobster

    def files(name, msg, book):
        m, b = tmp_path / f"{name}_m.csv", tmp_path / f"{name}_b.csv"
        m.write_text(msg)
        b.write_text(book)
        return str(m), str(b)

    def same(m, b, upt, every):
        got = DS.load_lobster(m, b, upt, every)
        o = orc.lobster(m, b, upt, every)
        want = DS(HostStore.from_messages(o.messages(), o.states()), 0)
        assert got.messages().tobytes() == want.messages().tobytes()
        assert got.states() == want.states() == o.states()
        return got, o

    for name, msg, book, upt, every in ACCEPTED:
        same(*files(name, msg, book), upt, every)
    for name, msg, book, upt, every in MALFORMED:
        m, b = files(name, msg, book)
        errs = []
        for load in (lambda: DS.load_lobster(m, b, upt, every), lambda: orc.lobster(m, b, upt, every)):
            with pytest.raises(Exception) as ei:
                load()
            errs.append((type(ei.value), str(ei.value)))
        assert errs[0] == errs[1], name
    with pytest.raises(ValueError):
        DS.load_lobster(m, b, 0, 1)
    # a synthetic day: parse on the GPU, then replay through the env
    synth = orc.synth(abi.synth_config(n_messages=20000, state_sample_every=100), 2)
    m, b = str(tmp_path / "day_m.csv"), str(tmp_path / "day_b.csv")
    write_lobster(orc, synth.messages(), m, b, upt=100, depth=10)
    dev, ost = same(m, b, 100, 100)
    cfg = abi.env_config([abi.agent_spec(abi.MARKET_MAKER), abi.agent_spec(abi.EXECUTOR)],
                         steps_per_episode=20, messages_per_step=50, start_stride_steps=4)
    bt = MarketEnvBatch(dev, cfg, n_envs=4, seed=3, env_indices=[0, 1, 2, 3])
    refs = [OEnv(orc, ost, cfg, 3, i) for i in range(4)]
    eps = [0, 5, 17, 30]
    bt.reset(eps)
    for r, ep in zip(refs, eps):
        r.reset(ep)
    rng = kat.CounterRng(kat.make_key(9, 9))
    for t in range(20):
        ids = [[rng.below(abi.action_arity(cfg.specs[s])) for s in bt.flat] for _ in range(4)]
        bt.step_ids(np.array(ids, dtype=np.int32))
        for i, r in enumerate(refs):
            r.step_ids(ids[i])
            compare_env_state(bt.view(i), r)


def test_ppo_update_matches_reference(ref):
    """Device train_loop iterations (collect_rollout + ppo_update per type,
    rollout.hpp:127-145 / ppo.hpp:263-310) against the reference's: metrics and
    parameters after each update, and the next rollout with the updated nets.
    Reductions are ordered differently (GEMMs over T x streams), so the bar is
    1e-8 relative (+1e-12 absolute)."""
    from tests.common import rollout_case
    cfg, synth_kw, nets = rollout_case(ref)
    g = MarketVecEnv(dev_store(synth_kw), cfg, seed=3, n_envs=5)
    o = OVecEnv(ref, small_store(ref, synth_kw), cfg, 3, 5)
    g.reset_all()
    o.reset_all()
    g.set_nets(nets)
    pcfg = abi.ppo_config(minibatches=2)
    for upd in (1, 2):
        g.collect_rollout(12, 0.99, 0.95, seed=77, update_index=upd)
        o.collect_rollout(nets if upd == 1 else None, 12, 0.99, 0.95, 77, upd)
        assert g.rollout(0, abi.RB_ACTIONS).tobytes() == o.rollout(0, abi.RB_ACTIONS).tobytes()
        assert g.rollout(1, abi.RB_ACTIONS).tobytes() == o.rollout(1, abi.RB_ACTIONS).tobytes()
        for t in range(cfg.n_specs):
            gm = g.ppo_update(t, pcfg, seed=77, update_index=upd)
            om = o.ppo_update(t, pcfg, 77, upd)
            for f, _ in abi.UpdateMetrics._fields_:
                np.testing.assert_allclose(getattr(gm, f), getattr(om, f), rtol=1e-8, atol=1e-12,
                                           err_msg=f"{upd} {t} {f}")
            np.testing.assert_allclose(g.read_net(t), o.read_net(t), rtol=1e-8, atol=1e-12,
                                       err_msg=f"params {upd} {t}")


def test_rollout_graph_replay_matches_plain_launches(monkeypatch):
    """collect_rollout replayed from its captured CUDA graph (seed / update read
    from device memory, odd T flipping the hidden-buffer parity, weights
    re-uploaded and PPO-updated between rollouts) equals plain launches."""
    from oracle.oracle import Oracle
    from tests.common import rollout_case
    orc = Oracle("orc")
    cfg, synth_kw, nets = rollout_case(orc)
    envs = []
    for _ in range(2):
        v = MarketVecEnv(dev_store(synth_kw), cfg, seed=3, n_envs=7)
        v.reset_all()
        v.set_nets(nets)
        envs.append(v)
    outs = [[], []]
    for i, v in enumerate(envs):
        if i == 1:
            monkeypatch.setenv("MLOB_NO_GRAPH", "1")
        for upd, T in ((1, 5), (2, 5), (3, 6), (4, 5)):
            v.collect_rollout(T, 0.99, 0.95, seed=11, update_index=upd)
            outs[i] += [v.rollout(t, f).tobytes() for t in range(2) for f in range(11)]
            if upd == 2:
                v.ppo_update(0, abi.ppo_config(epochs=1, minibatches=1), seed=5, update_index=upd)
        monkeypatch.delenv("MLOB_NO_GRAPH", raising=False)
    assert outs[0] == outs[1]


@pytest.mark.parametrize("workload", ["C", "D", "E"])
def test_bench_workload_sampled_envs_match_oracle(orc, workload):
    """Full bench sizes (config C: 65,536 envs; config D's shape: 262,144
    deep-book envs, untrimmed store; config E: 2^20 envs): the whole batch steps through the bench
    harness (device-drawn actions, bench.hpp:53-70) across an episode
    boundary; sampled envs — block-round edges, the middle, the last, random
    picks — are replayed one by one in the oracle and compared bit-exactly."""
    import bench
    n, cfg, synth, _ = bench.workload(workload)
    dev = DeviceStore(HostStore.synth(synth, 0), 0)
    ost = orc.synth(synth, 0)
    g = MarketVecEnv(dev, cfg, seed=0, n_envs=n)
    g.reset_all()
    T = cfg.steps_per_episode + 6
    for s in range(T):
        g.step_random(0, s)
    arities = [abi.action_arity(cfg.specs[t]) for t in abi.flat_specs(cfg)]
    rng = np.random.default_rng(7)
    sample = sorted({0, 1, 31, 3551, 3552, n // 2, n - 2, n - 1,
                     *rng.integers(0, n, size=4).tolist()})
    for e in sample:
        o = OEnv(orc, ost, cfg, 0, e)
        n_ep = o.n_episodes
        o.reset(e % n_ep)
        cursor = 1
        for s in range(T):
            o.step_ids(kat.bench_actions(0, e, s, arities))
            if o.scalars().terminal:
                o.reset((e + cursor * n) % n_ep)
                cursor += 1
        compare_env_state(g.view(e), o, trades=False)  # the bench runs without the trade log


@pytest.mark.parametrize("scenario", ["mm_fixed_exec", "deep_evict"])
def test_step_io_chunked_matches_oracle(orc, scenario, monkeypatch):
    """mlob_venv_step_io split into env chunks on two streams (every per-env
    hand-off buffer offset by the chunk, the fill-overflow pool shared out per
    chunk), for a register book and a 4-word-slot deep book, across an
    episode boundary: every env equals its oracle replay (MarketVecEnv
    auto-reset, rollout.hpp:290-318)."""
    monkeypatch.setenv("MLOB_IO_CHUNKS", "3")
    cfg, synth_kw, _ = scenario_configs()[scenario]
    dev = dev_store(synth_kw)
    ost = small_store(orc, synth_kw)
    n = 9
    g = MarketVecEnv(dev, cfg, seed=4, n_envs=n)
    g.reset_all()
    refs = [OEnv(orc, ost, cfg, 4, e) for e in range(n)]
    n_ep = refs[0].n_episodes
    for e, r in enumerate(refs):
        r.reset(e % n_ep)
    cursor = [1] * n
    arities = [abi.action_arity(cfg.specs[t]) for t in abi.flat_specs(cfg)]
    rew = np.zeros((n, g.n_agents))
    dn = np.zeros((n, g.n_agents), dtype=np.uint8)
    for t in range(cfg.steps_per_episode + 3):
        acts = np.array([kat.bench_actions(0, e, t, arities) for e in range(n)], dtype=np.int32)
        g.step_io(actions=acts, rewards=rew, dones=dn)
        for e, r in enumerate(refs):
            r.step_ids(list(acts[e]))
            for a in range(g.n_agents):
                assert rew[e, a] == r.reward(a) and dn[e, a] == r.done(a)
            if r.scalars().terminal:  # the device env has auto-reset already
                r.reset((e + cursor[e] * n) % n_ep)
                cursor[e] += 1
                for side in (0, 1):
                    assert g.view(e).book(side).tobytes() == r.book(side).tobytes()
            else:
                compare_env_state(g.view(e), r, trades=False)


@pytest.mark.parametrize("n", [6, 5000])
def test_trade_log_instantiation_gate(n):
    """The trade log is its own book_kernel instantiation (REC = true when
    MLOB_VENV_RECORD_TRADES is set): both instantiations evolve identical
    books (one round of warps, and 5,000 envs: more envs than one round of
    the persistent grid); the one without the log refuses
    mlob_venv_read_trades (MarketEnv::step_trades, env.hpp:139-141), the
    other returns the step's TradeRecords."""
    cfg, synth_kw, _ = scenario_configs()["mm_fixed_exec"]
    dev = dev_store(synth_kw)
    plain = MarketVecEnv(dev, cfg, seed=2, n_envs=n)
    logged = MarketVecEnv(dev, cfg, seed=2, n_envs=n, record_trades=True)
    for v in (plain, logged):
        v.reset_all()
    n_trades = 0
    for t in range(cfg.steps_per_episode - 1):
        for v in (plain, logged):
            v.step_random(3, t)
        for e in (range(n) if n <= 64 else sorted({0, 1, 4143, 4144, n - 1, *range(0, n, 397)})):
            for side in (0, 1):
                assert plain.view(e).book(side).tobytes() == logged.view(e).book(side).tobytes()
            n_trades += len(logged.view(e).trades())
        assert plain.rewards().tobytes() == logged.rewards().tobytes()
    assert n_trades > 0
    with pytest.raises(LogicError, match="trade log disabled"):
        plain.view(0).trades()
