"""Shared test scenarios and comparators (used by the oracle tests and the GPU
parity tests alike)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2511_02136_b200 import abi

INT64_MIN = -(1 << 63)


def small_store(o, synth_kw, seed=0):
    kw = {"n_messages": 20000, "state_sample_every": 100}
    kw.update(synth_kw)
    return o.synth(abi.synth_config(**kw), seed)


DEEP_SYNTH = {"initial_mid": 100000, "band": 2000, "p_new_passive": 0.46, "p_new_cross": 0.04,
              "p_cancel": 0.30, "p_delete": 0.16, "p_execute": 0.02, "state_depth": 1000}


def scenario_configs():
    """name -> (EnvConfig, synth kwargs, steps per episode run)."""
    A = abi
    mm = A.agent_spec(A.MARKET_MAKER)
    ex = A.agent_spec(A.EXECUTOR)
    out = {}
    out["mm_fixed_exec"] = (A.env_config([mm, ex], steps_per_episode=20, messages_per_step=100,
                                         start_stride_steps=20), {}, 20)
    out["spread_buysell_full"] = (A.env_config(
        [A.agent_spec(A.MARKET_MAKER, mm_space=A.SPREAD_SKEW, obs_space=A.OBS_MM_FULL,
                      reward=A.REWARD_BUYSELL, ref_price=A.REF_FAR_TOUCH, quadratic_penalty=0,
                      reward_scale=0.01),
         A.agent_spec(A.EXECUTOR, task_size=120, reward_scale=0.001, ref_price=A.REF_FAR_TOUCH)],
        steps_per_episode=16, messages_per_step=50, start_stride_steps=8, obs_depth=3), {}, 16)
    out["avst_spooner"] = (A.env_config(
        [A.agent_spec(A.MARKET_MAKER, mm_space=A.AVST, lambda_=0.2, order_size=7),
         A.agent_spec(A.MARKET_MAKER, mm_space=A.FIXED_QUANT, fixed_quant_from_mid=1)],
        steps_per_episode=24, messages_per_step=25, start_stride_steps=24), {}, 24)
    out["directional_simple_exec"] = (A.env_config(
        [A.agent_spec(A.DIRECTIONAL), A.agent_spec(A.EXECUTOR, exec_complex=0, task_size=40,
                                                   order_size=3)],
        steps_per_episode=12, messages_per_step=10, start_stride_steps=12),
        {"state_sample_every": 40}, 12)
    out["small_capacity_eviction"] = (A.env_config(
        [A.agent_spec(A.MARKET_MAKER, count=2), A.agent_spec(A.EXECUTOR, count=2)],
        steps_per_episode=10, messages_per_step=40, start_stride_steps=10, book_capacity=6,
        obs_depth=2), {"state_depth": 5}, 10)
    out["zero_agents"] = (A.env_config([], steps_per_episode=16, messages_per_step=100,
                                       start_stride_steps=16), {}, 16)
    out["one_msg_per_step"] = (A.env_config([mm, ex], steps_per_episode=64, messages_per_step=1,
                                            start_stride_steps=64),
                               {"state_sample_every": 64}, 64)
    out["many_agents"] = (A.env_config(
        [A.agent_spec(A.MARKET_MAKER, count=5), A.agent_spec(A.EXECUTOR, count=5, task_size=200)],
        steps_per_episode=10, messages_per_step=100, start_stride_steps=10), {}, 10)
    # 200 msgs/step (two replay chunks), MMFull at depth 64, 8 agents: ~15 KB of
    # shared memory per warp forces the step kernel below its full block width
    out["wide_smem"] = (A.env_config(
        [A.agent_spec(A.MARKET_MAKER, count=4, obs_space=A.OBS_MM_FULL),
         A.agent_spec(A.EXECUTOR, count=4, task_size=300)],
        steps_per_episode=5, messages_per_step=200, start_stride_steps=5, obs_depth=64),
        {"state_sample_every": 1000, "n_messages": 40000}, 5)
    # shared-memory book (capacity 300 -> 16 rows/lane) that runs full: every
    # better-priced newcomer evicts (book.hpp:174-181) through the cached worst
    out["deep_evict"] = (A.env_config([mm, ex], steps_per_episode=16, messages_per_step=100,
                                      start_stride_steps=32, book_capacity=300),
                         dict(DEEP_SYNTH, n_messages=40000, state_sample_every=3200, state_depth=200), 16)
    out["deep_book"] = (A.env_config([mm, ex], steps_per_episode=8, messages_per_step=100,
                                     start_stride_steps=64, book_capacity=1000),
                        dict(DEEP_SYNTH, n_messages=80000, state_sample_every=6400), 8)
    return out


def random_direct_action(rng) -> abi.AgentAction:
    """Direct-quote AgentAction (env.hpp:66-72) with 0-2 random quotes."""
    a = abi.AgentAction()
    a.direct = 1
    a.n_quotes = rng.below(3)
    for i in range(a.n_quotes):
        a.quotes[i].side = rng.below(2)
        a.quotes[i].price = 990 + rng.below(25)
        a.quotes[i].quantity = rng.below(30) - 2
    return a


def compare_env_state(a, b, ref_side=False, trades=True):
    """Bit-exact comparison of every observable of two single-env readers
    (trades=False: a vec env built without the per-step trade log)."""
    sa, sb = a.scalars(), b.scalars()
    for f, _ in abi.EnvScalars._fields_:
        va, vb = getattr(sa, f), getattr(sb, f)
        if f in ("last_bid", "last_ask", "last_time") and INT64_MIN in (va, vb):
            continue
        assert va == vb, (f, va, vb)
    for side in (0, 1):
        ba, bb = a.book(side), b.book(side)
        assert ba.tobytes() == bb.tobytes(), ("book", side, ba, bb)
    if trades:
        ta, tb = a.trades(), b.trades()
        assert ta.tobytes() == tb.tobytes(), ("trades", ta, tb)
    for ag in range(a.n_agents):
        xa, xb = a.agent(ag), b.agent(ag)
        assert bytes(xa) == bytes(xb), ("agent", ag, state_dict(xa), state_dict(xb))
        ia, ib = a.info(ag), b.info(ag)
        assert bytes(ia) == bytes(ib), ("info", ag, struct_dict(ia), struct_dict(ib))
        assert a.reward(ag) == b.reward(ag) or (np.isnan(a.reward(ag)) and np.isnan(b.reward(ag))), \
            ("reward", ag, a.reward(ag), b.reward(ag))
        assert a.done(ag) == b.done(ag)
        oa, ob = a.obs(ag), b.obs(ag)
        assert oa.tobytes() == ob.tobytes(), ("obs", ag, oa, ob)


def struct_dict(s):
    return {f: getattr(s, f) for f, _ in s._fields_ if not f.startswith("_")}


def state_dict(s: abi.AgentState):
    d = struct_dict(s)
    d["active"] = [struct_dict(s.active[i]) for i in range(min(s.n_active, abi.MAX_ACTIVE))]
    return d


def crossplay_case():
    """A two-type cross-play grid over every scripted policy kind
    (evaluate.hpp:17): MM (AvSt space) vs Executor, 3 episodes."""
    A = abi
    cfg = A.env_config([A.agent_spec(A.MARKET_MAKER, count=2, mm_space=A.AVST),
                        A.agent_spec(A.EXECUTOR, task_size=120, order_size=4)],
                       steps_per_episode=12, messages_per_step=25, start_stride_steps=12)
    synth_kw = {"state_sample_every": 25 * 12, "n_messages": 20000}
    type0 = [A.policy(A.POLICY_NOOP), A.policy(A.POLICY_AVST),
             A.policy(A.POLICY_AVST, gamma_index=3, kappa=2.5, sigma=1.0, horizon=12.0),
             A.policy(A.POLICY_RANDOM), A.policy(A.POLICY_TWAP)]
    type1 = [A.policy(A.POLICY_TWAP), A.policy(A.POLICY_TWAP, twap_mode=A.TWAP_PASSIVE),
             A.policy(A.POLICY_RANDOM), A.policy(A.POLICY_NOOP), A.policy(A.POLICY_AVST)]
    return cfg, synth_kw, [2, 0, 5], type0, type1


def rollout_case(o):
    """(cfg, synth kwargs, nets) for rollout parity: MM x2 (FixedQuant) + Executor,
    short episodes so auto-resets fall inside the rollout."""
    A = abi
    cfg = A.env_config([A.agent_spec(A.MARKET_MAKER, count=2), A.agent_spec(A.EXECUTOR)],
                       steps_per_episode=8, messages_per_step=20, start_stride_steps=3)
    nets = [o.make_policy_net(A.observation_size(cfg.specs[0].obs_space, cfg.obs_depth), 16,
                              A.action_arity(cfg.specs[0]), 11),
            o.make_policy_net(A.observation_size(cfg.specs[1].obs_space, cfg.obs_depth), 32,
                              A.action_arity(cfg.specs[1]), 12)]
    return cfg, {"state_sample_every": 20}, nets


def crossplay_learned_case(o):
    """crossplay_case plus Learned options (GRU nets from `o`'s make_policy_net)."""
    A = abi
    cfg, synth_kw, eps, t0, t1 = crossplay_case()
    nets = [o.make_policy_net(A.observation_size(cfg.specs[t].obs_space, cfg.obs_depth), h,
                              A.action_arity(cfg.specs[t]), 40 + t) for t, h in ((0, 16), (1, 32))]
    t0 = [A.policy(A.POLICY_LEARNED, net=nets[0]), t0[1], t0[3]]
    t1 = [t1[0], A.policy(A.POLICY_LEARNED, net=nets[1]), t1[2]]
    return cfg, synth_kw, eps, t0, t1
