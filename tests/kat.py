"""Known-answer digests (SURVEY §8c recipe), computed identically for any
implementation exposing the single-env reader interface (step_ids, trades,
reward, obs, scalars, book): the C restatement, the compiled reference, or the
CUDA product's single-env facade."""
from __future__ import annotations

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def splitmix64(z: int) -> int:
    """core/rng.hpp:11-16"""
    z = (z + GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def make_key(seed: int, *words: int) -> int:
    """core/rng.hpp:18-27"""
    h = splitmix64(seed & M64)
    for w in words:
        w &= M64
        h = splitmix64(h ^ ((w + GAMMA + ((h << 6) & M64) + (h >> 2)) & M64))
    return h


class CounterRng:
    """core/rng.hpp:41-61"""

    def __init__(self, key: int):
        self.state = key

    def next(self) -> int:
        self.state = (self.state + GAMMA) & M64
        return splitmix64(self.state)

    def below(self, n: int) -> int:
        return self.next() % n

    def uniform(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53


BENCH_ACTION = 7


def bench_actions(seed: int, env_index: int, step: int, arities) -> list[int]:
    """bench.hpp:57-60"""
    r = CounterRng(make_key(seed, BENCH_ACTION, env_index, step))
    return [r.below(a) for a in arities]


def env_digest(env, n_steps: int, arities, seed: int = 0, env_index: int = 0) -> dict:
    from oracle.oracle import book_bytes, fnv1a, trade_bytes
    tb = b""
    n_trades = 0
    s_rew = 0.0
    s_obs = 0.0
    for t in range(n_steps):
        env.step_ids(bench_actions(seed, env_index, t, arities))
        tr = env.trades()
        n_trades += len(tr)
        tb += trade_bytes(tr)
        for a in range(len(arities)):
            s_rew += env.reward(a)
            for x in env.obs(a):
                s_obs += float(x)
    s = env.scalars()
    bids, asks = env.book(0), env.book(1)
    return {"messages": int(s.messages_processed), "trades": n_trades,
            "trade_fnv": "%016x" % fnv1a(tb),
            "book_fnv": "%016x" % fnv1a(book_bytes(bids, asks, s.next_seq)),
            "live_bid": len(bids), "live_ask": len(asks), "next_seq": int(s.next_seq),
            "mid_half": int(s.mid_half), "sum_reward": s_rew, "sum_obs": s_obs}


def config_a(name: str):
    """Config A of BASELINE.json / SURVEY §8d: default synth, 10k messages, one
    episode of 100 steps x 100 messages, capacity 100, obs depth 5."""
    from paper_2511_02136_b200 import abi
    synth = abi.synth_config(n_messages=10000, state_sample_every=10000)
    ex = abi.agent_spec(abi.EXECUTOR)
    specs = {"exec_only": [ex], "mm_exec": [abi.agent_spec(abi.MARKET_MAKER), ex]}[name]
    cfg = abi.env_config(specs, steps_per_episode=100, messages_per_step=100,
                         start_stride_steps=100)
    return synth, cfg


def config_a_digest(kind: str, name: str) -> dict:
    from oracle.oracle import OEnv, Oracle
    from paper_2511_02136_b200 import abi
    o = Oracle(kind)
    synth, cfg = config_a(name)
    st = o.synth(synth, 0)
    e = OEnv(o, st, cfg, 0, 0)
    e.reset(0)
    ar = [abi.action_arity(cfg.specs[s]) for s in abi.flat_specs(cfg)]
    return env_digest(e, 100, ar)
