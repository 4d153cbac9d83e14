"""TEST INFRASTRUCTURE ONLY — Python loader for the parity oracle.

Loads either implementation of oracle/oracle_api.h:
  * ``Oracle("orc")`` — the plain-C restatement (oracle/libmarlob_oracle.so);
  * ``Oracle("ref")`` — the reference headers compiled in place
    (oracle/_ref/libmarlob_ref.so, built from /root/reference by oracle/Makefile).
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2511_02136_b200 import abi
from paper_2511_02136_b200.abi import (AgentAction, AgentInfo, AgentState, EnvConfig,
                                       EnvScalars, EpisodeStats, Level, Message, RestingOrder,
                                       SynthConfig, Trade)

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {"orc": os.path.join(HERE, "libmarlob_oracle.so"),
        "ref": os.path.join(HERE, "_ref", "libmarlob_ref.so")}


class BenchRow(C.Structure):
    _fields_ = [("messages_per_step", C.c_int32), ("agents_per_type", C.c_int32),
                ("workers", C.c_int32), ("_pad", C.c_int32), ("env_steps", C.c_uint64),
                ("messages", C.c_uint64), ("wall_seconds", C.c_double),
                ("steps_per_sec", C.c_double), ("messages_per_sec", C.c_double),
                ("worker_utilization", C.c_double)]


class StreamConfig(C.Structure):
    _fields_ = [("n_messages", C.c_uint64), ("initial_ref", C.c_int64), ("band", C.c_int32),
                ("_pad", C.c_int32), ("max_qty", C.c_int64), ("p_new", C.c_double),
                ("p_marketable", C.c_double), ("p_cancel", C.c_double),
                ("p_delete", C.c_double), ("p_execute", C.c_double), ("p_absent", C.c_double)]


def stream_config(**kw) -> StreamConfig:
    """testing::RandomStreamConfig defaults, tests/reference/random_messages.hpp:16-28."""
    c = StreamConfig(100000, 10000, 25, 0, 50, 0.40, 0.35, 0.16, 0.26, 0.10, 0.05)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def build(force: bool = False) -> None:
    """Builds the oracle libraries (no-op when present and not forced)."""
    if force or not all(os.path.exists(p) for p in LIBS.values()):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


class OracleError(Exception):
    pass


_EXC = {abi.MLOB_E_INVALID_ARGUMENT: ValueError, abi.MLOB_E_OUT_OF_RANGE: IndexError,
        abi.MLOB_E_LOGIC: RuntimeError, abi.MLOB_E_RUNTIME: RuntimeError}

_P = C.POINTER
_SIG = {
    "last_error": (C.c_char_p, []),
    "store_synth": (C.c_void_p, [_P(SynthConfig), C.c_uint64]),
    "store_create": (C.c_void_p, [_P(Message), C.c_uint64, _P(abi.BookStates)]),
    "store_n_messages": (C.c_uint64, [C.c_void_p]),
    "store_messages": (_P(Message), [C.c_void_p]),
    "store_n_states": (C.c_uint64, [C.c_void_p]),
    "store_state": (C.c_int, [C.c_void_p, C.c_uint64, _P(C.c_uint64), _P(Level), _P(C.c_uint32),
                              _P(Level), _P(C.c_uint32), C.c_uint32]),
    "store_free": (None, [C.c_void_p]),
    "load_lobster": (C.c_void_p, [C.c_char_p, C.c_char_p, C.c_int64, C.c_uint64, _P(C.c_int)]),
    "book_create": (C.c_void_p, [C.c_uint64]),
    "book_init_from_l2": (C.c_int, [C.c_void_p, _P(Level), C.c_uint32, _P(Level), C.c_uint32,
                                    C.c_uint64]),
    "book_process": (C.c_uint64, [C.c_void_p, _P(Message), _P(Trade), C.c_uint64]),
    "book_orders": (C.c_uint64, [C.c_void_p, C.c_int, _P(RestingOrder), C.c_uint64]),
    "book_next_seq": (C.c_uint64, [C.c_void_p]),
    "book_mid_half": (C.c_int64, [C.c_void_p, C.c_int64]),
    "book_l2": (None, [C.c_void_p, C.c_uint64, _P(Level), _P(C.c_uint32), _P(Level),
                       _P(C.c_uint32)]),
    "book_free": (None, [C.c_void_p]),
    "env_create": (C.c_void_p, [C.c_void_p, _P(EnvConfig), C.c_uint64, C.c_int, _P(C.c_int)]),
    "env_n_episodes": (C.c_uint64, [C.c_void_p]),
    "env_episode_start": (C.c_uint64, [C.c_void_p, C.c_uint64]),
    "env_n_agents": (C.c_int, [C.c_void_p]),
    "env_reset": (C.c_int, [C.c_void_p, C.c_uint64]),
    "env_step_ids": (C.c_int, [C.c_void_p, _P(C.c_int32), C.c_uint64]),
    "env_step": (C.c_int, [C.c_void_p, _P(AgentAction), C.c_uint64]),
    "env_scalars": (None, [C.c_void_p, _P(EnvScalars)]),
    "env_book": (C.c_uint64, [C.c_void_p, C.c_int, _P(RestingOrder), C.c_uint64]),
    "env_agent": (None, [C.c_void_p, C.c_int, _P(AgentState)]),
    "env_info": (None, [C.c_void_p, C.c_int, _P(AgentInfo)]),
    "env_reward": (C.c_double, [C.c_void_p, C.c_int]),
    "env_done": (C.c_int, [C.c_void_p, C.c_int]),
    "env_obs": (C.c_uint64, [C.c_void_p, C.c_int, _P(C.c_double), C.c_uint64]),
    "env_trades": (C.c_uint64, [C.c_void_p, _P(Trade), C.c_uint64]),
    "env_free": (None, [C.c_void_p]),
    "venv_create": (C.c_void_p, [C.c_void_p, _P(EnvConfig), _P(C.c_uint64), C.c_uint64,
                                 C.c_uint64, C.c_int, C.c_int, _P(C.c_int)]),
    "venv_reset_all": (C.c_int, [C.c_void_p]),
    "venv_set_action": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.c_int]),
    "venv_step_all": (C.c_int, [C.c_void_p]),
    "venv_gather": (None, [C.c_void_p, C.c_int, _P(C.c_double), _P(C.c_uint8)]),
    "venv_reward": (C.c_double, [C.c_void_p, C.c_int, C.c_uint64]),
    "venv_done": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64]),
    "venv_episode_stats": (None, [C.c_void_p, C.c_int, _P(EpisodeStats)]),
    "venv_clear_episode_stats": (None, [C.c_void_p]),
    "venv_instance": (C.c_void_p, [C.c_void_p, C.c_uint64]),
    "venv_free": (None, [C.c_void_p]),
    "bench_run": (C.c_int, [C.c_void_p, _P(EnvConfig), C.c_int, C.c_int, C.c_int, C.c_int,
                            C.c_uint64, C.c_int, C.c_int, _P(BenchRow)]),
    "random_stream": (None, [_P(StreamConfig), C.c_uint64, _P(Message)]),
    "make_policy_net": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, _P(C.c_double)]),
    "venv_collect_rollout": (C.c_int, [C.c_void_p, _P(abi.PolicyNetC), _P(abi.RolloutConfig),
                                       C.c_uint64]),
    "venv_rollout_field": (C.c_uint64, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_uint64]),
    "evaluate_matrix": (C.c_int, [C.c_void_p, _P(EnvConfig), _P(C.c_uint64), C.c_uint64,
                                  _P(abi.Policy), C.c_int, _P(abi.Policy), C.c_int, C.c_uint64,
                                  _P(abi.CellStats)]),
}
_REF_ONLY = {
    "venv_ppo_update": (C.c_int, [C.c_void_p, C.c_int, _P(abi.PpoConfig), C.c_uint64, C.c_uint64,
                                  _P(abi.UpdateMetrics)]),
    "venv_read_net": (C.c_uint64, [C.c_void_p, C.c_int, _P(C.c_double), C.c_uint64]),
    "naive_create": (C.c_void_p, []),
    "naive_process": (C.c_uint64, [C.c_void_p, _P(Message), _P(Trade), C.c_uint64]),
    "naive_best": (C.c_int, [C.c_void_p, C.c_int, _P(C.c_int64)]),
    "naive_l2_full": (C.c_uint32, [C.c_void_p, C.c_int, _P(Level), C.c_uint32]),
    "naive_free": (None, [C.c_void_p]),
}
_ORC_ONLY = {
    "splitmix64": (C.c_uint64, [C.c_uint64]),
    "make_key": (C.c_uint64, [C.c_uint64, C.c_int, _P(C.c_uint64)]),
    "crng_draws": (None, [C.c_uint64, C.c_uint64, _P(C.c_uint64)]),
    "choose_action": (C.c_int, [C.c_void_p, C.c_int, _P(abi.Policy), C.c_int, C.c_uint64,
                                C.c_uint64, C.c_uint64, _P(AgentAction)]),
}

_cache: dict[str, "Oracle"] = {}


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


class Oracle:
    """Thin ctypes facade over one oracle implementation ("orc" or "ref")."""

    def __new__(cls, kind: str = "orc"):
        if kind in _cache:
            return _cache[kind]
        self = super().__new__(cls)
        if not available(kind):
            build()
        self.kind = kind
        self.lib = C.CDLL(LIBS[kind])
        sigs = dict(_SIG)
        sigs.update(_REF_ONLY if kind == "ref" else _ORC_ONLY)
        for name, (res, args) in sigs.items():
            fn = getattr(self.lib, f"{kind}_{name}")
            fn.restype = res
            fn.argtypes = args
            setattr(self, name + "_" if name == "make_policy_net" else name, fn)
        _cache[kind] = self
        return self

    def check(self, rc: int) -> None:
        if rc != abi.MLOB_OK:
            raise _EXC.get(rc, OracleError)(self.last_error().decode())

    def make_policy_net(self, obs_dim: int, hidden: int, n_actions: int, seed: int) -> abi.NetParams:
        """ippo::make_policy_net (net.hpp:80-104)."""
        out = np.zeros(abi.NetParams.param_count(obs_dim, hidden, n_actions), dtype=np.float64)
        self.check(self.make_policy_net_(obs_dim, hidden, n_actions, seed,
                                         out.ctypes.data_as(_P(C.c_double))))
        return abi.NetParams(obs_dim, hidden, n_actions, out)

    def evaluate(self, store: "OStore", cfg: EnvConfig, episodes, type0, type1, seed: int):
        """evaluate_matrix (evaluate.hpp:104-217) -> list of CellStats, row-major."""
        eps = np.ascontiguousarray(episodes, dtype=np.uint64)
        t0 = (abi.Policy * max(1, len(type0)))(*type0)
        t1 = (abi.Policy * max(1, len(type1)))(*type1)
        out = (abi.CellStats * max(1, len(type0) * len(type1)))()
        self.check(self.evaluate_matrix(store.h, C.byref(cfg), eps.ctypes.data_as(_P(C.c_uint64)),
                                        len(eps), t0, len(type0), t1, len(type1), seed, out))
        return list(out)[:len(type0) * len(type1)]

    # ---- stores ----
    def synth(self, cfg: SynthConfig, seed: int) -> "OStore":
        h = self.store_synth(C.byref(cfg), seed)
        if not h:
            raise ValueError(self.last_error().decode())
        return OStore(self, h)

    def lobster(self, message_path: str, orderbook_path: str, units_per_tick: int,
                sample_every: int) -> "OStore":
        """data::load_lobster (lobster.hpp:119-193)."""
        st = C.c_int()
        h = self.load_lobster(str(message_path).encode(), str(orderbook_path).encode(), units_per_tick,
                              sample_every, C.byref(st))
        self.check(st.value)
        return OStore(self, h)

    def store_from(self, msgs: np.ndarray, states=None) -> "OStore":
        """msgs: structured array of Message records; states: list of
        (message_index, [(p,q)...] bids, [(p,q)...] asks)."""
        msgs = np.ascontiguousarray(msgs)
        bs, keep = make_book_states(states or [])
        h = self.store_create(msgs.ctypes.data_as(C.POINTER(Message)), len(msgs), C.byref(bs))
        return OStore(self, h)


# Record dtypes with explicit padding fields so tobytes() is fully defined.
MESSAGE_DTYPE = np.dtype([("time", "<i8"), ("order_id", "<u8"), ("price", "<i8"),
                          ("quantity", "<i8"), ("kind", "u1"), ("side", "u1"), ("_pad", "V2"),
                          ("trader_id", "<i4")])
TRADE_DTYPE = np.dtype([("price", "<i8"), ("quantity", "<i8"), ("time", "<i8"),
                        ("passive_order_id", "<u8"), ("aggressor_order_id", "<u8"),
                        ("passive_trader_id", "<i4"), ("aggressor_trader_id", "<i4"),
                        ("aggressor_side", "u1"), ("_pad", "V7")])
ORDER_DTYPE = np.dtype([("price", "<i8"), ("quantity", "<i8"), ("order_id", "<u8"),
                        ("arrival_seq", "<u8"), ("trader_id", "<i4"), ("_pad", "<i4")])


def make_book_states(states):
    """Flattens [(message_index, bids, asks), ...] into an mlob_book_states
    (returns the struct and the arrays it points into)."""
    n = len(states)
    mi = np.array([s[0] for s in states], dtype=np.uint64)
    nb = np.array([len(s[1]) for s in states], dtype=np.uint32)
    off = np.zeros(n + 1, dtype=np.uint64)
    lv = []
    for i, (_, b, a) in enumerate(states):
        lv += list(b) + list(a)
        off[i + 1] = off[i] + len(b) + len(a)
    levels = np.array(lv if lv else [(0, 0)], dtype=np.int64).reshape(-1, 2)
    levels = np.ascontiguousarray(levels)
    bs = abi.BookStates()
    bs.n_states = n
    bs.message_index = mi.ctypes.data_as(C.POINTER(C.c_uint64))
    bs.level_offset = off.ctypes.data_as(C.POINTER(C.c_uint64))
    bs.n_bids = nb.ctypes.data_as(C.POINTER(C.c_uint32))
    bs.levels = levels.ctypes.data_as(C.POINTER(Level))
    return bs, (mi, nb, off, levels)


class OStore:
    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h

    def __del__(self):
        if getattr(self, "h", None):
            self.o.store_free(self.h)
            self.h = None

    @property
    def n_messages(self) -> int:
        return self.o.store_n_messages(self.h)

    def messages(self) -> np.ndarray:
        n = self.n_messages
        p = self.o.store_messages(self.h)
        buf = (C.c_char * (n * 40)).from_address(C.addressof(p.contents)) if n else b""
        return np.frombuffer(bytes(buf), dtype=MESSAGE_DTYPE).copy()

    def states(self, cap: int = 4096):
        out = []
        bids, asks = (Level * cap)(), (Level * cap)()
        mi, nb, na = C.c_uint64(), C.c_uint32(), C.c_uint32()
        for i in range(self.o.store_n_states(self.h)):
            self.o.check(self.o.store_state(self.h, i, C.byref(mi), bids, C.byref(nb), asks,
                                            C.byref(na), cap))
            out.append((mi.value, [(bids[k].price, bids[k].quantity) for k in range(nb.value)],
                        [(asks[k].price, asks[k].quantity) for k in range(na.value)]))
        return out


def _records(arr, n, dtype):
    return np.frombuffer(bytes(arr)[: n * dtype.itemsize], dtype=dtype).copy()


class OBook:
    def __init__(self, o: Oracle, capacity: int):
        self.o = o
        self.h = o.book_create(capacity)
        if not self.h:
            raise ValueError(o.last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.o.book_free(self.h)

    def init_from_l2(self, bids, asks, id_base):
        b = (Level * max(1, len(bids)))(*[Level(*x) for x in bids])
        a = (Level * max(1, len(asks)))(*[Level(*x) for x in asks])
        self.o.check(self.o.book_init_from_l2(self.h, b, len(bids), a, len(asks), id_base))

    def process(self, m) -> np.ndarray:
        msg = m if isinstance(m, Message) else Message(int(m["time"]), int(m["order_id"]),
                                                          int(m["price"]), int(m["quantity"]),
                                                          int(m["kind"]), int(m["side"]),
                                                          (C.c_uint8 * 2)(), int(m["trader_id"]))
        cap = 4096
        out = (Trade * cap)()
        n = self.o.book_process(self.h, C.byref(msg), out, cap)
        return _records(out, n, TRADE_DTYPE)

    def orders(self, side) -> np.ndarray:
        cap = 1 << 16
        out = (RestingOrder * cap)()
        n = self.o.book_orders(self.h, side, out, cap)
        return _records(out, n, ORDER_DTYPE)

    @property
    def next_seq(self):
        return self.o.book_next_seq(self.h)

    def mid_half(self, fallback):
        return self.o.book_mid_half(self.h, fallback)

    def l2(self, depth):
        b, a = (Level * (depth + 1))(), (Level * (depth + 1))()
        nb, na = C.c_uint32(), C.c_uint32()
        self.o.book_l2(self.h, depth, b, C.byref(nb), a, C.byref(na))
        return ([(b[i].price, b[i].quantity) for i in range(nb.value)],
                [(a[i].price, a[i].quantity) for i in range(na.value)])


class OEnv:
    """One MarketEnv instance (env/env.hpp:98-282) in either oracle."""

    def __init__(self, o: Oracle, store: OStore, cfg: EnvConfig, seed: int, env_index: int,
                 handle=None):
        self.o, self.store, self.cfg = o, store, cfg
        if handle is not None:
            self.h, self.owned = handle, False
        else:
            st = C.c_int()
            self.h = o.env_create(store.h, C.byref(cfg), seed, env_index, C.byref(st))
            o.check(st.value)
            self.owned = True
        self.n_agents = o.env_n_agents(self.h)
        self.flat = abi.flat_specs(cfg)

    def __del__(self):
        if getattr(self, "h", None) and getattr(self, "owned", False):
            self.o.env_free(self.h)
            self.h = None

    @property
    def n_episodes(self):
        return self.o.env_n_episodes(self.h)

    def reset(self, episode: int):
        self.o.check(self.o.env_reset(self.h, episode))

    def step_ids(self, ids):
        arr = (C.c_int32 * max(1, len(ids)))(*ids)
        self.o.check(self.o.env_step_ids(self.h, arr, len(ids)))

    def policy_action(self, a: int, pol, step: int, seed: int, cell: int, episode: int):
        """choose_action (evaluate.hpp:56-99) for a scripted policy (orc only)."""
        out = AgentAction()
        self.o.check(self.o.choose_action(self.h, a, C.byref(pol), step, seed, cell, episode,
                                          C.byref(out)))
        return out

    def step(self, actions):
        arr = (AgentAction * max(1, len(actions)))(*actions)
        self.o.check(self.o.env_step(self.h, arr, len(actions)))

    def scalars(self) -> EnvScalars:
        s = EnvScalars()
        self.o.env_scalars(self.h, C.byref(s))
        return s

    def book(self, side) -> np.ndarray:
        cap = 1 << 16
        out = (RestingOrder * cap)()
        n = self.o.env_book(self.h, side, out, cap)
        return _records(out, n, ORDER_DTYPE)

    def agent(self, a) -> AgentState:
        s = AgentState()
        self.o.env_agent(self.h, a, C.byref(s))
        return s

    def info(self, a) -> AgentInfo:
        s = AgentInfo()
        self.o.env_info(self.h, a, C.byref(s))
        return s

    def reward(self, a) -> float:
        return self.o.env_reward(self.h, a)

    def done(self, a) -> int:
        return self.o.env_done(self.h, a)

    def obs(self, a) -> np.ndarray:
        out = (C.c_double * 512)()
        n = self.o.env_obs(self.h, a, out, 512)
        return np.array(out[:n], dtype=np.float64)

    def trades(self) -> np.ndarray:
        n = self.o.env_trades(self.h, None, 0)
        out = (Trade * max(1, n))()
        self.o.env_trades(self.h, out, n)
        return _records(out, n, TRADE_DTYPE)


class OVecEnv:
    """ippo::MarketVecEnv (rollout.hpp:151-336) in either oracle."""

    def __init__(self, o: Oracle, store: OStore, cfg: EnvConfig, seed: int, n_envs: int,
                 pool=None, workers: int = 1):
        self.o, self.store, self.cfg = o, store, cfg
        st = C.c_int()
        p = None
        if pool is not None:
            self._pool = (C.c_uint64 * len(pool))(*pool)
            p = self._pool
        self.h = o.venv_create(store.h, C.byref(cfg), p, len(pool) if pool else 0, seed, n_envs,
                               workers, C.byref(st))
        o.check(st.value)
        self.n_envs = n_envs

    def __del__(self):
        if getattr(self, "h", None):
            self.o.venv_free(self.h)
            self.h = None

    def reset_all(self):
        self.o.check(self.o.venv_reset_all(self.h))

    def set_action(self, t, s, a):
        self.o.check(self.o.venv_set_action(self.h, t, s, a))

    def step_all(self):
        self.o.check(self.o.venv_step_all(self.h))

    def collect_rollout(self, nets, rollout_len: int, discount: float, gae_lambda: float,
                        seed: int, update_index: int):
        """ippo::collect_rollout (rollout.hpp:41-124); nets: one abi.NetParams per type."""
        arr = None if nets is None else (abi.PolicyNetC * len(nets))(*[n.to_c() for n in nets])
        c = abi.RolloutConfig(rollout_len=rollout_len, discount=discount, gae_lambda=gae_lambda,
                              seed=seed)
        self.o.check(self.o.venv_collect_rollout(self.h, arr, C.byref(c), update_index))

    def ppo_update(self, t: int, cfg, seed: int, update_index: int):
        """ippo::ppo_update (ppo.hpp:263-310) of type t (reference only)."""
        m = abi.UpdateMetrics()
        self.o.check(self.o.venv_ppo_update(self.h, t, C.byref(cfg), seed, update_index, C.byref(m)))
        return m

    def read_net(self, t: int) -> np.ndarray:
        n = self.o.venv_read_net(self.h, t, None, 0)
        out = np.zeros(n, dtype=np.float64)
        self.o.venv_read_net(self.h, t, out.ctypes.data_as(_P(C.c_double)), n)
        return out

    def rollout(self, t: int, field: int) -> np.ndarray:
        n = self.o.venv_rollout_field(self.h, t, field, None, 0)
        out = np.zeros(n, dtype=np.uint8)
        self.o.venv_rollout_field(self.h, t, field, out.ctypes.data, n)
        return out.view(abi.RB_DTYPES[field])

    def gather(self, t):
        count = self.cfg.specs[t].count
        dim = abi.observation_size(self.cfg.specs[t].obs_space, self.cfg.obs_depth)
        n = self.n_envs * count
        obs = np.zeros(n * dim, dtype=np.float64)
        rs = np.zeros(n, dtype=np.uint8)
        self.o.venv_gather(self.h, t, obs.ctypes.data_as(C.POINTER(C.c_double)),
                           rs.ctypes.data_as(C.POINTER(C.c_uint8)))
        return obs.reshape(n, dim), rs

    def reward(self, t, s):
        return self.o.venv_reward(self.h, t, s)

    def done(self, t, s):
        return self.o.venv_done(self.h, t, s)

    def episode_stats(self, t) -> EpisodeStats:
        s = EpisodeStats()
        self.o.venv_episode_stats(self.h, t, C.byref(s))
        return s

    def clear_episode_stats(self):
        self.o.venv_clear_episode_stats(self.h)

    def instance(self, e) -> OEnv:
        return OEnv(self.o, self.store, self.cfg, 0, 0, handle=self.o.venv_instance(self.h, e))


def bench_run(o: Oracle, store: OStore, cfg: EnvConfig, n_envs: int, n_steps: int, warmup: int,
              workers: int, seed: int, messages_per_step: int, agents_per_type: int) -> BenchRow:
    row = BenchRow()
    o.check(o.bench_run(store.h, C.byref(cfg), n_envs, n_steps, warmup, workers, seed,
                        messages_per_step, agents_per_type, C.byref(row)))
    return row


def random_stream(o: Oracle, seed: int, **kw) -> np.ndarray:
    cfg = stream_config(**kw)
    out = np.zeros(cfg.n_messages, dtype=MESSAGE_DTYPE)
    o.random_stream(C.byref(cfg), seed, out.ctypes.data_as(C.POINTER(Message)))
    return out


def dup_id_stream(o: Oracle, seed: int, n_ids: int = 5, **kw) -> np.ndarray:
    """A random_stream whose order ids are folded onto n_ids values, so resting
    orders share ids and cancels / deletes / executes hit duplicate live ids
    (the first-match-in-storage-order rule of book.hpp:191-206)."""
    msgs = random_stream(o, seed, **kw).copy()
    msgs["order_id"] = msgs["order_id"] % n_ids + 1
    return msgs


def fnv1a(data: bytes, h: int = 1469598103934665603) -> int:
    """FNV-1a 64 (SURVEY §8c digest recipe)."""
    for b in data:
        h ^= b
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def trade_bytes(trades: np.ndarray) -> bytes:
    """Digest byte layout of a trade list: price, qty, time (i64), passive, aggressor id
    (u64), passive/aggressor trader (i32), (int)aggressor_side (i32)."""
    rec = np.zeros(len(trades), dtype=[("p", "<i8"), ("q", "<i8"), ("t", "<i8"), ("pi", "<u8"),
                                       ("ai", "<u8"), ("pt", "<i4"), ("at", "<i4"),
                                       ("s", "<i4")])
    rec["p"], rec["q"], rec["t"] = trades["price"], trades["quantity"], trades["time"]
    rec["pi"], rec["ai"] = trades["passive_order_id"], trades["aggressor_order_id"]
    rec["pt"], rec["at"] = trades["passive_trader_id"], trades["aggressor_trader_id"]
    rec["s"] = trades["aggressor_side"]
    return rec.tobytes()


def book_bytes(bids: np.ndarray, asks: np.ndarray, next_seq: int) -> bytes:
    out = b""
    for side in (bids, asks):
        rec = np.zeros(len(side), dtype=[("p", "<i8"), ("q", "<i8"), ("i", "<u8"), ("s", "<u8"),
                                         ("t", "<i4")])
        rec["p"], rec["q"], rec["i"] = side["price"], side["quantity"], side["order_id"]
        rec["s"], rec["t"] = side["arrival_seq"], side["trader_id"]
        out += rec.tobytes()
    return out + np.uint64(next_seq).tobytes()
