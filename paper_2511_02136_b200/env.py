"""Python host mirror of the reference environment API over the C ABI.

* ``MarketVecEnv`` — ippo::MarketVecEnv (ippo/rollout.hpp:151-336): the VecEnv
  concept (n_types, n_streams, obs_dim, n_actions, reset_all, gather,
  set_action, step_all, reward, done, episode_stats, clear_episode_stats) plus
  batched numpy entry points (set_actions, rewards, dones, infos).
* ``MarketEnvBatch`` / ``EnvView`` — N independent env::MarketEnv instances
  (env/env.hpp:98-282) stepped together; ``EnvView`` exposes one instance's
  reset/step/book/agent_state/output/step_trades readers.
* ``synth_store`` / ``HostStore`` / ``DeviceStore`` — data::synth_generate and
  the device-resident message store.

Every step and reset runs on the GPU through libmlob.so.  There is no CPU
fallback: constructing an environment without the library or without a CUDA
device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi
from .abi import (AgentAction, AgentInfo, AgentState, EnvConfig, EnvScalars, EpisodeStats, Level,
                  Message, RestingOrder, SynthConfig, Trade, VenvDesc)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmlob.so")  # the in-tree product library, nothing else

_EXC = {abi.MLOB_E_INVALID_ARGUMENT: ValueError, abi.MLOB_E_OUT_OF_RANGE: IndexError,
        abi.MLOB_E_LOGIC: RuntimeError, abi.MLOB_E_RUNTIME: RuntimeError,
        abi.MLOB_E_CUDA: RuntimeError}


class LogicError(RuntimeError):
    """std::logic_error (e.g. stepping a terminal env, env.hpp:195)."""


_EXC[abi.MLOB_E_LOGIC] = LogicError

_P = C.POINTER
_vp = C.c_void_p
_SIGS = {
    "mlob_last_error": (C.c_char_p, []),
    "mlob_abi_version": (C.c_int, []),
    "mlob_default_env_config": (None, [_P(EnvConfig)]),
    "mlob_default_agent_spec": (None, [_P(abi.AgentSpec)]),
    "mlob_default_synth_config": (None, [_P(SynthConfig)]),
    "mlob_action_arity": (C.c_int, [_P(abi.AgentSpec)]),
    "mlob_observation_size": (C.c_int, [C.c_int, C.c_uint64]),
    "mlob_validate_env_config": (C.c_int, [_P(EnvConfig)]),
    "mlob_host_store_synth": (C.c_int, [_P(SynthConfig), C.c_uint64, _P(_vp)]),
    "mlob_host_store_create": (C.c_int, [_P(Message), C.c_uint64, _P(abi.BookStates), _P(_vp)]),
    "mlob_host_store_trim_front": (C.c_int, [_vp, C.c_uint64]),
    "mlob_host_store_save": (C.c_int, [_vp, C.c_char_p]),
    "mlob_host_store_load": (C.c_int, [C.c_char_p, _vp]),
    "mlob_host_store_n_messages": (C.c_uint64, [_vp]),
    "mlob_host_store_messages": (_P(Message), [_vp]),
    "mlob_host_store_n_states": (C.c_uint64, [_vp]),
    "mlob_host_store_state": (C.c_int, [_vp, C.c_uint64, _P(C.c_uint64), _P(Level), _P(C.c_uint32),
                                        _P(Level), _P(C.c_uint32), C.c_uint32]),
    "mlob_host_store_free": (None, [_vp]),
    "mlob_build_episode_index": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int, _P(C.c_uint64),
                                           C.c_uint64, _P(C.c_uint64)]),
    "mlob_store_upload": (C.c_int, [_vp, C.c_int, _P(_vp)]),
    "mlob_store_upload_raw": (C.c_int, [_P(Message), C.c_uint64, _P(abi.BookStates), C.c_int,
                                        _P(_vp)]),
    "mlob_store_n_messages": (C.c_uint64, [_vp]),
    "mlob_store_load_lobster": (C.c_int, [C.c_char_p, C.c_char_p, C.c_int64, C.c_uint64, C.c_int,
                                          _P(_vp)]),
    "mlob_store_read_messages": (C.c_int, [_vp, C.c_uint64, C.c_uint64, _P(Message)]),
    "mlob_store_n_states": (C.c_uint64, [_vp]),
    "mlob_store_state": (C.c_int, [_vp, C.c_uint64, _P(C.c_uint64), _P(Level), _P(C.c_uint32),
                                   _P(Level), _P(C.c_uint32), C.c_uint32]),
    "mlob_store_device_bytes": (C.c_uint64, [_vp]),
    "mlob_store_free": (None, [_vp]),
    "mlob_venv_create": (C.c_int, [_P(VenvDesc), _P(_vp)]),
    "mlob_venv_destroy": (None, [_vp]),
    "mlob_venv_n_envs": (C.c_uint64, [_vp]),
    "mlob_venv_n_agents": (C.c_int, [_vp]),
    "mlob_venv_n_types": (C.c_int, [_vp]),
    "mlob_venv_n_streams": (C.c_uint64, [_vp, C.c_int]),
    "mlob_venv_obs_dim": (C.c_int, [_vp, C.c_int]),
    "mlob_venv_n_actions": (C.c_int, [_vp, C.c_int]),
    "mlob_venv_n_episodes": (C.c_uint64, [_vp]),
    "mlob_venv_reset_all": (C.c_int, [_vp]),
    "mlob_venv_reset_envs": (C.c_int, [_vp, _P(C.c_uint64)]),
    "mlob_venv_set_actions": (C.c_int, [_vp, _vp, C.c_int]),
    "mlob_venv_set_direct_actions": (C.c_int, [_vp, _P(AgentAction)]),
    "mlob_venv_step": (C.c_int, [_vp]),
    "mlob_venv_step_random": (C.c_int, [_vp, C.c_uint64, C.c_uint64]),
    "mlob_venv_gather": (C.c_int, [_vp, C.c_int, _vp, _vp]),
    "mlob_venv_obs_device": (_vp, [_vp, C.c_int]),
    "mlob_venv_rewards": (C.c_int, [_vp, _vp]),
    "mlob_venv_dones": (C.c_int, [_vp, _vp]),
    "mlob_venv_rewards_device": (_vp, [_vp]),
    "mlob_venv_dones_device": (_vp, [_vp]),
    "mlob_venv_infos": (C.c_int, [_vp, _vp]),
    "mlob_venv_step_io": (C.c_int, [_vp, _P(abi.StepIO)]),
    "mlob_default_policy": (None, [C.c_int, _P(abi.Policy)]),
    "mlob_venv_set_nets": (C.c_int, [_vp, _P(abi.PolicyNetC)]),
    "mlob_venv_ppo_update": (C.c_int, [_vp, C.c_int, _P(abi.PpoConfig), C.c_uint64, C.c_uint64,
                                       _P(abi.UpdateMetrics)]),
    "mlob_venv_read_net": (C.c_int, [_vp, C.c_int, _P(C.c_double), C.c_uint64]),
    "mlob_default_ppo_config": (None, [_P(abi.PpoConfig)]),
    "mlob_venv_collect_rollout": (C.c_int, [_vp, _P(abi.RolloutConfig), C.c_uint64]),
    "mlob_venv_rollout_read": (C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_uint64]),
    "mlob_venv_rollout_device": (_vp, [_vp, C.c_int, C.c_int]),
    "mlob_venv_set_policies": (C.c_int, [_vp, _P(abi.Policy), C.c_int, _vp, _vp]),
    "mlob_evaluate_matrix": (C.c_int, [_vp, _P(EnvConfig), _P(C.c_uint64), C.c_uint64,
                                       _P(abi.Policy), C.c_int, _P(abi.Policy), C.c_int,
                                       C.c_uint64, C.c_int, _P(abi.CellStats)]),
    "mlob_venv_env_obs": (C.c_int, [_vp, C.c_uint64, _P(C.c_double), C.c_uint64]),
    "mlob_venv_episode_stats": (C.c_int, [_vp, C.c_int, _P(EpisodeStats)]),
    "mlob_venv_episode_stats_device": (C.c_int, [_vp, _vp]),
    "mlob_venv_allreduce_episode_stats": (C.c_int, [_vp, _vp, _vp]),
    "mlob_venv_profile": (C.c_int, [_vp, C.c_int]),
    "mlob_venv_kernel_ms": (C.c_int, [_vp, _vp, _vp]),
    "mlob_venv_clear_episode_stats": (C.c_int, [_vp]),
    "mlob_venv_read_scalars": (C.c_int, [_vp, C.c_uint64, _P(EnvScalars)]),
    "mlob_venv_read_book": (C.c_int, [_vp, C.c_uint64, C.c_int, _P(RestingOrder), C.c_uint64,
                                      _P(C.c_uint64)]),
    "mlob_venv_read_agent": (C.c_int, [_vp, C.c_uint64, C.c_int, _P(AgentState)]),
    "mlob_venv_read_trades": (C.c_int, [_vp, C.c_uint64, _P(Trade), C.c_uint64, _P(C.c_uint64)]),
    "mlob_venv_messages_processed": (C.c_int, [_vp, _P(C.c_uint64)]),
    "mlob_venv_synchronize": (C.c_int, [_vp]),
    "mlob_venv_stream": (_vp, [_vp]),
    "mlob_venv_launch_count": (C.c_uint64, [_vp]),
}

_lib = None


def lib():
    """Loads libmlob.so (built by ``make -C paper_2511_02136_b200`` /
    __graft_entry__.build()); raises if it is missing — no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                               "(the environment step has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.mlob_abi_version() != abi.ABI_VERSION:
            raise RuntimeError("libmlob ABI version mismatch")
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != abi.MLOB_OK:
        raise _EXC.get(rc, RuntimeError)(lib().mlob_last_error().decode())


MESSAGE_DTYPE = np.dtype([("time", "<i8"), ("order_id", "<u8"), ("price", "<i8"),
                          ("quantity", "<i8"), ("kind", "u1"), ("side", "u1"), ("_pad", "V2"),
                          ("trader_id", "<i4")])
TRADE_DTYPE = np.dtype([("price", "<i8"), ("quantity", "<i8"), ("time", "<i8"),
                        ("passive_order_id", "<u8"), ("aggressor_order_id", "<u8"),
                        ("passive_trader_id", "<i4"), ("aggressor_trader_id", "<i4"),
                        ("aggressor_side", "u1"), ("_pad", "V7")])
ORDER_DTYPE = np.dtype([("price", "<i8"), ("quantity", "<i8"), ("order_id", "<u8"),
                        ("arrival_seq", "<u8"), ("trader_id", "<i4"), ("_pad", "<i4")])
INFO_DTYPE = np.dtype([("inventory", "<i8"), ("cash", "<i8"), ("portfolio_value", "<f8"),
                       ("slippage_step", "<f8"), ("slippage_total", "<f8"),
                       ("task_remaining", "<i8"), ("step_filled", "<i8"),
                       ("step_fill_count", "<i4"), ("_pad", "<i4")])


# ---- stores --------------------------------------------------------------------

def _host_ptr(x, dtype, n):
    """Address of a contiguous host buffer of n elements of `dtype` (numpy
    array or CPU torch tensor); None -> NULL."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):  # torch tensor
        if x.is_cuda or not x.is_contiguous() or x.numel() != n or x.element_size() != np.dtype(dtype).itemsize:
            raise ValueError(f"expected a contiguous host tensor of {n} x {np.dtype(dtype)}")
        return x.data_ptr()
    if not isinstance(x, np.ndarray) or not x.flags.c_contiguous or x.size != n or x.dtype != np.dtype(dtype):
        raise ValueError(f"expected a C-contiguous {np.dtype(dtype)} array of {n} elements")
    return x.ctypes.data


class HostStore:
    """data::MessageStore in host memory (contiguous messages + sampled states)."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mlob_host_store_free(self.h)
            self.h = None

    @classmethod
    def synth(cls, cfg: SynthConfig, seed: int) -> "HostStore":
        """data::synth_generate (data/synth.hpp:39-177)."""
        h = _vp()
        _check(lib().mlob_host_store_synth(C.byref(cfg), seed, C.byref(h)))
        return cls(h)

    @classmethod
    def from_messages(cls, msgs: np.ndarray, states=()) -> "HostStore":
        msgs = np.ascontiguousarray(msgs, dtype=MESSAGE_DTYPE)
        bs, keep = make_book_states(states)
        h = _vp()
        _check(lib().mlob_host_store_create(msgs.ctypes.data_as(_P(Message)), len(msgs),
                                            C.byref(bs), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "HostStore":
        """A store saved by save() (one writer per node)."""
        h = _vp()
        _check(lib().mlob_host_store_load(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        _check(lib().mlob_host_store_save(self.h, path.encode()))

    def trim_front(self, n: int) -> None:
        _check(lib().mlob_host_store_trim_front(self.h, n))

    @property
    def n_messages(self) -> int:
        return lib().mlob_host_store_n_messages(self.h)

    def messages(self) -> np.ndarray:
        n = self.n_messages
        if n == 0:
            return np.zeros(0, dtype=MESSAGE_DTYPE)
        p = lib().mlob_host_store_messages(self.h)
        buf = (C.c_char * (n * 40)).from_address(C.addressof(p.contents))
        return np.frombuffer(buf, dtype=MESSAGE_DTYPE).copy()

    def states(self, cap: int = 4096):
        out = []
        b, a = (Level * cap)(), (Level * cap)()
        mi, nb, na = C.c_uint64(), C.c_uint32(), C.c_uint32()
        for i in range(lib().mlob_host_store_n_states(self.h)):
            _check(lib().mlob_host_store_state(self.h, i, C.byref(mi), b, C.byref(nb), a,
                                               C.byref(na), cap))
            out.append((mi.value, [(b[k].price, b[k].quantity) for k in range(nb.value)],
                        [(a[k].price, a[k].quantity) for k in range(na.value)]))
        return out


def make_book_states(states):
    n = len(states)
    mi = np.array([s[0] for s in states], dtype=np.uint64)
    nb = np.array([len(s[1]) for s in states], dtype=np.uint32)
    off = np.zeros(n + 1, dtype=np.uint64)
    lv = []
    for i, (_, b, a) in enumerate(states):
        lv += list(b) + list(a)
        off[i + 1] = off[i] + len(b) + len(a)
    levels = np.ascontiguousarray(np.array(lv if lv else [(0, 0)], dtype=np.int64).reshape(-1, 2))
    bs = abi.BookStates()
    bs.n_states = n
    bs.message_index = mi.ctypes.data_as(_P(C.c_uint64))
    bs.level_offset = off.ctypes.data_as(_P(C.c_uint64))
    bs.n_bids = nb.ctypes.data_as(_P(C.c_uint32))
    bs.levels = levels.ctypes.data_as(_P(Level))
    return bs, (mi, nb, off, levels)


def synth_store(seed: int = 0, **kw) -> HostStore:
    return HostStore.synth(abi.synth_config(**kw), seed)


def episode_index(n_messages: int, steps: int, mps: int, stride: int) -> np.ndarray:
    """data::build_episode_index (data/store.hpp:52-72)."""
    n = C.c_uint64()
    _check(lib().mlob_build_episode_index(n_messages, steps, mps, stride, None, 0, C.byref(n)))
    out = np.zeros(max(1, n.value), dtype=np.uint64)
    _check(lib().mlob_build_episode_index(n_messages, steps, mps, stride,
                                          out.ctypes.data_as(_P(C.c_uint64)), n.value,
                                          C.byref(n)))
    return out[: n.value]


class DeviceStore:
    """The message store resident in HBM (uploaded once, shared read-only)."""

    def __init__(self, host: HostStore, device: int = 0):
        self.h = _vp()
        self.device = device
        _check(lib().mlob_store_upload(host.h, device, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mlob_store_free(self.h)
            self.h = None

    @property
    def n_messages(self) -> int:
        return lib().mlob_store_n_messages(self.h)

    @property
    def device_bytes(self) -> int:
        return lib().mlob_store_device_bytes(self.h)

    @classmethod
    def load_lobster(cls, message_path: str, orderbook_path: str, units_per_tick: int,
                     sample_every: int, device: int = 0) -> "DeviceStore":
        """data::load_lobster (lobster.hpp:119-193) parsed on the GPU straight into HBM."""
        self = cls.__new__(cls)
        self.h = _vp()
        self.device = device
        _check(lib().mlob_store_load_lobster(str(message_path).encode(), str(orderbook_path).encode(),
                                             units_per_tick, sample_every, device, C.byref(self.h)))
        return self

    def messages(self) -> np.ndarray:
        """Device records widened to lob::Message (price / qty as the device keeps them)."""
        n = self.n_messages
        out = np.zeros(n, dtype=MESSAGE_DTYPE)
        if n:
            _check(lib().mlob_store_read_messages(self.h, 0, n, out.ctypes.data_as(_P(Message))))
        return out

    def states(self, cap: int = 4096):
        out = []
        bids, asks = (Level * cap)(), (Level * cap)()
        mi, nb, na = C.c_uint64(), C.c_uint32(), C.c_uint32()
        for i in range(lib().mlob_store_n_states(self.h)):
            _check(lib().mlob_store_state(self.h, i, C.byref(mi), bids, C.byref(nb), asks, C.byref(na), cap))
            out.append((mi.value, [(bids[k].price, bids[k].quantity) for k in range(nb.value)],
                        [(asks[k].price, asks[k].quantity) for k in range(na.value)]))
        return out


# ---- batched environments ------------------------------------------------------

class _Venv:
    def __init__(self, store: DeviceStore, cfg: EnvConfig, n_envs: int, seed: int = 0, *,
                 pool=None, n_envs_global: int | None = None, env_index_base: int = 0,
                 env_seeds=None, env_indices=None, auto_reset: bool = True,
                 record_trades: bool = False, trade_capacity: int = 4096, device: int | None = None,
                 stream: int | None = None):
        self.store, self.cfg = store, cfg
        d = VenvDesc()
        d.store = store.h
        d.cfg = cfg
        self._keep = []
        if pool is not None:
            arr = np.ascontiguousarray(pool, dtype=np.uint64)
            self._keep.append(arr)
            d.episode_pool = arr.ctypes.data_as(_P(C.c_uint64))
            d.pool_len = len(arr)
        d.seed = seed
        d.n_envs_global = n_envs_global or n_envs
        d.env_index_base = env_index_base
        d.n_envs_local = n_envs
        for name, v in (("env_seeds", env_seeds), ("env_indices", env_indices)):
            if v is not None:
                arr = np.ascontiguousarray(v, dtype=np.uint64)
                self._keep.append(arr)
                setattr(d, name, arr.ctypes.data_as(_P(C.c_uint64)))
        d.flags = (abi.VENV_AUTO_RESET if auto_reset else 0) | \
                  (abi.VENV_RECORD_TRADES if record_trades else 0)
        d.trade_capacity = trade_capacity
        d.device = store.device if device is None else device
        d.stream = stream
        self.h = _vp()
        _check(lib().mlob_venv_create(C.byref(d), C.byref(self.h)))
        self.n_envs = n_envs
        self.n_agents = lib().mlob_venv_n_agents(self.h)
        self.flat = abi.flat_specs(cfg)
        self.type_offset = []
        off = 0
        for t in range(cfg.n_specs):
            self.type_offset.append(off)
            off += cfg.specs[t].count

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.mlob_venv_destroy(self.h)
            self.h = None

    # VecEnv concept, rollout.hpp:16-28 / 180-191
    def n_types(self) -> int:
        return self.cfg.n_specs

    def n_streams(self, t: int) -> int:
        return lib().mlob_venv_n_streams(self.h, t)

    def obs_dim(self, t: int) -> int:
        return lib().mlob_venv_obs_dim(self.h, t)

    def n_actions(self, t: int) -> int:
        return lib().mlob_venv_n_actions(self.h, t)

    @property
    def n_episodes(self) -> int:
        return lib().mlob_venv_n_episodes(self.h)

    def set_actions(self, ids) -> None:
        """Action ids [n_envs, n_agents] (flat agent order); numpy host array or a
        torch CUDA int32 tensor on the handle's device."""
        if hasattr(ids, "is_cuda") and ids.is_cuda:
            assert ids.dtype.__str__() == "torch.int32" and ids.is_contiguous()
            _check(lib().mlob_venv_set_actions(self.h, _vp(ids.data_ptr()), 1))
            return
        a = np.ascontiguousarray(ids, dtype=np.int32).reshape(-1)
        if a.size != self.n_envs * self.n_agents:
            raise ValueError(f"expected {self.n_envs * self.n_agents} actions, got {a.size}")
        _check(lib().mlob_venv_set_actions(self.h, _vp(a.ctypes.data), 0))

    def set_direct_actions(self, actions) -> None:
        n = self.n_envs * self.n_agents
        if len(actions) != n:
            raise ValueError(f"expected {n} actions, got {len(actions)}")
        arr = (AgentAction * max(1, n))(*actions)
        _check(lib().mlob_venv_set_direct_actions(self.h, arr))

    def step(self) -> None:
        _check(lib().mlob_venv_step(self.h))

    def step_random(self, bench_seed: int, global_step: int) -> None:
        """bench::RandomStepHarness semantics: actions drawn on the device."""
        _check(lib().mlob_venv_step_random(self.h, bench_seed, global_step))

    def synchronize(self) -> None:
        _check(lib().mlob_venv_synchronize(self.h))

    def set_nets(self, nets) -> None:
        """One abi.NetParams per agent type (mlob_venv_set_nets)."""
        arr = (abi.PolicyNetC * len(nets))(*[n.to_c() for n in nets])
        _check(lib().mlob_venv_set_nets(self.h, arr))
        self._hidden = [n.hidden for n in nets]

    def collect_rollout(self, rollout_len: int, discount: float = 0.99, gae_lambda: float = 0.95,
                        seed: int = 0, update_index: int = 1) -> None:
        """collect_rollout (rollout.hpp:41-124) on the device (mlob_venv_collect_rollout)."""
        c = abi.RolloutConfig(rollout_len=rollout_len, discount=discount, gae_lambda=gae_lambda,
                              seed=seed)
        _check(lib().mlob_venv_collect_rollout(self.h, C.byref(c), update_index))
        self._rollout_len = rollout_len

    def ppo_update(self, t: int, cfg=None, seed: int = 0, update_index: int = 1) -> abi.UpdateMetrics:
        """ppo_update (ppo.hpp:263-310) of type t on the device (mlob_venv_ppo_update)."""
        cfg = cfg if cfg is not None else abi.ppo_config()
        m = abi.UpdateMetrics()
        _check(lib().mlob_venv_ppo_update(self.h, t, C.byref(cfg), seed, update_index, C.byref(m)))
        return m

    def read_net(self, t: int) -> np.ndarray:
        """Type t's parameters, PolicyNet::for_each_param order."""
        D, H, A = self.obs_dim(t), self._hidden[t], self.n_actions(t)
        out = np.zeros(abi.NetParams.param_count(D, H, A), dtype=np.float64)
        _check(lib().mlob_venv_read_net(self.h, t, out.ctypes.data_as(_P(C.c_double)), out.size))
        return out

    def rollout(self, t: int, field: int) -> np.ndarray:
        """One RolloutBatch field of type t (time-major, flat) in host memory."""
        T, B = self._rollout_len, self.n_streams(t)
        n = {abi.RB_OBS: T * B * self.obs_dim(t), abi.RB_VALUES: (T + 1) * B,
             abi.RB_H0: B * self._hidden[t], abi.RB_HIDDEN: B * self._hidden[t]}.get(field, T * B)
        out = np.zeros(n, dtype=np.dtype(abi.RB_DTYPES[field]))
        _check(lib().mlob_venv_rollout_read(self.h, t, field, _vp(out.ctypes.data), out.nbytes))
        return out

    def set_policies(self, policies, env_policy, env_cell=None) -> None:
        """Scripted actions (mlob_venv_set_policies): env e's type-t agents act by
        policies[env_policy[e, t]]; Random draws are keyed by env_cell[e]."""
        pol = (abi.Policy * max(1, len(policies)))(*policies)
        ep = np.ascontiguousarray(env_policy, dtype=np.uint8).reshape(-1)
        if ep.size != self.n_envs * self.n_types():
            raise ValueError(f"env_policy: expected {self.n_envs} x {self.n_types()} entries")
        cell = None if env_cell is None else np.ascontiguousarray(env_cell, dtype=np.uint64)
        _check(lib().mlob_venv_set_policies(self.h, pol, len(policies), _vp(ep.ctypes.data),
                                            None if cell is None else _vp(cell.ctypes.data)))

    def step_io(self, actions=None, rewards=None, dones=None, infos=None, obs=None, resets=None) -> None:
        """Fused set_actions + step + rewards/dones/infos + per-type gather
        (mlob_venv_step_io).  Buffers are C-contiguous host numpy arrays or
        (page-locked, for overlapped copies) CPU torch tensors of the layouts
        the separate calls use; obs / resets are per-type lists, None skips."""
        key = (id(actions), id(rewards), id(dones), id(infos),
               tuple(map(id, obs)) if obs is not None else None,
               tuple(map(id, resets)) if resets is not None else None)
        cached = getattr(self, "_io_cache", None)
        if cached is not None and cached[0] == key:  # same buffers as the last call
            _check(lib().mlob_venv_step_io(self.h, C.byref(cached[1])))
            return
        io = abi.StepIO()
        io.actions = _host_ptr(actions, np.int32, self.n_envs * self.n_agents)
        io.rewards = _host_ptr(rewards, np.float64, self.n_envs * self.n_agents)
        io.dones = _host_ptr(dones, np.uint8, self.n_envs * self.n_agents)
        io.infos = _host_ptr(infos, INFO_DTYPE, self.n_envs * self.n_agents)
        for t in range(self.n_types()):
            if obs is not None and obs[t] is not None:
                io.obs[t] = _host_ptr(obs[t], np.float64, self.n_streams(t) * self.obs_dim(t))
            if resets is not None and resets[t] is not None:
                io.resets[t] = _host_ptr(resets[t], np.uint8, self.n_streams(t))
        # keep the buffers alive with the cached descriptor (ids stay unique)
        self._io_cache = (key, io, (actions, rewards, dones, infos, obs, resets))
        _check(lib().mlob_venv_step_io(self.h, C.byref(io)))

    def rewards(self) -> np.ndarray:
        out = np.zeros((self.n_envs, self.n_agents), dtype=np.float64)
        _check(lib().mlob_venv_rewards(self.h, _vp(out.ctypes.data)))
        return out

    def dones(self) -> np.ndarray:
        out = np.zeros((self.n_envs, self.n_agents), dtype=np.uint8)
        _check(lib().mlob_venv_dones(self.h, _vp(out.ctypes.data)))
        return out

    def infos(self) -> np.ndarray:
        out = np.zeros((self.n_envs, self.n_agents), dtype=INFO_DTYPE)
        _check(lib().mlob_venv_infos(self.h, _vp(out.ctypes.data)))
        return out

    def obs_type(self, t: int) -> np.ndarray:
        dim = self.obs_dim(t)
        out = np.zeros((self.n_streams(t), dim), dtype=np.float64)
        _check(lib().mlob_venv_gather(self.h, t, _vp(out.ctypes.data), None))
        return out

    def messages_processed(self) -> int:
        n = C.c_uint64()
        _check(lib().mlob_venv_messages_processed(self.h, C.byref(n)))
        return n.value

    @property
    def stream(self) -> int:
        return lib().mlob_venv_stream(self.h) or 0

    @property
    def launches(self) -> int:
        return lib().mlob_venv_launch_count(self.h)

    def episode_stats(self, t: int) -> EpisodeStats:
        s = EpisodeStats()
        _check(lib().mlob_venv_episode_stats(self.h, t, C.byref(s)))
        return s

    def episode_stats_device(self, out_ptr: int) -> None:
        """K4: per-type sums into a device buffer of STAT_WORDS*n_types doubles
        (pv, slippage, completion, inventory², episodes, Σ remaining)."""
        _check(lib().mlob_venv_episode_stats_device(self.h, _vp(out_ptr)))

    def allreduce_episode_stats(self, nccl_comm: int = 0) -> list:
        """K4 + ncclAllReduce over `nccl_comm` (an ncclComm_t; 0 = this handle
        alone) -> per-type EpisodeStats with the exact completion sum."""
        out = (EpisodeStats * self.n_types())()
        _check(lib().mlob_venv_allreduce_episode_stats(self.h, _vp(nccl_comm), out))
        return list(out)

    def profile(self, on: bool) -> None:
        """Per-kernel event timing of the following steps (measurement only)."""
        _check(lib().mlob_venv_profile(self.h, 1 if on else 0))

    def kernel_ms(self):
        """([act, book, outcome] summed ms, steps timed) since profile(True)."""
        out = (C.c_double * 3)()
        n = C.c_uint64()
        _check(lib().mlob_venv_kernel_ms(self.h, out, C.byref(n)))
        return list(out), n.value

    def clear_episode_stats(self) -> None:
        _check(lib().mlob_venv_clear_episode_stats(self.h))

    def view(self, e: int) -> "EnvView":
        return EnvView(self, e)


def evaluate_matrix(store: "DeviceStore", cfg: EnvConfig, episodes, type0, type1, seed: int,
                    device: int = 0):
    """ippo::evaluate_matrix (evaluate.hpp:104-217) on the GPU: the whole
    cross-play grid as one batch (mlob_evaluate_matrix).  type0 / type1 are
    lists of abi.Policy; returns the CellStats list, row-major."""
    eps = np.ascontiguousarray(episodes, dtype=np.uint64)
    t0 = (abi.Policy * max(1, len(type0)))(*type0)
    t1 = (abi.Policy * max(1, len(type1)))(*type1)
    out = (abi.CellStats * max(1, len(type0) * len(type1)))()
    _check(lib().mlob_evaluate_matrix(store.h, C.byref(cfg), eps.ctypes.data_as(_P(C.c_uint64)),
                                      len(eps), t0, len(type0), t1, len(type1), seed, device, out))
    return list(out)[:len(type0) * len(type1)]


class MarketVecEnv(_Venv):
    """ippo::MarketVecEnv (rollout.hpp:151-336) on the GPU: env-major streams,
    auto-reset with round-robin episodes from the pool, cached rewards/dones."""

    def __init__(self, store: DeviceStore, cfg: EnvConfig, episode_pool=None, seed: int = 0,
                 n_envs: int = 1, **kw):
        kw.setdefault("auto_reset", True)
        super().__init__(store, cfg, n_envs, seed, pool=episode_pool, **kw)
        self._actions = np.zeros((n_envs, self.n_agents), dtype=np.int32)
        self._rewards = np.zeros((n_envs, self.n_agents), dtype=np.float64)
        self._dones = np.zeros((n_envs, self.n_agents), dtype=np.uint8)

    def reset_all(self) -> None:  # rollout.hpp:194-200
        _check(lib().mlob_venv_reset_all(self.h))

    def gather(self, t: int, obs_out: np.ndarray | None = None,
               reset_out: np.ndarray | None = None):  # rollout.hpp:202-213
        n, dim = self.n_streams(t), self.obs_dim(t)
        if obs_out is None:
            obs_out = np.zeros((n, dim), dtype=np.float64)
        if reset_out is None:
            reset_out = np.zeros(n, dtype=np.uint8)
        _check(lib().mlob_venv_gather(self.h, t, _vp(obs_out.ctypes.data),
                                      _vp(reset_out.ctypes.data)))
        return obs_out, reset_out

    def set_action(self, t: int, stream: int, action: int) -> None:  # rollout.hpp:215-222
        count = self.cfg.specs[t].count
        self._actions[stream // count, self.type_offset[t] + stream % count] = action

    def step_all(self) -> None:  # rollout.hpp:224-234 (+ the reward/done caches)
        self.step_io(actions=self._actions, rewards=self._rewards, dones=self._dones)

    def _locate(self, t, s):
        count = self.cfg.specs[t].count
        return s // count, self.type_offset[t] + s % count

    def reward(self, t: int, stream: int) -> float:  # rollout.hpp:236-239
        e, a = self._locate(t, stream)
        return float(self._rewards[e, a])

    def done(self, t: int, stream: int) -> bool:  # rollout.hpp:240-243
        e, a = self._locate(t, stream)
        return bool(self._dones[e, a])


class MarketEnvBatch(_Venv):
    """N independent env::MarketEnv instances (env.hpp:98-282) stepped together
    (no auto-reset: stepping a terminal env raises LogicError like env.hpp:195)."""

    def __init__(self, store: DeviceStore, cfg: EnvConfig, n_envs: int = 1, seed: int = 0, **kw):
        kw.setdefault("auto_reset", False)
        kw.setdefault("record_trades", True)
        super().__init__(store, cfg, n_envs, seed, **kw)

    def reset(self, episodes) -> None:
        """MarketEnv::reset(episode) per env (env.hpp:143-192)."""
        eps = np.ascontiguousarray(np.broadcast_to(np.asarray(episodes, dtype=np.uint64),
                                                   (self.n_envs,)))
        _check(lib().mlob_venv_reset_envs(self.h, eps.ctypes.data_as(_P(C.c_uint64))))

    def step_ids(self, ids) -> None:
        """MarketEnv::step_ids for every env; ids shape [n_envs, n_agents]."""
        ids = np.asarray(ids, dtype=np.int32).reshape(self.n_envs, -1)
        if ids.shape[1] != self.n_agents:
            raise ValueError(f"MarketEnv::step: expected {self.n_agents} actions, "
                             f"got {ids.shape[1]}")
        self.set_actions(ids)
        self.step()

    def step_actions(self, actions) -> None:
        """MarketEnv::step(span<const AgentAction>) for every env."""
        self.set_direct_actions(actions)
        self.step()


class EnvView:
    """Readers of one env of a batch in reference record formats (the
    single-env interface the parity tests compare against the oracle)."""

    def __init__(self, venv: _Venv, e: int):
        self.v, self.e = venv, e
        self.n_agents = venv.n_agents
        self.flat = venv.flat

    def scalars(self) -> EnvScalars:
        s = EnvScalars()
        _check(lib().mlob_venv_read_scalars(self.v.h, self.e, C.byref(s)))
        return s

    def book(self, side: int) -> np.ndarray:
        cap = 1 << 12
        out = (RestingOrder * cap)()
        n = C.c_uint64()
        _check(lib().mlob_venv_read_book(self.v.h, self.e, side, out, cap, C.byref(n)))
        return np.frombuffer(bytes(out)[: n.value * 40], dtype=ORDER_DTYPE).copy()

    def agent(self, a: int) -> AgentState:
        s = AgentState()
        _check(lib().mlob_venv_read_agent(self.v.h, self.e, a, C.byref(s)))
        return s

    def info(self, a: int) -> AgentInfo:
        return AgentInfo.from_buffer_copy(self.v.infos()[self.e, a].tobytes())

    def reward(self, a: int) -> float:
        return float(self.v.rewards()[self.e, a])

    def done(self, a: int) -> int:
        return int(self.v.dones()[self.e, a])

    def obs(self, a: int) -> np.ndarray:
        t = self.flat[a]
        k = a - self.v.type_offset[t]
        dim = self.v.obs_dim(t)
        count = self.v.cfg.specs[t].count
        allobs = self.v.obs_type(t)
        return allobs[self.e * count + k].copy()

    def trades(self) -> np.ndarray:
        cap = 1 << 14
        out = (Trade * cap)()
        n = C.c_uint64()
        _check(lib().mlob_venv_read_trades(self.v.h, self.e, out, cap, C.byref(n)))
        return np.frombuffer(bytes(out)[: n.value * 56], dtype=TRADE_DTYPE).copy()
