"""ctypes mirror of include/mlob.h (record and config PODs).

Field order and widths match the C header exactly; layouts of the record types
equal the reference structs (lob/types.hpp:31-80, env/env.hpp:20-57), which
tests/test_host.py checks through sizeof/offsetof exported by the library.
"""
from __future__ import annotations

import ctypes as C

i8, u8, i32, u32, i64, u64, f64 = (C.c_int8, C.c_uint8, C.c_int32, C.c_uint32, C.c_int64,
                                   C.c_uint64, C.c_double)

ABI_VERSION = 1
MLOB_OK, MLOB_E_INVALID_ARGUMENT, MLOB_E_OUT_OF_RANGE, MLOB_E_LOGIC, MLOB_E_RUNTIME, MLOB_E_CUDA = range(6)

# lob::MsgKind / Side (lob/types.hpp:8-22)
NEW_LIMIT, CANCEL_PARTIAL, DELETE, EXECUTE_VISIBLE, EXECUTE_HIDDEN, CROSS, HALT = range(7)
BID, ASK = 0, 1
# env/config.hpp enums
MARKET_MAKER, EXECUTOR, DIRECTIONAL = 0, 1, 2
SPREAD_SKEW, FIXED_QUANT, AVST = 0, 1, 2
REWARD_BUYSELL, REWARD_SPOONER, REWARD_EXEC = 0, 1, 2
REF_MID, REF_FAR_TOUCH = 0, 1
OBS_MM_BASIC, OBS_MM_FULL, OBS_EXEC = 0, 1, 2
TASK_BUY, TASK_SELL = 0, 1

MAX_SPREAD_SKEW_ROWS = 32
MAX_GAMMA = 16
MAX_ACTIVE = 8
MAX_SPECS = 8
MAX_AGENTS = 32
STAT_WORDS = 6  # MLOB_STAT_WORDS: pv, slippage, completion, inventory², episodes, Σ remaining

VENV_AUTO_RESET = 1 << 0
VENV_RECORD_TRADES = 1 << 1
# ippo::PolicyKind (evaluate.hpp:17), baselines::TwapPriceMode (twap.hpp:11)
POLICY_LEARNED, POLICY_TWAP, POLICY_AVST, POLICY_RANDOM, POLICY_NOOP = range(5)
TWAP_AGGRESSIVE, TWAP_PASSIVE = 0, 1


class Message(C.Structure):
    _fields_ = [("time", i64), ("order_id", u64), ("price", i64), ("quantity", i64),
                ("kind", u8), ("side", u8), ("_pad", u8 * 2), ("trader_id", i32)]


class RestingOrder(C.Structure):
    _fields_ = [("price", i64), ("quantity", i64), ("order_id", u64), ("arrival_seq", u64),
                ("trader_id", i32), ("_pad", i32)]


class Trade(C.Structure):
    _fields_ = [("price", i64), ("quantity", i64), ("time", i64), ("passive_order_id", u64),
                ("aggressor_order_id", u64), ("passive_trader_id", i32),
                ("aggressor_trader_id", i32), ("aggressor_side", u8), ("_pad", u8 * 7)]


class Level(C.Structure):
    _fields_ = [("price", i64), ("quantity", i64)]


class BookStates(C.Structure):
    _fields_ = [("n_states", u64), ("message_index", C.POINTER(u64)),
                ("level_offset", C.POINTER(u64)), ("n_bids", C.POINTER(u32)),
                ("levels", C.POINTER(Level))]


class AgentParams(C.Structure):
    _fields_ = [("order_size", i64), ("inventory_cap", i64), ("rho", f64),
                ("quadratic_penalty", i32), ("ref_price", i32), ("lambda_", f64),
                ("unfilled_penalty_coef", f64), ("lambda_exec", f64), ("task_size", i64),
                ("exec_complex", i32), ("default_half_spread", i32), ("reward_scale", f64),
                ("fixed_quant_from_mid", i32), ("n_spread_skew", i32),
                ("spread_skew_half", i32 * MAX_SPREAD_SKEW_ROWS),
                ("spread_skew_skew", i32 * MAX_SPREAD_SKEW_ROWS),
                ("n_gamma", i32), ("_pad", i32), ("gamma_grid", f64 * MAX_GAMMA),
                ("kappa", f64), ("sigma", f64), ("horizon", f64)]


class AgentSpec(C.Structure):
    _fields_ = [("type", i32), ("count", i32), ("mm_space", i32), ("obs_space", i32),
                ("reward", i32), ("_pad", i32), ("params", AgentParams)]


class EnvConfig(C.Structure):
    _fields_ = [("steps_per_episode", i32), ("messages_per_step", i32),
                ("start_stride_steps", i32), ("n_specs", i32), ("book_capacity", u64),
                ("obs_depth", u64), ("fallback_mid_half", i64),
                ("synthetic_init_id_base", u64), ("agent_id_base", u64),
                ("agent_id_range", u64), ("fill_reserve", u64),
                ("specs", AgentSpec * MAX_SPECS)]


class Quote(C.Structure):
    _fields_ = [("side", u8), ("_pad", u8 * 7), ("price", i64), ("quantity", i64)]


class AgentAction(C.Structure):
    _fields_ = [("id", i32), ("direct", i32), ("n_quotes", i32), ("_pad", i32),
                ("quotes", Quote * 2)]


class ActiveOrder(C.Structure):
    _fields_ = [("order_id", u64), ("price", i64), ("quantity", i64), ("side", u8),
                ("_pad", u8 * 7)]


class AgentState(C.Structure):
    _fields_ = [("inventory", i64), ("cash", i64), ("task_remaining", i64), ("task_dir", i32),
                ("n_active", i32), ("p_init", f64), ("order_nonce", u64),
                ("filled_total", i64), ("slippage_total", f64),
                ("active", ActiveOrder * MAX_ACTIVE)]


class AgentInfo(C.Structure):
    _fields_ = [("inventory", i64), ("cash", i64), ("portfolio_value", f64),
                ("slippage_step", f64), ("slippage_total", f64), ("task_remaining", i64),
                ("step_filled", i64), ("step_fill_count", i32), ("_pad", i32)]


class EnvScalars(C.Structure):
    _fields_ = [("step", i32), ("terminal", i32), ("episode", u64), ("mid_half", i64),
                ("prev_mid_half", i64), ("mean_mid_ticks", f64), ("last_bid", i64),
                ("last_ask", i64), ("last_time", i64), ("messages_processed", u64),
                ("next_seq", u64), ("live_bid", u64), ("live_ask", u64)]


class EpisodeStats(C.Structure):
    _fields_ = [("pv_sum", f64), ("slippage_sum", f64), ("completion_sum", f64),
                ("inventory_sq_sum", f64), ("episodes", i64)]


class SynthConfig(C.Structure):
    _fields_ = [("n_messages", u64), ("initial_mid", i64), ("volatility", f64),
                ("p_new_passive", f64), ("p_new_cross", f64), ("p_cancel", f64),
                ("p_delete", f64), ("p_execute", f64), ("band", i32), ("seed_levels", i32),
                ("max_qty", i64), ("seed_qty", i64), ("state_sample_every", u64),
                ("state_depth", u64)]


class PolicyNetC(C.Structure):
    """mlob_policy_net: ippo::PolicyNet (net.hpp:18-30) as host array pointers."""
    _P = C.POINTER(f64)
    _fields_ = [("obs_dim", i32), ("hidden", i32), ("n_actions", i32), ("_pad", i32),
                ("w_ih", _P), ("w_hh", _P), ("b_ih", _P), ("b_hh", _P), ("w_actor", _P),
                ("b_actor", _P), ("w_critic", _P), ("b_critic", f64)]


class RolloutConfig(C.Structure):  # TrainLoopConfig (rollout.hpp:30-37)
    _fields_ = [("rollout_len", i32), ("_pad", i32), ("discount", f64), ("gae_lambda", f64),
                ("seed", u64)]


# RolloutBatch fields (ppo.hpp:33-48) + the persistent hidden state
(RB_OBS, RB_ACTIONS, RB_LOG_PROBS, RB_VALUES, RB_REWARDS, RB_DONES, RB_RESETS, RB_H0,
 RB_ADVANTAGES, RB_RETURNS, RB_HIDDEN) = range(11)
RB_DTYPES = {RB_OBS: "<f8", RB_ACTIONS: "<i4", RB_LOG_PROBS: "<f8", RB_VALUES: "<f8",
             RB_REWARDS: "<f8", RB_DONES: "u1", RB_RESETS: "u1", RB_H0: "<f8",
             RB_ADVANTAGES: "<f8", RB_RETURNS: "<f8", RB_HIDDEN: "<f8"}


class NetParams:
    """A PolicyNet's parameters as numpy arrays, flat order of
    PolicyNet::for_each_param (net.hpp:36-41): w_ih, w_hh, b_ih, b_hh, w_actor,
    b_actor, w_critic, b_critic."""

    def __init__(self, obs_dim: int, hidden: int, n_actions: int, flat):
        import numpy as np
        D, H, A = obs_dim, hidden, n_actions
        self.obs_dim, self.hidden, self.n_actions = D, H, A
        self.flat = np.ascontiguousarray(flat, dtype=np.float64).copy()
        sizes = [3 * H * D, 3 * H * H, 3 * H, 3 * H, A * H, A, H, 1]
        if self.flat.size != sum(sizes):
            raise ValueError(f"expected {sum(sizes)} parameters, got {self.flat.size}")
        offs = np.cumsum([0] + sizes)
        self.parts = [self.flat[offs[i]:offs[i + 1]] for i in range(8)]

    @staticmethod
    def param_count(obs_dim: int, hidden: int, n_actions: int) -> int:
        return 3 * hidden * (obs_dim + hidden + 2) + n_actions * hidden + n_actions + hidden + 1

    def to_c(self) -> PolicyNetC:
        n = PolicyNetC()
        n.obs_dim, n.hidden, n.n_actions = self.obs_dim, self.hidden, self.n_actions
        P = C.POINTER(f64)
        for name, arr in zip(("w_ih", "w_hh", "b_ih", "b_hh", "w_actor", "b_actor", "w_critic"),
                             self.parts[:7]):
            setattr(n, name, arr.ctypes.data_as(P))
        n.b_critic = float(self.parts[7][0])
        return n


class PpoConfig(C.Structure):  # ippo::PpoConfig (ppo.hpp:19-28)
    _fields_ = [("epochs", i32), ("minibatches", i32), ("clip_eps", f64), ("vf_coef", f64),
                ("ent_coef", f64), ("lr", f64), ("max_grad_norm", f64), ("normalize_adv", i32),
                ("_pad", i32)]


def ppo_config(**kw) -> PpoConfig:
    """PpoConfig with the reference defaults (ppo.hpp:19-28), overridden by kw."""
    c = PpoConfig(epochs=4, minibatches=4, clip_eps=0.2, vf_coef=0.5, ent_coef=0.01, lr=3e-4,
                  max_grad_norm=0.5, normalize_adv=1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class UpdateMetrics(C.Structure):  # ippo::UpdateMetrics (ppo.hpp:69-77)
    _fields_ = [("pg_loss", f64), ("v_loss", f64), ("entropy", f64), ("approx_kl", f64),
                ("clip_frac", f64), ("grad_norm", f64), ("mean_reward", f64)]


class Policy(C.Structure):
    """mlob_policy = ippo::PolicyChoice without the network (evaluate.hpp:19-25)."""
    _fields_ = [("kind", i32), ("twap_mode", i32), ("avst_gamma_index", i32), ("n_gamma", i32),
                ("gamma_grid", f64 * MAX_GAMMA), ("kappa", f64), ("sigma", f64), ("horizon", f64),
                ("net", C.POINTER(PolicyNetC))]


class TypeCellStats(C.Structure):  # evaluate.hpp:27-35
    _fields_ = [("pv_mean", f64), ("pv_stderr", f64), ("slippage_mean", f64),
                ("slippage_stderr", f64), ("completion_mean", f64), ("filled_total", i64),
                ("no_fills", i32), ("_pad", i32)]


class CellStats(C.Structure):  # evaluate.hpp:37-42 (labels omitted)
    _fields_ = [("per_type", TypeCellStats * 2), ("episodes", i64)]


def policy(kind: int, twap_mode: int = TWAP_AGGRESSIVE, gamma_index: int = 1,
           gamma_grid=(0.05, 0.1, 0.5, 1.0), kappa: float = 1.5, sigma: float = 2.0,
           horizon: float = 64.0, net: "NetParams | None" = None) -> Policy:
    """A policy option with the reference defaults (AvStBaseline avst.hpp:14-17 over
    AvStParams actions.hpp:142-147; TwapPriceMode::Aggressive evaluate.hpp:24);
    `net` = the network of a POLICY_LEARNED option (kept alive by the returned
    object)."""
    p = Policy()
    if net is not None:
        p._net_c = net.to_c()
        p._net_params = net
        p.net = C.pointer(p._net_c)
    p.kind, p.twap_mode, p.avst_gamma_index = kind, twap_mode, gamma_index
    if len(gamma_grid) > MAX_GAMMA:
        raise ValueError(f"at most {MAX_GAMMA} gamma values")
    p.n_gamma = len(gamma_grid)
    for i, g in enumerate(gamma_grid):
        p.gamma_grid[i] = g
    p.kappa, p.sigma, p.horizon = kappa, sigma, horizon
    return p


class StepIO(C.Structure):
    """mlob_step_io: host buffers of one fused step (NULL = skip)."""
    _fields_ = [("actions", C.c_void_p), ("rewards", C.c_void_p), ("dones", C.c_void_p),
                ("infos", C.c_void_p), ("obs", C.c_void_p * MAX_SPECS),
                ("resets", C.c_void_p * MAX_SPECS)]


class VenvDesc(C.Structure):
    _fields_ = [("store", C.c_void_p), ("cfg", EnvConfig), ("episode_pool", C.POINTER(u64)),
                ("pool_len", u64), ("seed", u64), ("n_envs_global", u64),
                ("env_index_base", u64), ("n_envs_local", u64), ("env_seeds", C.POINTER(u64)),
                ("env_indices", C.POINTER(u64)), ("flags", u32), ("trade_capacity", u32),
                ("device", i32), ("_pad", i32), ("stream", C.c_void_p)]


# ---- struct defaults (mirrors of the reference struct initialisers) ----------

def default_agent_params() -> AgentParams:
    """env::AgentParams defaults, env/config.hpp:32-48 (+ SpreadSkewTable::standard
    actions.hpp:117-124 and AvStParams actions.hpp:142-147)."""
    p = AgentParams()
    p.order_size = 10
    p.inventory_cap = 30
    p.rho = 50.0
    p.quadratic_penalty = 1
    p.lambda_ = 0.5
    p.ref_price = REF_MID
    p.unfilled_penalty_coef = 0.1
    p.lambda_exec = 0.0
    p.task_size = 600
    p.exec_complex = 1
    p.reward_scale = 1.0
    p.default_half_spread = 2
    p.fixed_quant_from_mid = 0
    rows = [(s, k) for s in (1, 2, 3) for k in (-1, 0, 1)]
    p.n_spread_skew = len(rows)
    for i, (s, k) in enumerate(rows):
        p.spread_skew_half[i] = s
        p.spread_skew_skew[i] = k
    grid = [0.05, 0.1, 0.5, 1.0]
    p.n_gamma = len(grid)
    for i, g in enumerate(grid):
        p.gamma_grid[i] = g
    p.kappa = 1.5
    p.sigma = 2.0
    p.horizon = 64.0
    return p


def agent_spec(type_: int = MARKET_MAKER, count: int = 1, mm_space: int = FIXED_QUANT,
               obs_space: int | None = None, reward: int | None = None, **params) -> AgentSpec:
    """env::AgentSpec (env/config.hpp:50-57).  obs_space / reward default to the
    struct defaults (MMBasic / Spooner) unless the type is Executor, in which
    case the reference tests' executor spec (Exec / Exec) is used."""
    s = AgentSpec()
    s.type = type_
    s.count = count
    s.mm_space = mm_space
    if obs_space is None:
        obs_space = OBS_EXEC if type_ == EXECUTOR else OBS_MM_BASIC
    if reward is None:
        reward = REWARD_EXEC if type_ == EXECUTOR else REWARD_SPOONER
    s.obs_space = obs_space
    s.reward = reward
    s.params = default_agent_params()
    for k, v in params.items():
        if k == "lambda":
            k = "lambda_"
        if k == "spread_skew":
            s.params.n_spread_skew = len(v)
            for i, (h, kk) in enumerate(v):
                s.params.spread_skew_half[i] = h
                s.params.spread_skew_skew[i] = kk
            continue
        if k == "gamma_grid":
            s.params.n_gamma = len(v)
            for i, g in enumerate(v):
                s.params.gamma_grid[i] = g
            continue
        if not hasattr(s.params, k):
            raise AttributeError(f"unknown agent param {k}")
        setattr(s.params, k, v)
    return s


def env_config(specs=(), steps_per_episode: int = 64, messages_per_step: int = 100,
               start_stride_steps: int = 64, book_capacity: int = 100, obs_depth: int = 5,
               fallback_mid_half: int = 2000, synthetic_init_id_base: int = 1 << 36,
               agent_id_base: int = 1 << 40, agent_id_range: int = 1 << 20,
               fill_reserve: int = 512) -> EnvConfig:
    """env::EnvConfig defaults, env/config.hpp:59-71."""
    if len(specs) > MAX_SPECS:
        raise ValueError(f"at most {MAX_SPECS} agent specs")
    c = EnvConfig()
    c.steps_per_episode = steps_per_episode
    c.messages_per_step = messages_per_step
    c.start_stride_steps = start_stride_steps
    c.book_capacity = book_capacity
    c.obs_depth = obs_depth
    c.fallback_mid_half = fallback_mid_half
    c.synthetic_init_id_base = synthetic_init_id_base
    c.agent_id_base = agent_id_base
    c.agent_id_range = agent_id_range
    c.fill_reserve = fill_reserve
    c.n_specs = len(specs)
    for i, s in enumerate(specs):
        c.specs[i] = s
    return c


def synth_config(**kw) -> SynthConfig:
    """data::SynthConfig defaults, data/synth.hpp:18-36."""
    c = SynthConfig()
    c.n_messages = 100000
    c.initial_mid = 1000
    c.volatility = 0.02
    c.p_new_passive = 0.44
    c.p_new_cross = 0.14
    c.p_cancel = 0.08
    c.p_delete = 0.18
    c.p_execute = 0.14
    c.band = 8
    c.max_qty = 20
    c.seed_levels = 5
    c.seed_qty = 10
    c.state_sample_every = 1600
    c.state_depth = 10
    for k, v in kw.items():
        if not hasattr(c, k):
            raise AttributeError(f"unknown synth field {k}")
        setattr(c, k, v)
    return c


def action_arity(spec: AgentSpec) -> int:
    """env::action_arity, env/config.hpp:73-90."""
    if spec.type == EXECUTOR:
        return 12 if spec.params.exec_complex else 4
    if spec.type == DIRECTIONAL:
        return 3
    if spec.mm_space == SPREAD_SKEW:
        return spec.params.n_spread_skew
    if spec.mm_space == FIXED_QUANT:
        return 8
    return spec.params.n_gamma


def observation_size(obs_space: int, depth: int) -> int:
    """agents::observation_size, observations.hpp:69-76."""
    return {OBS_MM_BASIC: 8, OBS_MM_FULL: 8 + 4 * depth, OBS_EXEC: 10}[obs_space]


def flat_specs(cfg: EnvConfig) -> list[int]:
    """Spec index of every flat agent (env.hpp:105-106)."""
    out = []
    for s in range(cfg.n_specs):
        out += [s] * cfg.specs[s].count
    return out
