// mlob_dev.h — device data layout shared by the kernels (mlob_kernels.cu) and
// the host runtime (mlob_runtime.cu).  See DESIGN.md "Data layout in HBM".
#pragma once

#include <cstdint>
#include <cstdio>

#include "../../include/mlob.h"

// Checked builds (libmlob_checked.so, -DMLOB_CHECKS=1): device-side bounds
// and invariant assertions on the hand-off buffers, the book rows, the fill
// log and the mbarrier waits; a failure prints its site and traps (the test
// harness's stand-in for compute-sanitizer, which is closed on this pool).
#ifndef MLOB_CHECKS
#define MLOB_CHECKS 0
#endif
#if MLOB_CHECKS
#define MLOB_CHECK(c)                                                            \
  do {                                                                           \
    if (!(c)) {                                                                  \
      printf("MLOB_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);           \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define MLOB_CHECK(c) \
  do {                \
  } while (0)
#endif

namespace mlob {

constexpr int kWarp = 32;
constexpr int kMaxAgents = MLOB_MAX_AGENTS;
constexpr int kMaxSpecs = MLOB_MAX_SPECS;
constexpr int kMaxActive = MLOB_MAX_ACTIVE;
constexpr int kMaxObsDepth = 64;
constexpr int kChunk = 128;       // replay messages staged per bulk copy
constexpr uint32_t kEmptySt = 0xffffffffu;
constexpr uint32_t kMaxSeq = 1u << 24;  // arrival_seq lives in the top 24 bits of `st`

// 32-byte device message record (repacked from the 40-byte lob::Message,
// lob/types.hpp:31-41).  32-byte records keep every per-step slice 16-byte
// aligned for cp.async.bulk whatever the slice offset.
struct DevMsg {
  int64_t time;
  uint64_t order_id;
  int32_t price;
  int32_t qty;
  uint8_t kind;
  uint8_t side;
  uint16_t _pad;
  int32_t trader;
};
static_assert(sizeof(DevMsg) == 32, "DevMsg must be 32 bytes");

// Initial-book reference for an episode (data::MessageStore::state_before,
// store.hpp:29-36, resolved once on the host).  valid == 0: no sampled state.
struct EpState {
  uint64_t level_offset;  // into the store's level table (bids then asks)
  uint32_t nb, na;
  uint32_t valid;
  uint32_t _pad;
};

// One agent-side fill of the step, in fill order (env.hpp:381-396: the
// passive agent's entry first, then the aggressor's).  The outcome kernel
// replays the log for the agent accounting, the slippage sums and the MM
// rewards (rewards.hpp:22-36), so every sum keeps the reference's order.
struct FillEnt {
  int32_t price;
  int32_t qty;
  int32_t agent;
  int32_t side;
};
constexpr int kStatWords = 6;            // K4 doubles per agent type (stats_kernel)
constexpr int kFillInline = 16;          // per-env inline fill-log entries
constexpr int kFillChunk = 32;           // overflow chunk: entry 0 links the next chunk
constexpr uint32_t kNoChunk = 0xffffffffu;

// One aggregated L2 level (book.hpp:209-220).
struct L2Lvl {
  int32_t price;
  int32_t _pad;
  int64_t qty;
};
// Step summary of the book for the observations (observations.hpp:42-148):
// level counts within obs_depth, top-of-book and top-D quantities per side.
struct L2Sum {
  int32_t nb, na;
  int64_t sumq0, sumq1, topq0, topq1;
  int64_t _pad;
};
static_assert(sizeof(L2Sum) == 48, "L2Sum must be 48 bytes");

struct DevLevel {
  int32_t price;
  int32_t qty;
};

// Per agent spec, env/config.hpp:32-57 (+ precomputed AvSt spread terms).
struct DevSpec {
  int32_t type, mm_space, obs_space, reward;
  int32_t count, flat_offset, obs_dim, arity;
  int64_t order_size, inventory_cap, task_size;
  double rho, lambda, unfilled_penalty_coef, reward_scale;
  int32_t quadratic_penalty, ref_price, exec_complex, default_half_spread;
  int32_t fixed_quant_from_mid, n_spread_skew, n_gamma, _pad;
  double sigma, horizon;
  int32_t ss_half[MLOB_MAX_SPREAD_SKEW_ROWS];
  int32_t ss_skew[MLOB_MAX_SPREAD_SKEW_ROWS];
  double gamma[MLOB_MAX_GAMMA];
  double avst_term[MLOB_MAX_GAMMA];  // (2.0 / gamma) * log1p(gamma / kappa), host glibc
};

struct DevCfg {
  int32_t steps_per_episode, mps, capacity, obs_depth;
  int32_t n_specs, n_agents, max_obs_dim, full_l2;  // full_l2: some agent uses MMFull levels
  int64_t fallback_mid_half;
  uint64_t synth_id_base, agent_id_base, agent_id_range;
  uint8_t flat_spec[kMaxAgents];
  DevSpec specs[kMaxSpecs];
};

// Per-env scalar state, 128 bytes (MarketEnv members env.hpp:505-525 plus
// the book's counts/next_seq and the VecEnv's per-env bookkeeping).
struct EnvHdr {
  int64_t mid_half, prev_mid_half;
  double mbar;
  int64_t last_bid, last_ask, last_time;
  uint64_t episode, msgs_processed, cursor;
  int64_t episodes_finished;
  uint32_t next_seq;
  int32_t step;
  uint16_t live[2];
  uint16_t hwm[2];
  int32_t best[2];
  uint32_t n_trades;
  uint8_t terminal, just_reset, _pad8[2];
  // split-step hand-offs: agent messages of this step (act_kernel ->
  // book_kernel), agent fills logged (book_kernel -> outcome_kernel) and the
  // first overflow chunk of the fill log (kNoChunk: none)
  uint32_t n_amsg, n_fills, fill_head, _pad32;
};
static_assert(sizeof(EnvHdr) == 128, "EnvHdr must be 128 bytes");

// Per (env, agent) state, env::AgentState (env.hpp:29-46) minus the active list.
struct AgentRec {
  int64_t inventory, cash, task_remaining, filled_total;
  double p_init, slippage_total;
  uint64_t nonce;
  int32_t task_dir, n_active;
};
static_assert(sizeof(AgentRec) == 64, "AgentRec must be 64 bytes");

// env::ActiveOrder (env.hpp:20-27), 16 bytes; side in bit 31 of qty_side.
struct ActiveRec {
  uint64_t order_id;
  int32_t price;
  uint32_t qty_side;
};

enum ActionMode : int32_t { kActIds = 0, kActDirect = 1, kActBench = 2, kActScripted = 3 };

// A scripted policy (mlob_policy) resolved for the device: AvSt's gamma and
// log1p term are taken on the host (glibc), as for the AvSt action space.
struct DevPolicy {
  int32_t kind, twap_mode;
  double gamma, sigma, horizon, avst_term;
};
constexpr int kMaxPolicies = 64;

enum DevError : uint32_t {
  kErrMissingState = 1u << 0,   // runtime_error, env.hpp:149-153
  kErrTooDeep = 1u << 1,        // invalid_argument, book.hpp:42-43
  kErrActiveOverflow = 1u << 2, // more than MLOB_MAX_ACTIVE resting orders for one agent
  kErrPriceRange = 1u << 3,     // an agent quote does not fit the int32 device book
  kErrSeqRange = 1u << 4,       // arrival_seq beyond 2^24
  kErrBadAction = 1u << 5,      // device-resident action id out of range (actions.hpp:69-70)
  kErrBadTrader = 1u << 6,      // replay trader_id names a non-existent agent
  kErrFillPool = 1u << 7,       // agent-fill overflow pool exhausted in one step
  kErrAmsgCap = 1u << 8,        // more agent messages in one step than the hand-off buffer holds
  kErrDeepRange = 1u << 9,      // deep-book 4-word slot: qty >= 2^24, order id >= 2^44 or seq >= 2^20
};

struct __align__(16) KParams {
  // store (read-only, shared by every handle on the device)
  const DevMsg* msgs;
  const uint64_t* ep_start;
  const EpState* ep_state;
  const DevLevel* levels;
  uint64_t n_episodes;
  // book, SoA: [(env * 2 + side) * SPL + k] * 32 + lane
  int32_t* bk_p;
  int32_t* bk_q;
  uint2* bk_id;
  uint32_t* bk_st;
  EnvHdr* hdr;
  AgentRec* agents;   // [env * A + a]
  ActiveRec* active;  // [(env * A + a) * kMaxActive + i]
  // actions
  const int32_t* action_ids;               // [env * A + a]
  const mlob_agent_action* action_direct;  // [env * A + a]
  int32_t action_mode;
  int32_t flags;
  uint64_t bench_seed, global_step;
  // outputs
  double* obs[kMaxSpecs];  // per type: [(env * count + k) * dim + j]
  double* rewards;         // [env * A + a]
  uint8_t* dones;
  mlob_agent_info* infos;
  uint8_t* just_reset;     // [env]
  double* t_pv;
  double* t_slip;
  double* t_comp;
  double* t_inv;
  int64_t* t_rem;          // Σ task_remaining of finished executor episodes [env * A + a]
  mlob_trade* trades;      // [env * trade_cap + i]
  uint32_t trade_cap;
  uint32_t _pad_tc;
  // env identity / episode pool
  const uint64_t* env_seed;   // optional
  const uint64_t* env_index;  // optional
  uint64_t seed, env_index_base;
  const uint64_t* pool;
  uint64_t pool_len, n_envs_global, n_envs;
  const uint64_t* reset_episodes;  // reset kernel: per-env episode
  uint32_t* error;
  const DevCfg* cfg;  // device copy; staged into shared memory by each block
  const uint32_t* gate;  // optional: non-zero word = skip the launch (rejected actions)
  // kActScripted: policies[env_policy[env * n_specs + type]], Random keyed by env_cell[env]
  const DevPolicy* policies;
  const uint8_t* env_policy;
  const uint64_t* env_cell;
  // split step hand-offs (per env, offset with the launch's env range)
  DevMsg* amsg;              // [env * amsg_cap + i] agent messages in processing order
  FillEnt* fills;            // [env * kFillInline + i] inline agent-fill log
  L2Sum* l2sum;              // [env]
  L2Lvl* l2lv;               // [env * 2 * obs_depth] MMFull levels (null unless some agent uses them)
  FillEnt* fill_pool;        // overflow chunks of this launch's env range
  uint32_t* fill_pool_ctr;   // chunks taken (zeroed by the launch's act_kernel)
  uint32_t fill_pool_chunks;
  uint32_t amsg_cap;
};

}  // namespace mlob
