/*
 * mlob.h — C ABI of the B200-native batched limit-order-book environment.
 *
 * This is the drop-in boundary for the reference's batched environment step
 * (marlob `ippo::MarketVecEnv` / `env::MarketEnv`).  Every
 * entry point takes plain pointers and sizes; no C++ or torch types cross it.
 * Each function below names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/marlob/).
 *
 * Error model (replaces the reference's C++ exceptions, env.hpp:195-199,
 * env/config.hpp:96-120, actions.hpp:69-70, env.hpp:144-153): every function
 * returns an mlob_status; the thread-local message is read with
 * mlob_last_error().  The C++ wrapper (include/mlob/vec_env.hpp) and the Python
 * host mirror rethrow the same exception classes as the reference:
 *   MLOB_E_INVALID_ARGUMENT -> std::invalid_argument / ValueError
 *   MLOB_E_OUT_OF_RANGE     -> std::out_of_range     / IndexError
 *   MLOB_E_LOGIC            -> std::logic_error      / RuntimeError(logic)
 *   MLOB_E_RUNTIME          -> std::runtime_error    / RuntimeError
 *   MLOB_E_CUDA             -> std::runtime_error (CUDA failure, no GPU, ...)
 */
#ifndef MLOB_H_
#define MLOB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLOB_ABI_VERSION 1

typedef enum mlob_status {
  MLOB_OK = 0,
  MLOB_E_INVALID_ARGUMENT = 1,
  MLOB_E_OUT_OF_RANGE = 2,
  MLOB_E_LOGIC = 3,
  MLOB_E_RUNTIME = 4,
  MLOB_E_CUDA = 5,
} mlob_status;

/* ---- Record types (layouts identical to the reference structs) ---------- */

/* lob::MsgKind, lob/types.hpp:14-22 */
enum { MLOB_NEW_LIMIT = 0, MLOB_CANCEL_PARTIAL = 1, MLOB_DELETE = 2, MLOB_EXECUTE_VISIBLE = 3,
       MLOB_EXECUTE_HIDDEN = 4, MLOB_CROSS = 5, MLOB_HALT = 6 };
/* lob::Side, lob/types.hpp:8 */
enum { MLOB_BID = 0, MLOB_ASK = 1 };

/* lob::Message, lob/types.hpp:31-41 — 40 bytes, same field offsets, so a
 * std::vector<lob::Message> can be passed as-is. */
typedef struct mlob_message {
  int64_t time;
  uint64_t order_id;
  int64_t price;
  int64_t quantity;
  uint8_t kind;
  uint8_t side;
  uint8_t _pad[2];
  int32_t trader_id;
} mlob_message;

/* lob::RestingOrder, lob/types.hpp:43-51 — 40 bytes. */
typedef struct mlob_resting_order {
  int64_t price;
  int64_t quantity;
  uint64_t order_id;
  uint64_t arrival_seq;
  int32_t trader_id;
  int32_t _pad;
} mlob_resting_order;

/* lob::TradeRecord, lob/types.hpp:54-65 — 56 bytes. */
typedef struct mlob_trade {
  int64_t price;
  int64_t quantity;
  int64_t time;
  uint64_t passive_order_id;
  uint64_t aggressor_order_id;
  int32_t passive_trader_id;
  int32_t aggressor_trader_id;
  uint8_t aggressor_side;
  uint8_t _pad[7];
} mlob_trade;

/* lob::L2Level, lob/types.hpp:67-72 */
typedef struct mlob_level {
  int64_t price;
  int64_t quantity;
} mlob_level;

/* data::BookState list (data/store.hpp:16-21), flattened.  State i covers
 * levels[level_offset[i] .. level_offset[i+1]): its n_bids[i] bid levels
 * (best-first) followed by its ask levels (best-first). */
typedef struct mlob_book_states {
  uint64_t n_states;
  const uint64_t* message_index; /* [n_states], strictly increasing */
  const uint64_t* level_offset;  /* [n_states + 1] */
  const uint32_t* n_bids;        /* [n_states] */
  const mlob_level* levels;
} mlob_book_states;

/* ---- Configuration (env/config.hpp:13-71, agents/actions.hpp) ------------ */

enum { MLOB_MARKET_MAKER = 0, MLOB_EXECUTOR = 1, MLOB_DIRECTIONAL = 2 };      /* AgentType */
enum { MLOB_SPREAD_SKEW = 0, MLOB_FIXED_QUANT = 1, MLOB_AVST = 2 };           /* MMActionSpace */
enum { MLOB_REWARD_BUYSELL = 0, MLOB_REWARD_SPOONER = 1, MLOB_REWARD_EXEC = 2 }; /* RewardId */
enum { MLOB_REF_MID = 0, MLOB_REF_FAR_TOUCH = 1 };                            /* RefPriceMode */
enum { MLOB_OBS_MM_BASIC = 0, MLOB_OBS_MM_FULL = 1, MLOB_OBS_EXEC = 2 };      /* ObsSpaceId */
enum { MLOB_TASK_BUY = 0, MLOB_TASK_SELL = 1 };                               /* TaskDir */

#define MLOB_MAX_SPREAD_SKEW_ROWS 32
#define MLOB_MAX_GAMMA 16
#define MLOB_MAX_ACTIVE 8

/* env::AgentParams, env/config.hpp:32-48 (+ SpreadSkewTable, AvStParams).
 * mlob_default_agent_params() fills the reference struct defaults. */
typedef struct mlob_agent_params {
  int64_t order_size;
  int64_t inventory_cap;
  double rho;
  int32_t quadratic_penalty;
  int32_t ref_price;
  double lambda;
  double unfilled_penalty_coef;
  double lambda_exec;
  int64_t task_size;
  int32_t exec_complex;
  int32_t default_half_spread;
  double reward_scale;
  int32_t fixed_quant_from_mid;
  int32_t n_spread_skew;
  int32_t spread_skew_half[MLOB_MAX_SPREAD_SKEW_ROWS];
  int32_t spread_skew_skew[MLOB_MAX_SPREAD_SKEW_ROWS];
  int32_t n_gamma;
  int32_t _pad;
  double gamma_grid[MLOB_MAX_GAMMA];
  double kappa;
  double sigma;
  double horizon;
} mlob_agent_params;

/* env::AgentSpec, env/config.hpp:50-57 */
typedef struct mlob_agent_spec {
  int32_t type;
  int32_t count;
  int32_t mm_space;
  int32_t obs_space;
  int32_t reward;
  int32_t _pad;
  mlob_agent_params params;
} mlob_agent_spec;

#define MLOB_MAX_SPECS 8
#define MLOB_MAX_AGENTS 32

/* env::EnvConfig, env/config.hpp:59-71 */
typedef struct mlob_env_config {
  int32_t steps_per_episode;
  int32_t messages_per_step;
  int32_t start_stride_steps;
  int32_t n_specs;
  uint64_t book_capacity;
  uint64_t obs_depth;
  int64_t fallback_mid_half;
  uint64_t synthetic_init_id_base;
  uint64_t agent_id_base;
  uint64_t agent_id_range;
  uint64_t fill_reserve;
  mlob_agent_spec specs[MLOB_MAX_SPECS];
} mlob_env_config;

/* agents::Quote / QuoteList / env::AgentAction, actions.hpp:14-40, env.hpp:66-72 */
typedef struct mlob_quote {
  uint8_t side;
  uint8_t _pad[7];
  int64_t price;
  int64_t quantity;
} mlob_quote;

typedef struct mlob_agent_action {
  int32_t id;
  int32_t direct;
  int32_t n_quotes;
  int32_t _pad;
  mlob_quote quotes[2];
} mlob_agent_action;

/* env::ActiveOrder / AgentState, env.hpp:20-46 */
typedef struct mlob_active_order {
  uint64_t order_id;
  int64_t price;
  int64_t quantity;
  uint8_t side;
  uint8_t _pad[7];
} mlob_active_order;

typedef struct mlob_agent_state {
  int64_t inventory;
  int64_t cash;
  int64_t task_remaining;
  int32_t task_dir;
  int32_t n_active;
  double p_init;
  uint64_t order_nonce;
  int64_t filled_total;
  double slippage_total;
  mlob_active_order active[MLOB_MAX_ACTIVE];
} mlob_agent_state;

/* env::AgentInfo, env.hpp:48-57 */
typedef struct mlob_agent_info {
  int64_t inventory;
  int64_t cash;
  double portfolio_value;
  double slippage_step;
  double slippage_total;
  int64_t task_remaining;
  int64_t step_filled;
  int32_t step_fill_count;
  int32_t _pad;
} mlob_agent_info;

/* MarketEnv scalar accessors, env.hpp:131-137 (+ book next_seq / live counts) */
typedef struct mlob_env_scalars {
  int32_t step;
  int32_t terminal;
  uint64_t episode;
  int64_t mid_half;
  int64_t prev_mid_half;
  double mean_mid_ticks;
  int64_t last_bid;
  int64_t last_ask;
  int64_t last_time;
  uint64_t messages_processed;
  uint64_t next_seq;
  uint64_t live_bid;
  uint64_t live_ask;
} mlob_env_scalars;

/* ippo::MarketVecEnv::EpisodeStats, rollout.hpp:248-254 */
typedef struct mlob_episode_stats {
  double pv_sum;
  double slippage_sum;
  double completion_sum;
  double inventory_sq_sum;
  int64_t episodes;
} mlob_episode_stats;

/* data::SynthConfig, data/synth.hpp:18-36 */
typedef struct mlob_synth_config {
  uint64_t n_messages;
  int64_t initial_mid;
  double volatility;
  double p_new_passive;
  double p_new_cross;
  double p_cancel;
  double p_delete;
  double p_execute;
  int32_t band;
  int32_t seed_levels;
  int64_t max_qty;
  int64_t seed_qty;
  uint64_t state_sample_every;
  uint64_t state_depth;
} mlob_synth_config;

/* ---- Defaults ------------------------------------------------------------ */

void mlob_default_agent_params(mlob_agent_params* out);            /* env/config.hpp:32-48 */
void mlob_default_agent_spec(mlob_agent_spec* out);                /* env/config.hpp:50-57 */
void mlob_default_env_config(mlob_env_config* out);                /* env/config.hpp:59-71 */
void mlob_default_synth_config(mlob_synth_config* out);            /* data/synth.hpp:18-36 */
int mlob_action_arity(const mlob_agent_spec* spec);                /* env/config.hpp:73-90 */
int mlob_observation_size(int obs_space, uint64_t depth);          /* observations.hpp:69-76 */
mlob_status mlob_validate_env_config(const mlob_env_config* cfg);  /* env/config.hpp:96-120 */

const char* mlob_last_error(void);
int mlob_abi_version(void);

/* ---- Host message stores (data/store.hpp, data/synth.hpp) ---------------- */

typedef struct mlob_host_store mlob_host_store;

/* data::synth_generate, data/synth.hpp:39-177: deterministic synthetic MBO
 * stream (host C++, identical output to the reference generator). */
mlob_status mlob_host_store_synth(const mlob_synth_config* cfg, uint64_t seed,
                                  mlob_host_store** out);
/* Wraps caller-provided records (copied). */
mlob_status mlob_host_store_create(const mlob_message* msgs, uint64_t n_msgs,
                                   const mlob_book_states* states, mlob_host_store** out);
/* Drops the first `n` messages and every state before index n; shifts the
 * remaining states' message_index by -n (SURVEY §8d config D trim). */
mlob_status mlob_host_store_trim_front(mlob_host_store* s, uint64_t n);
uint64_t mlob_host_store_n_messages(const mlob_host_store* s);
const mlob_message* mlob_host_store_messages(const mlob_host_store* s);
uint64_t mlob_host_store_n_states(const mlob_host_store* s);
/* Copies state i; writes level counts; fails with OUT_OF_RANGE if cap is short. */
mlob_status mlob_host_store_state(const mlob_host_store* s, uint64_t i, uint64_t* message_index,
                                  mlob_level* bids, uint32_t* n_bids, mlob_level* asks,
                                  uint32_t* n_asks, uint32_t cap);
void mlob_host_store_free(mlob_host_store* s);
/* Binary image of a host store (messages + sampled states).  One process per
 * node synthesises and saves, the other ranks load: the store is built once
 * per node, not once per GPU (new; the reference builds one store per
 * process, util/config.hpp:382-419). */
mlob_status mlob_host_store_save(const mlob_host_store* s, const char* path);
mlob_status mlob_host_store_load(const char* path, mlob_host_store** out);

/* data::build_episode_index, data/store.hpp:52-72.  Writes up to `cap` starts
 * and the full count to *n_out. */
mlob_status mlob_build_episode_index(uint64_t n_messages, int steps_per_episode,
                                     int messages_per_step, int start_stride_steps,
                                     uint64_t* starts, uint64_t cap, uint64_t* n_out);

/* ---- Device store -------------------------------------------------------- */

typedef struct mlob_store mlob_store;

/* Uploads a message store (and its sampled book states) to `device` once; it
 * is shared read-only by every env handle on that device (store.hpp:23-24).
 * Messages are repacked to 32-byte device records; prices, quantities must
 * fit in int32 and replay trader ids in [0, 255] (INVALID_ARGUMENT if not). */
mlob_status mlob_store_upload(const mlob_host_store* host, int device, mlob_store** out);
mlob_status mlob_store_upload_raw(const mlob_message* msgs, uint64_t n_msgs,
                                  const mlob_book_states* states, int device, mlob_store** out);
uint64_t mlob_store_n_messages(const mlob_store* s);
uint64_t mlob_store_device_bytes(const mlob_store* s);
void mlob_store_free(mlob_store* s);

/* data::load_lobster (data/lobster.hpp:119-193) straight into a device store:
 * the message / orderbook CSV pair is read once and parsed on the GPU (one
 * thread per row; sampled orderbook rows -> book states at offsets 0,
 * sample_every, 2*sample_every, ...).  Same acceptance rules and error texts
 * as the reference (first failing row wins); invalid_argument for
 * units_per_tick < 1 / sample_every == 0, runtime_error for file and format
 * errors, invalid_argument when a value exceeds the device int32 layout. */
mlob_status mlob_store_load_lobster(const char* message_path, const char* orderbook_path,
                                    int64_t units_per_tick, uint64_t sample_every, int device,
                                    mlob_store** out);
/* Readback of a device store (parity checks): messages widened to the
 * reference record (price / quantity as the device keeps them: zero for
 * kinds that do not use them), and book states. */
mlob_status mlob_store_read_messages(const mlob_store* s, uint64_t first, uint64_t n, mlob_message* out);
uint64_t mlob_store_n_states(const mlob_store* s);
mlob_status mlob_store_state(const mlob_store* s, uint64_t i, uint64_t* message_index, mlob_level* bids,
                             uint32_t* n_bids, mlob_level* asks, uint32_t* n_asks, uint32_t cap);

/* ---- Batched environment (ippo::MarketVecEnv + env::MarketEnv) ----------- */

typedef struct mlob_venv mlob_venv;

enum {
  MLOB_VENV_AUTO_RESET = 1u << 0,    /* MarketVecEnv semantics: reset on terminal (rollout.hpp:299-317) */
  MLOB_VENV_RECORD_TRADES = 1u << 1, /* keep MarketEnv::step_trades() per env (env.hpp:139-141) */
};

typedef struct mlob_venv_desc {
  const mlob_store* store;
  mlob_env_config cfg;
  const uint64_t* episode_pool; /* MarketVecEnv episode pool (rollout.hpp:153-156); NULL = all episodes */
  uint64_t pool_len;
  uint64_t seed;                /* global seed (env.hpp:100-101) */
  uint64_t n_envs_global;       /* auto-reset round-robin uses the global count (rollout.hpp:286-288) */
  uint64_t env_index_base;      /* first global env index owned by this handle (GPU shard) */
  uint64_t n_envs_local;
  const uint64_t* env_seeds;    /* optional per-env seed override [n_envs_local] */
  const uint64_t* env_indices;  /* optional per-env env-index override [n_envs_local] */
  uint32_t flags;
  uint32_t trade_capacity;      /* per-env per-step trade log capacity when RECORD_TRADES */
  int32_t device;
  int32_t _pad;
  void* stream;                 /* cudaStream_t to launch on (NULL = handle-owned stream) */
} mlob_venv_desc;

/* MarketVecEnv ctor (rollout.hpp:153-178) / MarketEnv ctor (env.hpp:100-122). */
mlob_status mlob_venv_create(const mlob_venv_desc* desc, mlob_venv** out);
void mlob_venv_destroy(mlob_venv* v);

uint64_t mlob_venv_n_envs(const mlob_venv* v);
int mlob_venv_n_agents(const mlob_venv* v);
int mlob_venv_n_types(const mlob_venv* v);
uint64_t mlob_venv_n_streams(const mlob_venv* v, int type);  /* rollout.hpp:182-184 */
int mlob_venv_obs_dim(const mlob_venv* v, int type);         /* rollout.hpp:185-188 */
int mlob_venv_n_actions(const mlob_venv* v, int type);       /* rollout.hpp:189-191 */
uint64_t mlob_venv_n_episodes(const mlob_venv* v);

/* MarketVecEnv::reset_all (rollout.hpp:194-200). */
mlob_status mlob_venv_reset_all(mlob_venv* v);
/* MarketEnv::reset(episode) for every env: episodes[n_envs_local]. */
mlob_status mlob_venv_reset_envs(mlob_venv* v, const uint64_t* episodes);

/* Action ids, env-major [n_envs_local * n_agents] (flat agent order).  With
 * on_device != 0 `ids` is a device pointer already on the handle's device.
 * MarketVecEnv::set_action (rollout.hpp:215-222) per element; ids are
 * validated against the action arity before launch (actions.hpp:69-70). */
mlob_status mlob_venv_set_actions(mlob_venv* v, const int32_t* ids, int on_device);
/* Direct-quote actions (env.hpp:290-298), [n_envs_local * n_agents]. */
mlob_status mlob_venv_set_direct_actions(mlob_venv* v, const mlob_agent_action* actions);

/* MarketVecEnv::step_all (rollout.hpp:224-234) / MarketEnv::step (env.hpp:194-254)
 * for every env, stream-ordered: returns once the kernels are enqueued. */
mlob_status mlob_venv_step(mlob_venv* v);
/* bench::RandomStepHarness::step_env (bench.hpp:53-70): actions drawn on the
 * device from CounterRng(make_key(bench_seed, BenchAction, e, global_step)). */
mlob_status mlob_venv_step_random(mlob_venv* v, uint64_t bench_seed, uint64_t global_step);

/* MarketVecEnv::gather (rollout.hpp:202-213): obs [n_streams(type) * obs_dim]
 * and reset flags [n_streams(type)] into host memory (NULL skips either). */
mlob_status mlob_venv_gather(mlob_venv* v, int type, double* obs_out, uint8_t* reset_out);
/* Device pointers of the same buffers (valid until destroy; contents until the next step). */
const double* mlob_venv_obs_device(const mlob_venv* v, int type);
/* Rewards/dones [n_envs_local * n_agents] (rollout.hpp:236-243, cached pre-reset). */
mlob_status mlob_venv_rewards(mlob_venv* v, double* out);
mlob_status mlob_venv_dones(mlob_venv* v, uint8_t* out);
const double* mlob_venv_rewards_device(const mlob_venv* v);
const uint8_t* mlob_venv_dones_device(const mlob_venv* v);
/* MarketEnv::output().infos, [n_envs_local * n_agents] (env.hpp:445-464). */
mlob_status mlob_venv_infos(mlob_venv* v, mlob_agent_info* out);

/* One collect_rollout iteration's env I/O in a single call (set_action,
 * step_all, reward/done, then the next gather: rollout.hpp:72-98): host action ids in,
 * host rewards / dones / infos / per-type obs + reset flags out, same layouts
 * as the separate calls.  Any pointer may be NULL (actions NULL = step with
 * the current actions).  Actions are range-checked on the device before any
 * env steps (actions.hpp:69-70; a bad id fails with MLOB_E_OUT_OF_RANGE and
 * leaves every env unchanged).  The step runs in env chunks on two streams
 * while a copy stream returns each finished chunk's outputs, so the
 * transfers overlap the step.  Host buffers should be page-locked for the
 * overlap.  Returns when every output is in host memory. */
typedef struct mlob_step_io {
  const int32_t* actions;                  /* [n_envs_local * n_agents] */
  double* rewards;                         /* [n_envs_local * n_agents] */
  uint8_t* dones;                          /* [n_envs_local * n_agents] */
  mlob_agent_info* infos;                  /* [n_envs_local * n_agents] */
  double* obs[MLOB_MAX_SPECS];             /* per type [n_streams(t) * obs_dim(t)] */
  uint8_t* resets[MLOB_MAX_SPECS];         /* per type [n_streams(t)] */
} mlob_step_io;
mlob_status mlob_venv_step_io(mlob_venv* v, const mlob_step_io* io);

/* ---- On-device policy inference and rollouts (ippo/net.hpp, rollout.hpp) -- */

/* ippo::PolicyNet (net.hpp:18-30): host arrays in the reference's layout,
 * gate order [reset, update, candidate]. */
typedef struct mlob_policy_net {
  int32_t obs_dim;
  int32_t hidden;
  int32_t n_actions;
  int32_t _pad;
  const double* w_ih;     /* (3H, obs_dim) */
  const double* w_hh;     /* (3H, H) */
  const double* b_ih;     /* 3H */
  const double* b_hh;     /* 3H */
  const double* w_actor;  /* (n_actions, H) */
  const double* b_actor;  /* n_actions */
  const double* w_critic; /* H */
  double b_critic;
} mlob_policy_net;

/* One network per agent type (obs_dim / n_actions must match the type's;
 * hidden <= 512, net.hpp:86-87).  Uploads the weights and zeroes the
 * per-stream hidden states, as train_loop does before its first rollout
 * (rollout.hpp:132-135).  Re-uploading weights keeps the hidden states when
 * the shapes are unchanged (the learner's update between rollouts). */
mlob_status mlob_venv_set_nets(mlob_venv* v, const mlob_policy_net* nets);

/* TrainLoopConfig fields used by collect_rollout (rollout.hpp:30-37). */
typedef struct mlob_rollout_config {
  int32_t rollout_len;
  int32_t _pad;
  double discount;
  double gae_lambda;
  uint64_t seed;
} mlob_rollout_config;

/* collect_rollout (rollout.hpp:41-124) on the device: per step, for each type
 * the GRU forward of every stream (net.hpp:120-188) and the categorical draw
 * keyed (seed, ActionSample, type, update_index, t, stream) (ppo.hpp:80-98),
 * then the env step with auto-reset; after T steps the bootstrap values and
 * GAE (gae.hpp:14-32).  The rollout batch (ppo.hpp:33-48) stays in HBM; read
 * it with mlob_venv_rollout_read / _device.  Hidden states persist across
 * calls.  Needs MLOB_VENV_AUTO_RESET, set_nets and a reset. */
mlob_status mlob_venv_collect_rollout(mlob_venv* v, const mlob_rollout_config* cfg, uint64_t update_index);

/* RolloutBatch fields (ppo.hpp:33-48), time-major; HIDDEN = the persistent
 * hidden state after the rollout, (B, H). */
enum { MLOB_RB_OBS = 0, MLOB_RB_ACTIONS = 1, MLOB_RB_LOG_PROBS = 2, MLOB_RB_VALUES = 3,
       MLOB_RB_REWARDS = 4, MLOB_RB_DONES = 5, MLOB_RB_RESETS = 6, MLOB_RB_H0 = 7,
       MLOB_RB_ADVANTAGES = 8, MLOB_RB_RETURNS = 9, MLOB_RB_HIDDEN = 10 };
/* Copies one field of type `type`'s batch to host memory (cap_bytes checked). */
mlob_status mlob_venv_rollout_read(mlob_venv* v, int type, int field, void* out, uint64_t cap_bytes);
/* Device pointer of the same field (NULL before the first rollout). */
const void* mlob_venv_rollout_device(const mlob_venv* v, int type, int field);

/* ippo::PpoConfig (ppo.hpp:19-28) */
typedef struct mlob_ppo_config {
  int32_t epochs;
  int32_t minibatches;
  double clip_eps;
  double vf_coef;
  double ent_coef;
  double lr;
  double max_grad_norm;
  int32_t normalize_adv;
  int32_t _pad;
} mlob_ppo_config;
void mlob_default_ppo_config(mlob_ppo_config* out);

/* ippo::UpdateMetrics (ppo.hpp:69-77) */
typedef struct mlob_update_metrics {
  double pg_loss;
  double v_loss;
  double entropy;
  double approx_kl;
  double clip_frac;
  double grad_norm;
  double mean_reward;
} mlob_update_metrics;

/* ppo_update (ppo.hpp:263-310) of type `type` on the device over the batch of
 * the last collect_rollout: `epochs` passes over a CounterRng-shuffled
 * partition of the streams (key (seed, Minibatch, update_index, epoch,
 * type)), each minibatch a BPTT forward/backward of the GRU, global-norm
 * clipping and an Adam step (net.hpp:281-331; the Adam state lives in the
 * handle, reset by set_nets).  The updated weights are used by the next
 * rollout; read them with mlob_venv_read_net.  runtime_error on a non-finite
 * loss, as the reference. */
mlob_status mlob_venv_ppo_update(mlob_venv* v, int type, const mlob_ppo_config* cfg, uint64_t seed,
                                 uint64_t update_index, mlob_update_metrics* out);
/* The type's current parameters, PolicyNet::for_each_param order (net.hpp:36-41). */
mlob_status mlob_venv_read_net(mlob_venv* v, int type, double* flat, uint64_t cap);

/* ---- Scripted policies and cross-play evaluation (ippo/evaluate.hpp) ------ */

/* ippo::PolicyKind (evaluate.hpp:17); Learned is not available on the device. */
enum { MLOB_POLICY_LEARNED = 0, MLOB_POLICY_TWAP = 1, MLOB_POLICY_AVST = 2, MLOB_POLICY_RANDOM = 3,
       MLOB_POLICY_NOOP = 4 };
/* baselines::TwapPriceMode (twap.hpp:11) */
enum { MLOB_TWAP_AGGRESSIVE = 0, MLOB_TWAP_PASSIVE = 1 };

/* ippo::PolicyChoice (evaluate.hpp:19-25) without the network pointer:
 * AvSt = baselines::AvStBaseline (avst.hpp:14-17), TWAP = the price mode of
 * baselines::make_twap_plan (twap.hpp:21-33).  mlob_default_policy() fills
 * the reference defaults (AvStParams actions.hpp:142-147, gamma_index 1). */
typedef struct mlob_policy {
  int32_t kind;
  int32_t twap_mode;
  int32_t avst_gamma_index;
  int32_t n_gamma;
  double gamma_grid[MLOB_MAX_GAMMA];
  double kappa;
  double sigma;
  double horizon;
  const struct mlob_policy_net* net; /* Learned: argmax of the GRU policy (evaluate.hpp:80-90) */
} mlob_policy;
void mlob_default_policy(int kind, mlob_policy* out);

/* Scripted actions for the next steps (evaluate.hpp:56-99 choose_action; Learned
 * options only through mlob_evaluate_matrix),
 * twap.hpp:37-58, avst.hpp:19-32): env e's agents of type t act by
 * policies[env_policy[e * n_types + t]] from the env's own state on the
 * device; Random draws CounterRng(make_key(env seed, EpisodeDraw, env_cell[e],
 * episode, step, agent)).below(arity) (env_cell NULL = 0).  Stays in force
 * until set_actions / set_direct_actions. */
mlob_status mlob_venv_set_policies(mlob_venv* v, const mlob_policy* policies, int n_policies,
                                   const uint8_t* env_policy, const uint64_t* env_cell);

/* ippo::TypeCellStats / CellStats (evaluate.hpp:27-42), labels omitted. */
typedef struct mlob_type_cell_stats {
  double pv_mean;
  double pv_stderr;
  double slippage_mean;
  double slippage_stderr;
  double completion_mean;
  int64_t filled_total;
  int32_t no_fills;
  int32_t _pad;
} mlob_type_cell_stats;
typedef struct mlob_cell_stats {
  mlob_type_cell_stats per_type[2];
  int64_t episodes;
} mlob_cell_stats;

/* ippo::evaluate_matrix (evaluate.hpp:104-217) for scripted policies: every
 * (row, col, episode) of the cross-play grid is one environment of a single
 * device batch (env seed = `seed`, env index 0, as the reference's one
 * MarketEnv), stepped to the episode end; the per-cell statistics are then
 * formed on the host in the reference's order.  out[n_rows * n_cols],
 * row-major.  Learned options run their network on the device each step
 * (hidden state zeroed at the episode start, argmax action).  Errors:
 * invalid_argument as the reference (two types, episodes non-empty, a
 * Learned option without a network or with the wrong shape). */
mlob_status mlob_evaluate_matrix(const mlob_store* store, const mlob_env_config* cfg,
                                 const uint64_t* episodes, uint64_t n_episodes,
                                 const mlob_policy* type0, int n_type0, const mlob_policy* type1,
                                 int n_type1, uint64_t seed, int device, mlob_cell_stats* out);
/* MarketEnv::output().obs for one env, all agents concatenated. */
mlob_status mlob_venv_env_obs(mlob_venv* v, uint64_t env, double* out, uint64_t cap);

/* MarketVecEnv::episode_stats / clear_episode_stats (rollout.hpp:255-278).
 * episode_stats sums this handle's envs in env order (bit-identical to the
 * reference); episode_stats_device reduces on the GPU (K4) into `out_device`,
 * MLOB_STAT_WORDS doubles per type (layout below), ready for an all-reduce.
 * PV, slippage and inventory² are multiples of 0.5 and the remaining-quantity
 * sum is an integer, so their sums are exact in any order; the exact
 * completion sum is episodes·count − Σremaining / task_size (executors). */
#define MLOB_STAT_WORDS 6
enum { MLOB_STAT_PV = 0, MLOB_STAT_SLIPPAGE = 1, MLOB_STAT_COMPLETION = 2, MLOB_STAT_INVENTORY_SQ = 3,
       MLOB_STAT_EPISODES = 4, MLOB_STAT_REMAINING = 5 };
mlob_status mlob_venv_episode_stats(mlob_venv* v, int type, mlob_episode_stats* out);
mlob_status mlob_venv_episode_stats_device(mlob_venv* v, double* out_device);
mlob_status mlob_venv_clear_episode_stats(mlob_venv* v);
/* The episode statistics of every type summed over all ranks of a NCCL
 * communicator — the one collective of the path: K4 on this
 * GPU, one ncclAllReduce(sum) of MLOB_STAT_WORDS doubles per type on the
 * handle's stream, then per-type stats (completion formed exactly as above).
 * Replaces MarketVecEnv::episode_stats (rollout.hpp:255-270) as the trainer
 * consumes it per update (train.hpp:200-219) when the envs are sharded over
 * GPUs.  nccl_comm: an ncclComm_t (one rank per GPU) or NULL for this handle
 * alone; ncclAllReduce is resolved at run time from the process's
 * libnccl.so.2 (MLOB_E_RUNTIME if absent).  out: [n_types]. */
mlob_status mlob_venv_allreduce_episode_stats(mlob_venv* v, void* nccl_comm, mlob_episode_stats* out);

/* Parity readers in reference record formats. */
mlob_status mlob_venv_read_scalars(mlob_venv* v, uint64_t env, mlob_env_scalars* out);
/* OrderBook::orders(side), book.hpp:122-126: worst-to-best storage order. */
mlob_status mlob_venv_read_book(mlob_venv* v, uint64_t env, int side, mlob_resting_order* out,
                                uint64_t cap, uint64_t* n_out);
/* MarketEnv::agent_state, env.hpp:129 (active orders rebuilt as env.hpp:398-407). */
mlob_status mlob_venv_read_agent(mlob_venv* v, uint64_t env, int agent, mlob_agent_state* out);
/* MarketEnv::step_trades, env.hpp:139-141 (needs MLOB_VENV_RECORD_TRADES). */
mlob_status mlob_venv_read_trades(mlob_venv* v, uint64_t env, mlob_trade* out, uint64_t cap,
                                  uint64_t* n_out);
/* Σ messages_processed over the handle's envs (bench.hpp:133-154). */
mlob_status mlob_venv_messages_processed(mlob_venv* v, uint64_t* out);

mlob_status mlob_venv_synchronize(mlob_venv* v);
void* mlob_venv_stream(const mlob_venv* v);
/* Kernel launches issued by this handle so far (bench evidence). */
uint64_t mlob_venv_launch_count(const mlob_venv* v);
/* Per-kernel timing of the step (measurement only): with profiling on, every
 * mlob_venv_step / _step_random records CUDA events around its three kernels
 * on the handle's stream; kernel_ms returns the summed milliseconds of
 * [act_kernel, book_kernel, outcome_kernel] since profiling was switched on
 * and the number of steps timed. */
mlob_status mlob_venv_profile(mlob_venv* v, int on);
mlob_status mlob_venv_kernel_ms(mlob_venv* v, double* out3, uint64_t* steps);

#ifdef __cplusplus
}
#endif

#endif /* MLOB_H_ */
