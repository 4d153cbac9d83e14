/*
 * oracle_api.h — TEST INFRASTRUCTURE ONLY.
 *
 * One C API, implemented twice:
 *   orc_*  by oracle/marlob_oracle.c  — a plain-C restatement of the reference
 *                                       algorithm (each function cites the
 *                                       reference file:line it follows);
 *   ref_*  by oracle/ref_shim.cpp     — the unmodified reference headers under
 *                                       /root/reference/proj/include compiled in
 *                                       place into oracle/_ref/libmarlob_ref.so.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load these
 * libraries; the product (paper_2511_02136_b200/) never links them.
 */
#ifndef MLOB_ORACLE_API_H_
#define MLOB_ORACLE_API_H_

#include "../include/mlob.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_bench_row {
  int32_t messages_per_step;
  int32_t agents_per_type;
  int32_t workers;
  int32_t _pad;
  uint64_t env_steps;
  uint64_t messages;
  double wall_seconds;
  double steps_per_sec;
  double messages_per_sec;
  double worker_utilization;
} orc_bench_row;

#define ORACLE_DECLARE(P)                                                                      \
  const char* P##last_error(void);                                                             \
  /* stores (data/store.hpp, data/synth.hpp) */                                                \
  void* P##store_synth(const mlob_synth_config* cfg, uint64_t seed);                          \
  void* P##store_create(const mlob_message* msgs, uint64_t n, const mlob_book_states* st);    \
  uint64_t P##store_n_messages(void* s);                                                       \
  const mlob_message* P##store_messages(void* s);                                              \
  uint64_t P##store_n_states(void* s);                                                         \
  int P##store_state(void* s, uint64_t i, uint64_t* msg_index, mlob_level* bids,              \
                     uint32_t* nb, mlob_level* asks, uint32_t* na, uint32_t cap);              \
  void P##store_free(void* s);                                                                 \
  /* data/lobster.hpp load_lobster */                                                          \
  void* P##load_lobster(const char* message_path, const char* orderbook_path,                  \
                        int64_t units_per_tick, uint64_t sample_every, int* status);           \
  /* book (lob/book.hpp) */                                                                    \
  void* P##book_create(uint64_t capacity);                                                     \
  int P##book_init_from_l2(void* b, const mlob_level* bids, uint32_t nb,                      \
                           const mlob_level* asks, uint32_t na, uint64_t id_base);            \
  uint64_t P##book_process(void* b, const mlob_message* m, mlob_trade* out, uint64_t cap);    \
  uint64_t P##book_orders(void* b, int side, mlob_resting_order* out, uint64_t cap);          \
  uint64_t P##book_next_seq(void* b);                                                          \
  int64_t P##book_mid_half(void* b, int64_t fallback);                                         \
  void P##book_l2(void* b, uint64_t depth, mlob_level* bids, uint32_t* nb, mlob_level* asks,   \
                  uint32_t* na);                                                               \
  void P##book_free(void* b);                                                                  \
  /* single environment (env/env.hpp) */                                                       \
  void* P##env_create(void* store, const mlob_env_config* cfg, uint64_t seed, int env_index,   \
                      int* status);                                                            \
  uint64_t P##env_n_episodes(void* e);                                                         \
  uint64_t P##env_episode_start(void* e, uint64_t episode);                                    \
  int P##env_n_agents(void* e);                                                                \
  int P##env_reset(void* e, uint64_t episode);                                                 \
  int P##env_step_ids(void* e, const int32_t* ids, uint64_t n);                                \
  int P##env_step(void* e, const mlob_agent_action* actions, uint64_t n);                      \
  void P##env_scalars(void* e, mlob_env_scalars* out);                                         \
  uint64_t P##env_book(void* e, int side, mlob_resting_order* out, uint64_t cap);             \
  void P##env_agent(void* e, int a, mlob_agent_state* out);                                    \
  void P##env_info(void* e, int a, mlob_agent_info* out);                                      \
  double P##env_reward(void* e, int a);                                                        \
  int P##env_done(void* e, int a);                                                             \
  uint64_t P##env_obs(void* e, int a, double* out, uint64_t cap);                              \
  uint64_t P##env_trades(void* e, mlob_trade* out, uint64_t cap);                              \
  void P##env_free(void* e);                                                                   \
  /* batched env (ippo/rollout.hpp MarketVecEnv) */                                            \
  void* P##venv_create(void* store, const mlob_env_config* cfg, const uint64_t* pool,          \
                       uint64_t pool_len, uint64_t seed, int n_envs, int workers, int* status);\
  int P##venv_reset_all(void* v);                                                              \
  int P##venv_set_action(void* v, int type, uint64_t stream, int action);                      \
  int P##venv_step_all(void* v);                                                               \
  void P##venv_gather(void* v, int type, double* obs, uint8_t* resets);                        \
  double P##venv_reward(void* v, int type, uint64_t stream);                                   \
  int P##venv_done(void* v, int type, uint64_t stream);                                        \
  void P##venv_episode_stats(void* v, int type, mlob_episode_stats* out);                      \
  void P##venv_clear_episode_stats(void* v);                                                   \
  void* P##venv_instance(void* v, uint64_t e);                                                 \
  void P##venv_free(void* v);                                                                  \
  /* throughput harness (bench/bench.hpp run_throughput, one grid cell) */                     \
  int P##bench_run(void* store, const mlob_env_config* base, int n_envs, int n_steps,          \
                   int warmup, int workers, uint64_t seed, int messages_per_step,              \
                   int agents_per_type, orc_bench_row* out);                                   \
  /* networks and rollouts (ippo/net.hpp make_policy_net, rollout.hpp collect_rollout) */     \
  int P##make_policy_net(int obs_dim, int hidden, int n_actions, uint64_t seed, double* out);  \
  int P##venv_collect_rollout(void* v, const mlob_policy_net* nets,                           \
                              const mlob_rollout_config* cfg, uint64_t update_index);         \
  uint64_t P##venv_rollout_field(void* v, int type, int field, void* out, uint64_t cap);      \
  /* cross-play grid (ippo/evaluate.hpp evaluate_matrix, scripted policies) */                \
  int P##evaluate_matrix(void* store, const mlob_env_config* cfg, const uint64_t* episodes,   \
                         uint64_t n_episodes, const mlob_policy* type0, int n0,               \
                         const mlob_policy* type1, int n1, uint64_t seed, mlob_cell_stats* out);

ORACLE_DECLARE(orc_)
ORACLE_DECLARE(ref_)

/* RNG known-answer exports and the reference test-stream generator
 * (tests/reference/random_messages.hpp:16-119). */
typedef struct orc_stream_config {
  uint64_t n_messages;
  int64_t initial_ref;
  int32_t band;
  int32_t _pad;
  int64_t max_qty;
  double p_new, p_marketable, p_cancel, p_delete, p_execute, p_absent;
} orc_stream_config;

uint64_t orc_splitmix64(uint64_t z);
uint64_t orc_make_key(uint64_t seed, int n, const uint64_t* words);
void orc_crng_draws(uint64_t key, uint64_t n, uint64_t* out);
void orc_random_stream(const orc_stream_config* cfg, uint64_t seed, mlob_message* out);
/* ppo_update (ppo.hpp:263-310) over the last ref_venv_collect_rollout batch; the
 * device update is pinned to the reference directly (reference-side only) */
int ref_venv_ppo_update(void* v, int type, const mlob_ppo_config* cfg, uint64_t seed, uint64_t update_index,
                        mlob_update_metrics* out);
uint64_t ref_venv_read_net(void* v, int type, double* out, uint64_t cap);
/* evaluate.hpp:56-99 choose_action (scripted kinds) on an orc env */
int orc_choose_action(void* env, int agent, const mlob_policy* p, int step, uint64_t seed,
                      uint64_t cell_id, uint64_t episode, mlob_agent_action* out);
void ref_random_stream(const orc_stream_config* cfg, uint64_t seed, mlob_message* out);
/* tests/reference/naive_book.hpp:16-134 (reference-side only) */
void* ref_naive_create(void);
uint64_t ref_naive_process(void* b, const mlob_message* m, mlob_trade* out, uint64_t cap);
int ref_naive_best(void* b, int side, int64_t* price);
uint32_t ref_naive_l2_full(void* b, int side, mlob_level* out, uint32_t cap);
void ref_naive_free(void* b);

#ifdef __cplusplus
}
#endif

#endif
