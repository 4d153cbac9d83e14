// mlob/vec_env.hpp — the C++ drop-in for the reference's batched
// environment: CudaMarketVecEnv satisfies the VecEnv concept that
// ippo::collect_rollout / ippo::train_loop are templated over
// (marlob/ippo/rollout.hpp:16-28) with the member set and layouts of
// ippo::MarketVecEnv (rollout.hpp:151-336), running every env step on the GPU
// through the C ABI (include/mlob.h, libmlob.so).
//
// Include it after (or instead of) "marlob/ippo/rollout.hpp" with
// -I<reference>/proj/include -I<this repo>/include and link -lmlob:
//
//   marlob::ippo::CudaMarketVecEnv env(store, index, cfg, pool, seed, n_envs);
//   marlob::ippo::train_loop(env, nets, adams, loop_cfg, per_update);
//
// Multi-GPU: one process per GPU, each constructing the env over its shard
// (env_index_base / n_envs_global); episode statistics are summed
// across ranks with allreduce_episode_stats(ncclComm_t) — the path's one
// collective (rollout.hpp:255-270 as consumed by train.hpp:200-219).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../mlob.h"
#include "marlob/data/store.hpp"
#include "marlob/env/config.hpp"
#include "marlob/ippo/rollout.hpp"

namespace marlob::ippo {

// mlob_status -> the reference's exception classes (include/mlob.h header).
inline void mlob_throw(mlob_status s) {
  if (s == MLOB_OK) return;
  const std::string m = mlob_last_error();
  switch (s) {
    case MLOB_E_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case MLOB_E_OUT_OF_RANGE: throw std::out_of_range(m);
    case MLOB_E_LOGIC: throw std::logic_error(m);
    default: throw std::runtime_error(m);
  }
}

// env::EnvConfig (env/config.hpp:59-71) -> mlob_env_config, field by field.
inline mlob_env_config to_mlob_config(const env::EnvConfig& c) {
  mlob_env_config r;
  mlob_default_env_config(&r);
  if (c.specs.size() > MLOB_MAX_SPECS) throw std::invalid_argument("CudaMarketVecEnv: too many agent specs");
  r.steps_per_episode = c.steps_per_episode;
  r.messages_per_step = c.messages_per_step;
  r.start_stride_steps = c.start_stride_steps;
  r.n_specs = static_cast<int32_t>(c.specs.size());
  r.book_capacity = c.book_capacity;
  r.obs_depth = c.obs_depth;
  r.fallback_mid_half = c.fallback_mid_half;
  r.synthetic_init_id_base = c.synthetic_init_id_base;
  r.agent_id_base = c.agent_id_base;
  r.agent_id_range = c.agent_id_range;
  r.fill_reserve = c.fill_reserve;
  for (size_t s = 0; s < c.specs.size(); ++s) {
    const env::AgentSpec& a = c.specs[s];
    mlob_agent_spec& o = r.specs[s];
    mlob_default_agent_spec(&o);
    o.type = static_cast<int32_t>(a.type);
    o.count = a.count;
    o.mm_space = static_cast<int32_t>(a.mm_space);
    o.obs_space = static_cast<int32_t>(a.obs_space);
    o.reward = static_cast<int32_t>(a.reward);
    const env::AgentParams& p = a.params;
    mlob_agent_params& q = o.params;
    q.order_size = p.order_size;
    q.inventory_cap = p.inventory_cap;
    q.rho = p.rho;
    q.quadratic_penalty = p.quadratic_penalty ? 1 : 0;
    q.ref_price = static_cast<int32_t>(p.ref_price);
    q.lambda = p.lambda;
    q.unfilled_penalty_coef = p.unfilled_penalty_coef;
    q.lambda_exec = p.lambda_exec;
    q.task_size = p.task_size;
    q.exec_complex = p.exec_complex ? 1 : 0;
    q.default_half_spread = p.default_half_spread;
    q.reward_scale = p.reward_scale;
    q.fixed_quant_from_mid = p.fixed_quant_from_mid ? 1 : 0;
    if (p.spread_skew.rows.size() > MLOB_MAX_SPREAD_SKEW_ROWS || p.avst.gamma_grid.size() > MLOB_MAX_GAMMA)
      throw std::invalid_argument("CudaMarketVecEnv: action table above the device limit");
    q.n_spread_skew = static_cast<int32_t>(p.spread_skew.rows.size());
    for (size_t i = 0; i < p.spread_skew.rows.size(); ++i) {
      q.spread_skew_half[i] = p.spread_skew.rows[i].half_spread;
      q.spread_skew_skew[i] = p.spread_skew.rows[i].skew;
    }
    q.n_gamma = static_cast<int32_t>(p.avst.gamma_grid.size());
    for (size_t i = 0; i < p.avst.gamma_grid.size(); ++i) q.gamma_grid[i] = p.avst.gamma_grid[i];
    q.kappa = p.avst.kappa;
    q.sigma = p.avst.sigma;
    q.horizon = p.avst.horizon;
  }
  return r;
}

// data::MessageStore (data/store.hpp:23-39) uploaded once to `device`; shared
// read-only by every CudaMarketVecEnv built on it (store.hpp:23-24).
class CudaMessageStore {
 public:
  CudaMessageStore(const data::MessageStore& store, int device = 0) {
    std::vector<mlob_level> lv;
    std::vector<uint64_t> idx, off{0};
    std::vector<uint32_t> nb;
    for (const auto& s : store.book_states) {
      idx.push_back(s.message_index);
      nb.push_back(static_cast<uint32_t>(s.snapshot.bids.size()));
      for (const auto& l : s.snapshot.bids) lv.push_back({l.price, l.quantity});
      for (const auto& l : s.snapshot.asks) lv.push_back({l.price, l.quantity});
      off.push_back(lv.size());
    }
    mlob_book_states st{idx.size(), idx.data(), off.data(), nb.data(), lv.data()};
    static_assert(sizeof(lob::Message) == sizeof(mlob_message), "lob::Message layout");
    mlob_throw(mlob_store_upload_raw(reinterpret_cast<const mlob_message*>(store.messages.data()),
                                     store.messages.size(), &st, device, &s_));
  }
  ~CudaMessageStore() { mlob_store_free(s_); }
  CudaMessageStore(const CudaMessageStore&) = delete;
  CudaMessageStore& operator=(const CudaMessageStore&) = delete;
  const mlob_store* get() const { return s_; }

 private:
  mlob_store* s_ = nullptr;
};

// Same member set as MarketVecEnv (rollout.hpp:151-336).  The episode pool
// holds indices into `index` (build_episode_index with the config's episode
// shape, as MarketVecEnv's callers pass it, train.hpp:160-168).
class CudaMarketVecEnv {
 public:
  CudaMarketVecEnv(const CudaMessageStore& store, const data::EpisodeIndex& index, const env::EnvConfig& cfg,
                   std::span<const std::size_t> episode_pool, std::uint64_t seed, int n_envs, int device = 0,
                   std::uint64_t n_envs_global = 0, std::uint64_t env_index_base = 0)
      : cfg_(cfg) {
    if (n_envs < 1) throw std::invalid_argument("MarketVecEnv: n_envs >= 1");
    if (episode_pool.empty()) throw std::invalid_argument("MarketVecEnv: empty episode pool");
    if (index.steps_per_episode != cfg.steps_per_episode || index.messages_per_step != cfg.messages_per_step ||
        index.start_stride_steps != cfg.start_stride_steps)
      throw std::invalid_argument("CudaMarketVecEnv: episode index built with another episode shape");
    std::vector<uint64_t> pool(episode_pool.begin(), episode_pool.end());
    mlob_venv_desc d{};
    d.store = store.get();
    d.cfg = to_mlob_config(cfg);
    d.episode_pool = pool.data();
    d.pool_len = pool.size();
    d.seed = seed;
    d.n_envs_local = static_cast<uint64_t>(n_envs);
    d.n_envs_global = n_envs_global ? n_envs_global : d.n_envs_local;
    d.env_index_base = env_index_base;
    d.flags = MLOB_VENV_AUTO_RESET;
    d.device = device;
    mlob_throw(mlob_venv_create(&d, &v_));
    n_envs_ = static_cast<std::size_t>(n_envs);
    agents_ = static_cast<std::size_t>(mlob_venv_n_agents(v_));
    actions_.assign(n_envs_ * agents_, 0);
    rewards_.assign(n_envs_ * agents_, 0.0);
    dones_.assign(n_envs_ * agents_, 0);
    std::size_t o = 0;
    for (const auto& s : cfg.specs) {
      offset_.push_back(o);
      o += static_cast<std::size_t>(s.count);
    }
  }
  ~CudaMarketVecEnv() { mlob_venv_destroy(v_); }
  CudaMarketVecEnv(const CudaMarketVecEnv&) = delete;
  CudaMarketVecEnv& operator=(const CudaMarketVecEnv&) = delete;

  int n_types() const { return mlob_venv_n_types(v_); }
  std::size_t n_envs() const { return n_envs_; }
  std::size_t n_streams(int t) const { return static_cast<std::size_t>(mlob_venv_n_streams(v_, t)); }
  std::size_t obs_dim(int t) const { return static_cast<std::size_t>(mlob_venv_obs_dim(v_, t)); }
  int n_actions(int t) const { return mlob_venv_n_actions(v_, t); }

  void reset_all() { mlob_throw(mlob_venv_reset_all(v_)); }
  void gather(int t, double* obs_out, std::uint8_t* reset_out) {
    mlob_throw(mlob_venv_gather(v_, t, obs_out, reset_out));
  }
  void set_action(int t, std::size_t stream, int action) { actions_[slot(t, stream)] = action; }
  // set_action'ed ids in, reward/done caches out (actions range-checked on
  // the device before any env steps, actions.hpp:69-70)
  void step_all() {
    mlob_step_io io{};
    io.actions = actions_.data();
    io.rewards = rewards_.data();
    io.dones = dones_.data();
    mlob_throw(mlob_venv_step_io(v_, &io));
  }
  double reward(int t, std::size_t stream) const { return rewards_[slot(t, stream)]; }
  bool done(int t, std::size_t stream) const { return dones_[slot(t, stream)] != 0; }

  MarketVecEnv::EpisodeStats episode_stats(int t) const {
    mlob_episode_stats e;
    mlob_throw(mlob_venv_episode_stats(v_, t, &e));
    return {e.pv_sum, e.slippage_sum, e.completion_sum, e.inventory_sq_sum, e.episodes};
  }
  // episode_stats summed over every rank of `nccl_comm` (an ncclComm_t; NULL:
  // this shard only), one ncclAllReduce for all types
  std::vector<MarketVecEnv::EpisodeStats> allreduce_episode_stats(void* nccl_comm) const {
    std::vector<mlob_episode_stats> e(static_cast<std::size_t>(n_types()));
    mlob_throw(mlob_venv_allreduce_episode_stats(v_, nccl_comm, e.data()));
    std::vector<MarketVecEnv::EpisodeStats> out;
    for (const auto& x : e) out.push_back({x.pv_sum, x.slippage_sum, x.completion_sum, x.inventory_sq_sum, x.episodes});
    return out;
  }
  void clear_episode_stats() { mlob_throw(mlob_venv_clear_episode_stats(v_)); }

  mlob_venv* handle() const { return v_; }

 private:
  std::size_t slot(int t, std::size_t stream) const {  // rollout.hpp:280-284 locate()
    const auto count = static_cast<std::size_t>(cfg_.specs[static_cast<std::size_t>(t)].count);
    return (stream / count) * agents_ + offset_[static_cast<std::size_t>(t)] + stream % count;
  }
  env::EnvConfig cfg_;
  mlob_venv* v_ = nullptr;
  std::size_t n_envs_ = 0, agents_ = 0;
  std::vector<int32_t> actions_;
  std::vector<double> rewards_;
  std::vector<uint8_t> dones_;
  std::vector<std::size_t> offset_;
};

}  // namespace marlob::ippo
