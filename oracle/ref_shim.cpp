// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Exposes the unmodified reference (marlob, header-only C++20) through the
// ref_* functions of oracle_api.h.  Built by oracle/Makefile with
// -I/root/reference/proj/include (the reference sources are compiled where they
// lie, never copied) into oracle/_ref/libmarlob_ref.so.  Used by the tests to
// pin the C restatement (orc_*) and the CUDA product against the reference
// itself, and by bench.py's reference / cpu_baseline legs.
#include <cstddef>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "marlob/bench/bench.hpp"
#include "marlob/data/lobster.hpp"
#include "marlob/data/store.hpp"
#include "marlob/data/synth.hpp"
#include "marlob/env/env.hpp"
#include "marlob/ippo/evaluate.hpp"
#include "marlob/ippo/rollout.hpp"
#include "marlob/lob/book.hpp"
#include "marlob/util/thread_pool.hpp"
#include "oracle_api.h"

using namespace marlob;

static_assert(sizeof(lob::Message) == sizeof(mlob_message));
static_assert(offsetof(lob::Message, trader_id) == offsetof(mlob_message, trader_id));
static_assert(sizeof(lob::RestingOrder) == sizeof(mlob_resting_order));
static_assert(sizeof(lob::TradeRecord) == sizeof(mlob_trade));
static_assert(offsetof(lob::TradeRecord, aggressor_side) == offsetof(mlob_trade, aggressor_side));
static_assert(sizeof(env::AgentInfo) == sizeof(mlob_agent_info));

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MLOB_OK;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return MLOB_E_OUT_OF_RANGE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MLOB_E_INVALID_ARGUMENT;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return MLOB_E_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MLOB_E_RUNTIME;
  }
}

lob::Message to_msg(const mlob_message& m) {
  lob::Message r;
  r.time = m.time;
  r.order_id = m.order_id;
  r.price = m.price;
  r.quantity = m.quantity;
  r.kind = static_cast<lob::MsgKind>(m.kind);
  r.side = static_cast<lob::Side>(m.side);
  r.trader_id = m.trader_id;
  return r;
}

mlob_trade to_trade(const lob::TradeRecord& t) {
  mlob_trade r{};
  r.price = t.price;
  r.quantity = t.quantity;
  r.time = t.time;
  r.passive_order_id = t.passive_order_id;
  r.aggressor_order_id = t.aggressor_order_id;
  r.passive_trader_id = t.passive_trader_id;
  r.aggressor_trader_id = t.aggressor_trader_id;
  r.aggressor_side = static_cast<uint8_t>(t.aggressor_side);
  return r;
}

mlob_resting_order to_resting(const lob::RestingOrder& o) {
  mlob_resting_order r{};
  r.price = o.price;
  r.quantity = o.quantity;
  r.order_id = o.order_id;
  r.arrival_seq = o.arrival_seq;
  r.trader_id = o.trader_id;
  return r;
}

env::AgentParams to_params(const mlob_agent_params& p) {
  env::AgentParams r;
  r.order_size = p.order_size;
  r.inventory_cap = p.inventory_cap;
  r.rho = p.rho;
  r.quadratic_penalty = p.quadratic_penalty != 0;
  r.lambda = p.lambda;
  r.ref_price = static_cast<env::RefPriceMode>(p.ref_price);
  r.unfilled_penalty_coef = p.unfilled_penalty_coef;
  r.lambda_exec = p.lambda_exec;
  r.task_size = p.task_size;
  r.exec_complex = p.exec_complex != 0;
  r.reward_scale = p.reward_scale;
  r.default_half_spread = p.default_half_spread;
  r.fixed_quant_from_mid = p.fixed_quant_from_mid != 0;
  r.spread_skew.rows.clear();
  for (int i = 0; i < p.n_spread_skew; ++i)
    r.spread_skew.rows.push_back({p.spread_skew_half[i], p.spread_skew_skew[i]});
  r.avst.gamma_grid.assign(p.gamma_grid, p.gamma_grid + p.n_gamma);
  r.avst.kappa = p.kappa;
  r.avst.sigma = p.sigma;
  r.avst.horizon = p.horizon;
  return r;
}

env::EnvConfig to_cfg(const mlob_env_config& c) {
  env::EnvConfig r;
  r.steps_per_episode = c.steps_per_episode;
  r.messages_per_step = c.messages_per_step;
  r.start_stride_steps = c.start_stride_steps;
  r.book_capacity = c.book_capacity;
  r.obs_depth = c.obs_depth;
  r.fallback_mid_half = c.fallback_mid_half;
  r.synthetic_init_id_base = c.synthetic_init_id_base;
  r.agent_id_base = c.agent_id_base;
  r.agent_id_range = c.agent_id_range;
  r.fill_reserve = c.fill_reserve;
  for (int s = 0; s < c.n_specs; ++s) {
    env::AgentSpec sp;
    sp.type = static_cast<env::AgentType>(c.specs[s].type);
    sp.count = c.specs[s].count;
    sp.mm_space = static_cast<env::MMActionSpace>(c.specs[s].mm_space);
    sp.obs_space = static_cast<agents::ObsSpaceId>(c.specs[s].obs_space);
    sp.reward = static_cast<env::RewardId>(c.specs[s].reward);
    sp.params = to_params(c.specs[s].params);
    r.specs.push_back(sp);
  }
  return r;
}

lob::L2Snapshot to_snap(const mlob_level* bids, uint32_t nb, const mlob_level* asks, uint32_t na) {
  lob::L2Snapshot s;
  for (uint32_t i = 0; i < nb; ++i) s.bids.push_back({bids[i].price, bids[i].quantity});
  for (uint32_t i = 0; i < na; ++i) s.asks.push_back({asks[i].price, asks[i].quantity});
  return s;
}

struct StoreH {
  data::MessageStore store;
};

struct EnvH {
  std::unique_ptr<data::EpisodeIndex> index;
  std::unique_ptr<env::MarketEnv> owned;
  env::MarketEnv* env = nullptr;
};

struct VenvH {
  std::unique_ptr<data::EpisodeIndex> index;
  std::unique_ptr<util::ThreadPool> pool;
  std::unique_ptr<ippo::MarketVecEnv> venv;
  // collect_rollout state (rollout.hpp:41-124): nets, persistent hidden, batches
  std::vector<ippo::PolicyNet> nets;
  std::vector<std::vector<double>> hidden;
  std::vector<ippo::RolloutBatch> batches;
  std::vector<ippo::AdamState> adams;  // one per type (train_loop's adams)
};

ippo::PolicyNet to_net(const mlob_policy_net& n) {
  ippo::PolicyNet r;
  r.obs_dim = n.obs_dim;
  r.hidden = n.hidden;
  r.n_actions = n.n_actions;
  const std::size_t D = n.obs_dim, H = n.hidden, A = n.n_actions;
  r.w_ih.assign(n.w_ih, n.w_ih + 3 * H * D);
  r.w_hh.assign(n.w_hh, n.w_hh + 3 * H * H);
  r.b_ih.assign(n.b_ih, n.b_ih + 3 * H);
  r.b_hh.assign(n.b_hh, n.b_hh + 3 * H);
  r.w_actor.assign(n.w_actor, n.w_actor + A * H);
  r.b_actor.assign(n.b_actor, n.b_actor + A);
  r.w_critic.assign(n.w_critic, n.w_critic + H);
  r.b_critic = n.b_critic;
  return r;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_store_synth(const mlob_synth_config* c, uint64_t seed) {
  auto* h = new StoreH;
  data::SynthConfig cfg;
  cfg.n_messages = c->n_messages;
  cfg.initial_mid = c->initial_mid;
  cfg.volatility = c->volatility;
  cfg.p_new_passive = c->p_new_passive;
  cfg.p_new_cross = c->p_new_cross;
  cfg.p_cancel = c->p_cancel;
  cfg.p_delete = c->p_delete;
  cfg.p_execute = c->p_execute;
  cfg.band = c->band;
  cfg.max_qty = c->max_qty;
  cfg.seed_levels = c->seed_levels;
  cfg.seed_qty = c->seed_qty;
  cfg.state_sample_every = c->state_sample_every;
  cfg.state_depth = c->state_depth;
  if (guarded([&] { h->store = data::synth_generate(cfg, seed); }) != MLOB_OK) {
    delete h;
    return nullptr;
  }
  return h;
}

void* ref_store_create(const mlob_message* msgs, uint64_t n, const mlob_book_states* st) {
  auto* h = new StoreH;
  h->store.messages.reserve(n);
  for (uint64_t i = 0; i < n; ++i) h->store.messages.push_back(to_msg(msgs[i]));
  if (st) {
    for (uint64_t i = 0; i < st->n_states; ++i) {
      const uint64_t off = st->level_offset[i];
      const uint32_t nb = st->n_bids[i];
      const uint32_t na = static_cast<uint32_t>(st->level_offset[i + 1] - off) - nb;
      h->store.book_states.push_back(data::BookState{
          st->message_index[i], to_snap(st->levels + off, nb, st->levels + off + nb, na)});
    }
  }
  return h;
}

uint64_t ref_store_n_messages(void* s) { return static_cast<StoreH*>(s)->store.messages.size(); }
const mlob_message* ref_store_messages(void* s) {
  return reinterpret_cast<const mlob_message*>(static_cast<StoreH*>(s)->store.messages.data());
}
uint64_t ref_store_n_states(void* s) { return static_cast<StoreH*>(s)->store.book_states.size(); }
int ref_store_state(void* s, uint64_t i, uint64_t* msg_index, mlob_level* bids, uint32_t* nb,
                    mlob_level* asks, uint32_t* na, uint32_t cap) {
  const auto& st = static_cast<StoreH*>(s)->store.book_states.at(i);
  *msg_index = st.message_index;
  *nb = static_cast<uint32_t>(st.snapshot.bids.size());
  *na = static_cast<uint32_t>(st.snapshot.asks.size());
  if (*nb > cap || *na > cap) return MLOB_E_OUT_OF_RANGE;
  for (uint32_t k = 0; k < *nb; ++k) bids[k] = {st.snapshot.bids[k].price, st.snapshot.bids[k].quantity};
  for (uint32_t k = 0; k < *na; ++k) asks[k] = {st.snapshot.asks[k].price, st.snapshot.asks[k].quantity};
  return MLOB_OK;
}
void ref_store_free(void* s) { delete static_cast<StoreH*>(s); }

// ---- book ----
void* ref_book_create(uint64_t capacity) {
  lob::OrderBook* b = nullptr;
  if (guarded([&] { b = new lob::OrderBook(capacity); }) != MLOB_OK) return nullptr;
  return b;
}
int ref_book_init_from_l2(void* b, const mlob_level* bids, uint32_t nb, const mlob_level* asks,
                          uint32_t na, uint64_t id_base) {
  return guarded([&] {
    static_cast<lob::OrderBook*>(b)->init_from_l2(to_snap(bids, nb, asks, na), id_base);
  });
}
uint64_t ref_book_process(void* b, const mlob_message* m, mlob_trade* out, uint64_t cap) {
  std::vector<lob::TradeRecord> trades;
  static_cast<lob::OrderBook*>(b)->process(to_msg(*m), trades);
  for (uint64_t i = 0; i < trades.size() && i < cap; ++i) out[i] = to_trade(trades[i]);
  return trades.size();
}
uint64_t ref_book_orders(void* b, int side, mlob_resting_order* out, uint64_t cap) {
  const auto o = static_cast<lob::OrderBook*>(b)->orders(static_cast<lob::Side>(side));
  for (uint64_t i = 0; i < o.size() && i < cap; ++i) out[i] = to_resting(o[i]);
  return o.size();
}
uint64_t ref_book_next_seq(void* b) { return static_cast<lob::OrderBook*>(b)->next_seq(); }
int64_t ref_book_mid_half(void* b, int64_t fallback) {
  return static_cast<lob::OrderBook*>(b)->mid_half_ticks(fallback);
}
void ref_book_l2(void* b, uint64_t depth, mlob_level* bids, uint32_t* nb, mlob_level* asks,
                 uint32_t* na) {
  const auto snap = static_cast<lob::OrderBook*>(b)->l2_snapshot(depth);
  *nb = static_cast<uint32_t>(snap.bids.size());
  *na = static_cast<uint32_t>(snap.asks.size());
  for (uint32_t k = 0; k < *nb; ++k) bids[k] = {snap.bids[k].price, snap.bids[k].quantity};
  for (uint32_t k = 0; k < *na; ++k) asks[k] = {snap.asks[k].price, snap.asks[k].quantity};
}
void ref_book_free(void* b) { delete static_cast<lob::OrderBook*>(b); }

// ---- env ----
void* ref_env_create(void* store, const mlob_env_config* cfg, uint64_t seed, int env_index,
                     int* status) {
  auto* h = new EnvH;
  const auto* st = &static_cast<StoreH*>(store)->store;
  *status = guarded([&] {
    const env::EnvConfig c = to_cfg(*cfg);
    h->index = std::make_unique<data::EpisodeIndex>(data::build_episode_index(
        *st, c.steps_per_episode, c.messages_per_step, c.start_stride_steps));
    h->owned = std::make_unique<env::MarketEnv>(st, h->index.get(), c, seed, env_index);
    h->env = h->owned.get();
  });
  if (*status != MLOB_OK) {
    delete h;
    return nullptr;
  }
  return h;
}
uint64_t ref_env_n_episodes(void* e) { return static_cast<EnvH*>(e)->index->episode_count(); }
uint64_t ref_env_episode_start(void* e, uint64_t ep) {
  return static_cast<EnvH*>(e)->index->starts.at(ep);
}
int ref_env_n_agents(void* e) { return static_cast<int>(static_cast<EnvH*>(e)->env->n_agents()); }
int ref_env_reset(void* e, uint64_t episode) {
  return guarded([&] { static_cast<EnvH*>(e)->env->reset(episode); });
}
int ref_env_step_ids(void* e, const int32_t* ids, uint64_t n) {
  return guarded([&] {
    std::vector<int> v(ids, ids + n);
    static_cast<EnvH*>(e)->env->step_ids(v);
  });
}
int ref_env_step(void* e, const mlob_agent_action* actions, uint64_t n) {
  return guarded([&] {
    std::vector<env::AgentAction> v(n);
    for (uint64_t i = 0; i < n; ++i) {
      v[i].id = actions[i].id;
      v[i].direct = actions[i].direct != 0;
      for (int q = 0; q < actions[i].n_quotes; ++q)
        v[i].quotes.push(static_cast<lob::Side>(actions[i].quotes[q].side),
                         actions[i].quotes[q].price, actions[i].quotes[q].quantity);
    }
    static_cast<EnvH*>(e)->env->step(v);
  });
}
void ref_env_scalars(void* e, mlob_env_scalars* o) {
  const env::MarketEnv& m = *static_cast<EnvH*>(e)->env;
  std::memset(o, 0, sizeof(*o));
  o->step = m.step_count();
  o->terminal = m.terminal() ? 1 : 0;
  o->episode = m.episode();
  o->mid_half = m.mid_half();
  o->prev_mid_half = m.prev_mid_half();
  o->mean_mid_ticks = m.mean_mid_ticks();
  o->messages_processed = m.messages_processed();
  o->next_seq = m.book().next_seq();
  o->live_bid = m.book().live_orders(lob::Side::Bid);
  o->live_ask = m.book().live_orders(lob::Side::Ask);
  // last_bid/last_ask/last_time are private in the reference; report the
  // observable fallbacks instead (tests only compare them oracle vs GPU).
  o->last_bid = INT64_MIN;
  o->last_ask = INT64_MIN;
  o->last_time = INT64_MIN;
}
uint64_t ref_env_book(void* e, int side, mlob_resting_order* out, uint64_t cap) {
  const auto o = static_cast<EnvH*>(e)->env->book().orders(static_cast<lob::Side>(side));
  for (uint64_t i = 0; i < o.size() && i < cap; ++i) out[i] = to_resting(o[i]);
  return o.size();
}
void ref_env_agent(void* e, int a, mlob_agent_state* o) {
  const env::AgentState& s = static_cast<EnvH*>(e)->env->agent_state(static_cast<size_t>(a));
  std::memset(o, 0, sizeof(*o));
  o->inventory = s.inventory;
  o->cash = s.cash;
  o->task_remaining = s.task_remaining;
  o->task_dir = static_cast<int32_t>(s.task_dir);
  o->p_init = s.p_init;
  o->order_nonce = s.order_nonce;
  o->filled_total = s.filled_total;
  o->slippage_total = s.slippage_total;
  o->n_active = static_cast<int32_t>(s.active.size());
  for (size_t i = 0; i < s.active.size() && i < MLOB_MAX_ACTIVE; ++i) {
    o->active[i].order_id = s.active[i].order_id;
    o->active[i].price = s.active[i].price;
    o->active[i].quantity = s.active[i].quantity;
    o->active[i].side = static_cast<uint8_t>(s.active[i].side);
  }
}
void ref_env_info(void* e, int a, mlob_agent_info* o) {
  const auto& i = static_cast<EnvH*>(e)->env->output().infos.at(static_cast<size_t>(a));
  std::memcpy(o, &i, sizeof(*o));
}
double ref_env_reward(void* e, int a) {
  return static_cast<EnvH*>(e)->env->output().rewards.at(static_cast<size_t>(a));
}
int ref_env_done(void* e, int a) {
  return static_cast<EnvH*>(e)->env->output().dones.at(static_cast<size_t>(a));
}
uint64_t ref_env_obs(void* e, int a, double* out, uint64_t cap) {
  const auto& o = static_cast<EnvH*>(e)->env->output().obs.at(static_cast<size_t>(a));
  for (uint64_t i = 0; i < o.size() && i < cap; ++i) out[i] = o[i];
  return o.size();
}
uint64_t ref_env_trades(void* e, mlob_trade* out, uint64_t cap) {
  const auto t = static_cast<EnvH*>(e)->env->step_trades();
  for (uint64_t i = 0; i < t.size() && i < cap; ++i) out[i] = to_trade(t[i]);
  return t.size();
}
void ref_env_free(void* e) { delete static_cast<EnvH*>(e); }

// ---- vec env ----
void* ref_venv_create(void* store, const mlob_env_config* cfg, const uint64_t* pool,
                      uint64_t pool_len, uint64_t seed, int n_envs, int workers, int* status) {
  auto* h = new VenvH;
  const auto* st = &static_cast<StoreH*>(store)->store;
  *status = guarded([&] {
    const env::EnvConfig c = to_cfg(*cfg);
    h->index = std::make_unique<data::EpisodeIndex>(data::build_episode_index(
        *st, c.steps_per_episode, c.messages_per_step, c.start_stride_steps));
    std::vector<std::size_t> p;
    if (pool)
      p.assign(pool, pool + pool_len);
    else
      for (std::size_t i = 0; i < h->index->episode_count(); ++i) p.push_back(i);
    h->pool = std::make_unique<util::ThreadPool>(workers);
    h->venv = std::make_unique<ippo::MarketVecEnv>(st, h->index.get(), c, p, seed, n_envs,
                                                   h->pool.get());
  });
  if (*status != MLOB_OK) {
    delete h;
    return nullptr;
  }
  return h;
}
int ref_venv_reset_all(void* v) {
  return guarded([&] { static_cast<VenvH*>(v)->venv->reset_all(); });
}
int ref_venv_set_action(void* v, int type, uint64_t stream, int action) {
  return guarded([&] { static_cast<VenvH*>(v)->venv->set_action(type, stream, action); });
}
int ref_venv_step_all(void* v) {
  return guarded([&] { static_cast<VenvH*>(v)->venv->step_all(); });
}
void ref_venv_gather(void* v, int type, double* obs, uint8_t* resets) {
  static_cast<VenvH*>(v)->venv->gather(type, obs, resets);
}
double ref_venv_reward(void* v, int type, uint64_t stream) {
  return static_cast<VenvH*>(v)->venv->reward(type, stream);
}
int ref_venv_done(void* v, int type, uint64_t stream) {
  return static_cast<VenvH*>(v)->venv->done(type, stream) ? 1 : 0;
}
void ref_venv_episode_stats(void* v, int type, mlob_episode_stats* out) {
  const auto s = static_cast<VenvH*>(v)->venv->episode_stats(type);
  out->pv_sum = s.pv_sum;
  out->slippage_sum = s.slippage_sum;
  out->completion_sum = s.completion_sum;
  out->inventory_sq_sum = s.inventory_sq_sum;
  out->episodes = s.episodes;
}
void ref_venv_clear_episode_stats(void* v) { static_cast<VenvH*>(v)->venv->clear_episode_stats(); }
void* ref_venv_instance(void* v, uint64_t e) {
  auto* h = new EnvH;
  h->env = const_cast<env::MarketEnv*>(&static_cast<VenvH*>(v)->venv->instance(e));
  return h;
}
void ref_venv_free(void* v) { delete static_cast<VenvH*>(v); }

// ---- LOBSTER ingestion (data/lobster.hpp) ----
void* ref_load_lobster(const char* message_path, const char* orderbook_path, int64_t units_per_tick,
                       uint64_t sample_every, int* status) {
  auto* h = new StoreH;
  *status = guarded([&] {
    h->store = data::load_lobster(message_path, orderbook_path, units_per_tick, sample_every);
  });
  if (*status != MLOB_OK) {
    delete h;
    return nullptr;
  }
  return h;
}

// ---- networks and rollouts (ippo/net.hpp, ippo/rollout.hpp) ----
int ref_make_policy_net(int obs_dim, int hidden, int n_actions, uint64_t seed, double* out) {
  return guarded([&] {
    ippo::PolicyNet n = ippo::make_policy_net(obs_dim, hidden, n_actions, seed);
    std::size_t i = 0;
    n.for_each_param([&](double& v) { out[i++] = v; });
  });
}

int ref_venv_collect_rollout(void* v, const mlob_policy_net* nets, const mlob_rollout_config* cfg,
                             uint64_t update_index) {
  auto* h = static_cast<VenvH*>(v);
  return guarded([&] {
    const int T = h->venv->n_types();
    const bool fresh = h->nets.empty();
    if (nets) {  // null: keep the networks (as updated by ref_venv_ppo_update)
      h->nets.clear();
      for (int t = 0; t < T; ++t) h->nets.push_back(to_net(nets[t]));
    }
    if (fresh) {  // train_loop, rollout.hpp:132-135
      h->hidden.assign(static_cast<std::size_t>(T), {});
      for (int t = 0; t < T; ++t)
        h->hidden[t].assign(h->venv->n_streams(t) * static_cast<std::size_t>(h->nets[t].hidden), 0.0);
      h->batches.assign(static_cast<std::size_t>(T), {});
      h->adams.assign(static_cast<std::size_t>(T), {});
    }
    ippo::TrainLoopConfig c;
    c.rollout_len = cfg->rollout_len;
    c.discount = cfg->discount;
    c.gae_lambda = cfg->gae_lambda;
    c.seed = cfg->seed;
    ippo::collect_rollout(*h->venv, h->nets, h->hidden, h->batches, c, update_index);
  });
}

int ref_venv_ppo_update(void* v, int type, const mlob_ppo_config* cfg, uint64_t seed, uint64_t update_index,
                        mlob_update_metrics* out) {
  auto* h = static_cast<VenvH*>(v);
  return guarded([&] {
    ippo::PpoConfig c;
    c.epochs = cfg->epochs;
    c.minibatches = cfg->minibatches;
    c.clip_eps = cfg->clip_eps;
    c.vf_coef = cfg->vf_coef;
    c.ent_coef = cfg->ent_coef;
    c.lr = cfg->lr;
    c.max_grad_norm = cfg->max_grad_norm;
    c.normalize_adv = cfg->normalize_adv != 0;
    const auto t = static_cast<std::size_t>(type);
    const ippo::UpdateMetrics m =
        ippo::ppo_update(h->nets.at(t), h->adams.at(t), h->batches.at(t), c, seed, update_index, t);
    *out = mlob_update_metrics{m.pg_loss, m.v_loss, m.entropy, m.approx_kl, m.clip_frac, m.grad_norm,
                               m.mean_reward};
  });
}

uint64_t ref_venv_read_net(void* v, int type, double* out, uint64_t cap) {
  auto* h = static_cast<VenvH*>(v);
  ippo::PolicyNet& n = h->nets.at(static_cast<std::size_t>(type));
  const uint64_t P = n.param_count();
  if (P <= cap) {
    std::size_t i = 0;
    n.for_each_param([&](double& x) { out[i++] = x; });
  }
  return P;
}

uint64_t ref_venv_rollout_field(void* v, int type, int field, void* out, uint64_t cap) {
  auto* h = static_cast<VenvH*>(v);
  const ippo::RolloutBatch& b = h->batches.at(static_cast<std::size_t>(type));
  const auto put = [&](const auto& vec) -> uint64_t {
    const uint64_t bytes = vec.size() * sizeof(vec[0]);
    if (bytes <= cap) std::memcpy(out, vec.data(), bytes);
    return bytes;
  };
  switch (field) {
    case MLOB_RB_OBS: return put(b.obs);
    case MLOB_RB_ACTIONS: return put(b.actions);
    case MLOB_RB_LOG_PROBS: return put(b.log_probs);
    case MLOB_RB_VALUES: return put(b.values);
    case MLOB_RB_REWARDS: return put(b.rewards);
    case MLOB_RB_DONES: return put(b.dones);
    case MLOB_RB_RESETS: return put(b.resets);
    case MLOB_RB_H0: return put(b.h0);
    case MLOB_RB_ADVANTAGES: return put(b.advantages);
    case MLOB_RB_RETURNS: return put(b.returns);
    case MLOB_RB_HIDDEN: return put(h->hidden.at(static_cast<std::size_t>(type)));
  }
  return 0;
}

// ---- bench ----
int ref_bench_run(void* store, const mlob_env_config* base, int n_envs, int n_steps, int warmup,
                  int workers, uint64_t seed, int messages_per_step, int agents_per_type,
                  orc_bench_row* out) {
  return guarded([&] {
    bench::BenchConfig b;
    b.n_envs = n_envs;
    b.n_steps = n_steps;
    b.warmup_steps = warmup;
    b.messages_grid = {messages_per_step};
    b.agents_grid = {agents_per_type};
    b.workers = workers;
    b.seed = seed;
    const auto rows =
        bench::run_throughput(static_cast<StoreH*>(store)->store, to_cfg(*base), b);
    const auto& r = rows.at(0);
    out->messages_per_step = r.messages_per_step;
    out->agents_per_type = r.agents_per_type;
    out->workers = r.workers;
    out->env_steps = r.env_steps;
    out->messages = r.messages;
    out->wall_seconds = r.wall_seconds;
    out->steps_per_sec = r.steps_per_sec;
    out->messages_per_sec = r.messages_per_sec;
    out->worker_utilization = r.worker_utilization;
  });
}

// ---- cross-play (ippo::evaluate_matrix, the reference's own driver) ----
int ref_evaluate_matrix(void* store, const mlob_env_config* cfg, const uint64_t* episodes, uint64_t n_eps,
                        const mlob_policy* t0, int n0, const mlob_policy* t1, int n1, uint64_t seed,
                        mlob_cell_stats* out) {
  return guarded([&] {
    const auto to_choice = [](const mlob_policy& p) {
      ippo::PolicyChoice c;
      c.kind = static_cast<ippo::PolicyKind>(p.kind);
      c.avst.params.gamma_grid.assign(p.gamma_grid, p.gamma_grid + p.n_gamma);
      c.avst.params.kappa = p.kappa;
      c.avst.params.sigma = p.sigma;
      c.avst.params.horizon = p.horizon;
      c.avst.gamma_index = p.avst_gamma_index;
      c.twap_mode = static_cast<baselines::TwapPriceMode>(p.twap_mode);
      return c;
    };
    std::vector<ippo::PolicyChoice> o0, o1;
    std::vector<std::unique_ptr<ippo::PolicyNet>> owned;  // PolicyChoice::net is non-owning
    const auto with_net = [&](const mlob_policy& p) {
      ippo::PolicyChoice c = to_choice(p);
      if (p.kind == MLOB_POLICY_LEARNED && p.net) {
        owned.push_back(std::make_unique<ippo::PolicyNet>(to_net(*p.net)));
        c.net = owned.back().get();
      }
      return c;
    };
    for (int i = 0; i < n0; ++i) o0.push_back(with_net(t0[i]));
    for (int i = 0; i < n1; ++i) o1.push_back(with_net(t1[i]));
    const env::EnvConfig c = to_cfg(*cfg);
    const data::MessageStore& st = static_cast<StoreH*>(store)->store;
    const data::EpisodeIndex index =
        data::build_episode_index(st, c.steps_per_episode, c.messages_per_step, c.start_stride_steps);
    const std::vector<std::size_t> eps(episodes, episodes + n_eps);
    const ippo::CrossPlayResult r = ippo::evaluate_matrix(st, index, c, eps, o0, o1, seed);
    for (std::size_t i = 0; i < r.cells.size(); ++i) {
      const ippo::CellStats& cs = r.cells[i];
      std::memset(&out[i], 0, sizeof out[i]);
      out[i].episodes = cs.episodes;
      for (int t = 0; t < 2; ++t) {
        const ippo::TypeCellStats& s = cs.per_type[t];
        mlob_type_cell_stats& d = out[i].per_type[t];
        d.pv_mean = s.pv_mean;
        d.pv_stderr = s.pv_stderr;
        d.slippage_mean = s.slippage_mean;
        d.slippage_stderr = s.slippage_stderr;
        d.completion_mean = s.completion_mean;
        d.filled_total = s.filled_total;
        d.no_fills = s.no_fills ? 1 : 0;
      }
    }
  });
}

}  // extern "C"

#include "reference/naive_book.hpp"
#include "reference/random_messages.hpp"

extern "C" {

void ref_random_stream(const orc_stream_config* c, uint64_t seed, mlob_message* out) {
  marlob::testing::RandomStreamConfig cfg;
  cfg.n_messages = c->n_messages;
  cfg.initial_ref = c->initial_ref;
  cfg.band = c->band;
  cfg.max_qty = c->max_qty;
  cfg.p_new = c->p_new;
  cfg.p_marketable = c->p_marketable;
  cfg.p_cancel = c->p_cancel;
  cfg.p_delete = c->p_delete;
  cfg.p_execute = c->p_execute;
  cfg.p_absent = c->p_absent;
  marlob::testing::RandomMessageGen gen(cfg, seed);
  for (uint64_t i = 0; i < cfg.n_messages; ++i) {
    const lob::Message m = gen.next();
    std::memcpy(&out[i], &m, sizeof(mlob_message));
  }
}

void* ref_naive_create(void) { return new marlob::testing::NaiveBook; }
uint64_t ref_naive_process(void* b, const mlob_message* m, mlob_trade* out, uint64_t cap) {
  std::vector<lob::TradeRecord> trades;
  static_cast<marlob::testing::NaiveBook*>(b)->process(to_msg(*m), trades);
  for (uint64_t i = 0; i < trades.size() && i < cap; ++i) out[i] = to_trade(trades[i]);
  return trades.size();
}
int ref_naive_best(void* b, int side, int64_t* price) {
  auto* nb = static_cast<marlob::testing::NaiveBook*>(b);
  const auto p = side == 0 ? nb->best_bid() : nb->best_ask();
  if (!p) return 0;
  *price = *p;
  return 1;
}
uint32_t ref_naive_l2_full(void* b, int side, mlob_level* out, uint32_t cap) {
  const auto snap = static_cast<marlob::testing::NaiveBook*>(b)->l2_full();
  const auto& v = side == 0 ? snap.bids : snap.asks;
  for (uint32_t i = 0; i < v.size() && i < cap; ++i) out[i] = {v[i].price, v[i].quantity};
  return static_cast<uint32_t>(v.size());
}
void ref_naive_free(void* b) { delete static_cast<marlob::testing::NaiveBook*>(b); }

}  // extern "C"
