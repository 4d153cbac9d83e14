// mlob_runtime.cu — host runtime behind include/mlob.h: device stores, batched
// environment handles, launches, parity readers and the error model.
// There is no CPU execution path for the environment step: every step/reset
// is a kernel launch; without a CUDA device every call fails with MLOB_E_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <dlfcn.h>
#include <memory>
#include <string>
#include <vector>

#include "mlob_dev.h"
#include "mlob_host.h"
#include "mlob_lobster.h"
#include "mlob_policy.h"
#include "mlob_ppo.h"

#include <sstream>

namespace mlob {
size_t step_min_smem_bytes(const DevCfg& c);
uint32_t step_amsg_cap(const DevCfg& c);
int step_launches();
int slots_per_lane(int capacity);
cudaError_t launch_step(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s, cudaEvent_t* ev = nullptr);
cudaError_t launch_reset(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s);
cudaError_t launch_stats(const KParams& kp, const DevCfg& cfg, double* out, cudaStream_t s);
cudaError_t launch_sum_msgs(const EnvHdr* hdr, uint64_t n, unsigned long long* out, cudaStream_t s);
cudaError_t launch_validate_actions(const int32_t* ids, uint64_t n, const DevCfg* cfg, uint32_t* error,
                                    uint32_t* gate, cudaStream_t s);
cudaError_t launch_expand_resets(const uint8_t* just_reset, uint64_t n_envs, int count, uint8_t* out,
                                 cudaStream_t s);
cudaError_t launch_clear_finished(EnvHdr* hdr, uint64_t n, cudaStream_t s);
}  // namespace mlob

using namespace mlob;

namespace {

thread_local std::string g_err;

template <class F>
mlob_status guarded(F&& f) {
  try {
    f();
    return MLOB_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return MLOB_E_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MLOB_E_RUNTIME;
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(MLOB_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dalloc(size_t n, const char* what) {
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), what);
  cuda_check(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)), what);
  return static_cast<T*>(p);
}

uint64_t host_splitmix(uint64_t z) {  // rng.hpp:11-16
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
uint64_t host_fold(uint64_t h, uint64_t w) {  // rng.hpp:18-20
  return host_splitmix(h ^ (w + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2)));
}

int64_t fits32(int64_t v, const char* what) {
  if (v <= INT32_MIN || v >= INT32_MAX)
    fail(MLOB_E_INVALID_ARGUMENT, std::string(what) + " outside the device int32 range");
  return v;
}

}  // namespace

struct mlob_store {
  int device = 0;
  uint64_t n_msgs = 0;
  DevMsg* d_msgs = nullptr;
  DevLevel* d_levels = nullptr;
  std::vector<uint64_t> st_index, st_offset;
  std::vector<uint32_t> st_nb;
  uint64_t bytes = 0;
  ~mlob_store() {
    cudaSetDevice(device);
    if (d_msgs) cudaFree(d_msgs);
    if (d_levels) cudaFree(d_levels);
  }
  int64_t state_before(uint64_t idx) const {
    const auto it = std::lower_bound(st_index.begin(), st_index.end(), idx);
    if (it == st_index.end() || *it != idx) return -1;
    return it - st_index.begin();
  }
};

constexpr uint64_t kMaxIoChunks = 16;  // step_io env chunks (each owns a share of the fill pool)

struct mlob_venv {
  const mlob_store* store = nullptr;
  mlob_env_config cfg{};
  DevCfg dcfg{};
  int spl = 0, A = 0, device = 0;
  uint64_t n_envs = 0, n_envs_global = 0, env_index_base = 0, seed = 0;
  uint32_t flags = 0, trade_cap = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // step_io pipeline: second compute stream, copy stream, per-chunk events
  cudaStream_t stream2 = nullptr, copy_stream = nullptr;
  std::vector<cudaEvent_t> io_events;
  uint32_t* d_gate = nullptr;
  uint8_t* d_resets[MLOB_MAX_SPECS] = {};
  // scripted policies (kActScripted)
  DevPolicy* d_policies = nullptr;
  uint8_t* d_env_policy = nullptr;
  uint64_t* d_env_cell = nullptr;
  bool has_cells = false;
  // on-device rollouts (mlob_policy.cu): one network + hidden state per type,
  // one RolloutBatch arena per type
  struct NetState {
    DevNet dn{};
    double* w = nullptr;  // all weights, transposed layout (mlob_policy.h)
    double* hidden[2] = {};
    int cur = 0;
    // reference layout + gradient + Adam moments (ppo_update), P doubles each
    double *p = nullptr, *g = nullptr, *m = nullptr, *v = nullptr;
    uint64_t P = 0;
    int64_t adam_t = 0;
  };
  static void free_net(NetState& n) {
    cudaFree(n.w);
    cudaFree(n.hidden[0]);
    cudaFree(n.hidden[1]);
    cudaFree(n.p);
    cudaFree(n.g);
    cudaFree(n.m);
    cudaFree(n.v);
    n = NetState{};
  }
  // ppo_update workspace (mlob_ppo.cu), grown on demand
  char* ppo_ws = nullptr;
  uint64_t ppo_ws_bytes = 0;
  struct Batch {
    uint64_t T = 0, B = 0;
    char* arena = nullptr;
    double *obs = nullptr, *log_probs = nullptr, *values = nullptr, *rewards = nullptr, *h0 = nullptr,
           *adv = nullptr, *ret = nullptr;
    int32_t* actions = nullptr;
    uint8_t *dones = nullptr, *resets = nullptr;
  };
  NetState nets[MLOB_MAX_SPECS];
  Batch batch[MLOB_MAX_SPECS];
  bool has_nets = false;
  // collect_rollout as a CUDA graph: captured once per (T, hidden-buffer
  // parities, buffer version), replayed with {seed, update} in device memory
  cudaGraphExec_t roll_graph = nullptr;
  uint64_t roll_key = ~0ull;
  uint64_t buf_version = 0;  // bumped whenever a net / batch buffer is reallocated
  uint64_t* d_seed_update = nullptr;
  std::vector<NetState> eval_nets;  // evaluate_matrix: one per Learned option
  std::vector<uint64_t> starts;
  std::vector<EpState> ep_state;
  std::vector<uint64_t> pool;  // empty = identity
  std::vector<uint64_t> genv;  // global env index per local env
  // host mirror of the per-env step: resets reset every env and steps step every
  // env, so all envs share it (-1 = never reset)
  int32_t step_ctr = -1;
  int action_mode = kActIds;
  uint64_t launches = 0;
  std::vector<void*> allocs;
  // device buffers
  uint64_t* d_ep_start = nullptr;
  EpState* d_ep_state = nullptr;
  uint64_t* d_pool = nullptr;
  int32_t* d_bk_p = nullptr;
  int32_t* d_bk_q = nullptr;
  uint2* d_bk_id = nullptr;
  uint32_t* d_bk_st = nullptr;
  EnvHdr* d_hdr = nullptr;
  AgentRec* d_agents = nullptr;
  ActiveRec* d_active = nullptr;
  int32_t* d_actions = nullptr;
  mlob_agent_action* d_direct = nullptr;
  double* d_obs[MLOB_MAX_SPECS] = {};
  double* d_rewards = nullptr;
  uint8_t* d_dones = nullptr;
  mlob_agent_info* d_infos = nullptr;
  uint8_t* d_just_reset = nullptr;
  double* d_t[4] = {};
  mlob_trade* d_trades = nullptr;
  // split-step hand-offs (mlob_kernels.cu): agent messages, fill log + overflow pool, L2 summary
  DevMsg* d_amsg = nullptr;
  uint32_t amsg_cap = 0;
  FillEnt* d_fills = nullptr;
  FillEnt* d_fill_pool = nullptr;
  uint32_t* d_fill_pool_ctr = nullptr;  // one counter per step_io chunk
  uint64_t fill_pool_chunks = 0;
  L2Sum* d_l2sum = nullptr;
  L2Lvl* d_l2lv = nullptr;
  int64_t* d_t_rem = nullptr;
  uint64_t* d_env_seed = nullptr;
  uint64_t* d_env_index = nullptr;
  uint64_t* d_reset_eps = nullptr;
  uint32_t* d_error = nullptr;
  unsigned long long* d_scratch = nullptr;
  DevCfg* d_cfg = nullptr;

  double* d_stats = nullptr;  // K4 output for mlob_venv_allreduce_episode_stats
  // per-kernel timing of step launches (mlob_venv_profile): 4 events per step
  bool profiling = false;
  std::vector<cudaEvent_t> prof_ev;
  size_t prof_steps = 0;
  cudaEvent_t* prof_slot() {
    if (!profiling) return nullptr;
    while (prof_ev.size() < 4 * (prof_steps + 1)) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "event");
      prof_ev.push_back(e);
    }
    return prof_ev.data() + 4 * prof_steps++;
  }
  double* alloc_scratch_stats() {
    if (!d_stats) d_stats = alloc<double>(static_cast<size_t>(MLOB_MAX_SPECS) * kStatWords, "stats");
    return d_stats;
  }
  template <class T>
  T* alloc(size_t n, const char* what) {
    T* p = dalloc<T>(n, what);
    allocs.push_back(p);
    return p;
  }
  ~mlob_venv() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (cudaStream_t s : {stream2, copy_stream})
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    for (cudaEvent_t e : io_events) cudaEventDestroy(e);
    for (cudaEvent_t e : prof_ev) cudaEventDestroy(e);
    for (int t = 0; t < MLOB_MAX_SPECS; ++t) {
      free_net(nets[t]);
      cudaFree(batch[t].arena);
    }
    for (NetState& n : eval_nets) free_net(n);
    if (roll_graph) cudaGraphExecDestroy(roll_graph);
    cudaFree(ppo_ws);
    for (void* p : allocs) cudaFree(p);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  KParams params() const {
    KParams k;
    std::memset(&k, 0, sizeof k);
    k.msgs = store->d_msgs;
    k.ep_start = d_ep_start;
    k.ep_state = d_ep_state;
    k.levels = store->d_levels;
    k.n_episodes = starts.size();
    k.bk_p = d_bk_p;
    k.bk_q = d_bk_q;
    k.bk_id = d_bk_id;
    k.bk_st = d_bk_st;
    k.hdr = d_hdr;
    k.agents = d_agents;
    k.active = d_active;
    k.action_ids = d_actions;
    k.action_direct = d_direct;
    k.action_mode = action_mode;
    k.flags = static_cast<int32_t>(flags);
    for (int t = 0; t < cfg.n_specs; ++t) k.obs[t] = d_obs[t];
    k.rewards = d_rewards;
    k.dones = d_dones;
    k.infos = d_infos;
    k.just_reset = d_just_reset;
    k.t_pv = d_t[0];
    k.t_slip = d_t[1];
    k.t_comp = d_t[2];
    k.t_inv = d_t[3];
    k.trades = d_trades;
    k.trade_cap = trade_cap;
    k.t_rem = d_t_rem;
    k.amsg = d_amsg;
    k.amsg_cap = amsg_cap;
    k.fills = d_fills;
    k.l2sum = d_l2sum;
    k.l2lv = d_l2lv;
    k.fill_pool = d_fill_pool;
    k.fill_pool_ctr = d_fill_pool_ctr;
    k.fill_pool_chunks = static_cast<uint32_t>(fill_pool_chunks);
    k.env_seed = d_env_seed;
    k.env_index = d_env_index;
    k.seed = seed;
    k.env_index_base = env_index_base;
    k.pool = d_pool;
    k.pool_len = pool.empty() ? starts.size() : pool.size();
    k.n_envs_global = n_envs_global;
    k.n_envs = n_envs;
    k.reset_episodes = d_reset_eps;
    k.error = d_error;
    k.cfg = d_cfg;
    k.policies = d_policies;
    k.env_policy = d_env_policy;
    k.env_cell = has_cells ? d_env_cell : nullptr;
    return k;
  }

  void set_device() const { cuda_check(cudaSetDevice(device), "cudaSetDevice"); }

  // Maps device-side error bits onto the reference's exception classes.
  void check_device_errors() {
    uint32_t e = 0;
    cuda_check(cudaMemcpyAsync(&e, d_error, sizeof e, cudaMemcpyDeviceToHost, stream), "error word");
    cuda_check(cudaStreamSynchronize(stream), "stream sync");
    if (!e) return;
    cuda_check(cudaMemsetAsync(d_error, 0, sizeof e, stream), "error reset");
    if (e & kErrMissingState)
      fail(MLOB_E_RUNTIME,
           "MarketEnv::reset: no book state sampled at an episode start offset; reload the data "
           "with a matching sample stride");
    if (e & kErrTooDeep) fail(MLOB_E_INVALID_ARGUMENT, "OrderBook: snapshot deeper than book capacity");
    if (e & kErrBadAction) fail(MLOB_E_OUT_OF_RANGE, "action id out of range for its action space");
    if (e & kErrPriceRange) fail(MLOB_E_RUNTIME, "agent quote outside the device int32 price range");
    if (e & kErrSeqRange) fail(MLOB_E_RUNTIME, "arrival sequence beyond 2^24 in one episode");
    if (e & kErrActiveOverflow) fail(MLOB_E_RUNTIME, "more than MLOB_MAX_ACTIVE resting orders for one agent");
    if (e & kErrBadTrader) fail(MLOB_E_RUNTIME, "replay trader_id names a non-existent agent");
    if (e & kErrFillPool) fail(MLOB_E_RUNTIME, "agent-fill log overflow pool exhausted in one step");
    if (e & kErrAmsgCap) fail(MLOB_E_RUNTIME, "more agent messages in one step than the hand-off buffer holds");
    if (e & kErrDeepRange)
      fail(MLOB_E_RUNTIME, "deep book (capacity > 256): resting quantity >= 2^24, order id >= 2^44 or more than "
                           "2^20 arrivals in an episode");
    fail(MLOB_E_RUNTIME, "device error");
  }

  void check_episode(uint64_t ep) const {
    if (ep >= starts.size())
      fail(MLOB_E_OUT_OF_RANGE, "MarketEnv::reset: episode " + std::to_string(ep) +
                                    " out of range (count " + std::to_string(starts.size()) + ")");
    const EpState& s = ep_state[ep];
    if (!s.valid)
      fail(MLOB_E_RUNTIME, "MarketEnv::reset: no book state sampled at episode start offset " +
                               std::to_string(starts[ep]) +
                               "; reload the data with a matching sample stride");
    if (s.nb > cfg.book_capacity || s.na > cfg.book_capacity)
      fail(MLOB_E_INVALID_ARGUMENT, "OrderBook: snapshot deeper than book capacity");
  }

  uint64_t episode_for(uint64_t e, uint64_t k) const {  // rollout.hpp:286-288
    const uint64_t n = pool.empty() ? starts.size() : pool.size();
    const uint64_t i = (genv[e] + k * n_envs_global) % n;
    return pool.empty() ? i : pool[i];
  }
};

// ===========================================================================
// Binary store file: magic, counts, then the five arrays as they sit in
// memory (one writer per node, every rank reads: SURVEY §8e builds the
// store once per node instead of once per GPU).
namespace {
constexpr uint64_t kStoreMagic = 0x31454f5453424f4dull;  // "MOBSTOE1"
template <class T>
void write_vec(std::FILE* f, const std::vector<T>& v) {
  const uint64_t n = v.size();
  if (std::fwrite(&n, 8, 1, f) != 1 || (n && std::fwrite(v.data(), sizeof(T), n, f) != n))
    mlob::fail(MLOB_E_RUNTIME, "store file: write failed");
}
template <class T>
void read_vec(std::FILE* f, std::vector<T>& v) {
  uint64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) mlob::fail(MLOB_E_RUNTIME, "store file: truncated");
  v.resize(n);
  if (n && std::fread(v.data(), sizeof(T), n, f) != n) mlob::fail(MLOB_E_RUNTIME, "store file: truncated");
}
}  // namespace

extern "C" {

const char* mlob_last_error(void) { return g_err.c_str(); }
int mlob_abi_version(void) { return MLOB_ABI_VERSION; }

void mlob_default_agent_params(mlob_agent_params* p) {  // env/config.hpp:32-48
  std::memset(p, 0, sizeof *p);
  p->order_size = 10;
  p->inventory_cap = 30;
  p->rho = 50.0;
  p->quadratic_penalty = 1;
  p->lambda = 0.5;
  p->ref_price = MLOB_REF_MID;
  p->unfilled_penalty_coef = 0.1;
  p->lambda_exec = 0.0;
  p->task_size = 600;
  p->exec_complex = 1;
  p->reward_scale = 1.0;
  p->default_half_spread = 2;
  p->fixed_quant_from_mid = 0;
  int r = 0;
  for (int s : {1, 2, 3})  // SpreadSkewTable::standard, actions.hpp:117-124
    for (int k : {-1, 0, 1}) {
      p->spread_skew_half[r] = s;
      p->spread_skew_skew[r] = k;
      ++r;
    }
  p->n_spread_skew = r;
  const double g[4] = {0.05, 0.1, 0.5, 1.0};  // AvStParams, actions.hpp:142-147
  p->n_gamma = 4;
  for (int i = 0; i < 4; ++i) p->gamma_grid[i] = g[i];
  p->kappa = 1.5;
  p->sigma = 2.0;
  p->horizon = 64.0;
}

void mlob_default_agent_spec(mlob_agent_spec* s) {  // env/config.hpp:50-57
  std::memset(s, 0, sizeof *s);
  s->type = MLOB_MARKET_MAKER;
  s->count = 1;
  s->mm_space = MLOB_FIXED_QUANT;
  s->obs_space = MLOB_OBS_MM_BASIC;
  s->reward = MLOB_REWARD_SPOONER;
  mlob_default_agent_params(&s->params);
}

void mlob_default_env_config(mlob_env_config* c) {  // env/config.hpp:59-71
  std::memset(c, 0, sizeof *c);
  c->steps_per_episode = 64;
  c->messages_per_step = 100;
  c->start_stride_steps = 64;
  c->n_specs = 0;
  c->book_capacity = 100;
  c->obs_depth = 5;
  c->fallback_mid_half = 2000;
  c->synthetic_init_id_base = 1ull << 36;
  c->agent_id_base = 1ull << 40;
  c->agent_id_range = 1ull << 20;
  c->fill_reserve = 512;
}

void mlob_default_synth_config(mlob_synth_config* c) {  // data/synth.hpp:18-36
  std::memset(c, 0, sizeof *c);
  c->n_messages = 100000;
  c->initial_mid = 1000;
  c->volatility = 0.02;
  c->p_new_passive = 0.44;
  c->p_new_cross = 0.14;
  c->p_cancel = 0.08;
  c->p_delete = 0.18;
  c->p_execute = 0.14;
  c->band = 8;
  c->max_qty = 20;
  c->seed_levels = 5;
  c->seed_qty = 10;
  c->state_sample_every = 1600;
  c->state_depth = 10;
}

int mlob_action_arity(const mlob_agent_spec* s) {  // env/config.hpp:73-90
  switch (s->type) {
    case MLOB_EXECUTOR: return s->params.exec_complex ? 12 : 4;
    case MLOB_DIRECTIONAL: return 3;
    case MLOB_MARKET_MAKER:
      switch (s->mm_space) {
        case MLOB_SPREAD_SKEW: return s->params.n_spread_skew;
        case MLOB_FIXED_QUANT: return 8;
        case MLOB_AVST: return s->params.n_gamma;
      }
  }
  return 0;
}

int mlob_observation_size(int obs_space, uint64_t depth) {  // observations.hpp:69-76
  switch (obs_space) {
    case MLOB_OBS_MM_BASIC: return 8;
    case MLOB_OBS_MM_FULL: return static_cast<int>(8 + 4 * depth);
    case MLOB_OBS_EXEC: return 10;
  }
  return 0;
}

mlob_status mlob_validate_env_config(const mlob_env_config* cfg) {
  return guarded([&] { validate_config(*cfg); });
}

// ---- host stores ------------------------------------------------------------
mlob_status mlob_host_store_synth(const mlob_synth_config* cfg, uint64_t seed, mlob_host_store** out) {
  *out = nullptr;
  return guarded([&] {
    auto s = std::make_unique<mlob_host_store>();
    synth_generate(*cfg, seed, *s);
    *out = s.release();
  });
}

mlob_status mlob_host_store_create(const mlob_message* msgs, uint64_t n, const mlob_book_states* st,
                                   mlob_host_store** out) {
  *out = nullptr;
  return guarded([&] {
    auto s = std::make_unique<mlob_host_store>();
    s->msgs.assign(msgs, msgs + n);
    s->st_offset.push_back(0);
    if (st)
      for (uint64_t i = 0; i < st->n_states; ++i) {
        if (i > 0 && st->message_index[i] <= st->message_index[i - 1])
          fail(MLOB_E_INVALID_ARGUMENT, "book states must be sorted by message_index");
        const uint64_t off = st->level_offset[i];
        const uint32_t nb = st->n_bids[i];
        const uint32_t na = static_cast<uint32_t>(st->level_offset[i + 1] - off) - nb;
        s->push_state(st->message_index[i], st->levels + off, nb, st->levels + off + nb, na);
      }
    *out = s.release();
  });
}

mlob_status mlob_host_store_trim_front(mlob_host_store* s, uint64_t n) {
  return guarded([&] {
    if (n > s->msgs.size()) fail(MLOB_E_OUT_OF_RANGE, "trim beyond the store");
    s->msgs.erase(s->msgs.begin(), s->msgs.begin() + static_cast<std::ptrdiff_t>(n));
    mlob_host_store t;
    t.st_offset.push_back(0);
    for (size_t i = 0; i < s->st_index.size(); ++i) {
      if (s->st_index[i] < n) continue;
      t.push_state(s->st_index[i] - n, s->state_levels(i), s->st_nb[i], s->state_levels(i) + s->st_nb[i],
                   s->state_na(i));
    }
    t.msgs.swap(s->msgs);
    *s = std::move(t);
  });
}

uint64_t mlob_host_store_n_messages(const mlob_host_store* s) { return s->msgs.size(); }
const mlob_message* mlob_host_store_messages(const mlob_host_store* s) { return s->msgs.data(); }
uint64_t mlob_host_store_n_states(const mlob_host_store* s) { return s->st_index.size(); }
mlob_status mlob_host_store_state(const mlob_host_store* s, uint64_t i, uint64_t* message_index,
                                  mlob_level* bids, uint32_t* n_bids, mlob_level* asks,
                                  uint32_t* n_asks, uint32_t cap) {
  return guarded([&] {
    if (i >= s->st_index.size()) fail(MLOB_E_OUT_OF_RANGE, "state index out of range");
    *message_index = s->st_index[i];
    *n_bids = s->st_nb[i];
    *n_asks = s->state_na(i);
    if (*n_bids > cap || *n_asks > cap) fail(MLOB_E_OUT_OF_RANGE, "level buffer too small");
    std::memcpy(bids, s->state_levels(i), *n_bids * sizeof(mlob_level));
    std::memcpy(asks, s->state_levels(i) + *n_bids, *n_asks * sizeof(mlob_level));
  });
}
void mlob_host_store_free(mlob_host_store* s) { delete s; }


mlob_status mlob_host_store_save(const mlob_host_store* s, const char* path) {
  return guarded([&] {
    std::FILE* f = std::fopen(path, "wb");
    if (!f) fail(MLOB_E_RUNTIME, std::string("store file: cannot create ") + path);
    try {
      if (std::fwrite(&kStoreMagic, 8, 1, f) != 1) fail(MLOB_E_RUNTIME, "store file: write failed");
      write_vec(f, s->msgs);
      write_vec(f, s->st_index);
      write_vec(f, s->st_offset);
      write_vec(f, s->st_nb);
      write_vec(f, s->levels);
    } catch (...) {
      std::fclose(f);
      throw;
    }
    if (std::fclose(f) != 0) fail(MLOB_E_RUNTIME, "store file: write failed");
  });
}

mlob_status mlob_host_store_load(const char* path, mlob_host_store** out) {
  *out = nullptr;
  return guarded([&] {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) fail(MLOB_E_RUNTIME, std::string("store file: cannot open ") + path);
    auto s = std::make_unique<mlob_host_store>();
    try {
      uint64_t magic = 0;
      if (std::fread(&magic, 8, 1, f) != 1 || magic != kStoreMagic) fail(MLOB_E_RUNTIME, "store file: bad magic");
      read_vec(f, s->msgs);
      read_vec(f, s->st_index);
      read_vec(f, s->st_offset);
      read_vec(f, s->st_nb);
      read_vec(f, s->levels);
    } catch (...) {
      std::fclose(f);
      throw;
    }
    std::fclose(f);
    if (s->st_offset.size() != s->st_index.size() + 1 || s->st_nb.size() != s->st_index.size())
      fail(MLOB_E_RUNTIME, "store file: inconsistent state arrays");
    *out = s.release();
  });
}

mlob_status mlob_build_episode_index(uint64_t n_messages, int steps, int mps, int stride,
                                     uint64_t* starts, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    const auto v = build_episode_index(n_messages, steps, mps, stride);
    *n_out = v.size();
    for (uint64_t i = 0; i < v.size() && i < cap; ++i) starts[i] = v[i];
  });
}

// ---- device store -------------------------------------------------------------
static mlob_status upload(const mlob_message* msgs, uint64_t n, const mlob_host_store* hs,
                          int device, mlob_store** out) {
  *out = nullptr;
  return guarded([&] {
    auto s = std::make_unique<mlob_store>();
    s->device = device;
    s->n_msgs = n;
    std::vector<DevMsg> dm(n);
    for (uint64_t i = 0; i < n; ++i) {  // repack 40 B lob::Message -> 32 B DevMsg
      const mlob_message& m = msgs[i];
      if (m.kind > MLOB_HALT) fail(MLOB_E_INVALID_ARGUMENT, "message kind out of range");
      if (m.side > MLOB_ASK) fail(MLOB_E_INVALID_ARGUMENT, "message side out of range");
      if (m.trader_id < 0 || m.trader_id > 255)
        fail(MLOB_E_INVALID_ARGUMENT, "replay trader_id must lie in [0, 255]");
      DevMsg d;
      d.time = m.time;
      d.order_id = m.order_id;
      d.kind = m.kind;
      d.side = m.side;
      d._pad = 0;
      d.trader = m.trader_id;
      d.price = 0;
      d.qty = 0;
      if (m.kind == MLOB_NEW_LIMIT) {
        if (m.quantity > 0) {
          d.price = static_cast<int32_t>(fits32(m.price, "NewLimit price"));
          d.qty = static_cast<int32_t>(fits32(m.quantity, "NewLimit quantity"));
        }
      } else if (m.kind == MLOB_CANCEL_PARTIAL || m.kind == MLOB_EXECUTE_VISIBLE) {
        if (m.quantity < 0) fail(MLOB_E_INVALID_ARGUMENT, "negative cancel/execute quantity");
        d.qty = static_cast<int32_t>(std::min<int64_t>(m.quantity, INT32_MAX));  // min(q, by), q < 2^31
      }
      dm[i] = d;
    }
    std::vector<DevLevel> lv(hs->levels.size());
    for (size_t i = 0; i < lv.size(); ++i) {
      lv[i].price = static_cast<int32_t>(fits32(hs->levels[i].price, "book-state price"));
      if (hs->levels[i].quantity <= 0 || hs->levels[i].quantity >= INT32_MAX)
        fail(MLOB_E_INVALID_ARGUMENT, "book-state quantity outside (0, 2^31)");
      lv[i].qty = static_cast<int32_t>(hs->levels[i].quantity);
    }
    s->st_index = hs->st_index;
    s->st_offset = hs->st_offset;
    s->st_nb = hs->st_nb;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaMalloc(&s->d_msgs, std::max<uint64_t>(n, 1) * sizeof(DevMsg)), "cudaMalloc(store)");
    cuda_check(cudaMalloc(&s->d_levels, std::max<size_t>(lv.size(), 1) * sizeof(DevLevel)),
               "cudaMalloc(levels)");
    if (n) cuda_check(cudaMemcpy(s->d_msgs, dm.data(), n * sizeof(DevMsg), cudaMemcpyHostToDevice), "upload");
    if (!lv.empty())
      cuda_check(cudaMemcpy(s->d_levels, lv.data(), lv.size() * sizeof(DevLevel), cudaMemcpyHostToDevice),
                 "upload");
    s->bytes = n * sizeof(DevMsg) + lv.size() * sizeof(DevLevel);
    *out = s.release();
  });
}

mlob_status mlob_store_upload(const mlob_host_store* host, int device, mlob_store** out) {
  return upload(host->msgs.data(), host->msgs.size(), host, device, out);
}

mlob_status mlob_store_upload_raw(const mlob_message* msgs, uint64_t n, const mlob_book_states* st,
                                  int device, mlob_store** out) {
  mlob_host_store* hs = nullptr;
  mlob_status r = mlob_host_store_create(msgs, 0, st, &hs);
  if (r != MLOB_OK) return r;
  r = upload(msgs, n, hs, device, out);
  delete hs;
  return r;
}

mlob_status mlob_store_load_lobster(const char* message_path, const char* orderbook_path, int64_t units_per_tick,
                                    uint64_t sample_every, int device, mlob_store** out) {
  *out = nullptr;
  return guarded([&] {
    if (!message_path || !orderbook_path) fail(MLOB_E_INVALID_ARGUMENT, "load_lobster: null path");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cudaStream_t st = nullptr;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    lobster::LobsterStore ls;
    try {
      lobster::load(message_path, orderbook_path, units_per_tick, sample_every, st, ls);
    } catch (const lobster::LobsterError& e) {
      cudaStreamDestroy(st);
      fail(static_cast<mlob_status>(e.status), e.what());
    }
    cudaStreamDestroy(st);
    auto s = std::make_unique<mlob_store>();
    s->device = device;
    s->n_msgs = ls.n_msgs;
    s->d_msgs = ls.d_msgs;
    s->d_levels = ls.d_levels;
    s->st_index = std::move(ls.st_index);
    s->st_offset = std::move(ls.st_offset);
    s->st_nb = std::move(ls.st_nb);
    s->bytes = ls.n_msgs * sizeof(DevMsg) + ls.n_levels * sizeof(DevLevel);
    *out = s.release();
  });
}

mlob_status mlob_store_read_messages(const mlob_store* s, uint64_t first, uint64_t n, mlob_message* out) {
  return guarded([&] {
    if (first > s->n_msgs || n > s->n_msgs - first) fail(MLOB_E_OUT_OF_RANGE, "read_messages: range");
    cuda_check(cudaSetDevice(s->device), "cudaSetDevice");
    std::vector<DevMsg> d(n);
    if (n) cuda_check(cudaMemcpy(d.data(), s->d_msgs + first, n * sizeof(DevMsg), cudaMemcpyDeviceToHost), "D2H");
    for (uint64_t i = 0; i < n; ++i) {
      mlob_message& m = out[i];
      std::memset(&m, 0, sizeof m);
      m.time = d[i].time;
      m.order_id = d[i].order_id;
      m.price = d[i].price;
      m.quantity = d[i].qty;
      m.kind = d[i].kind;
      m.side = d[i].side;
      m.trader_id = d[i].trader;
    }
  });
}

uint64_t mlob_store_n_states(const mlob_store* s) { return s->st_index.size(); }

mlob_status mlob_store_state(const mlob_store* s, uint64_t i, uint64_t* message_index, mlob_level* bids,
                             uint32_t* n_bids, mlob_level* asks, uint32_t* n_asks, uint32_t cap) {
  return guarded([&] {
    if (i >= s->st_index.size()) fail(MLOB_E_OUT_OF_RANGE, "state index out of range");
    const uint64_t b = s->st_offset[i], e = s->st_offset[i + 1];
    const uint32_t nb = s->st_nb[i], na = static_cast<uint32_t>(e - b) - nb;
    *message_index = s->st_index[i];
    *n_bids = nb;
    *n_asks = na;
    if (nb > cap || na > cap) fail(MLOB_E_OUT_OF_RANGE, "state: capacity too small");
    std::vector<DevLevel> lv(e - b);
    cuda_check(cudaSetDevice(s->device), "cudaSetDevice");
    if (e > b) cuda_check(cudaMemcpy(lv.data(), s->d_levels + b, (e - b) * sizeof(DevLevel), cudaMemcpyDeviceToHost),
                          "D2H");
    for (uint32_t k = 0; k < nb; ++k) bids[k] = mlob_level{lv[k].price, lv[k].qty};
    for (uint32_t k = 0; k < na; ++k) asks[k] = mlob_level{lv[nb + k].price, lv[nb + k].qty};
  });
}

uint64_t mlob_store_n_messages(const mlob_store* s) { return s->n_msgs; }
uint64_t mlob_store_device_bytes(const mlob_store* s) { return s->bytes; }
void mlob_store_free(mlob_store* s) { delete s; }

// ---- venv -----------------------------------------------------------------------
static void build_devcfg(mlob_venv& v) {
  const mlob_env_config& c = v.cfg;
  DevCfg& d = v.dcfg;
  std::memset(&d, 0, sizeof d);
  d.steps_per_episode = c.steps_per_episode;
  d.mps = c.messages_per_step;
  d.capacity = static_cast<int32_t>(c.book_capacity);
  d.obs_depth = static_cast<int32_t>(c.obs_depth);
  d.n_specs = c.n_specs;
  d.fallback_mid_half = c.fallback_mid_half;
  d.synth_id_base = c.synthetic_init_id_base;
  d.agent_id_base = c.agent_id_base;
  d.agent_id_range = c.agent_id_range;
  int a = 0, maxdim = 0;
  for (int s = 0; s < c.n_specs; ++s) {
    const mlob_agent_spec& sp = c.specs[s];
    DevSpec& ds = d.specs[s];
    ds.type = sp.type;
    ds.mm_space = sp.mm_space;
    ds.obs_space = sp.obs_space;
    ds.reward = sp.reward;
    ds.count = sp.count;
    ds.flat_offset = a;
    ds.obs_dim = mlob_observation_size(sp.obs_space, c.obs_depth);
    ds.arity = mlob_action_arity(&sp);
    ds.order_size = sp.params.order_size;
    ds.inventory_cap = sp.params.inventory_cap;
    ds.task_size = sp.params.task_size;
    ds.rho = sp.params.rho;
    ds.lambda = sp.params.lambda;
    ds.unfilled_penalty_coef = sp.params.unfilled_penalty_coef;
    ds.reward_scale = sp.params.reward_scale;
    ds.quadratic_penalty = sp.params.quadratic_penalty;
    ds.ref_price = sp.params.ref_price;
    ds.exec_complex = sp.params.exec_complex;
    ds.default_half_spread = sp.params.default_half_spread;
    ds.fixed_quant_from_mid = sp.params.fixed_quant_from_mid;
    ds.n_spread_skew = sp.params.n_spread_skew;
    ds.n_gamma = sp.params.n_gamma;
    ds.sigma = sp.params.sigma;
    ds.horizon = sp.params.horizon;
    for (int i = 0; i < MLOB_MAX_SPREAD_SKEW_ROWS; ++i) {
      ds.ss_half[i] = sp.params.spread_skew_half[i];
      ds.ss_skew[i] = sp.params.spread_skew_skew[i];
    }
    for (int i = 0; i < sp.params.n_gamma; ++i) {
      const double g = sp.params.gamma_grid[i];
      ds.gamma[i] = g;
      // actions.hpp:157: (2.0 / gamma) * std::log1p(gamma / kappa), evaluated with the
      // host libm so the device reproduces the reference's bits exactly.
      ds.avst_term[i] = (2.0 / g) * std::log1p(g / sp.params.kappa);
    }
    for (int k = 0; k < sp.count; ++k) d.flat_spec[a++] = static_cast<uint8_t>(s);
    maxdim = std::max(maxdim, ds.obs_dim);
    if (sp.obs_space == MLOB_OBS_MM_FULL) d.full_l2 = 1;
  }
  d.n_agents = a;
  d.max_obs_dim = maxdim;
}

mlob_status mlob_venv_create(const mlob_venv_desc* desc, mlob_venv** out) {
  *out = nullptr;
  return guarded([&] {
    if (!desc->store) fail(MLOB_E_INVALID_ARGUMENT, "venv: null store");
    const mlob_env_config& c = desc->cfg;
    validate_config(c);
    auto v = std::make_unique<mlob_venv>();
    v->store = desc->store;
    v->cfg = c;
    v->device = desc->device;
    v->n_envs = desc->n_envs_local;
    v->n_envs_global = desc->n_envs_global ? desc->n_envs_global : desc->n_envs_local;
    v->env_index_base = desc->env_index_base;
    v->seed = desc->seed;
    v->flags = desc->flags;
    v->trade_cap = (desc->flags & MLOB_VENV_RECORD_TRADES) ? std::max<uint32_t>(desc->trade_capacity, 1) : 0;
    if (v->n_envs < 1) fail(MLOB_E_INVALID_ARGUMENT, "MarketVecEnv: n_envs >= 1");
    // device limits (stricter than the reference)
    v->spl = slots_per_lane(static_cast<int>(std::min<uint64_t>(c.book_capacity, 1u << 20)));
    if (v->spl < 0) fail(MLOB_E_INVALID_ARGUMENT, "book_capacity above the device limit (1024)");
    if (c.obs_depth > static_cast<uint64_t>(kMaxObsDepth))
      fail(MLOB_E_INVALID_ARGUMENT, "obs_depth above the device limit (64)");
    int A = 0;
    for (int s = 0; s < c.n_specs; ++s) {
      A += c.specs[s].count;
      if (c.specs[s].type == MLOB_EXECUTOR && c.specs[s].obs_space == MLOB_OBS_MM_BASIC)
        fail(MLOB_E_INVALID_ARGUMENT,
             "executor agents need the exec (or mm_full) observation space: the reference writes "
             "10 executor features (env.hpp:499-500) into the 8-wide mm_basic vector");
      if (c.specs[s].params.order_size > (INT32_MAX / 5))
        fail(MLOB_E_INVALID_ARGUMENT, "order_size outside the device int32 range");
    }
    if (A > MLOB_MAX_AGENTS) fail(MLOB_E_INVALID_ARGUMENT, "more than 32 agents per env");
    v->A = A;
    v->starts = build_episode_index(v->store->n_msgs, c.steps_per_episode, c.messages_per_step,
                                    c.start_stride_steps);
    if (v->starts.empty()) fail(MLOB_E_INVALID_ARGUMENT, "MarketVecEnv: empty episode pool");
    uint64_t max_depth = 0;
    v->ep_state.resize(v->starts.size());
    for (size_t i = 0; i < v->starts.size(); ++i) {
      EpState& e = v->ep_state[i];
      std::memset(&e, 0, sizeof e);
      const int64_t si = v->store->state_before(v->starts[i]);
      if (si < 0) continue;
      e.valid = 1;
      e.level_offset = v->store->st_offset[si];
      e.nb = v->store->st_nb[si];
      e.na = static_cast<uint32_t>(v->store->st_offset[si + 1] - e.level_offset) - e.nb;
      max_depth = std::max<uint64_t>(max_depth, std::max(e.nb, e.na));
    }
    const uint64_t seq_bound = static_cast<uint64_t>(c.steps_per_episode) *
                                   (static_cast<uint64_t>(c.messages_per_step) + 4ull * A) +
                               2 * max_depth;
    if (seq_bound >= kMaxSeq)
      fail(MLOB_E_INVALID_ARGUMENT, "episode too long for the device's 24-bit arrival sequence");
    if (v->spl > 8 && seq_bound >= (1u << 20))
      fail(MLOB_E_INVALID_ARGUMENT, "episode too long for the deep book's 20-bit arrival sequence");
    if (desc->episode_pool) {
      if (desc->pool_len == 0) fail(MLOB_E_INVALID_ARGUMENT, "MarketVecEnv: empty episode pool");
      v->pool.assign(desc->episode_pool, desc->episode_pool + desc->pool_len);
      for (uint64_t ep : v->pool)
        if (ep >= v->starts.size())
          fail(MLOB_E_OUT_OF_RANGE, "episode pool entry " + std::to_string(ep) + " out of range");
    }
    v->genv.resize(v->n_envs);
    for (uint64_t e = 0; e < v->n_envs; ++e)
      v->genv[e] = desc->env_indices ? desc->env_indices[e] : desc->env_index_base + e;
    v->step_ctr = -1;
    build_devcfg(*v);

    v->set_device();
    if (desc->stream) {
      v->stream = static_cast<cudaStream_t>(desc->stream);
    } else {
      cuda_check(cudaStreamCreateWithFlags(&v->stream, cudaStreamNonBlocking), "cudaStreamCreate");
      v->own_stream = true;
    }
    const uint64_t n = v->n_envs;
    const uint64_t slots = n * 2 * v->spl * kWarp;
    v->d_cfg = v->alloc<DevCfg>(1, "cfg");
    cuda_check(cudaMemcpy(v->d_cfg, &v->dcfg, sizeof(DevCfg), cudaMemcpyHostToDevice), "H2D cfg");
    v->d_ep_start = v->alloc<uint64_t>(v->starts.size(), "ep_start");
    v->d_ep_state = v->alloc<EpState>(v->ep_state.size(), "ep_state");
    cuda_check(cudaMemcpy(v->d_ep_start, v->starts.data(), v->starts.size() * 8, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(v->d_ep_state, v->ep_state.data(), v->ep_state.size() * sizeof(EpState),
                          cudaMemcpyHostToDevice), "H2D");
    if (!v->pool.empty()) {
      v->d_pool = v->alloc<uint64_t>(v->pool.size(), "pool");
      cuda_check(cudaMemcpy(v->d_pool, v->pool.data(), v->pool.size() * 8, cudaMemcpyHostToDevice), "H2D");
    }
    v->d_bk_p = v->alloc<int32_t>(slots, "book");
    v->d_bk_q = v->alloc<int32_t>(slots, "book");
    v->d_bk_id = v->alloc<uint2>(slots, "book");
    v->d_bk_st = v->alloc<uint32_t>(slots, "book");
    v->d_hdr = v->alloc<EnvHdr>(n, "hdr");
    v->d_agents = v->alloc<AgentRec>(n * std::max(A, 1), "agents");
    v->d_active = v->alloc<ActiveRec>(n * std::max(A, 1) * kMaxActive, "active");
    v->d_actions = v->alloc<int32_t>(n * std::max(A, 1), "actions");
    for (int t = 0; t < c.n_specs; ++t)
      v->d_obs[t] = v->alloc<double>(n * c.specs[t].count * v->dcfg.specs[t].obs_dim, "obs");
    v->d_rewards = v->alloc<double>(n * std::max(A, 1), "rewards");
    v->d_dones = v->alloc<uint8_t>(n * std::max(A, 1), "dones");
    v->d_infos = v->alloc<mlob_agent_info>(n * std::max(A, 1), "infos");
    v->d_just_reset = v->alloc<uint8_t>(n, "just_reset");
    for (int i = 0; i < 4; ++i) v->d_t[i] = v->alloc<double>(n * std::max(A, 1), "stats");
    if (v->trade_cap) v->d_trades = v->alloc<mlob_trade>(n * v->trade_cap, "trades");
    v->d_t_rem = v->alloc<int64_t>(n * std::max(A, 1), "stats");
    v->d_scratch = v->alloc<unsigned long long>(8, "scratch");
    v->amsg_cap = step_amsg_cap(v->dcfg);
    v->d_amsg = v->alloc<DevMsg>(n * v->amsg_cap, "agent messages");
    v->d_fills = v->alloc<FillEnt>(n * kFillInline, "fill log");
    // overflow pool: enough chunks for every env of the step to log 32 more
    // agent fills than the inline part holds (beyond: MLOB_E_RUNTIME), split
    // evenly over the step_io chunks, >= 64 chunks each
    v->fill_pool_chunks = std::max<uint64_t>(n / 8, 64 * kMaxIoChunks);
    v->d_fill_pool = v->alloc<FillEnt>(v->fill_pool_chunks * kFillChunk, "fill pool");
    v->d_fill_pool_ctr = v->alloc<uint32_t>(kMaxIoChunks, "fill pool counters");
    v->d_l2sum = v->alloc<L2Sum>(n, "l2 summary");
    if (v->dcfg.full_l2) v->d_l2lv = v->alloc<L2Lvl>(n * 2 * c.obs_depth, "l2 levels");
    v->d_reset_eps = v->alloc<uint64_t>(n, "reset_eps");
    v->d_error = v->alloc<uint32_t>(1, "error");
    if (desc->env_seeds) {
      v->d_env_seed = v->alloc<uint64_t>(n, "env_seed");
      cuda_check(cudaMemcpy(v->d_env_seed, desc->env_seeds, n * 8, cudaMemcpyHostToDevice), "H2D");
    }
    {
      v->d_env_index = v->alloc<uint64_t>(n, "env_index");
      cuda_check(cudaMemcpy(v->d_env_index, v->genv.data(), n * 8, cudaMemcpyHostToDevice), "H2D");
    }
    if (step_min_smem_bytes(v->dcfg) > 226 * 1024)
      fail(MLOB_E_INVALID_ARGUMENT, "configuration needs more shared memory per env than an SM has");
    cuda_check(cudaDeviceSynchronize(), "create");
    *out = v.release();
  });
}

void mlob_venv_destroy(mlob_venv* v) { delete v; }
uint64_t mlob_venv_n_envs(const mlob_venv* v) { return v->n_envs; }
int mlob_venv_n_agents(const mlob_venv* v) { return v->A; }
int mlob_venv_n_types(const mlob_venv* v) { return v->cfg.n_specs; }
uint64_t mlob_venv_n_streams(const mlob_venv* v, int t) {
  return v->n_envs * static_cast<uint64_t>(v->cfg.specs[t].count);
}
int mlob_venv_obs_dim(const mlob_venv* v, int t) { return v->dcfg.specs[t].obs_dim; }
int mlob_venv_n_actions(const mlob_venv* v, int t) { return v->dcfg.specs[t].arity; }
uint64_t mlob_venv_n_episodes(const mlob_venv* v) { return v->starts.size(); }
void* mlob_venv_stream(const mlob_venv* v) { return v->stream; }
uint64_t mlob_venv_launch_count(const mlob_venv* v) { return v->launches; }

static void do_reset(mlob_venv* v, const std::vector<uint64_t>& eps) {
  for (uint64_t ep : eps) v->check_episode(ep);
  v->set_device();
  cuda_check(cudaMemcpyAsync(v->d_reset_eps, eps.data(), eps.size() * 8, cudaMemcpyHostToDevice, v->stream),
             "H2D");
  cuda_check(cudaStreamSynchronize(v->stream), "sync");  // eps is a host temporary
  const KParams kp = v->params();
  cuda_check(launch_reset(kp, v->dcfg, v->spl, v->stream), "reset kernel");
  ++v->launches;
  v->step_ctr = 0;
}

mlob_status mlob_venv_reset_all(mlob_venv* v) {
  return guarded([&] {
    std::vector<uint64_t> eps(v->n_envs);
    for (uint64_t e = 0; e < v->n_envs; ++e) eps[e] = v->episode_for(e, 0);
    do_reset(v, eps);
  });
}

mlob_status mlob_venv_reset_envs(mlob_venv* v, const uint64_t* episodes) {
  return guarded([&] { do_reset(v, std::vector<uint64_t>(episodes, episodes + v->n_envs)); });
}

// actions.hpp:69-70: the first out-of-range id, reported like set_action does
static void fail_bad_action(const mlob_venv* v, const int32_t* ids) {
  const uint64_t n = v->n_envs * v->A;
  for (uint64_t i = 0; i < n; ++i) {
    const int a = static_cast<int>(i % v->A);
    const int ar = v->dcfg.specs[v->dcfg.flat_spec[a]].arity;
    if (ids[i] < 0 || ids[i] >= ar)
      fail(MLOB_E_OUT_OF_RANGE, "action id " + std::to_string(ids[i]) + " out of range for agent " +
                                    std::to_string(a) + " (arity " + std::to_string(ar) + ")");
  }
  fail(MLOB_E_OUT_OF_RANGE, "action id out of range for its action space");
}

mlob_status mlob_venv_set_actions(mlob_venv* v, const int32_t* ids, int on_device) {
  return guarded([&] {
    const uint64_t n = v->n_envs * v->A;
    v->set_device();
    if (!on_device) {
      // actions.hpp:69-70 range check, env-major without per-element division
      uint32_t ar[MLOB_MAX_AGENTS];
      for (int a = 0; a < v->A; ++a) ar[a] = static_cast<uint32_t>(v->dcfg.specs[v->dcfg.flat_spec[a]].arity);
      bool bad = false;
      for (uint64_t e = 0, i = 0; e < v->n_envs; ++e)
        for (int a = 0; a < v->A; ++a, ++i) bad |= static_cast<uint32_t>(ids[i]) >= ar[a];
      if (bad) fail_bad_action(v, ids);
      cuda_check(cudaMemcpyAsync(v->d_actions, ids, n * 4, cudaMemcpyHostToDevice, v->stream), "H2D");
      // a page-locked `ids` is read asynchronously: the caller may reuse it on return
      cuda_check(cudaStreamSynchronize(v->stream), "sync");
    } else {
      cuda_check(cudaMemcpyAsync(v->d_actions, ids, n * 4, cudaMemcpyDeviceToDevice, v->stream), "D2D");
    }
    v->action_mode = kActIds;
  });
}

mlob_status mlob_venv_set_direct_actions(mlob_venv* v, const mlob_agent_action* acts) {
  return guarded([&] {
    const uint64_t n = v->n_envs * v->A;
    for (uint64_t i = 0; i < n; ++i) {
      const mlob_agent_action& a = acts[i];
      if (a.direct) {
        if (a.n_quotes < 0 || a.n_quotes > 2) fail(MLOB_E_INVALID_ARGUMENT, "direct action: 0..2 quotes");
        for (int q = 0; q < a.n_quotes; ++q) {
          fits32(a.quotes[q].price, "direct quote price");
          fits32(a.quotes[q].quantity, "direct quote quantity");
          if (a.quotes[q].side > 1) fail(MLOB_E_INVALID_ARGUMENT, "direct quote side");
        }
      } else {
        const int ag = static_cast<int>(i % v->A);
        const int ar = v->dcfg.specs[v->dcfg.flat_spec[ag]].arity;
        if (a.id < 0 || a.id >= ar)
          fail(MLOB_E_OUT_OF_RANGE, "action id " + std::to_string(a.id) + " out of range");
      }
    }
    v->set_device();
    if (!v->d_direct) v->d_direct = v->alloc<mlob_agent_action>(n, "direct actions");
    cuda_check(cudaMemcpyAsync(v->d_direct, acts, n * sizeof(mlob_agent_action), cudaMemcpyHostToDevice,
                               v->stream), "H2D");
    cuda_check(cudaStreamSynchronize(v->stream), "sync");
    v->action_mode = kActDirect;
  });
}

static void advance_step(mlob_venv* v) {
  if (++v->step_ctr >= v->cfg.steps_per_episode && (v->flags & MLOB_VENV_AUTO_RESET)) v->step_ctr = 0;
}

static void do_step(mlob_venv* v, int mode, uint64_t bench_seed, uint64_t global_step) {
  const bool auto_reset = (v->flags & MLOB_VENV_AUTO_RESET) != 0;
  if (v->step_ctr < 0 || (!auto_reset && v->step_ctr >= v->cfg.steps_per_episode))
    fail(MLOB_E_LOGIC, "MarketEnv::step: episode is terminal; reset first");
  v->set_device();
  KParams kp = v->params();
  kp.action_mode = mode;
  kp.bench_seed = bench_seed;
  kp.global_step = global_step;
  cuda_check(launch_step(kp, v->dcfg, v->spl, v->stream, v->prof_slot()), "step kernels");
  v->launches += step_launches();
  advance_step(v);
}

mlob_status mlob_venv_step(mlob_venv* v) {
  return guarded([&] { do_step(v, v->action_mode, 0, 0); });
}

mlob_status mlob_venv_step_random(mlob_venv* v, uint64_t bench_seed, uint64_t global_step) {
  return guarded([&] { do_step(v, kActBench, bench_seed, global_step); });
}

mlob_status mlob_venv_synchronize(mlob_venv* v) {
  return guarded([&] {
    v->set_device();
    v->check_device_errors();
  });
}

mlob_status mlob_venv_gather(mlob_venv* v, int type, double* obs, uint8_t* resets) {
  return guarded([&] {
    if (type < 0 || type >= v->cfg.n_specs) fail(MLOB_E_OUT_OF_RANGE, "gather: type out of range");
    v->set_device();
    const uint64_t cnt = v->cfg.specs[type].count;
    const uint64_t dim = v->dcfg.specs[type].obs_dim;
    if (obs)
      cuda_check(cudaMemcpyAsync(obs, v->d_obs[type], v->n_envs * cnt * dim * 8, cudaMemcpyDeviceToHost,
                                 v->stream), "D2H");
    if (resets) {  // per-stream flags (rollout.hpp:206-211), expanded on the device
      const uint8_t* src = v->d_just_reset;
      if (cnt > 1) {
        if (!v->d_resets[type]) v->d_resets[type] = v->alloc<uint8_t>(v->n_envs * cnt, "resets");
        cuda_check(launch_expand_resets(v->d_just_reset, v->n_envs, static_cast<int>(cnt), v->d_resets[type],
                                        v->stream), "resets");
        src = v->d_resets[type];
      }
      cuda_check(cudaMemcpyAsync(resets, src, v->n_envs * cnt, cudaMemcpyDeviceToHost, v->stream), "D2H");
    }
    v->check_device_errors();
  });
}

const double* mlob_venv_obs_device(const mlob_venv* v, int type) { return v->d_obs[type]; }
const double* mlob_venv_rewards_device(const mlob_venv* v) { return v->d_rewards; }
const uint8_t* mlob_venv_dones_device(const mlob_venv* v) { return v->d_dones; }

extern "C++" {
template <class T>
static void d2h(mlob_venv* v, T* out, const T* src, uint64_t n) {
  v->set_device();
  cuda_check(cudaMemcpyAsync(out, src, n * sizeof(T), cudaMemcpyDeviceToHost, v->stream), "D2H");
  v->check_device_errors();
}
}

mlob_status mlob_venv_rewards(mlob_venv* v, double* out) {
  return guarded([&] { d2h(v, out, v->d_rewards, v->n_envs * v->A); });
}
mlob_status mlob_venv_dones(mlob_venv* v, uint8_t* out) {
  return guarded([&] { d2h(v, out, v->d_dones, v->n_envs * v->A); });
}
mlob_status mlob_venv_infos(mlob_venv* v, mlob_agent_info* out) {
  return guarded([&] { d2h(v, out, v->d_infos, v->n_envs * v->A); });
}

// ---- on-device policy inference and rollouts -------------------------------

static void check_net(const mlob_venv* v, int t, const mlob_policy_net& n) {
  if (n.obs_dim != v->dcfg.specs[t].obs_dim || n.n_actions != v->dcfg.specs[t].arity)
    fail(MLOB_E_INVALID_ARGUMENT, "policy net for type " + std::to_string(t) + ": expected obs_dim " +
                                      std::to_string(v->dcfg.specs[t].obs_dim) + ", n_actions " +
                                      std::to_string(v->dcfg.specs[t].arity));
  if (n.hidden < 1 || n.hidden > kPolicyMaxHidden)
    fail(MLOB_E_INVALID_ARGUMENT, "make_policy_net: hidden size capped at 512");
  if (n.n_actions > kPolicyMaxActions || n.obs_dim > kPolicyMaxObs)
    fail(MLOB_E_INVALID_ARGUMENT, "policy net: shape beyond the device limits");
  if (!n.w_ih || !n.w_hh || !n.b_ih || !n.b_hh || !n.w_actor || !n.b_actor || !n.w_critic)
    fail(MLOB_E_INVALID_ARGUMENT, "policy net: null weight array");
}

// Uploads `n` into `ns` (transposed layout, mlob_policy.h) with hidden buffers
// for B streams; a shape change reallocates and zeroes the hidden state.
static void upload_net(mlob_venv* v, const mlob_policy_net& n, mlob_venv::NetState& ns, uint64_t B) {
  const size_t D = n.obs_dim, H = n.hidden, A = n.n_actions, H3 = 3 * H;
  std::vector<double> w(H3 * D + H3 * H + 2 * H3 + A * H + A + H);
  double* w_ihT = w.data();
  for (size_t r = 0; r < H3; ++r)
    for (size_t d = 0; d < D; ++d) w_ihT[d * H3 + r] = n.w_ih[r * D + d];
  double* w_hhT = w_ihT + H3 * D;
  for (size_t r = 0; r < H3; ++r)
    for (size_t j = 0; j < H; ++j) w_hhT[j * H3 + r] = n.w_hh[r * H + j];
  double* b_ih = w_hhT + H3 * H;
  std::memcpy(b_ih, n.b_ih, H3 * 8);
  double* b_hh = b_ih + H3;
  std::memcpy(b_hh, n.b_hh, H3 * 8);
  double* w_aT = b_hh + H3;
  for (size_t a = 0; a < A; ++a)
    for (size_t j = 0; j < H; ++j) w_aT[j * A + a] = n.w_actor[a * H + j];
  double* b_a = w_aT + A * H;
  std::memcpy(b_a, n.b_actor, A * 8);
  double* w_c = b_a + A;
  std::memcpy(w_c, n.w_critic, H * 8);
  const bool same_shape = ns.w && ns.dn.D == n.obs_dim && ns.dn.H == n.hidden && ns.dn.A == n.n_actions;
  // the reference layout (for_each_param order) for ppo_update
  const uint64_t P = H3 * D + H3 * H + 2 * H3 + A * H + A + H + 1;
  std::vector<double> flat;
  flat.reserve(P);
  flat.insert(flat.end(), n.w_ih, n.w_ih + H3 * D);
  flat.insert(flat.end(), n.w_hh, n.w_hh + H3 * H);
  flat.insert(flat.end(), n.b_ih, n.b_ih + H3);
  flat.insert(flat.end(), n.b_hh, n.b_hh + H3);
  flat.insert(flat.end(), n.w_actor, n.w_actor + A * H);
  flat.insert(flat.end(), n.b_actor, n.b_actor + A);
  flat.insert(flat.end(), n.w_critic, n.w_critic + H);
  flat.push_back(n.b_critic);
  if (!same_shape) {
    ++v->buf_version;
    mlob_venv::free_net(ns);
    cuda_check(cudaMalloc(&ns.p, P * 8), "cudaMalloc(params)");
    cuda_check(cudaMalloc(&ns.g, P * 8), "cudaMalloc(grad)");
    cuda_check(cudaMalloc(&ns.m, P * 8), "cudaMalloc(adam)");
    cuda_check(cudaMalloc(&ns.v, P * 8), "cudaMalloc(adam)");
    ns.P = P;
    cuda_check(cudaMalloc(&ns.w, w.size() * 8), "cudaMalloc(net)");
    cuda_check(cudaMalloc(&ns.hidden[0], std::max<uint64_t>(1, B * H) * 8), "cudaMalloc(hidden)");
    cuda_check(cudaMalloc(&ns.hidden[1], std::max<uint64_t>(1, B * H) * 8), "cudaMalloc(hidden)");
    cuda_check(cudaMemsetAsync(ns.hidden[0], 0, B * H * 8, v->stream), "memset");
  }
  cuda_check(cudaMemcpyAsync(ns.w, w.data(), w.size() * 8, cudaMemcpyHostToDevice, v->stream), "H2D");
  cuda_check(cudaMemcpyAsync(ns.p, flat.data(), P * 8, cudaMemcpyHostToDevice, v->stream), "H2D");
  cuda_check(cudaMemsetAsync(ns.m, 0, P * 8, v->stream), "memset");  // AdamState::init
  cuda_check(cudaMemsetAsync(ns.v, 0, P * 8, v->stream), "memset");
  ns.adam_t = 0;
  const double* base = ns.w;
  ns.dn.D = n.obs_dim;
  ns.dn.H = n.hidden;
  ns.dn.A = n.n_actions;
  ns.dn.w_ihT = base;
  ns.dn.w_hhT = base + (w_hhT - w.data());
  ns.dn.b_ih = base + (b_ih - w.data());
  ns.dn.b_hh = base + (b_hh - w.data());
  ns.dn.w_actorT = base + (w_aT - w.data());
  ns.dn.b_actor = base + (b_a - w.data());
  ns.dn.w_critic = base + (w_c - w.data());
  ns.dn.b_critic = n.b_critic;
  ns.dn.b_critic_dev = ns.p + (P - 1);  // the reference layout ends with b_critic
  cuda_check(cudaStreamSynchronize(v->stream), "sync");  // `w` is a host temporary
}

mlob_status mlob_venv_set_nets(mlob_venv* v, const mlob_policy_net* nets) {
  return guarded([&] {
    if (!nets) fail(MLOB_E_INVALID_ARGUMENT, "set_nets: null");
    for (int t = 0; t < v->cfg.n_specs; ++t) check_net(v, t, nets[t]);  // nothing changes on error
    v->set_device();
    for (int t = 0; t < v->cfg.n_specs; ++t)
      upload_net(v, nets[t], v->nets[t], v->n_envs * static_cast<uint64_t>(v->cfg.specs[t].count));
    v->has_nets = true;
  });
}

static void ensure_batch(mlob_venv* v, int t, uint64_t T) {
  mlob_venv::Batch& b = v->batch[t];
  const uint64_t B = v->n_envs * static_cast<uint64_t>(v->cfg.specs[t].count);
  if (b.arena && b.T == T && b.B == B) return;
  ++v->buf_version;
  cudaFree(b.arena);
  b = mlob_venv::Batch{};
  const uint64_t D = v->nets[t].dn.D, H = v->nets[t].dn.H, TB = T * B;
  const uint64_t sizes[10] = {TB * D * 8, TB * 8, (TB + B) * 8, TB * 8, B * H * 8, TB * 8, TB * 8, TB * 4, TB, TB};
  uint64_t total = 0;
  for (uint64_t z : sizes) total += (z + 255) / 256 * 256;
  cuda_check(cudaMalloc(&b.arena, std::max<uint64_t>(total, 256)), "cudaMalloc(rollout batch)");
  char* p = b.arena;
  void** dst[10] = {(void**)&b.obs, (void**)&b.log_probs, (void**)&b.values, (void**)&b.rewards, (void**)&b.h0,
                    (void**)&b.adv, (void**)&b.ret, (void**)&b.actions, (void**)&b.dones, (void**)&b.resets};
  for (int i = 0; i < 10; ++i) {
    *dst[i] = p;
    p += (sizes[i] + 255) / 256 * 256;
  }
  b.T = T;
  b.B = B;
}

static PolicyArgs policy_args(mlob_venv* v, int t, const mlob_rollout_config& c, uint64_t update) {
  PolicyArgs pa{};
  mlob_venv::NetState& ns = v->nets[t];
  pa.net = ns.dn;
  pa.B = v->n_envs * static_cast<uint64_t>(v->cfg.specs[t].count);
  pa.count = v->cfg.specs[t].count;
  pa.offset = v->dcfg.specs[t].flat_offset;
  pa.agents_per_env = v->A;
  pa.type = t;
  pa.seed = c.seed;
  pa.update_index = update;
  pa.obs_env = v->d_obs[t];
  pa.just_reset = v->d_just_reset;
  pa.env_rewards = v->d_rewards;
  pa.env_dones = v->d_dones;
  pa.env_actions = v->d_actions;
  const mlob_venv::Batch& b = v->batch[t];
  pa.actions = b.actions;
  pa.log_probs = b.log_probs;
  pa.values = b.values;
  pa.rewards = b.rewards;
  pa.dones = b.dones;
  pa.resets = b.resets;
  return pa;
}

// The launches of one rollout (rollout.hpp:64-123): per step, one policy
// launch per type then the env step; then bootstrap values and GAE.
static void enqueue_rollout(mlob_venv* v, const mlob_rollout_config& cfg, uint64_t update_index, uint64_t T,
                            const uint64_t* seed_update) {
  const int NT = v->cfg.n_specs;
  for (uint64_t step = 0; step < T; ++step) {
    for (int t = 0; t < NT; ++t) {  // gather + policy_forward + sample + set_action
      mlob_venv::NetState& ns = v->nets[t];
      mlob_venv::Batch& b = v->batch[t];
      PolicyArgs pa = policy_args(v, t, cfg, update_index);
      pa.seed_update = seed_update;
      pa.row = static_cast<int32_t>(step);
      pa.prev_row = static_cast<int32_t>(step) - 1;
      pa.sample = 1;
      pa.hidden_in = ns.hidden[ns.cur];
      pa.hidden_out = ns.hidden[ns.cur ^ 1];
      pa.h0_out = step == 0 ? b.h0 : nullptr;
      pa.obs_out = b.obs + step * b.B * static_cast<uint64_t>(ns.dn.D);
      cuda_check(launch_policy(pa, v->stream), "policy kernel");
      ns.cur ^= 1;
    }
    KParams kp = v->params();  // step_all (rollout.hpp:92)
    kp.action_mode = kActIds;
    cuda_check(launch_step(kp, v->dcfg, v->spl, v->stream), "step kernel");
  }
  for (int t = 0; t < NT; ++t) {  // bootstrap values (hidden untouched), then GAE
    mlob_venv::NetState& ns = v->nets[t];
    mlob_venv::Batch& b = v->batch[t];
    PolicyArgs pa = policy_args(v, t, cfg, update_index);
    pa.seed_update = seed_update;
    pa.row = static_cast<int32_t>(T);
    pa.prev_row = static_cast<int32_t>(T) - 1;
    pa.sample = 0;
    pa.hidden_in = ns.hidden[ns.cur];
    cuda_check(launch_policy(pa, v->stream), "policy kernel");
    cuda_check(launch_gae(b.rewards, b.values, b.dones, T, b.B, cfg.discount, cfg.gae_lambda, b.adv, b.ret,
                          v->stream), "gae kernel");
  }
}

mlob_status mlob_venv_collect_rollout(mlob_venv* v, const mlob_rollout_config* cfg, uint64_t update_index) {
  return guarded([&] {
    if (!cfg || cfg->rollout_len < 1) fail(MLOB_E_INVALID_ARGUMENT, "collect_rollout: rollout_len >= 1");
    if (!v->has_nets) fail(MLOB_E_LOGIC, "collect_rollout: set_nets first");
    if (!(v->flags & MLOB_VENV_AUTO_RESET)) fail(MLOB_E_LOGIC, "collect_rollout: needs an auto-reset handle");
    if (v->step_ctr < 0) fail(MLOB_E_LOGIC, "MarketEnv::step: episode is terminal; reset first");
    v->set_device();
    const uint64_t T = static_cast<uint64_t>(cfg->rollout_len);
    const int NT = v->cfg.n_specs;
    for (int t = 0; t < NT; ++t) ensure_batch(v, t, T);
    const uint64_t launches = T * (NT + step_launches()) + 2 * NT;
    if (std::getenv("MLOB_NO_GRAPH")) {  // diagnostics: plain launches
      enqueue_rollout(v, *cfg, update_index, T, nullptr);
    } else {
      if (!v->d_seed_update) v->d_seed_update = v->alloc<uint64_t>(2, "seed/update");
      const uint64_t su[2] = {cfg->seed, update_index};
      cuda_check(cudaMemcpyAsync(v->d_seed_update, su, sizeof su, cudaMemcpyHostToDevice, v->stream), "H2D");
      // graph key: T, the hidden-buffer parity of every type, the buffer version,
      // and the GAE constants baked into the captured launches
      uint64_t key = T * 1315423911ull ^ v->buf_version * 2654435761ull;
      for (int t = 0; t < NT; ++t) key ^= static_cast<uint64_t>(v->nets[t].cur) << (40 + t);
      uint64_t dbits, lbits;
      std::memcpy(&dbits, &cfg->discount, 8);
      std::memcpy(&lbits, &cfg->gae_lambda, 8);
      key ^= host_splitmix(dbits) ^ host_splitmix(lbits + 1);
      if (!v->roll_graph || v->roll_key != key) {
        if (v->roll_graph) cudaGraphExecDestroy(v->roll_graph);
        v->roll_graph = nullptr;
        int cur[MLOB_MAX_SPECS];
        for (int t = 0; t < NT; ++t) cur[t] = v->nets[t].cur;
        cudaGraph_t g = nullptr;
        cuda_check(cudaStreamSynchronize(v->stream), "sync");
        cuda_check(cudaStreamBeginCapture(v->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
          enqueue_rollout(v, *cfg, update_index, T, v->d_seed_update);
        } catch (...) {
          cudaStreamEndCapture(v->stream, &g);
          if (g) cudaGraphDestroy(g);
          throw;
        }
        cuda_check(cudaStreamEndCapture(v->stream, &g), "end capture");
        const cudaError_t e = cudaGraphInstantiate(&v->roll_graph, g, 0);
        cudaGraphDestroy(g);
        cuda_check(e, "graph instantiate");
        for (int t = 0; t < NT; ++t) v->nets[t].cur = cur[t];  // replay advances them below
        v->roll_key = key;
      }
      cuda_check(cudaGraphLaunch(v->roll_graph, v->stream), "graph launch");
      for (int t = 0; t < NT; ++t)
        if (T & 1) v->nets[t].cur ^= 1;
    }
    for (uint64_t i = 0; i < T; ++i) advance_step(v);
    v->launches += launches;
    v->action_mode = kActIds;
  });
}

static const void* rollout_field(const mlob_venv* v, int t, int field, uint64_t* bytes) {
  const mlob_venv::Batch& b = v->batch[t];
  const mlob_venv::NetState& ns = v->nets[t];
  const uint64_t TB = b.T * b.B;
  switch (field) {
    case MLOB_RB_OBS: *bytes = TB * ns.dn.D * 8; return b.obs;
    case MLOB_RB_ACTIONS: *bytes = TB * 4; return b.actions;
    case MLOB_RB_LOG_PROBS: *bytes = TB * 8; return b.log_probs;
    case MLOB_RB_VALUES: *bytes = (TB + b.B) * 8; return b.values;
    case MLOB_RB_REWARDS: *bytes = TB * 8; return b.rewards;
    case MLOB_RB_DONES: *bytes = TB; return b.dones;
    case MLOB_RB_RESETS: *bytes = TB; return b.resets;
    case MLOB_RB_H0: *bytes = b.B * ns.dn.H * 8; return b.h0;
    case MLOB_RB_ADVANTAGES: *bytes = TB * 8; return b.adv;
    case MLOB_RB_RETURNS: *bytes = TB * 8; return b.ret;
    case MLOB_RB_HIDDEN:
      *bytes = v->n_envs * static_cast<uint64_t>(v->cfg.specs[t].count) * ns.dn.H * 8;
      return ns.hidden[ns.cur];
  }
  return nullptr;
}

mlob_status mlob_venv_rollout_read(mlob_venv* v, int type, int field, void* out, uint64_t cap_bytes) {
  return guarded([&] {
    if (type < 0 || type >= v->cfg.n_specs) fail(MLOB_E_OUT_OF_RANGE, "rollout_read: type out of range");
    if (field < MLOB_RB_OBS || field > MLOB_RB_HIDDEN) fail(MLOB_E_OUT_OF_RANGE, "rollout_read: field");
    uint64_t bytes = 0;
    const void* src = rollout_field(v, type, field, &bytes);
    if (!src) fail(MLOB_E_LOGIC, "rollout_read: no rollout collected");
    if (cap_bytes < bytes) fail(MLOB_E_OUT_OF_RANGE, "rollout_read: buffer too small");
    v->set_device();
    cuda_check(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, v->stream), "D2H");
    v->check_device_errors();
  });
}

const void* mlob_venv_rollout_device(const mlob_venv* v, int type, int field) {
  if (type < 0 || type >= v->cfg.n_specs) return nullptr;
  uint64_t bytes = 0;
  return rollout_field(v, type, field, &bytes);
}

// ---- PPO update (ppo.hpp:263-310) --------------------------------------------

void mlob_default_ppo_config(mlob_ppo_config* c) {  // PpoConfig defaults, ppo.hpp:19-28
  std::memset(c, 0, sizeof *c);
  c->epochs = 4;
  c->minibatches = 4;
  c->clip_eps = 0.2;
  c->vf_coef = 0.5;
  c->ent_coef = 0.01;
  c->lr = 3e-4;
  c->max_grad_norm = 0.5;
  c->normalize_adv = 1;
}

mlob_status mlob_venv_ppo_update(mlob_venv* v, int type, const mlob_ppo_config* cfg, uint64_t seed,
                                 uint64_t update_index, mlob_update_metrics* out) {
  return guarded([&] {
    if (type < 0 || type >= v->cfg.n_specs) fail(MLOB_E_OUT_OF_RANGE, "ppo_update: type out of range");
    if (!v->has_nets) fail(MLOB_E_LOGIC, "ppo_update: set_nets first");
    mlob_venv::Batch& bt = v->batch[type];
    if (!bt.arena || bt.B == 0 || bt.T == 0) fail(MLOB_E_INVALID_ARGUMENT, "ppo_update: empty batch");
    v->set_device();
    mlob_venv::NetState& ns = v->nets[type];
    const int D = ns.dn.D, H = ns.dn.H, A = ns.dn.A, H3 = 3 * H;
    const uint64_t T = bt.T, B = bt.B;
    const int n_mb = std::max(1, std::min<int>(cfg->minibatches, static_cast<int>(std::min<uint64_t>(B, INT32_MAX))));
    // workspace for the largest minibatch + the contractions' per-block partials
    const uint64_t Kmax = T * ((B + n_mb - 1) / n_mb + 1);
    const uint64_t max_e = std::max<uint64_t>({static_cast<uint64_t>(H3) * std::max(D, H), static_cast<uint64_t>(A) * H,
                                               static_cast<uint64_t>(H3), 8});
    const uint64_t part_n = static_cast<uint64_t>(kGemmBlocks) * max_e;
    const uint64_t cols = static_cast<uint64_t>(D) + 6ull * H + A + 1 + 5 + 2ull * H3 + 1;  // per row
    const uint64_t need = (Kmax * cols + part_n + 16) * 8 + B * 4 + 4096;
    if (need > v->ppo_ws_bytes) {
      cudaFree(v->ppo_ws);
      v->ppo_ws = nullptr;
      cuda_check(cudaMalloc(&v->ppo_ws, need), "cudaMalloc(ppo workspace)");
      v->ppo_ws_bytes = need;
    }
    double* wsd = reinterpret_cast<double*>(v->ppo_ws);
    double* part = wsd;            // gemm_tn partials
    double* sums = part + part_n;  // [0..4] terms, [5] grad norm, [6] reward sum
    double* rows = sums + 16;
    int32_t* d_order = reinterpret_cast<int32_t*>(rows + Kmax * cols);
    // reference-layout offsets (PolicyGrad mirrors PolicyNet)
    const uint64_t o_wih = 0, o_whh = o_wih + static_cast<uint64_t>(H3) * D, o_bih = o_whh + static_cast<uint64_t>(H3) * H,
                   o_bhh = o_bih + H3, o_wa = o_bhh + H3, o_ba = o_wa + static_cast<uint64_t>(A) * H, o_wc = o_ba + A,
                   o_bc = o_wc + H;
    std::vector<int32_t> order(B);
    for (uint64_t i = 0; i < B; ++i) order[i] = static_cast<int32_t>(i);
    mlob_update_metrics mt{};
    int n_updates = 0;
    for (int epoch = 0; epoch < cfg->epochs; ++epoch) {
      // CounterRng(make_key(seed, Minibatch, update, epoch, type)) + fisher_yates (ppo.hpp:275-278, rng.hpp:63-71)
      uint64_t st = host_splitmix(seed);
      st = host_fold(host_fold(host_fold(host_fold(st, 6), update_index), static_cast<uint64_t>(epoch)),
                     static_cast<uint64_t>(type));
      for (uint64_t i = B - 1; i > 0; --i) {
        st += 0x9E3779B97F4A7C15ull;
        const uint64_t j = host_splitmix(st) % (i + 1);
        if (i != j) std::swap(order[i], order[j]);
      }
      cuda_check(cudaMemcpyAsync(d_order, order.data(), B * 4, cudaMemcpyHostToDevice, v->stream), "H2D");
      for (int mb = 0; mb < n_mb; ++mb) {
        const uint64_t begin = B * static_cast<uint64_t>(mb) / n_mb, end = B * static_cast<uint64_t>(mb + 1) / n_mb;
        if (end == begin) continue;
        const uint64_t S = end - begin, K = T * S;
        PpoArgs a{};
        a.D = D;
        a.H = H;
        a.A = A;
        a.T = T;
        a.B = B;
        a.S = S;
        a.mb = d_order + begin;
        a.obs = bt.obs;
        a.resets = bt.resets;
        a.actions = bt.actions;
        a.logp_old = bt.log_probs;
        a.returns = bt.ret;
        a.h0 = bt.h0;
        a.w_ihT = ns.dn.w_ihT;
        a.w_hhT = ns.dn.w_hhT;
        a.w_actorT = ns.dn.w_actorT;
        a.w_ih = ns.p + o_wih;
        a.w_hh = ns.p + o_whh;
        a.b_ih = ns.p + o_bih;
        a.b_hh = ns.p + o_bhh;
        a.w_actor = ns.p + o_wa;
        a.b_actor = ns.p + o_ba;
        a.w_critic = ns.p + o_wc;
        cuda_check(cudaMemcpyAsync(&a.b_critic, ns.p + o_bc, 8, cudaMemcpyDeviceToHost, v->stream), "D2H");
        cuda_check(cudaStreamSynchronize(v->stream), "sync");
        a.clip_eps = cfg->clip_eps;
        a.vf_coef = cfg->vf_coef;
        a.ent_coef = cfg->ent_coef;
        double* r = rows;
        const auto carve = [&](uint64_t n) {
          double* p = r;
          r += n;
          return p;
        };
        double* adv = carve(K);
        a.adv = adv;
        a.X = carve(K * D);
        a.Hin = carve(K * H);
        a.R = carve(K * H);
        a.Z = carve(K * H);
        a.N = carve(K * H);
        a.HN = carve(K * H);
        a.Hout = carve(K * H);
        a.dL = carve(K * A);
        a.dV = carve(K);
        a.terms = carve(K * 5);
        a.dA = carve(K * H3);
        a.dB = carve(K * H3);
        cuda_check(launch_gather_adv(bt.adv, a.mb, T, B, S, adv, cfg->normalize_adv != 0, v->stream), "advantages");
        cuda_check(launch_ppo_forward(a, v->stream), "ppo forward");
        cuda_check(launch_ppo_backward(a, v->stream), "ppo backward");
        double* g = ns.g;
        cudaStream_t st = v->stream;
        cuda_check(gemm_tn(a.dA, a.X, K, H3, D, g + o_wih, part, st), "gradient w_ih");
        cuda_check(gemm_tn(a.dB, a.Hin, K, H3, H, g + o_whh, part, st), "gradient w_hh");
        cuda_check(colsum(a.dA, K, H3, g + o_bih, part, st), "gradient b_ih");
        cuda_check(colsum(a.dB, K, H3, g + o_bhh, part, st), "gradient b_hh");
        cuda_check(gemm_tn(a.dL, a.Hout, K, A, H, g + o_wa, part, st), "gradient w_actor");
        cuda_check(colsum(a.dL, K, A, g + o_ba, part, st), "gradient b_actor");
        cuda_check(gemm_tn(a.dV, a.Hout, K, 1, H, g + o_wc, part, st), "gradient w_critic");
        cuda_check(colsum(a.dV, K, 1, g + o_bc, part, st), "gradient b_critic");
        cuda_check(colsum(a.terms, K, 5, sums, part, st), "loss terms");
        double tsum[5];
        cuda_check(cudaMemcpyAsync(tsum, sums, sizeof tsum, cudaMemcpyDeviceToHost, v->stream), "D2H");
        cuda_check(cudaStreamSynchronize(v->stream), "sync");
        const double n_el = static_cast<double>(K);
        const double pg = tsum[0] / n_el, vl = tsum[1] / n_el, ent = tsum[2] / n_el, kl = tsum[3] / n_el,
                     cf = tsum[4] / n_el;
        const double loss = pg + cfg->vf_coef * vl - cfg->ent_coef * ent;
        if (!std::isfinite(loss)) {  // ppo.hpp:233-238
          std::ostringstream oss;
          oss << "ppo_update: non-finite loss (pg=" << pg << " v=" << vl << " ent=" << ent << " kl=" << kl << ")";
          fail(MLOB_E_RUNTIME, oss.str());
        }
        ++ns.adam_t;
        const double c1 = 1.0 - std::pow(0.9, static_cast<double>(ns.adam_t));
        const double c2 = 1.0 - std::pow(0.999, static_cast<double>(ns.adam_t));
        cuda_check(launch_clip_adam(ns.p, ns.g, ns.m, ns.v, ns.P, cfg->max_grad_norm, cfg->lr, c1, c2, sums + 5,
                                    v->stream),
                   "adam");
        // the next minibatch's forward reads the transposed copy
        cuda_check(launch_to_inference(ns.p, D, H, A, ns.w, v->stream), "to_inference");
        double norm = 0.0;
        cuda_check(cudaMemcpyAsync(&norm, sums + 5, 8, cudaMemcpyDeviceToHost, v->stream), "D2H");
        cuda_check(cudaStreamSynchronize(v->stream), "sync");
        mt.grad_norm += norm;
        mt.pg_loss += pg;
        mt.v_loss += vl;
        mt.entropy += ent;
        mt.approx_kl += kl;
        mt.clip_frac += cf;
        ++n_updates;
        v->launches += 4;
      }
    }
    const double inv = 1.0 / static_cast<double>(std::max(1, n_updates));
    mt.pg_loss *= inv;
    mt.v_loss *= inv;
    mt.entropy *= inv;
    mt.approx_kl *= inv;
    mt.clip_frac *= inv;
    mt.grad_norm *= inv;
    cuda_check(colsum(bt.rewards, T * B, 1, sums + 6, part, v->stream), "reward sum");
    double rsum = 0.0;
    cuda_check(cudaMemcpyAsync(&rsum, sums + 6, 8, cudaMemcpyDeviceToHost, v->stream), "D2H");
    // the next rollout's network: transposed copy + b_critic
    cuda_check(launch_to_inference(ns.p, D, H, A, ns.w, v->stream), "to_inference");
    cuda_check(cudaMemcpyAsync(&ns.dn.b_critic, ns.p + o_bc, 8, cudaMemcpyDeviceToHost, v->stream), "D2H");
    cuda_check(cudaStreamSynchronize(v->stream), "sync");
    mt.mean_reward = rsum / static_cast<double>(T * B);
    if (out) *out = mt;
  });
}

mlob_status mlob_venv_read_net(mlob_venv* v, int type, double* flat, uint64_t cap) {
  return guarded([&] {
    if (type < 0 || type >= v->cfg.n_specs) fail(MLOB_E_OUT_OF_RANGE, "read_net: type out of range");
    const mlob_venv::NetState& ns = v->nets[type];
    if (!ns.p) fail(MLOB_E_LOGIC, "read_net: set_nets first");
    if (cap < ns.P) fail(MLOB_E_OUT_OF_RANGE, "read_net: buffer too small");
    v->set_device();
    cuda_check(cudaMemcpyAsync(flat, ns.p, ns.P * 8, cudaMemcpyDeviceToHost, v->stream), "D2H");
    cuda_check(cudaStreamSynchronize(v->stream), "sync");
  });
}

// ---- scripted policies and cross-play evaluation ----------------------------

void mlob_default_policy(int kind, mlob_policy* out) {
  std::memset(out, 0, sizeof *out);
  out->kind = kind;
  out->twap_mode = MLOB_TWAP_AGGRESSIVE;
  out->avst_gamma_index = 1;  // AvStBaseline, avst.hpp:14-17
  const double grid[4] = {0.05, 0.1, 0.5, 1.0};  // AvStParams, actions.hpp:142-147
  out->n_gamma = 4;
  for (int i = 0; i < 4; ++i) out->gamma_grid[i] = grid[i];
  out->kappa = 1.5;
  out->sigma = 2.0;
  out->horizon = 64.0;
}

static DevPolicy resolve_policy(const mlob_policy& p) {
  if (p.kind < MLOB_POLICY_LEARNED || p.kind > MLOB_POLICY_NOOP)
    fail(MLOB_E_INVALID_ARGUMENT, "policy: unknown kind " + std::to_string(p.kind));
  if (p.kind == MLOB_POLICY_LEARNED && !p.net)
    fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: learned policy without a network");
  if (p.kind == MLOB_POLICY_TWAP && p.twap_mode != MLOB_TWAP_AGGRESSIVE && p.twap_mode != MLOB_TWAP_PASSIVE)
    fail(MLOB_E_INVALID_ARGUMENT, "policy: twap_mode");
  DevPolicy d{};
  d.kind = p.kind;
  d.twap_mode = p.twap_mode;
  if (p.kind == MLOB_POLICY_AVST) {
    if (p.n_gamma < 0 || p.n_gamma > MLOB_MAX_GAMMA) fail(MLOB_E_INVALID_ARGUMENT, "policy: n_gamma");
    if (p.avst_gamma_index < 0 || p.avst_gamma_index >= p.n_gamma)  // avst.hpp:21-23
      fail(MLOB_E_OUT_OF_RANGE, "avst_policy: gamma_index out of range");
    const double g = p.gamma_grid[p.avst_gamma_index];
    d.gamma = g;
    d.sigma = p.sigma;
    d.horizon = p.horizon;
    d.avst_term = (2.0 / g) * std::log1p(g / p.kappa);  // actions.hpp:158, host libm
  }
  return d;
}

static void set_policies(mlob_venv* v, const mlob_policy* policies, int n_policies, const uint8_t* env_policy,
                         const uint64_t* env_cell, bool learned_ok = false) {
  if (n_policies < 1 || n_policies > kMaxPolicies)
    fail(MLOB_E_INVALID_ARGUMENT, "set_policies: 1.." + std::to_string(kMaxPolicies) + " policies");
  std::vector<DevPolicy> dp(n_policies);
  for (int i = 0; i < n_policies; ++i) {
    if (policies[i].kind == MLOB_POLICY_LEARNED && !learned_ok)
      fail(MLOB_E_INVALID_ARGUMENT, "set_policies: learned policies run through mlob_evaluate_matrix");
    dp[i] = resolve_policy(policies[i]);
  }
  const uint64_t n = v->n_envs * static_cast<uint64_t>(v->cfg.n_specs);
  for (uint64_t i = 0; i < n; ++i)
    if (env_policy[i] >= n_policies) fail(MLOB_E_OUT_OF_RANGE, "set_policies: policy index out of range");
  v->set_device();
  if (!v->d_policies) {
    v->d_policies = v->alloc<DevPolicy>(kMaxPolicies, "policies");
    v->d_env_policy = v->alloc<uint8_t>(n > 0 ? n : 1, "env_policy");
    v->d_env_cell = v->alloc<uint64_t>(v->n_envs, "env_cell");
  }
  cuda_check(cudaMemcpyAsync(v->d_policies, dp.data(), dp.size() * sizeof(DevPolicy), cudaMemcpyHostToDevice,
                             v->stream), "H2D");
  cuda_check(cudaMemcpyAsync(v->d_env_policy, env_policy, n, cudaMemcpyHostToDevice, v->stream), "H2D");
  v->has_cells = env_cell != nullptr;
  if (env_cell)
    cuda_check(cudaMemcpyAsync(v->d_env_cell, env_cell, v->n_envs * 8, cudaMemcpyHostToDevice, v->stream), "H2D");
  cuda_check(cudaStreamSynchronize(v->stream), "sync");  // host arrays may be temporaries
  v->action_mode = kActScripted;
}

mlob_status mlob_venv_set_policies(mlob_venv* v, const mlob_policy* policies, int n_policies,
                                   const uint8_t* env_policy, const uint64_t* env_cell) {
  return guarded([&] { set_policies(v, policies, n_policies, env_policy, env_cell); });
}

mlob_status mlob_evaluate_matrix(const mlob_store* store, const mlob_env_config* cfg, const uint64_t* episodes,
                                 uint64_t n_episodes, const mlob_policy* type0, int n_type0,
                                 const mlob_policy* type1, int n_type1, uint64_t seed, int device,
                                 mlob_cell_stats* out) {
  return guarded([&] {
    if (cfg->n_specs != 2) fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: exactly two agent types required");
    if (n_episodes == 0) fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: empty episode set");
    for (int i = 0; i < n_type0 + n_type1; ++i)
      if ((i < n_type0 ? type0[i] : type1[i - n_type0]).kind == MLOB_POLICY_LEARNED &&
          !(i < n_type0 ? type0[i] : type1[i - n_type0]).net)
        fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: learned policy without a network");
    if (n_type0 <= 0 || n_type1 <= 0) return;
    if (n_type0 + n_type1 > kMaxPolicies)
      fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: at most " + std::to_string(kMaxPolicies) + " options");
    std::vector<mlob_policy> table(type0, type0 + n_type0);
    table.insert(table.end(), type1, type1 + n_type1);
    for (const auto& p : table) resolve_policy(p);  // argument errors before any work
    // one env per (row, col, episode), cell-major; every env is the reference's
    // MarketEnv(seed, env index 0) (evaluate.hpp:128)
    const uint64_t cells = static_cast<uint64_t>(n_type0) * n_type1, n = cells * n_episodes;
    std::vector<uint64_t> zeros(n, 0), eps(n), cell(n);
    std::vector<uint8_t> pol(n * 2);
    for (uint64_t e = 0; e < n; ++e) {
      const uint64_t c = e / n_episodes, row = c / n_type1, col = c % n_type1;
      eps[e] = episodes[e % n_episodes];
      cell[e] = row * 1000 + col;  // evaluate.hpp:139
      pol[e * 2] = static_cast<uint8_t>(row);
      pol[e * 2 + 1] = static_cast<uint8_t>(n_type0 + col);
    }
    mlob_venv_desc d{};
    d.store = store;
    d.cfg = *cfg;
    d.seed = seed;
    d.n_envs_global = d.n_envs_local = n;
    d.env_indices = zeros.data();
    d.device = device;
    mlob_venv* raw = nullptr;
    const mlob_status st = mlob_venv_create(&d, &raw);
    if (st != MLOB_OK) fail(st, mlob_last_error());
    std::unique_ptr<mlob_venv> v(raw);
    // Learned options: network + per-stream hidden state, zeroed at the episode
    // start (evaluate.hpp:151-154); argmax ids are written before each step
    struct Learned {
      int option, type;
    };
    std::vector<Learned> learned;
    for (int i = 0; i < static_cast<int>(table.size()); ++i)
      if (table[i].kind == MLOB_POLICY_LEARNED) {
        const int tau = i < n_type0 ? 0 : 1;
        check_net(v.get(), tau, *table[i].net);
        learned.push_back({i, tau});
      }
    v->eval_nets.resize(learned.size());
    for (size_t k = 0; k < learned.size(); ++k)
      upload_net(v.get(), *table[learned[k].option].net, v->eval_nets[k],
                 n * static_cast<uint64_t>(cfg->specs[learned[k].type].count));
    do_reset(v.get(), eps);
    set_policies(v.get(), table.data(), static_cast<int>(table.size()), pol.data(), cell.data(), true);
    for (int t = 0; t < cfg->steps_per_episode; ++t) {
      for (size_t k = 0; k < learned.size(); ++k) {
        mlob_venv::NetState& ns = v->eval_nets[k];
        const int tau = learned[k].type;
        PolicyArgs pa{};
        pa.net = ns.dn;
        pa.B = n * static_cast<uint64_t>(cfg->specs[tau].count);
        pa.count = cfg->specs[tau].count;
        pa.offset = v->dcfg.specs[tau].flat_offset;
        pa.agents_per_env = v->A;
        pa.type = tau;
        pa.argmax = 1;
        pa.prev_row = -1;
        pa.env_policy = v->d_env_policy;
        pa.n_specs = cfg->n_specs;
        pa.filter = learned[k].option;
        pa.obs_env = v->d_obs[tau];
        pa.just_reset = nullptr;  // choose_action passes reset = 0 (evaluate.hpp:83)
        pa.env_actions = v->d_actions;
        pa.hidden_in = ns.hidden[ns.cur];
        pa.hidden_out = ns.hidden[ns.cur ^ 1];
        cuda_check(launch_policy(pa, v->stream), "policy kernel");
        ++v->launches;
        ns.cur ^= 1;
      }
      do_step(v.get(), kActScripted, 0, 0);
    }
    const int A = v->A;
    std::vector<mlob_agent_info> info(n * A);
    std::vector<AgentRec> ag(n * A);
    d2h(v.get(), info.data(), v->d_infos, n * A);
    d2h(v.get(), ag.data(), v->d_agents, n * A);
    // per-cell statistics in the reference's order (evaluate.hpp:171-213)
    const auto mean_stderr = [](const std::vector<double>& xs, double& mean, double& se) {
      const double k = static_cast<double>(xs.size());
      mean = 0.0;
      for (const double x : xs) mean += x;
      mean /= k;
      double var = 0.0;
      for (const double x : xs) var += (x - mean) * (x - mean);
      se = xs.size() > 1 ? std::sqrt(var / (k - 1.0) / k) : 0.0;
    };
    for (uint64_t c = 0; c < cells; ++c) {
      std::vector<double> pv[2], slip[2];
      double completion_sum[2] = {0.0, 0.0};
      int64_t filled[2] = {0, 0};
      for (uint64_t k = 0; k < n_episodes; ++k) {
        const uint64_t e = c * n_episodes + k;
        double ep_pv[2] = {0.0, 0.0}, ep_slip[2] = {0.0, 0.0};
        int type_agents[2] = {0, 0};
        for (int a = 0; a < A; ++a) {
          const int tau = v->dcfg.flat_spec[a];
          const mlob_agent_info& inf = info[e * A + a];
          ep_pv[tau] += inf.portfolio_value;
          ep_slip[tau] += inf.slippage_total;
          ++type_agents[tau];
          filled[tau] += ag[e * A + a].filled_total;
          const mlob_agent_spec& sp = cfg->specs[tau];
          if (sp.type == MLOB_EXECUTOR)
            completion_sum[tau] +=
                1.0 - static_cast<double>(inf.task_remaining) / static_cast<double>(sp.params.task_size);
          else
            completion_sum[tau] += 0.0;
        }
        for (int tau = 0; tau < 2; ++tau) {
          pv[tau].push_back(ep_pv[tau] / type_agents[tau]);
          slip[tau].push_back(ep_slip[tau] / type_agents[tau]);
        }
      }
      mlob_cell_stats& cs = out[c];
      std::memset(&cs, 0, sizeof cs);
      cs.episodes = static_cast<int64_t>(n_episodes);
      for (int tau = 0; tau < 2; ++tau) {
        mlob_type_cell_stats& t = cs.per_type[tau];
        mean_stderr(pv[tau], t.pv_mean, t.pv_stderr);
        t.filled_total = filled[tau];
        t.no_fills = filled[tau] == 0;
        if (!t.no_fills) mean_stderr(slip[tau], t.slippage_mean, t.slippage_stderr);
        t.completion_mean = completion_sum[tau] / (static_cast<double>(n_episodes) *
                                                   static_cast<double>(cfg->specs[tau].count));
      }
    }
  });
}

// ---- fused env I/O: chunked step with overlapped transfers -----------------

// KParams of the env range [c0, c0 + n): every per-env array offset by c0,
// the global env identity (RNG keys, episode pool) kept
static KParams chunk_params(const mlob_venv* v, const KParams& k0, uint64_t c0, uint64_t n, uint64_t idx,
                            uint64_t nchunks) {
  KParams k = k0;
  // hand-off buffers and this chunk's share of the fill-overflow pool
  k.amsg += c0 * v->amsg_cap;
  k.fills += c0 * kFillInline;
  k.l2sum += c0;
  if (k.l2lv) k.l2lv += c0 * 2 * v->cfg.obs_depth;
  k.t_rem += c0 * static_cast<uint64_t>(v->A);
  const uint64_t per = v->fill_pool_chunks / nchunks;
  k.fill_pool += idx * per * kFillChunk;
  k.fill_pool_chunks = static_cast<uint32_t>(per);
  k.fill_pool_ctr += idx;
  const uint64_t A = static_cast<uint64_t>(v->A);
  const size_t bs = static_cast<size_t>(2 * v->spl * kWarp) * c0;
  k.bk_p += bs;
  k.bk_q += bs;
  if (v->spl > 8)  // deep books: the id buffer holds u32 low words (SmemSide layout)
    k.bk_id = reinterpret_cast<uint2*>(reinterpret_cast<uint32_t*>(k.bk_id) + bs);
  else
    k.bk_id += bs;
  k.bk_st += bs;
  k.hdr += c0;
  k.agents += c0 * A;
  k.active += c0 * A * kMaxActive;
  if (k.action_ids) k.action_ids += c0 * A;
  if (k.action_direct) k.action_direct += c0 * A;
  for (int t = 0; t < v->cfg.n_specs; ++t)
    k.obs[t] += c0 * static_cast<uint64_t>(v->cfg.specs[t].count) * static_cast<uint64_t>(v->dcfg.specs[t].obs_dim);
  k.rewards += c0 * A;
  k.dones += c0 * A;
  k.infos += c0 * A;
  k.just_reset += c0;
  k.t_pv += c0 * A;
  k.t_slip += c0 * A;
  k.t_comp += c0 * A;
  k.t_inv += c0 * A;
  if (k.trades) k.trades += c0 * v->trade_cap;
  if (k.env_seed) k.env_seed += c0;
  if (k.env_index) k.env_index += c0;
  k.env_index_base += c0;
  k.n_envs = n;
  return k;
}

static uint64_t io_chunk_envs(uint64_t n) {
  if (const char* e = std::getenv("MLOB_IO_CHUNKS")) {  // diagnostics: fixed chunk count
    const uint64_t c = std::min<uint64_t>(std::strtoull(e, nullptr, 10), kMaxIoChunks);
    if (c > 0) return (n + c - 1) / c;
  }
  // ≤ 8 chunks of ≥ 16k envs: each chunk is several rounds of the step kernel,
  // so the per-chunk tail is small; the last chunk's copies are the only
  // exposed transfer (measured at 65,536 envs: 4 chunks +4 % e2e over 1)
  uint64_t c = (n + 7) / 8;
  if (c < 16384) c = 16384;
  return (c + 1279) / 1280 * 1280;
}

mlob_status mlob_venv_step_io(mlob_venv* v, const mlob_step_io* io) {
  return guarded([&] {
    if (!io) fail(MLOB_E_INVALID_ARGUMENT, "step_io: null descriptor");
    const bool auto_reset = (v->flags & MLOB_VENV_AUTO_RESET) != 0;
    if (v->step_ctr < 0 || (!auto_reset && v->step_ctr >= v->cfg.steps_per_episode))
      fail(MLOB_E_LOGIC, "MarketEnv::step: episode is terminal; reset first");
    v->set_device();
    const uint64_t n = v->n_envs, A = static_cast<uint64_t>(v->A);
    const uint64_t chunk = io_chunk_envs(n);
    const uint64_t nc = (n + chunk - 1) / chunk;
    if (!v->copy_stream) {
      cuda_check(cudaStreamCreateWithFlags(&v->stream2, cudaStreamNonBlocking), "stream");
      cuda_check(cudaStreamCreateWithFlags(&v->copy_stream, cudaStreamNonBlocking), "stream");
      v->d_gate = v->alloc<uint32_t>(1, "gate");
    }
    while (v->io_events.size() < nc + 3) {
      cudaEvent_t e;
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      v->io_events.push_back(e);
    }
    for (int t = 0; t < v->cfg.n_specs; ++t)
      if (io->resets[t] && v->cfg.specs[t].count > 1 && !v->d_resets[t])
        v->d_resets[t] = v->alloc<uint8_t>(n * static_cast<uint64_t>(v->cfg.specs[t].count), "resets");
    KParams k0 = v->params();
    if (io->actions) {  // stage + validate the whole batch before any env steps
      cuda_check(cudaMemcpyAsync(v->d_actions, io->actions, n * A * 4, cudaMemcpyHostToDevice, v->stream), "H2D");
      cuda_check(launch_validate_actions(v->d_actions, n * A, v->d_cfg, v->d_error, v->d_gate, v->stream),
                 "validate kernel");
      v->action_mode = kActIds;
      k0.gate = v->d_gate;
    }
    k0.action_mode = v->action_mode;
    cudaEvent_t* ev = v->io_events.data();
    // one chunk: nothing to overlap, so everything stays on the handle's stream
    const bool single = nc == 1;
    cudaStream_t cs = single ? v->stream : v->copy_stream;
    if (!single) {
      cuda_check(cudaEventRecord(ev[0], v->stream), "event");
      cuda_check(cudaStreamWaitEvent(v->stream2, ev[0], 0), "wait");
    }
    const auto d2h = [&](void* dst, const void* src, uint64_t bytes) {
      if (dst && bytes) cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, cs), "D2H");
    };
    for (uint64_t i = 0; i < nc; ++i) {
      const uint64_t c0 = i * chunk, m = std::min(chunk, n - c0);
      cudaStream_t s = (i & 1) ? v->stream2 : v->stream;
      cuda_check(launch_step(chunk_params(v, k0, c0, m, i, nc), v->dcfg, v->spl, s), "step kernels");
      v->launches += step_launches();
      for (int t = 0; t < v->cfg.n_specs; ++t)
        if (io->resets[t] && v->cfg.specs[t].count > 1) {
          const int cnt = v->cfg.specs[t].count;
          cuda_check(launch_expand_resets(v->d_just_reset + c0, m, cnt, v->d_resets[t] + c0 * cnt, s), "resets");
          ++v->launches;
        }
      if (!single) {
        cuda_check(cudaEventRecord(ev[1 + i], s), "event");
        cuda_check(cudaStreamWaitEvent(v->copy_stream, ev[1 + i], 0), "wait");
      }
      d2h(io->rewards ? io->rewards + c0 * A : nullptr, v->d_rewards + c0 * A, m * A * 8);
      d2h(io->dones ? io->dones + c0 * A : nullptr, v->d_dones + c0 * A, m * A);
      d2h(io->infos ? io->infos + c0 * A : nullptr, v->d_infos + c0 * A, m * A * sizeof(mlob_agent_info));
      for (int t = 0; t < v->cfg.n_specs; ++t) {
        const uint64_t cnt = static_cast<uint64_t>(v->cfg.specs[t].count);
        const uint64_t w = cnt * static_cast<uint64_t>(v->dcfg.specs[t].obs_dim);
        d2h(io->obs[t] ? io->obs[t] + c0 * w : nullptr, v->d_obs[t] + c0 * w, m * w * 8);
        if (io->resets[t])
          d2h(io->resets[t] + c0 * cnt, cnt > 1 ? v->d_resets[t] + c0 * cnt : v->d_just_reset + c0, m * cnt);
      }
    }
    if (!single) {  // join: later work on the handle's stream follows both streams and the copies
      cuda_check(cudaEventRecord(ev[nc + 1], v->stream2), "event");
      cuda_check(cudaEventRecord(ev[nc + 2], v->copy_stream), "event");
      cuda_check(cudaStreamWaitEvent(v->stream, ev[nc + 1], 0), "wait");
      cuda_check(cudaStreamWaitEvent(v->stream, ev[nc + 2], 0), "wait");
    }
    uint32_t e = 0;
    cuda_check(cudaMemcpyAsync(&e, v->d_error, sizeof e, cudaMemcpyDeviceToHost, v->stream), "error word");
    cuda_check(cudaStreamSynchronize(v->stream), "stream sync");
    if ((e & kErrBadAction) && io->actions) {  // gate closed: no env stepped
      cuda_check(cudaMemsetAsync(v->d_error, 0, sizeof e, v->stream), "error reset");
      cuda_check(cudaStreamSynchronize(v->stream), "stream sync");
      fail_bad_action(v, io->actions);
    }
    advance_step(v);
    if (e) v->check_device_errors();
  });
}

mlob_status mlob_venv_env_obs(mlob_venv* v, uint64_t env, double* out, uint64_t cap) {
  return guarded([&] {
    if (env >= v->n_envs) fail(MLOB_E_OUT_OF_RANGE, "env index out of range");
    uint64_t off = 0;
    for (int t = 0; t < v->cfg.n_specs; ++t) {
      const uint64_t cnt = v->cfg.specs[t].count, dim = v->dcfg.specs[t].obs_dim;
      if (off + cnt * dim > cap) fail(MLOB_E_OUT_OF_RANGE, "obs buffer too small");
      cuda_check(cudaMemcpyAsync(out + off, v->d_obs[t] + env * cnt * dim, cnt * dim * 8,
                                 cudaMemcpyDeviceToHost, v->stream), "D2H");
      off += cnt * dim;
    }
    v->check_device_errors();
  });
}

static std::vector<EnvHdr> read_hdrs(mlob_venv* v) {
  std::vector<EnvHdr> h(v->n_envs);
  d2h(v, h.data(), v->d_hdr, v->n_envs);
  return h;
}

mlob_status mlob_venv_episode_stats(mlob_venv* v, int type, mlob_episode_stats* out) {
  return guarded([&] {
    if (type < 0 || type >= v->cfg.n_specs) fail(MLOB_E_OUT_OF_RANGE, "type out of range");
    const uint64_t na = v->n_envs * v->A;
    std::vector<double> t[4];
    for (int i = 0; i < 4; ++i) {
      t[i].resize(na);
      d2h(v, t[i].data(), v->d_t[i], na);
    }
    const auto h = read_hdrs(v);
    std::memset(out, 0, sizeof *out);
    const int cnt = v->cfg.specs[type].count, off = v->dcfg.specs[type].flat_offset;
    for (uint64_t e = 0; e < v->n_envs; ++e) {  // rollout.hpp:255-270, env order
      for (int k = 0; k < cnt; ++k) {
        const uint64_t s = e * v->A + off + k;
        out->pv_sum += t[0][s];
        out->slippage_sum += t[1][s];
        out->completion_sum += t[2][s];
        out->inventory_sq_sum += t[3][s];
      }
      out->episodes += h[e].episodes_finished;
    }
  });
}

mlob_status mlob_venv_episode_stats_device(mlob_venv* v, double* out_device) {
  return guarded([&] {
    v->set_device();
    cuda_check(launch_stats(v->params(), v->dcfg, out_device, v->stream), "stats kernel");
    ++v->launches;
  });
}

// ncclAllReduce from the process's NCCL (the caller's communicator must come
// from the same library): an already-loaded libnccl.so.2 first, else load it.
using NcclAllReduceFn = int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t);
static NcclAllReduceFn nccl_allreduce() {
  static NcclAllReduceFn fn = [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    return h ? reinterpret_cast<NcclAllReduceFn>(dlsym(h, "ncclAllReduce")) : nullptr;
  }();
  return fn;
}
constexpr int kNcclFloat64 = 8, kNcclSum = 0;  // nccl.h ncclDataType_t / ncclRedOp_t

mlob_status mlob_venv_allreduce_episode_stats(mlob_venv* v, void* nccl_comm, mlob_episode_stats* out) {
  return guarded([&] {
    v->set_device();
    const int NT = v->cfg.n_specs;
    double* d = v->alloc_scratch_stats();
    cuda_check(launch_stats(v->params(), v->dcfg, d, v->stream), "stats kernel");
    ++v->launches;
    if (nccl_comm) {
      const NcclAllReduceFn f = nccl_allreduce();
      if (!f) fail(MLOB_E_RUNTIME, "ncclAllReduce not found (libnccl.so.2 not loadable)");
      const int r = f(d, d, static_cast<size_t>(NT) * kStatWords, kNcclFloat64, kNcclSum, nccl_comm, v->stream);
      if (r != 0) fail(MLOB_E_RUNTIME, "ncclAllReduce failed with ncclResult_t " + std::to_string(r));
    }
    std::vector<double> h(static_cast<size_t>(NT) * kStatWords);
    d2h(v, h.data(), d, h.size());
    for (int t = 0; t < NT; ++t) {
      const double* w = h.data() + t * kStatWords;
      mlob_episode_stats& o = out[t];
      std::memset(&o, 0, sizeof o);
      o.pv_sum = w[MLOB_STAT_PV];
      o.slippage_sum = w[MLOB_STAT_SLIPPAGE];
      o.inventory_sq_sum = w[MLOB_STAT_INVENTORY_SQ];
      o.episodes = static_cast<int64_t>(w[MLOB_STAT_EPISODES]);
      const mlob_agent_spec& sp = v->cfg.specs[t];
      o.completion_sum = sp.type == MLOB_EXECUTOR
                             ? w[MLOB_STAT_EPISODES] * sp.count -
                                   w[MLOB_STAT_REMAINING] / static_cast<double>(sp.params.task_size)
                             : 0.0;
    }
  });
}

mlob_status mlob_venv_profile(mlob_venv* v, int on) {
  return guarded([&] {
    v->profiling = on != 0;
    v->prof_steps = 0;
  });
}

mlob_status mlob_venv_kernel_ms(mlob_venv* v, double* out, uint64_t* steps) {
  return guarded([&] {
    v->set_device();
    cuda_check(cudaStreamSynchronize(v->stream), "sync");
    out[0] = out[1] = out[2] = 0.0;
    for (size_t i = 0; i < v->prof_steps; ++i)
      for (int k = 0; k < 3; ++k) {
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, v->prof_ev[4 * i + k], v->prof_ev[4 * i + k + 1]), "elapsed");
        out[k] += ms;
      }
    *steps = v->prof_steps;
  });
}

mlob_status mlob_venv_clear_episode_stats(mlob_venv* v) {
  return guarded([&] {
    v->set_device();
    const uint64_t na = v->n_envs * v->A;
    for (int i = 0; i < 4; ++i)
      cuda_check(cudaMemsetAsync(v->d_t[i], 0, std::max<uint64_t>(na, 1) * 8, v->stream), "memset");
    cuda_check(cudaMemsetAsync(v->d_t_rem, 0, std::max<uint64_t>(na, 1) * 8, v->stream), "memset");
    cuda_check(launch_clear_finished(v->d_hdr, v->n_envs, v->stream), "clear kernel");
    ++v->launches;
  });
}

mlob_status mlob_venv_read_scalars(mlob_venv* v, uint64_t env, mlob_env_scalars* o) {
  return guarded([&] {
    if (env >= v->n_envs) fail(MLOB_E_OUT_OF_RANGE, "env index out of range");
    EnvHdr h;
    d2h(v, &h, v->d_hdr + env, 1);
    std::memset(o, 0, sizeof *o);
    o->step = h.step;
    o->terminal = v->step_ctr < 0 ? 1 : h.terminal;
    o->episode = h.episode;
    o->mid_half = h.mid_half;
    o->prev_mid_half = h.prev_mid_half;
    o->mean_mid_ticks = h.mbar;
    o->last_bid = h.last_bid;
    o->last_ask = h.last_ask;
    o->last_time = h.last_time;
    o->messages_processed = h.msgs_processed;
    o->next_seq = h.next_seq;
    o->live_bid = h.live[0];
    o->live_ask = h.live[1];
  });
}

mlob_status mlob_venv_read_book(mlob_venv* v, uint64_t env, int side, mlob_resting_order* out,
                                uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    if (env >= v->n_envs) fail(MLOB_E_OUT_OF_RANGE, "env index out of range");
    if (side < 0 || side > 1) fail(MLOB_E_INVALID_ARGUMENT, "side must be 0 (bid) or 1 (ask)");
    const uint64_t m = static_cast<uint64_t>(v->spl) * kWarp;
    const uint64_t base = (env * 2 + side) * m;
    std::vector<int32_t> p(m), q(m);
    std::vector<uint2> id(m);
    std::vector<uint32_t> st(m);
    v->set_device();
    cuda_check(cudaMemcpyAsync(p.data(), v->d_bk_p + base, m * 4, cudaMemcpyDeviceToHost, v->stream), "D2H");
    cuda_check(cudaMemcpyAsync(q.data(), v->d_bk_q + base, m * 4, cudaMemcpyDeviceToHost, v->stream), "D2H");
    if (v->spl > 8)  // deep books keep the low id word as a u32 array in the id buffer
      cuda_check(cudaMemcpyAsync(id.data(), reinterpret_cast<const uint32_t*>(v->d_bk_id) + base, m * 4,
                                 cudaMemcpyDeviceToHost, v->stream), "D2H");
    else
      cuda_check(cudaMemcpyAsync(id.data(), v->d_bk_id + base, m * 8, cudaMemcpyDeviceToHost, v->stream), "D2H");
    cuda_check(cudaMemcpyAsync(st.data(), v->d_bk_st + base, m * 4, cudaMemcpyDeviceToHost, v->stream), "D2H");
    EnvHdr h;
    cuda_check(cudaMemcpyAsync(&h, v->d_hdr + env, sizeof h, cudaMemcpyDeviceToHost, v->stream), "D2H");
    v->check_device_errors();
    std::vector<mlob_resting_order> o;
    const bool deep = v->spl > 8;  // 4-word slots: qt = q << 8 | trader, lo, hs = id_hi << 20 | seq
    const uint32_t* lo = reinterpret_cast<const uint32_t*>(id.data());
    for (uint64_t s = 0; s < std::min<uint64_t>(m, h.hwm[side]); ++s) {
      // slot s = row k, lane l; deep books group four rows: (k / 4) * 128 + l * 4 + k % 4
      const uint64_t k = s / kWarp, l = s % kWarp;
      const uint64_t i = deep ? (k >> 2) * 128 + l * 4 + (k & 3) : s;
      const int64_t qi = deep ? static_cast<int64_t>(static_cast<uint32_t>(q[i]) >> 8) : q[i];
      if (qi <= 0) continue;
      mlob_resting_order r;
      std::memset(&r, 0, sizeof r);
      r.price = p[i];
      r.quantity = qi;
      if (deep) {
        r.order_id = (static_cast<uint64_t>(st[i] >> 20) << 32) | lo[i];
        r.arrival_seq = st[i] & 0xfffffu;
        r.trader_id = static_cast<int32_t>(static_cast<uint32_t>(q[i]) & 0xffu);
      } else {
        r.order_id = (static_cast<uint64_t>(id[i].y) << 32) | id[i].x;
        r.arrival_seq = st[i] >> 8;
        r.trader_id = static_cast<int32_t>(st[i] & 0xffu);
      }
      o.push_back(r);
    }
    // storage order of lob::OrderBook (book.hpp:134-143): worst-to-best, newer first at a price
    std::sort(o.begin(), o.end(), [side](const mlob_resting_order& a, const mlob_resting_order& b) {
      if (a.price != b.price) return side == MLOB_BID ? a.price < b.price : a.price > b.price;
      return a.arrival_seq > b.arrival_seq;
    });
    *n_out = o.size();
    for (uint64_t i = 0; i < o.size() && i < cap; ++i) out[i] = o[i];
  });
}

mlob_status mlob_venv_read_agent(mlob_venv* v, uint64_t env, int a, mlob_agent_state* o) {
  return guarded([&] {
    if (env >= v->n_envs || a < 0 || a >= v->A) fail(MLOB_E_OUT_OF_RANGE, "env/agent index out of range");
    AgentRec r;
    ActiveRec act[kMaxActive];
    v->set_device();
    cuda_check(cudaMemcpyAsync(&r, v->d_agents + env * v->A + a, sizeof r, cudaMemcpyDeviceToHost, v->stream),
               "D2H");
    cuda_check(cudaMemcpyAsync(act, v->d_active + (env * v->A + a) * kMaxActive, sizeof act,
                               cudaMemcpyDeviceToHost, v->stream), "D2H");
    v->check_device_errors();
    std::memset(o, 0, sizeof *o);
    o->inventory = r.inventory;
    o->cash = r.cash;
    o->task_remaining = r.task_remaining;
    o->task_dir = r.task_dir;
    o->p_init = r.p_init;
    o->order_nonce = r.nonce;
    o->filled_total = r.filled_total;
    o->slippage_total = r.slippage_total;
    o->n_active = r.n_active;
    for (int i = 0; i < r.n_active && i < kMaxActive; ++i) {
      o->active[i].order_id = act[i].order_id;
      o->active[i].price = act[i].price;
      o->active[i].quantity = static_cast<int64_t>(act[i].qty_side & 0x7fffffffu);
      o->active[i].side = static_cast<uint8_t>(act[i].qty_side >> 31);
    }
  });
}

mlob_status mlob_venv_read_trades(mlob_venv* v, uint64_t env, mlob_trade* out, uint64_t cap, uint64_t* n_out) {
  return guarded([&] {
    if (env >= v->n_envs) fail(MLOB_E_OUT_OF_RANGE, "env index out of range");
    EnvHdr h;
    d2h(v, &h, v->d_hdr + env, 1);
    if (!(v->flags & MLOB_VENV_RECORD_TRADES)) fail(MLOB_E_LOGIC, "trade log disabled (MLOB_VENV_RECORD_TRADES)");
    *n_out = h.n_trades;
    if (h.n_trades > v->trade_cap)
      fail(MLOB_E_RUNTIME, "trade log overflow: " + std::to_string(h.n_trades) + " trades > capacity " +
                               std::to_string(v->trade_cap));
    const uint64_t n = std::min<uint64_t>(h.n_trades, cap);
    if (n) d2h(v, out, v->d_trades + env * v->trade_cap, n);
  });
}

mlob_status mlob_venv_messages_processed(mlob_venv* v, uint64_t* out) {
  return guarded([&] {
    v->set_device();
    cuda_check(cudaMemsetAsync(v->d_scratch, 0, 8, v->stream), "memset");
    cuda_check(launch_sum_msgs(v->d_hdr, v->n_envs, v->d_scratch, v->stream), "sum kernel");
    ++v->launches;
    unsigned long long s = 0;
    d2h(v, &s, v->d_scratch, 1);
    *out = s;
  });
}

}  // extern "C"
