// mlob_kernels.cu — sm_100a kernels of the batched LOB environment step.
//
// One environment step (MarketEnv::step, env.hpp:194-254, for every env) is
// three launches on the handle's stream:
//   act_kernel     one THREAD per env  (mlob_thread.cuh): actions -> agent
//                  messages, shuffled (env.hpp:205-215)
//   book_kernel    one WARP per env    (mlob_step.cuh): agent + replay messages
//                  through the env's book (env.hpp:217-240), fill log, active
//                  orders, L2 summary
//   outcome_kernel one THREAD per env  (mlob_thread.cuh): fills -> agent
//                  accounting, rewards, infos, observations, episode stats,
//                  auto-reset (env.hpp:242-253, rollout.hpp:290-318)
// plus K3 reset_kernel (thread per env), K4 stats_kernel (episode-stat sums
// for the all-reduce) and the host launchers.
// Compiled with --fmad=false (bit-exact double rounding).
#include "mlob_thread.cuh"

namespace mlob {

__host__ __device__ inline size_t book_smem_bytes(int capacity) {
  return static_cast<size_t>(2) * 4 * spl_of(capacity) * kWarp * sizeof(uint32_t);  // SmemSide: 4 words a slot
}
// agent-message hand-off slots per env: every active order of every agent
// may be deleted and two quotes placed (env.hpp:338-369); the same smem
// region holds rebuild_active's scratch (<= kMaxActive orders per agent)
__host__ __device__ inline uint32_t amsg_cap_of(int n_agents) {
  return static_cast<uint32_t>(n_agents * (kMaxActive + 2) + 4);
}
__host__ __device__ inline bool smem_book(int capacity) { return capacity > 8 * kWarp; }

__host__ __device__ inline size_t warp_smem_bytes(const DevCfg& c) {
  const int chunk = c.mps < kChunk ? c.mps : kChunk;
  const int nbuf = c.mps > kChunk ? 2 : 1;
  size_t b = 0;
  b += static_cast<size_t>(nbuf) * chunk * sizeof(DevMsg);
  b += 32;  // 3 mbarriers
  b += static_cast<size_t>(amsg_cap_of(c.n_agents)) * sizeof(DevMsg);
  b += static_cast<size_t>(c.n_agents) * kMaxActive * sizeof(ActiveRec);
  b += static_cast<size_t>((c.n_agents + 3) / 4) * 16;  // active counts
  b += 32;  // scalars (WarpSmem::scal: mid anchor / segment base, Σmid)
  b += static_cast<size_t>(2 * c.obs_depth) * sizeof(L2Lvl);
  b = (b + 15) / 16 * 16;
  if (MLOB_PREFIX_WALK && !smem_book(c.capacity))  // register books: the price-level walk's scratch
    b += static_cast<size_t>(spl_of(c.capacity)) * kWarp * sizeof(WalkEnt);
  if (smem_book(c.capacity)) b += book_smem_bytes(c.capacity);
  return (b + 127) / 128 * 128;
}

// Per-warp region offsets (identical for every warp of a block): written by
// thread 0 before stage_params' block barrier.
__device__ void carve_block(const DevCfg& c) {
  const int chunk = c.mps < kChunk ? c.mps : kChunk;
  const int nbuf = c.mps > kChunk ? 2 : 1;
  uint32_t p = 0;
  SmemOff& o = g_smem_off;
  o.chunk0 = p;
  o.chunk1 = nbuf == 2 ? p + static_cast<uint32_t>(chunk * sizeof(DevMsg)) : p;
  p += static_cast<uint32_t>(nbuf * chunk * sizeof(DevMsg));
  o.bar = p;
  p += 32;
  o.amsg = p;
  p += static_cast<uint32_t>(amsg_cap_of(c.n_agents) * sizeof(DevMsg));
  o.act = p;
  p += static_cast<uint32_t>(c.n_agents * kMaxActive * sizeof(ActiveRec));
  o.nact = p;
  p += static_cast<uint32_t>((c.n_agents + 3) / 4 * 16);
  o.scal = p;
  p += 32;
  o.l2 = p;
  p += static_cast<uint32_t>(2 * c.obs_depth * sizeof(L2Lvl));
  p = (p + 15) / 16 * 16;
  o.walk = p;
}

// deep-book smem region of a warp (after the WarpSmem carve-out)
__device__ inline uint32_t* book_region(char* base, const DevCfg& c) {
  size_t b = warp_smem_bytes(c) - (smem_book(c.capacity) ? book_smem_bytes(c.capacity) : 0);
  b = b / 16 * 16;
  return reinterpret_cast<uint32_t*>(base + b);
}

// Register-book book_kernel blocks: one persistent block per SM walks the
// envs in rounds (no block barrier between rounds: measured -3 % once the step
// was split).  Shared-memory (deep) books: blocks of as many warps as the
// shared memory holds, one env per warp.
// warps per register-book block and the register budget they leave: C <= 128
// (SPL <= 4) 28 warps x 72 registers (+2.4 % on C over 24 x 80, after the
// header fields left the loop's registers); SPL = 8 keeps 80 book registers,
// so 16 warps x 128
#ifndef MLOB_SYNC_WARPS
#define MLOB_SYNC_WARPS 28
#endif
#ifndef MLOB_SYNC_REGS
#define MLOB_SYNC_REGS 72
#endif
// WAVES (register books, C <= 128, large batches): one env per warp in
// 7-warp blocks over a full grid, so the block scheduler backfills SMs as
// blocks finish (E +3.5 %, C +3.2 % over the persistent rounds, whose static
// env lists end on their slowest warp); small batches (under kWavesMinEnvs)
// keep the persistent grid with balanced rounds (B -5 % otherwise).
constexpr int kWaveWarps = 7;
constexpr uint64_t kWavesMinEnvs = 16384;
template <int SPL, bool WAVES>
__host__ __device__ constexpr bool rounds_of() {
  return SPL <= 8 && !WAVES;
}
template <int SPL, bool WAVES>
__host__ __device__ constexpr int warps_per_block() {
  return WAVES ? kWaveWarps : !rounds_of<SPL, WAVES>() ? 8 : SPL <= 4 ? MLOB_SYNC_WARPS : 16;
}
template <int SPL, bool WAVES>
__host__ __device__ constexpr int min_blocks() {
  return WAVES ? 65536 / (MLOB_SYNC_REGS * 32 * kWaveWarps)
         : rounds_of<SPL, WAVES>() && SPL <= 4 && 65536 / (MLOB_SYNC_REGS * 32 * MLOB_SYNC_WARPS) > 0
             ? 65536 / (MLOB_SYNC_REGS * 32 * MLOB_SYNC_WARPS)
             : 1;
}
constexpr int kThreadBlock = 128;  // thread-per-env kernels

// Kernel parameters and the env config staged into shared memory once per
// block (reads through the __grid_constant__ parameter compiled to slow
// generic loads).
struct StagedParams {
  KParams kp;
  DevCfg cfg;
};
template <bool CARVE>
__device__ __forceinline__ void stage_params(StagedParams& sp, const KParams& kp) {
  const int4* a = reinterpret_cast<const int4*>(&kp);
  int4* d = reinterpret_cast<int4*>(&sp.kp);
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(KParams) / 16); i += blockDim.x) d[i] = a[i];
  const int n_specs = kp.cfg->n_specs;
  const int bytes = static_cast<int>(offsetof(DevCfg, specs) + n_specs * sizeof(DevSpec));
  const int4* c = reinterpret_cast<const int4*>(kp.cfg);
  int4* dc = reinterpret_cast<int4*>(&sp.cfg);
  for (int i = threadIdx.x; i < (bytes + 15) / 16; i += blockDim.x) dc[i] = c[i];
  if constexpr (CARVE) {
    if (threadIdx.x == 0) carve_block(*kp.cfg);
  }
  __syncthreads();
}
static_assert(sizeof(KParams) % 16 == 0, "KParams must be int4-copyable");
// Deep-book blocks stage the parameters at the front of the dynamic shared
// memory with only the config's n_specs agent specs (a static StagedParams
// reserves all kMaxSpecs): that is what lets a fifth 45 KB warp fit at C = 1000.
__host__ __device__ inline size_t staged_dyn_bytes(int n_specs) {
  const size_t b = offsetof(StagedParams, cfg) + offsetof(DevCfg, specs) + static_cast<size_t>(n_specs) * sizeof(DevSpec);
  return (b + 127) / 128 * 128;
}

// ---------------------------------------------------------------------------
// act_kernel: MarketEnv::step stages (1)+(2), thread per env.
__global__ void __launch_bounds__(kThreadBlock) act_kernel(const __grid_constant__ KParams kparam) {
  __shared__ __align__(16) StagedParams sp;
  stage_params<false>(sp, kparam);
  const KParams& kp = sp.kp;
  if (blockIdx.x == 0 && threadIdx.x == 0 && kp.fill_pool_ctr) *kp.fill_pool_ctr = 0;
  if (kp.gate && *kp.gate) return;  // the batch's actions were rejected: no env steps
  const uint64_t env = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (env >= kp.n_envs) return;
  ThreadEnv t(kp, sp.cfg, env);
  t.actions();
  t.report_errors();
}

// outcome_kernel: stage (5) + MarketVecEnv::step_one's caches and auto-reset.
__global__ void __launch_bounds__(kThreadBlock) outcome_kernel(const __grid_constant__ KParams kparam) {
  __shared__ __align__(16) StagedParams sp;
  stage_params<false>(sp, kparam);
  const KParams& kp = sp.kp;
  if (kp.gate && *kp.gate) return;
  const uint64_t env = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (env >= kp.n_envs) return;
  ThreadEnv t(kp, sp.cfg, env);
  t.outcomes();
  t.report_errors();
}

// K3: MarketEnv::reset for every env (reset_all / reset_envs).
__global__ void __launch_bounds__(kThreadBlock) reset_kernel(const __grid_constant__ KParams kparam) {
  __shared__ __align__(16) StagedParams sp;
  stage_params<false>(sp, kparam);
  const KParams& kp = sp.kp;
  const uint64_t env = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (env >= kp.n_envs) return;
  ThreadEnv t(kp, sp.cfg, env);
  t.reset_env();
  t.report_errors();
}

// book_kernel: stages (3)+(4) of the step, one warp per env.  Register books
// (C <= 256): a grid of one persistent block per SM walks the envs in
// rounds (env = first + r * stride), the next round's first replay chunk
// staged while the current env finishes.  Deep books: one env per warp.
// REC: the trade log is on (MLOB_VENV_RECORD_TRADES) — a separate
// instantiation, so the fill loop of the plain step carries no log flag
template <int SPL, bool REC, bool WAVES>
__global__ void __launch_bounds__(warps_per_block<SPL, WAVES>() * kWarp, min_blocks<SPL, WAVES>())
    book_kernel(const __grid_constant__ KParams kparam) {
  const int kWarps = static_cast<int>(blockDim.x) / kWarp;
  extern __shared__ __align__(128) char dsmem[];
  StagedParams* spp;
  char* smem = dsmem;  // the warps' regions
  if constexpr (SPL <= 8) {
    __shared__ __align__(16) StagedParams sp_static;
    spp = &sp_static;
  } else {
    spp = reinterpret_cast<StagedParams*>(dsmem);
    smem = dsmem + staged_dyn_bytes(kparam.cfg->n_specs);
  }
  StagedParams& sp_ = *spp;
  stage_params<true>(sp_, kparam);
  const KParams& kp = sp_.kp;
  if (kp.gate && *kp.gate) return;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWarps;
  const uint64_t first = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
  constexpr bool rounds = rounds_of<SPL, WAVES>();
  bool idle = first >= kp.n_envs;
  if (idle && !rounds) return;  // rounds: an idle warp skips every round below
  const DevCfg& cfg = sp_.cfg;
  char* wbase = smem + warp * warp_smem_bytes(cfg);
  WarpSmem sm{wbase};
  WarpEnv<SPL, REC> w(kp, cfg, sm, idle ? 0 : first, lane, book_region(wbase, cfg));
  const int mps = cfg.mps;
  const int nch = (mps + kChunk - 1) / kChunk;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.bar()[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.bar()[1])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sm.bar()[2])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const auto slice_of = [&](uint64_t e) {
    const EnvHdr& h = kp.hdr[e];
    return kp.msgs + kp.ep_start[h.episode] + static_cast<uint64_t>(h.step) * mps;
  };
  if (!idle && mps > 0) w.stage(slice_of(first), min(kChunk, mps));
  const uint64_t n_rounds = rounds ? (kp.n_envs + stride - 1) / stride : 1;
  uint64_t nenv = rounds ? first + stride : kp.n_envs;
  for (uint64_t env = first, round = 0; round < n_rounds; ++round) {
    if (!idle) {
      const bool has_next = nenv < kp.n_envs;
      w.bind(env);
      const DevMsg* slice = slice_of(env);
      w.load_hdr();
      w.book_load_issue();  // shared-memory books: bulk loads in flight from here
      if (nch >= 2) w.stage(slice + kChunk, min(kChunk, mps - kChunk));
      const DevMsg* next_slice = has_next && mps > 0 ? slice_of(nenv) : nullptr;
      w.load_agent_msgs();
      w.book_load_wait();
      // (3) + (4): agent messages, then the replay slice
      w.n_trades = 0;
      w.n_fills = 0;
      w.fill_head = kNoChunk;
      w.process_messages(w.n_amsg, slice);
      if (next_slice) w.stage(next_slice, min(kChunk, mps));  // overlaps the step's tail
      // (5), book-dependent part
      w.rebuild_active();
      w.snapshot();
      w.store_book();
      w.store_hdr(slice);
    }
    env = nenv;
    nenv = env + stride;
    idle = env >= kp.n_envs;
  }
  w.book_store_drain();
  w.report_errors();
}

// K4: per-type episode-stat sums over this handle's envs (for the
// all-reduce), kStatWords doubles per type: pv, slippage, completion (env
// order is not kept: atomics), inventory², episodes, Σ task_remaining of the
// finished executor episodes.  PV, slippage and inventory² are multiples of
// 0.5 and Σ remaining is an integer, so those sums are exact in any order;
// the exact completion is episodes·count − Σremaining / task_size.
__global__ void stats_kernel(const __grid_constant__ KParams kp, double* out) {
  const int t = blockIdx.y;
  const DevCfg& cfg = *kp.cfg;
  const int A = cfg.n_agents;
  const int cnt = cfg.specs[t].count, off = cfg.specs[t].flat_offset;
  double s[kStatWords] = {0, 0, 0, 0, 0, 0};
  for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < kp.n_envs;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    for (int k = 0; k < cnt; ++k) {
      const size_t slot = e * A + off + k;
      s[0] += kp.t_pv[slot];
      s[1] += kp.t_slip[slot];
      s[2] += kp.t_comp[slot];
      s[3] += kp.t_inv[slot];
      s[5] += static_cast<double>(kp.t_rem[slot]);
    }
    s[4] += static_cast<double>(kp.hdr[e].episodes_finished);
  }
#pragma unroll
  for (int i = 0; i < kStatWords; ++i) {
    double v = s[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULLMASK, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&out[t * kStatWords + i], v);
  }
}

__global__ void sum_msgs_kernel(const EnvHdr* hdr, uint64_t n, unsigned long long* out) {
  unsigned long long s = 0;
  for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    s += hdr[e].msgs_processed;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(FULLMASK, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// actions.hpp:69-70 range check of a whole batch of action ids on the device;
// any failure sets kErrBadAction and closes the gate of the following step.
__global__ void validate_actions_kernel(const int32_t* ids, uint64_t n, const DevCfg* cfg, uint32_t* error,
                                        uint32_t* gate) {
  __shared__ uint32_t ar[MLOB_MAX_AGENTS];
  const int A = cfg->n_agents;
  if (threadIdx.x < A) ar[threadIdx.x] = static_cast<uint32_t>(cfg->specs[cfg->flat_spec[threadIdx.x]].arity);
  __syncthreads();
  bool bad = false;
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    bad |= static_cast<uint32_t>(ids[i]) >= ar[i % A];
  if (__any_sync(FULLMASK, bad) && (threadIdx.x & 31) == 0) {
    atomicOr(error, static_cast<uint32_t>(kErrBadAction));
    *gate = 1;
  }
}

// per-stream reset flags of one type: resets[e * count + k] = just_reset[e]
__global__ void expand_resets_kernel(const uint8_t* just_reset, uint64_t n_envs, int count, uint8_t* out) {
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_envs * count;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = just_reset[i / count];
}

__global__ void clear_finished_kernel(EnvHdr* hdr, uint64_t n) {
  for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    hdr[e].episodes_finished = 0;
}

// ---------------------------------------------------------------------------
// host-side launchers

static bool deep_book(const DevCfg& c) { return spl_of(c.capacity) > 8; }
static size_t book_staged_bytes(const DevCfg& c) {  // dynamic-smem prefix (deep books)
  return deep_book(c) ? staged_dyn_bytes(c.n_specs) : 0;
}
// warps per book_kernel block: the round width for register books, as many
// as the shared memory holds for deep books (<= 8)
static int book_warps(const DevCfg& c, bool waves) {
  const bool deep = deep_book(c);
  const int spl = spl_of(c.capacity);
  // deep books: 3-warp blocks, two per SM (finer backfill than one 6-warp
  // block: D +1.5 %; one-warp blocks fit only five per SM: -13 %)
  const int want = waves ? kWaveWarps : deep ? 3 : spl <= 4 ? MLOB_SYNC_WARPS : 16;
  const size_t per = warp_smem_bytes(c);
  const size_t limit = deep ? 227 * 1024 - sizeof(SmemOff) - book_staged_bytes(c) - 256
                            : 227 * 1024 - sizeof(StagedParams) - sizeof(SmemOff) - 1024;
  const int fit = static_cast<int>(limit / (per > 0 ? per : 1));
  return fit < 1 ? 1 : (fit < want ? fit : want);
}

size_t step_min_smem_bytes(const DevCfg& c) {  // book_kernel smem of a one-warp block (feasibility)
  return book_staged_bytes(c) + warp_smem_bytes(c);
}
uint32_t step_amsg_cap(const DevCfg& c) { return amsg_cap_of(c.n_agents); }
int step_launches() { return 3; }

static unsigned grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 1184 ? (b > 0 ? b : 1) : 1184);
}
// thread-per-env kernels: 128-thread blocks; small batches in narrower blocks
// so that they spread over every SM (the kernels are latency-bound per env;
// +0.5 % on B, +0.3 % on C)
static int thread_block(uint64_t n) {
  return n >= 148ull * 4 * 128 ? kThreadBlock : n >= 148ull * 4 * 64 ? 64 : 32;
}
static unsigned thread_grid(uint64_t n) {
  const uint64_t b = static_cast<uint64_t>(thread_block(n));
  return static_cast<unsigned>((n + b - 1) / b);
}

template <int SPL, bool REC, bool WAVES>
static cudaError_t launch_book_t(const KParams& kp, const DevCfg& cfg, cudaStream_t s) {
  int warps = book_warps(cfg, WAVES);
  const size_t staged = book_staged_bytes(cfg);
  const size_t full_sm = staged + warp_smem_bytes(cfg) * warps;
  // the dynamic-smem opt-in only grows (a per-process cache per instantiation:
  // small launches are host-bound, so no attribute call per launch)
  static size_t sm_set[64] = {};
  static int n_sm_of[64] = {}, per_sm_of[64] = {};
  int cur_dev = 0;
  cudaError_t e = cudaGetDevice(&cur_dev);
  if (e != cudaSuccess) return e;
  size_t& done = sm_set[cur_dev & 63];
  if (full_sm > done) {
    e = cudaFuncSetAttribute(book_kernel<SPL, REC, WAVES>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(full_sm));
    if (e != cudaSuccess) return e;
    done = full_sm;
    per_sm_of[cur_dev & 63] = 0;  // re-query the occupancy for the new block size
  }
  uint64_t blocks = (kp.n_envs + warps - 1) / warps;
  if (rounds_of<SPL, WAVES>()) {
    // persistent grid: every SM filled to its occupancy limit (cached per device)
    int& n_sm = n_sm_of[cur_dev & 63];
    int& per_sm = per_sm_of[cur_dev & 63];
    if (n_sm == 0 && (e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, cur_dev)) != cudaSuccess)
      return e;
    if (per_sm == 0) {
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, book_kernel<SPL, REC, WAVES>, warps * kWarp, full_sm)) !=
          cudaSuccess)
        return e;
      if (per_sm < 1) per_sm = 1;
    }
    const uint64_t cap = static_cast<uint64_t>(n_sm) * static_cast<uint64_t>(per_sm);
    // balanced rounds: the fewest rounds at full width, then the narrowest
    // block that still covers the envs in that many rounds
    const uint64_t per_round = cap * static_cast<uint64_t>(warps);
    const uint64_t rounds = (kp.n_envs + per_round - 1) / per_round;
    const uint64_t w = (kp.n_envs + cap * rounds - 1) / (cap * rounds);
    warps = static_cast<int>(w < static_cast<uint64_t>(warps) ? (w > 0 ? w : 1) : warps);
    const uint64_t need = (kp.n_envs + warps - 1) / warps;
    blocks = need < cap ? need : cap;
  }
  const size_t sm = staged + warp_smem_bytes(cfg) * warps;
  book_kernel<SPL, REC, WAVES><<<static_cast<unsigned>(blocks), warps * kWarp, sm, s>>>(kp);
  return cudaGetLastError();
}

template <bool REC>
static cudaError_t launch_book_r(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s) {
  const bool waves = kp.n_envs >= kWavesMinEnvs;
  switch (spl) {
    case 1: return waves ? launch_book_t<1, REC, true>(kp, cfg, s) : launch_book_t<1, REC, false>(kp, cfg, s);
    case 2: return waves ? launch_book_t<2, REC, true>(kp, cfg, s) : launch_book_t<2, REC, false>(kp, cfg, s);
    case 4: return waves ? launch_book_t<4, REC, true>(kp, cfg, s) : launch_book_t<4, REC, false>(kp, cfg, s);
    case 8: return launch_book_t<8, REC, false>(kp, cfg, s);
    case 16: return launch_book_t<16, REC, false>(kp, cfg, s);
    case 32: return launch_book_t<32, REC, false>(kp, cfg, s);
  }
  return cudaErrorInvalidValue;
}
static cudaError_t launch_book(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s) {
  return (kp.flags & MLOB_VENV_RECORD_TRADES) ? launch_book_r<true>(kp, cfg, spl, s)
                                              : launch_book_r<false>(kp, cfg, spl, s);
}

int slots_per_lane(int capacity) { return spl_of(capacity); }

// ev: optional 4 events recorded around the three kernels (per-kernel timing)
cudaError_t launch_step(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s, cudaEvent_t* ev) {
  cudaError_t e;
  if (ev && (e = cudaEventRecord(ev[0], s)) != cudaSuccess) return e;
  act_kernel<<<thread_grid(kp.n_envs), thread_block(kp.n_envs), 0, s>>>(kp);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (ev && (e = cudaEventRecord(ev[1], s)) != cudaSuccess) return e;
  if ((e = launch_book(kp, cfg, spl, s)) != cudaSuccess) return e;
  if (ev && (e = cudaEventRecord(ev[2], s)) != cudaSuccess) return e;
  outcome_kernel<<<thread_grid(kp.n_envs), thread_block(kp.n_envs), 0, s>>>(kp);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (ev && (e = cudaEventRecord(ev[3], s)) != cudaSuccess) return e;
  return cudaSuccess;
}

cudaError_t launch_reset(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s) {
  (void)cfg;
  (void)spl;
  reset_kernel<<<thread_grid(kp.n_envs), thread_block(kp.n_envs), 0, s>>>(kp);
  return cudaGetLastError();
}

cudaError_t launch_stats(const KParams& kp, const DevCfg& cfg, double* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * kStatWords * cfg.n_specs, s);
  if (e != cudaSuccess) return e;
  stats_kernel<<<dim3(grid_for(kp.n_envs), cfg.n_specs), 256, 0, s>>>(kp, out);
  return cudaGetLastError();
}

cudaError_t launch_validate_actions(const int32_t* ids, uint64_t n, const DevCfg* cfg, uint32_t* error,
                                    uint32_t* gate, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(gate, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return e;
  validate_actions_kernel<<<grid_for(n), 256, 0, s>>>(ids, n, cfg, error, gate);
  return cudaGetLastError();
}

cudaError_t launch_expand_resets(const uint8_t* just_reset, uint64_t n_envs, int count, uint8_t* out,
                                 cudaStream_t s) {
  expand_resets_kernel<<<grid_for(n_envs * count), 256, 0, s>>>(just_reset, n_envs, count, out);
  return cudaGetLastError();
}

cudaError_t launch_sum_msgs(const EnvHdr* hdr, uint64_t n, unsigned long long* out, cudaStream_t s) {
  sum_msgs_kernel<<<grid_for(n), 256, 0, s>>>(hdr, n, out);
  return cudaGetLastError();
}

cudaError_t launch_clear_finished(EnvHdr* hdr, uint64_t n, cudaStream_t s) {
  clear_finished_kernel<<<grid_for(n), 256, 0, s>>>(hdr, n);
  return cudaGetLastError();
}

}  // namespace mlob
