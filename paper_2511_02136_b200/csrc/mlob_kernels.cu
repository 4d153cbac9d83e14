// mlob_kernels.cu — sm_100a kernels of the batched LOB environment step:
// K1+K2 step_kernel (one warp per env, mlob_step.cuh), K3 reset_kernel,
// K4 stats_kernel (episode-stat sums for the NCCL all-reduce) and host
// launchers.  Compiled with --fmad=false (bit-exact double rounding).
#include "mlob_step.cuh"

namespace mlob {

__host__ __device__ inline int spl_of(int capacity) {
  const int need = (capacity + kWarp - 1) / kWarp;
  return need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : need <= 16 ? 16 : need <= 32 ? 32 : -1;
}
__host__ __device__ inline size_t book_smem_bytes(int capacity) {
  return static_cast<size_t>(2) * 5 * spl_of(capacity) * kWarp * sizeof(uint32_t);
}

__host__ __device__ inline size_t warp_smem_bytes(const DevCfg& c) {
  const int chunk = c.mps < kChunk ? c.mps : kChunk;
  const int nbuf = c.mps > kChunk ? 2 : 1;
  size_t b = 0;
  b += static_cast<size_t>(nbuf) * chunk * sizeof(DevMsg);
  b += 32;  // 3 mbarriers
  b += static_cast<size_t>(4 * c.n_agents + 4) * sizeof(DevMsg);
  b += static_cast<size_t>(c.n_agents) * sizeof(AgentRec);
  b += static_cast<size_t>(c.n_agents) * kMaxActive * sizeof(ActiveRec);
  b += static_cast<size_t>(c.n_agents) * sizeof(StepAcc);
  b += kFillLog * sizeof(FillEnt);
  b += 32;  // scalars (WarpSmem::scal: fill-log count / overflow, mid anchor / segment base, Σmid)
  b += static_cast<size_t>(2 * c.obs_depth) * sizeof(L2Lvl);
  b += static_cast<size_t>(c.max_obs_dim + 1) * sizeof(double);
  b = (b + 15) / 16 * 16;
  if (c.capacity > 8 * kWarp || MLOB_SMEM_BOOK) b += book_smem_bytes(c.capacity);  // smem book
  return (b + 127) / 128 * 128;
}

__device__ WarpSmem carve(char* base, const DevCfg& c) {
  // every warp writes the same offsets; the warp's own writes are visible to
  // it after the __syncwarp, other warps' writes carry identical values
  const int chunk = c.mps < kChunk ? c.mps : kChunk;
  const int nbuf = c.mps > kChunk ? 2 : 1;
  if ((threadIdx.x & 31) == 0) {
    uint32_t p = 0;
    SmemOff& o = g_smem_off;
    o.chunk0 = p;
    o.chunk1 = nbuf == 2 ? p + static_cast<uint32_t>(chunk * sizeof(DevMsg)) : p;
    p += static_cast<uint32_t>(nbuf * chunk * sizeof(DevMsg));
    o.bar = p;
    p += 32;
    o.amsg = p;
    p += static_cast<uint32_t>((4 * c.n_agents + 4) * sizeof(DevMsg));
    o.ag = p;
    p += static_cast<uint32_t>(c.n_agents * sizeof(AgentRec));
    o.act = p;
    p += static_cast<uint32_t>(c.n_agents * kMaxActive * sizeof(ActiveRec));
    o.acc = p;
    p += static_cast<uint32_t>(c.n_agents * sizeof(StepAcc));
    o.fills = p;
    p += static_cast<uint32_t>(kFillLog * sizeof(FillEnt));
    o.scal = p;
    p += 32;
    o.l2 = p;
    p += static_cast<uint32_t>(2 * c.obs_depth * sizeof(L2Lvl));
    o.obs = p;
  }
  __syncwarp();
  WarpSmem s;
  s.base = base;
  return s;
}

// deep-book smem region of a warp (after the WarpSmem carve-out)
__device__ inline uint32_t* book_region(char* base, const DevCfg& c) {
  size_t b = warp_smem_bytes(c) - ((c.capacity > 8 * kWarp || MLOB_SMEM_BOOK) ? book_smem_bytes(c.capacity) : 0);
  b = b / 16 * 16;
  return reinterpret_cast<uint32_t*>(base + b);
}

// Register-book kernels run one block of kSyncWarps warps per SM with block
// barriers between the step phases, so all warps of an SM execute the same
// phase's code at the same time: the unsynchronised kernel was front-end
// (instruction-cache) bound with warps spread over ~9.5k instructions
// (profiles/r1_*).  Deep (smem) books keep 4-warp blocks.
#ifndef MLOB_PHASE_SYNC
#define MLOB_PHASE_SYNC 1
#endif
#ifndef MLOB_SYNC_WARPS
#define MLOB_SYNC_WARPS 24
#endif
#ifndef MLOB_SYNC_A  // barrier before the message loop (measured: no gain)
#define MLOB_SYNC_A 0
#endif
#ifndef MLOB_SYNC_B  // barrier after the message loop
#define MLOB_SYNC_B 1
#endif
#ifndef MLOB_DEEP_SYNC  // phase barriers for the deep (smem) book too
#define MLOB_DEEP_SYNC 0
#endif
#ifndef MLOB_SYNC_REGS
#define MLOB_SYNC_REGS 80
#endif
template <int SPL>
__host__ __device__ constexpr bool phase_sync() {
  return MLOB_PHASE_SYNC && (SPL <= 8 || MLOB_DEEP_SYNC);
}
template <int SPL>
__host__ __device__ constexpr int warps_per_block() {
  // deep books: as many warps as the shared memory holds (5 at C = 1000), <= 8
  return (phase_sync<SPL>() && SPL <= 8) ? MLOB_SYNC_WARPS : (SPL > 8 ? 8 : 4);
}
template <int SPL>
__host__ __device__ constexpr int min_blocks() {
  // blocks per SM for the register budget MLOB_SYNC_REGS (65536 regs / SM)
  return (phase_sync<SPL>() && SPL <= 8) ? (65536 / (MLOB_SYNC_REGS * 32 * MLOB_SYNC_WARPS) > 0
                                  ? 65536 / (MLOB_SYNC_REGS * 32 * MLOB_SYNC_WARPS)
                                  : 1)
                           : (SPL > 8 ? 1 : 4);
}
constexpr int kWarpsPerBlock = 4;  // reset kernel

#ifdef MLOB_PHASE_TIMING
#define PHASE(i)                                                               \
  do {                                                                         \
    __syncwarp();                                                              \
    if (lane == 0 && kp.timing) kp.timing[env * 16 + (i)] = clock64();         \
  } while (0)
#else
#define PHASE(i) \
  do {           \
  } while (0)
#endif

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// K1+K2: persistent warps, one environment step per warp per iteration
// (MarketEnv::step, env.hpp:194-254, + MarketVecEnv::step_one auto-reset,
// rollout.hpp:290-318).  While env e is processed, the next env's first
// replay chunk is already in flight (cp.async.bulk) and its header, agent
// records and book rows are prefetched into L2.
// Kernel parameters and the env config are staged into shared memory once
// per block: reading them through a reference to the __grid_constant__
// parameter compiled to slow generic loads (profiles/r1 phase timing).
struct StagedParams {
  KParams kp;
  DevCfg cfg;
};
__device__ __forceinline__ void stage_params(StagedParams& sp, const KParams& kp) {
  const int4* a = reinterpret_cast<const int4*>(&kp);
  int4* d = reinterpret_cast<int4*>(&sp.kp);
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(KParams) / 16); i += blockDim.x) d[i] = a[i];
  const int n_specs = kp.cfg->n_specs;
  const int bytes = static_cast<int>(offsetof(DevCfg, specs) + n_specs * sizeof(DevSpec));
  const int4* c = reinterpret_cast<const int4*>(kp.cfg);
  int4* dc = reinterpret_cast<int4*>(&sp.cfg);
  for (int i = threadIdx.x; i < (bytes + 15) / 16; i += blockDim.x) dc[i] = c[i];
  __syncthreads();
}
static_assert(sizeof(KParams) % 16 == 0, "KParams must be int4-copyable");
// Deep-book step blocks stage the parameters at the front of the dynamic
// shared memory with only the config's n_specs agent specs (a static
// StagedParams reserves all kMaxSpecs = 5.2 KB): that is what lets a fifth
// 45 KB warp fit in the 227 KB block at C = 1000.
__host__ __device__ inline size_t staged_dyn_bytes(int n_specs) {
  const size_t b = offsetof(StagedParams, cfg) + offsetof(DevCfg, specs) + static_cast<size_t>(n_specs) * sizeof(DevSpec);
  return (b + 127) / 128 * 128;
}

template <int SPL>
__global__ void __launch_bounds__(warps_per_block<SPL>() * kWarp, min_blocks<SPL>())
    step_kernel(const __grid_constant__ KParams kparam) {
  // warps per block: warps_per_block<SPL>() unless the config's shared memory
  // per warp needs a smaller block (step_warps)
  const int kWarpsPerBlock = static_cast<int>(blockDim.x) / kWarp;
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
  stage_params(sp_, kparam);
  const KParams& kp = sp_.kp;
  if (kp.gate && *kp.gate) return;  // the batch's actions were rejected: no env steps
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWarpsPerBlock;
  // dynamic work distribution (MLOB_PERSIST): the first env of each warp is
  // static, later ones come from a global ticket counter fetched one env ahead
  // so the next env's data can be prefetched; kp.ticket is zeroed per launch.
  const uint64_t first = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + warp;
  // phase-sync builds keep idle warps alive for the block barriers
  bool idle = first >= kp.n_envs;
  if (idle && !phase_sync<SPL>()) return;
  const auto ticket = [&]() -> uint64_t {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(kp.ticket, 1ull);
    return stride + __shfl_sync(FULLMASK, t, 0);
  };
  const DevCfg& cfg = sp_.cfg;
  char* wbase = smem + warp * warp_smem_bytes(cfg);
  WarpSmem sm = carve(wbase, cfg);
  WarpEnv<SPL> w(kp, cfg, sm, idle ? 0 : first, lane, book_region(wbase, cfg));
  const int mps = cfg.mps;
  const int nch = (mps + kChunk - 1) / kChunk;
  const int A = cfg.n_agents;
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

  // MLOB_ROUNDS (phase-sync blocks): a grid of one block per SM walks the
  // envs in rounds (env = first + r * stride) with a block barrier at each
  // round start, so every round begins with all warps in phase 1 (like a
  // fresh block) while the next round's first replay chunk and header / book
  // rows are prefetched during this one; idle warps keep joining the barriers.
  constexpr bool rounds = MLOB_ROUNDS && phase_sync<SPL>();
  const uint64_t n_rounds = rounds ? (kp.n_envs + stride - 1) / stride : 1;
  uint64_t nenv = (MLOB_PERSIST && !phase_sync<SPL>()) ? ticket() : rounds ? first + stride : kp.n_envs;
  for (uint64_t env = first, round = 0; round < n_rounds && (env < kp.n_envs || phase_sync<SPL>()); ++round) {
    if constexpr (rounds) {
      if (round > 0) __syncthreads();
    }
    const DevMsg* slice = nullptr;
    const bool has_next = nenv < kp.n_envs;
    const DevMsg* next_slice = nullptr;
    int n_amsg = 0;
    if (!idle) {  // ---- phase 1: header, agents, actions -> agent messages
      w.bind(env);
      PHASE(0);
      w.load_hdr();
      w.book_load_issue();  // shared-memory books: bulk loads in flight during phase 1
      slice = kp.msgs + kp.ep_start[w.episode] + static_cast<uint64_t>(w.step) * mps;
      if (nch >= 2) w.stage(slice + kChunk, min(kChunk, mps - kChunk));
      if (has_next) {
        next_slice = mps > 0 ? slice_of(nenv) : nullptr;
#if MLOB_PREFETCH
        const EnvHdr& nh = kp.hdr[nenv];
        if (lane == 0) prefetch_l2(&nh);
        if (lane < A) prefetch_l2(kp.agents + nenv * A + lane);
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int k = 0; k < SPL; ++k)
            if (k * kWarp < (s ? nh.hwm[1] : nh.hwm[0])) {
              const size_t i = ((nenv * 2 + s) * SPL + k) * kWarp + lane;
              prefetch_l2(kp.bk_p + i);
              prefetch_l2(kp.bk_q + i);
              prefetch_l2(kp.bk_id + i);
              prefetch_l2(kp.bk_st + i);
            }
#endif
      }
      w.load_agents();
      w.clear_step_acc();
      const int64_t step_time = mps > 0 ? slice[0].time : w.last_time + 1;
      PHASE(1);
      // (1) actions -> agent messages, (2) Fisher-Yates (rng.hpp:63-71)
      for (int a = 0; a < A; ++a) w.convert_action(a, step_time, n_amsg);
      __syncwarp();
      if (n_amsg >= 2 && lane == 0) {
        uint64_t h = splitmix64(w.seed);
        h = key_fold(h, w.genv);
        h = key_fold(h, w.episode);
        h = key_fold(h, static_cast<uint64_t>(w.step));
        h = key_fold(h, kRngShuffle);
        Rng r{h};
        for (int i = n_amsg - 1; i > 0; --i) {
          const int j = static_cast<int>(r.below(static_cast<uint64_t>(i + 1)));
          if (i != j) {
            const DevMsg t = sm.amsg()[i];
            sm.amsg()[i] = sm.amsg()[j];
            sm.amsg()[j] = t;
          }
        }
      }
      __syncwarp();
      PHASE(2);
    }
    if constexpr (phase_sync<SPL>() && MLOB_SYNC_A) __syncthreads();
    if (!idle) {  // ---- phase 2: book in registers, message loop, book out
      // book registers are loaded only now: nothing above needs them (tops are
      // in the header) and they must not be live across subroutine calls
      w.book_load_wait();
      // (3) + (4): agent messages, then the replay slice
      w.prev_mid_half = w.mid_half;
      w.mid_sum = 0;
      w.mid_count = 0;
      w.n_trades = 0;
      PHASE(3);
      w.process_messages(n_amsg, slice);
      PHASE(4);
      if (has_next && mps > 0) w.stage(next_slice, min(kChunk, mps));  // overlaps the outcomes
      if (w.live0 > 0) w.last_bid = w.best0;
      if (w.live1 > 0) w.last_ask = w.best1;
      // (5) outcomes
      w.mbar = w.mid_count > 0 ? static_cast<double>(w.mid_sum) / (2.0 * static_cast<double>(w.mid_count))
                               : static_cast<double>(w.prev_mid_half) / 2.0;
      if (sm.scal()[1] && lane == 0) atomicAdd(kp.fill_overflow, 1ull);
      w.rebuild_active();
      PHASE(5);
      ++w.step;
      w.terminal = w.step >= cfg.steps_per_episode;
      w.snapshot();
      PHASE(6);
      w.store_book();  // book registers dead from here on
      PHASE(7);
    }
    if constexpr (phase_sync<SPL>() && MLOB_SYNC_B) __syncthreads();
    if (!idle) {  // ---- phase 3: rewards / infos / observations, auto-reset
      uint8_t just_reset = 0;
      for (int pass = 0;; ++pass) {  // pass 1: the auto-reset env's fresh outputs
        if (pass > 0) {
          w.snapshot();
          w.store_book();
        }
        w.outcomes(pass == 0);
        if (pass == 0) PHASE(8);
        if (pass > 0 || !(w.terminal && (kp.flags & MLOB_VENV_AUTO_RESET))) break;
        if (lane == 0)
          for (int a = 0; a < A; ++a) {  // rollout.hpp:300-313
            const mlob_agent_info& info = kp.infos[env * A + a];
            const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
            const size_t slot = env * A + a;
            kp.t_pv[slot] += info.portfolio_value;
            kp.t_slip[slot] += info.slippage_total;
            kp.t_comp[slot] += sp.type == MLOB_EXECUTOR
                                   ? 1.0 - static_cast<double>(info.task_remaining) /
                                               static_cast<double>(sp.task_size)
                                   : 0.0;
            kp.t_inv[slot] += static_cast<double>(info.inventory) * static_cast<double>(info.inventory);
          }
        ++w.ep_finished;
        const uint64_t ep = w.episode_for(w.cursor);
        ++w.cursor;
        if (!w.reset(ep, false)) break;
        just_reset = 1;
      }
      w.store_state(just_reset);
      PHASE(9);
    }
    if constexpr (rounds) {
      env = nenv;
      nenv = env + stride;
      idle = env >= kp.n_envs;
    } else {
      if (idle) break;
      env = nenv;
      if (has_next) nenv = ticket();
      if (MLOB_PERSIST && !phase_sync<SPL>()) --round;  // ticketed: runs until the envs run out
    }
  }
  w.book_store_drain();
  w.report_errors();
}

// K3: MarketEnv::reset for every env (reset_all / reset_envs).
template <int SPL>
__global__ void __launch_bounds__(kWarpsPerBlock * kWarp)
    reset_kernel(const __grid_constant__ KParams kparam) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(16) StagedParams sp_;
  stage_params(sp_, kparam);
  const KParams& kp = sp_.kp;
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const uint64_t env = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + warp;
  if (env >= kp.n_envs) return;
  const DevCfg& cfg = sp_.cfg;
  char* wbase = smem + warp * warp_smem_bytes(cfg);
  WarpSmem sm = carve(wbase, cfg);
  WarpEnv<SPL> w(kp, cfg, sm, env, lane, book_region(wbase, cfg));
  w.load_hdr();  // keeps last_time / messages_processed across resets
  w.load_agents();
  w.load_book();
  if (w.reset(kp.reset_episodes[env], true)) {
    w.snapshot();
    w.store_book();
    w.outcomes(false);
  } else {
    w.store_book();
  }
  w.cursor = 1;
  w.store_state(1);
  w.book_store_drain();
  w.report_errors();
}

// K4: per-type episode-stat sums over this handle's envs (for the NCCL
// all-reduce), 5 doubles per type: pv, slip, completion, inv², episodes.
__global__ void stats_kernel(const __grid_constant__ KParams kp, double* out) {
  const int t = blockIdx.y;
  const DevCfg& cfg = *kp.cfg;
  const int A = cfg.n_agents;
  const int cnt = cfg.specs[t].count, off = cfg.specs[t].flat_offset;
  double s[5] = {0, 0, 0, 0, 0};
  for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < kp.n_envs;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    for (int k = 0; k < cnt; ++k) {
      const size_t slot = e * A + off + k;
      s[0] += kp.t_pv[slot];
      s[1] += kp.t_slip[slot];
      s[2] += kp.t_comp[slot];
      s[3] += kp.t_inv[slot];
    }
    s[4] += static_cast<double>(kp.hdr[e].episodes_finished);
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    double v = s[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULLMASK, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&out[t * 5 + i], v);
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

// warps per step-kernel block: the phase-sync width for register books, 4 for
// shared-memory books, fewer when the config's per-warp shared memory
// (obs depth, agents) would not fit the 227 KB block limit
constexpr size_t kBlockSmemLimit = 227 * 1024 - sizeof(StagedParams) - 1024;
static bool deep_book(const DevCfg& c) { return spl_of(c.capacity) > 8; }
static size_t step_staged_bytes(const DevCfg& c) {  // dynamic-smem prefix (deep books)
  return deep_book(c) ? staged_dyn_bytes(c.n_specs) : 0;
}
static int step_warps(const DevCfg& c) {
  const bool deep = deep_book(c);
  const int want = deep ? 8 : (MLOB_PHASE_SYNC ? MLOB_SYNC_WARPS : 4);
  const size_t per = warp_smem_bytes(c);
  // deep: 227 KB less the static g_smem_off table, the staged prefix and a margin
  const size_t limit = deep ? 227 * 1024 - sizeof(SmemOff) - step_staged_bytes(c) - 256 : kBlockSmemLimit;
  const int fit = static_cast<int>(limit / (per > 0 ? per : 1));
  return fit < 1 ? 1 : (fit < want ? fit : want);
}

size_t step_smem_bytes(const DevCfg& c) {  // dynamic smem of the step kernel's block
  return step_staged_bytes(c) + warp_smem_bytes(c) * step_warps(c);
}
size_t step_min_smem_bytes(const DevCfg& c) {  // ... of a one-warp block (the feasibility bound)
  return step_staged_bytes(c) + warp_smem_bytes(c);
}

static unsigned grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 1184 ? (b > 0 ? b : 1) : 1184);
}

template <int SPL>
static cudaError_t launch_step_t(const KParams& kp, const DevCfg& cfg, cudaStream_t s) {
  int warps = step_warps(cfg);
  const size_t staged = step_staged_bytes(cfg);
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
    e = cudaFuncSetAttribute(step_kernel<SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(full_sm));
    if (e != cudaSuccess) return e;
    done = full_sm;
    per_sm_of[cur_dev & 63] = 0;  // re-query the occupancy for the new block size
  }
  uint64_t blocks = (kp.n_envs + warps - 1) / warps;
  if ((MLOB_PERSIST && !phase_sync<SPL>()) || (MLOB_ROUNDS && phase_sync<SPL>())) {
    // persistent grid: every SM filled to its occupancy limit (cached per device)
    int& n_sm = n_sm_of[cur_dev & 63];
    int& per_sm = per_sm_of[cur_dev & 63];
    if (n_sm == 0 &&
        (e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, cur_dev)) != cudaSuccess)
      return e;
    if (per_sm == 0) {
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel<SPL>, warps * kWarp,
                                                             full_sm)) != cudaSuccess)
        return e;
      if (per_sm < 1) per_sm = 1;
    }
    const uint64_t cap = static_cast<uint64_t>(n_sm) * static_cast<uint64_t>(per_sm);
    if (MLOB_ROUNDS && phase_sync<SPL>()) {
      // balanced rounds: the fewest rounds at full width, then the narrowest
      // block that still covers the envs in that many rounds (4,096 envs:
      // 2 rounds of 14 warps on every SM instead of 24 + a 3.7 %-full round)
      const uint64_t per_round = cap * static_cast<uint64_t>(warps);
      const uint64_t rounds = (kp.n_envs + per_round - 1) / per_round;
      const uint64_t w = (kp.n_envs + cap * rounds - 1) / (cap * rounds);
      warps = static_cast<int>(w < static_cast<uint64_t>(warps) ? (w > 0 ? w : 1) : warps);
    }
    const uint64_t need = (kp.n_envs + warps - 1) / warps;
    blocks = need < cap ? need : cap;
  }
  const size_t sm = staged + warp_smem_bytes(cfg) * warps;
  step_kernel<SPL><<<static_cast<unsigned>(blocks), warps * kWarp, sm, s>>>(kp);
  return cudaGetLastError();
}

template <int SPL>
static cudaError_t launch_reset_t(const KParams& kp, const DevCfg& cfg, cudaStream_t s) {
  const size_t sm = warp_smem_bytes(cfg) * kWarpsPerBlock;
  cudaError_t e = cudaFuncSetAttribute(reset_kernel<SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm));
  if (e != cudaSuccess) return e;
  const unsigned blocks = static_cast<unsigned>((kp.n_envs + kWarpsPerBlock - 1) / kWarpsPerBlock);
  reset_kernel<SPL><<<blocks, kWarpsPerBlock * kWarp, sm, s>>>(kp);
  return cudaGetLastError();
}

int slots_per_lane(int capacity) { return spl_of(capacity); }

cudaError_t launch_step(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s) {
  switch (spl) {
    case 1: return launch_step_t<1>(kp, cfg, s);
    case 2: return launch_step_t<2>(kp, cfg, s);
    case 4: return launch_step_t<4>(kp, cfg, s);
    case 8: return launch_step_t<8>(kp, cfg, s);
    case 16: return launch_step_t<16>(kp, cfg, s);
    case 32: return launch_step_t<32>(kp, cfg, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_reset(const KParams& kp, const DevCfg& cfg, int spl, cudaStream_t s) {
  switch (spl) {
    case 1: return launch_reset_t<1>(kp, cfg, s);
    case 2: return launch_reset_t<2>(kp, cfg, s);
    case 4: return launch_reset_t<4>(kp, cfg, s);
    case 8: return launch_reset_t<8>(kp, cfg, s);
    case 16: return launch_reset_t<16>(kp, cfg, s);
    case 32: return launch_reset_t<32>(kp, cfg, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_stats(const KParams& kp, const DevCfg& cfg, double* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * 5 * cfg.n_specs, s);
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
