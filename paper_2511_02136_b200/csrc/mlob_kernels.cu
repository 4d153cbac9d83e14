// mlob_kernels.cu — sm_100a kernels of the batched LOB environment step.
//
// One warp owns one environment for a whole step (K1+K2 fused):
//   * the env's book is loaded from HBM into registers (SoA rows of 32 slots,
//     lane l owns slots l, l+32, ...), processed, and stored back;
//   * the step's replay slice is staged global->shared with cp.async.bulk
//     (TMA bulk copy, mbarrier completion), overlapped with the book load and
//     the agent-order generation;
//   * every book operation is warp-cooperative: best price / oldest order by
//     redux.sync min/max, order-id lookup by ballot, free-slot search by ballot;
//   * step outcomes (rewards, infos, L2 top-D, observations) are computed in the
//     same launch; terminal envs are reset in place (MarketVecEnv auto-reset).
// Reference semantics followed (paths under /root/reference/proj/include/marlob):
//   lob/book.hpp:65-220, env/env.hpp:143-503, agents/*.hpp, core/rng.hpp,
//   ippo/rollout.hpp:290-318, bench/bench.hpp:53-70.
// Compiled with --fmad=false so every double expression rounds exactly like
// the reference's x86-64 build (no FMA contraction).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "mlob_dev.h"

namespace mlob {

#define FULLMASK 0xffffffffu

// ---------------------------------------------------------------------------
// core/rng.hpp:11-61
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t key_fold(uint64_t h, uint64_t w) {
  return splitmix64(h ^ (w + kGamma + (h << 6) + (h >> 2)));
}
struct Rng {
  uint64_t s;
  __device__ __forceinline__ uint64_t next() {
    s += kGamma;
    return splitmix64(s);
  }
  __device__ __forceinline__ uint64_t below(uint64_t n) { return next() % n; }
  __device__ __forceinline__ bool coin() { return (next() & 1ull) != 0; }
};
enum : uint64_t { kRngShuffle = 1, kRngTaskDir = 2, kRngBenchAction = 7 };

// ---------------------------------------------------------------------------
// Book side held in registers: SPL rows of 32 slots (lane-major).
// Empty slot: q == 0, p == side sentinel (bid INT_MIN, ask INT_MAX), st == ~0.
// st = arrival_seq << 8 | trader_id, so a u32 min over st is a min over seq.
template <int SPL>
struct RegSide {
  int32_t p_[SPL], q_[SPL];
  uint32_t lo_[SPL], hi_[SPL], st_[SPL];
  __device__ __forceinline__ int32_t P(int k) const { return p_[k]; }
  __device__ __forceinline__ int32_t Q(int k) const { return q_[k]; }
  __device__ __forceinline__ uint32_t LO(int k) const { return lo_[k]; }
  __device__ __forceinline__ uint32_t HI(int k) const { return hi_[k]; }
  __device__ __forceinline__ uint32_t ST(int k) const { return st_[k]; }
  __device__ __forceinline__ void put(int k, int32_t p, int32_t q, uint32_t lo, uint32_t hi,
                                      uint32_t st) {
    p_[k] = p;
    q_[k] = q;
    lo_[k] = lo;
    hi_[k] = hi;
    st_[k] = st;
  }
  // dynamic-index read / predicated write (select chains, no local memory)
  __device__ __forceinline__ void get(int k, int32_t& p, int32_t& q, uint32_t& lo,
                                      uint32_t& hi) const {
    p = p_[0];
    q = q_[0];
    lo = lo_[0];
    hi = hi_[0];
#pragma unroll
    for (int kk = 1; kk < SPL; ++kk)
      if (k == kk) {
        p = p_[kk];
        q = q_[kk];
        lo = lo_[kk];
        hi = hi_[kk];
      }
  }
  __device__ __forceinline__ void set(int k, bool pred, int32_t p, int32_t q, uint32_t lo,
                                      uint32_t hi, uint32_t st) {
#pragma unroll
    for (int kk = 0; kk < SPL; ++kk)
      if (pred && k == kk) put(kk, p, q, lo, hi, st);
  }
  __device__ __forceinline__ void setq(int k, bool pred, int32_t q) {
#pragma unroll
    for (int kk = 0; kk < SPL; ++kk)
      if (pred && k == kk) q_[kk] = q;
  }
  __device__ __forceinline__ void clear(int k, bool pred, int32_t empty_p) {
#pragma unroll
    for (int kk = 0; kk < SPL; ++kk)
      if (pred && k == kk) {
        p_[kk] = empty_p;
        q_[kk] = 0;
        st_[kk] = kEmptySt;
      }
  }
};

template <int S>
__device__ __forceinline__ int32_t empty_price() {
  return S == 0 ? INT_MIN : INT_MAX;
}
template <int S>
__device__ __forceinline__ int32_t better_of(int32_t a, int32_t b) {
  return S == 0 ? max(a, b) : min(a, b);
}
template <int S>
__device__ __forceinline__ int32_t redux_best(int32_t v) {
  return S == 0 ? __reduce_max_sync(FULLMASK, v) : __reduce_min_sync(FULLMASK, v);
}

// Per-agent per-step accumulators (fills of this step, env.hpp:222, 381-396).
struct StepAcc {
  double slip;          // slippage(fills, p_init, dir) accumulated in fill order
  int64_t filled;       // Σ qty
  int64_t sq[2];        // Σ qty by side (fallback MM reward)
  int64_t spq[2];       // Σ price*qty by side
  int32_t count;
  int32_t _pad;
};
struct FillEnt {
  int32_t price;
  int32_t qty;
  int32_t agent;
  int32_t side;
};

struct L2Lvl {
  int32_t price;
  int32_t _pad;
  int64_t qty;
};

struct BestOrder {
  int owner;   // lane owning the order
  int k;       // slot row in the owner lane (valid in the owner lane only)
  int32_t q;   // uniform
  uint32_t lo, hi, st;
};

struct WarpSmem {
  DevMsg* chunk[2];
  uint64_t* bar;  // 2 mbarriers
  DevMsg* amsg;   // agent messages (<= 4 * A)
  AgentRec* ag;
  ActiveRec* act;
  StepAcc* acc;
  FillEnt* fills;
  L2Lvl* l2;      // [2][obs_depth]
  double* obs;    // staging, max_obs_dim
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------------------
template <int SPL>
struct WarpEnv {
  using SideT = RegSide<SPL>;
  SideT bid, ask;
  const KParams& kp;
  const DevCfg& cfg;
  WarpSmem sm;
  int lane;
  uint64_t env, genv, seed;
  // uniform state (identical in every lane)
  int live0, live1;
  int32_t best0, best1;
  uint32_t next_seq;
  int64_t mid_half, prev_mid_half, last_bid, last_ask, last_time;
  double mbar;
  uint64_t episode, msgs, cursor;
  int64_t ep_finished;
  int step;
  bool terminal;
  int64_t mid_sum, mid_count;
  uint32_t n_trades;
  int n_fills;
  bool fill_overflow;
  uint32_t err;

  __device__ WarpEnv(const KParams& p, const WarpSmem& s, uint64_t e, int ln)
      : kp(p), cfg(p.cfg), sm(s), lane(ln), env(e) {
    genv = kp.env_index ? kp.env_index[e] : kp.env_index_base + e;
    seed = kp.env_seed ? kp.env_seed[e] : kp.seed;
    err = 0;
  }

  template <int S>
  __device__ __forceinline__ SideT& sd() {
    if constexpr (S == 0)
      return bid;
    else
      return ask;
  }
  template <int S>
  __device__ __forceinline__ int& live() {
    if constexpr (S == 0)
      return live0;
    else
      return live1;
  }
  template <int S>
  __device__ __forceinline__ int32_t& best() {
    if constexpr (S == 0)
      return best0;
    else
      return best1;
  }

  // ---- HBM <-> registers --------------------------------------------------
  __device__ __forceinline__ size_t row_index(int s, int k) const {
    return ((env * 2 + static_cast<uint64_t>(s)) * SPL + static_cast<uint64_t>(k)) * kWarp + lane;
  }
  template <int S>
  __device__ __forceinline__ void load_side(int hwm) {
    SideT& d = sd<S>();
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      if (k * kWarp < hwm) {
        const size_t i = row_index(S, k);
        const uint2 id = kp.bk_id[i];
        d.put(k, kp.bk_p[i], kp.bk_q[i], id.x, id.y, kp.bk_st[i]);
      } else {
        d.put(k, empty_price<S>(), 0, 0, 0, kEmptySt);
      }
    }
  }
  template <int S>
  __device__ __forceinline__ int store_side() {
    SideT& d = sd<S>();
    int hwm = 0;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const uint32_t b = __ballot_sync(FULLMASK, d.Q(k) > 0);
      if (b) hwm = k * kWarp + 32 - __clz(b);
    }
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      if (k * kWarp < hwm) {
        const size_t i = row_index(S, k);
        kp.bk_p[i] = d.P(k);
        kp.bk_q[i] = d.Q(k);
        kp.bk_id[i] = make_uint2(d.LO(k), d.HI(k));
        kp.bk_st[i] = d.ST(k);
      }
    }
    return hwm;
  }

  __device__ void load_hdr() {
    const EnvHdr& h = kp.hdr[env];
    mid_half = h.mid_half;
    prev_mid_half = h.prev_mid_half;
    mbar = h.mbar;
    last_bid = h.last_bid;
    last_ask = h.last_ask;
    last_time = h.last_time;
    episode = h.episode;
    msgs = h.msgs_processed;
    cursor = h.cursor;
    ep_finished = h.episodes_finished;
    next_seq = h.next_seq;
    step = h.step;
    live0 = h.live[0];
    live1 = h.live[1];
    best0 = h.best[0];
    best1 = h.best[1];
    terminal = h.terminal != 0;
    n_trades = h.n_trades;
  }
  __device__ void load_book() {
    const EnvHdr& h = kp.hdr[env];
    load_side<0>(h.hwm[0]);
    load_side<1>(h.hwm[1]);
  }
  __device__ void store_all(uint8_t just_reset) {
    const int h0 = store_side<0>();
    const int h1 = store_side<1>();
    if (lane == 0) {
      EnvHdr h;
      h.mid_half = mid_half;
      h.prev_mid_half = prev_mid_half;
      h.mbar = mbar;
      h.last_bid = last_bid;
      h.last_ask = last_ask;
      h.last_time = last_time;
      h.episode = episode;
      h.msgs_processed = msgs;
      h.cursor = cursor;
      h.episodes_finished = ep_finished;
      h.next_seq = next_seq;
      h.step = step;
      h.live[0] = static_cast<uint16_t>(live0);
      h.live[1] = static_cast<uint16_t>(live1);
      h.hwm[0] = static_cast<uint16_t>(h0);
      h.hwm[1] = static_cast<uint16_t>(h1);
      h.best[0] = best0;
      h.best[1] = best1;
      h.n_trades = n_trades;
      h.terminal = terminal ? 1 : 0;
      h.just_reset = just_reset;
      h._pad8[0] = h._pad8[1] = 0;
      h._pad64[0] = h._pad64[1] = 0;
      kp.hdr[env] = h;
      kp.just_reset[env] = just_reset;
    }
    // agent records and active lists (written by lanes cooperatively)
    const int A = cfg.n_agents;
    const int words = A * static_cast<int>(sizeof(AgentRec) / 8);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(sm.ag);
    uint64_t* dst = reinterpret_cast<uint64_t*>(kp.agents + env * A);
    for (int i = lane; i < words; i += kWarp) dst[i] = src[i];
    for (int a = 0; a < A; ++a) {
      const int n = sm.ag[a].n_active;
      if (lane < n) kp.active[(env * A + a) * kMaxActive + lane] = sm.act[a * kMaxActive + lane];
    }
    if (err && lane == 0) atomicOr(kp.error, err);
  }
  __device__ void load_agents() {
    const int A = cfg.n_agents;
    const int words = A * static_cast<int>(sizeof(AgentRec) / 8);
    const uint64_t* src = reinterpret_cast<const uint64_t*>(kp.agents + env * A);
    uint64_t* dst = reinterpret_cast<uint64_t*>(sm.ag);
    for (int i = lane; i < words; i += kWarp) dst[i] = src[i];
    __syncwarp();
    for (int a = 0; a < A; ++a) {
      const int n = sm.ag[a].n_active;
      if (lane < n) sm.act[a * kMaxActive + lane] = kp.active[(env * A + a) * kMaxActive + lane];
    }
    __syncwarp();
  }

  // ---- book primitives (lob/book.hpp) -------------------------------------
  template <int S>
  __device__ __forceinline__ int32_t side_best() {
    SideT& d = sd<S>();
    int32_t b = d.P(0);
#pragma unroll
    for (int k = 1; k < SPL; ++k) b = better_of<S>(b, d.P(k));
    return redux_best<S>(b);
  }

  // Oldest order (min arrival_seq) at `price` on side S: the book.hpp back()
  // element when price is the best price, the eviction victim
  // (book.hpp:176-181) when price is the worst price.
  template <int S>
  __device__ __forceinline__ BestOrder oldest_at(int32_t price) {
    SideT& d = sd<S>();
    uint32_t m = kEmptySt;
    int lk = 0;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const bool c = d.P(k) == price && d.ST(k) < m;
      m = c ? d.ST(k) : m;
      lk = c ? k : lk;
    }
    BestOrder r;
    r.st = __reduce_min_sync(FULLMASK, m);
    r.owner = __ffs(__ballot_sync(FULLMASK, m == r.st)) - 1;
    r.k = lk;
    int32_t p, q;
    uint32_t lo, hi;
    d.get(lk, p, q, lo, hi);
    r.q = __shfl_sync(FULLMASK, q, r.owner);
    r.lo = __shfl_sync(FULLMASK, lo, r.owner);
    r.hi = __shfl_sync(FULLMASK, hi, r.owner);
    return r;
  }

  __device__ __forceinline__ void update_mid() {
    const bool hb = live0 > 0, ha = live1 > 0;
    if (hb && ha)
      mid_half = static_cast<int64_t>(best0) + best1;
    else if (hb)
      mid_half = 2 * static_cast<int64_t>(best0);
    else if (ha)
      mid_half = 2 * static_cast<int64_t>(best1);
  }

  // env.hpp:372-396
  __device__ void apply_fill(int a, int32_t price, int32_t qty, int side) {
    const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
    AgentRec& st = sm.ag[a];
    StepAcc& ac = sm.acc[a];
    const int64_t pq = static_cast<int64_t>(price) * qty;
    int64_t inv = st.inventory, cash = st.cash, rem = st.task_remaining;
    if (side == MLOB_BID) {
      inv += qty;
      cash -= pq;
    } else {
      inv -= qty;
      cash += pq;
    }
    if (sp.type == MLOB_EXECUTOR) {
      const bool task_side = (st.task_dir == MLOB_TASK_BUY) == (side == MLOB_BID);
      if (task_side) rem = max(static_cast<int64_t>(0), rem - qty);
    }
    // slippage term, rewards.hpp:69-75: (sign * q) * (price - p_init)
    const double sign = st.task_dir == MLOB_TASK_BUY ? 1.0 : -1.0;
    const double term = sign * static_cast<double>(qty) * (static_cast<double>(price) - st.p_init);
    __syncwarp();
    if (lane == 0) {
      st.inventory = inv;
      st.cash = cash;
      st.task_remaining = rem;
      st.filled_total += qty;
      ac.slip += term;
      ac.filled += qty;
      ac.count += 1;
      ac.sq[side] += qty;
      ac.spq[side] += pq;
      if (n_fills < kFillLog) sm.fills[n_fills] = FillEnt{price, qty, a, side};
    }
    if (n_fills < kFillLog)
      ++n_fills;
    else
      fill_overflow = true;
    __syncwarp();
  }

  __device__ __forceinline__ void emit_trade(int32_t price, int32_t qty, const DevMsg& m,
                                             const BestOrder& o, int aside) {
    if ((kp.flags & MLOB_VENV_RECORD_TRADES) && lane == 0 && n_trades < kp.trade_cap) {
      mlob_trade t;
      t.price = price;
      t.quantity = qty;
      t.time = m.time;
      t.passive_order_id = (static_cast<uint64_t>(o.hi) << 32) | o.lo;
      t.aggressor_order_id = m.order_id;
      t.passive_trader_id = static_cast<int32_t>(o.st & 0xffu);
      t.aggressor_trader_id = m.trader;
      t.aggressor_side = static_cast<uint8_t>(aside);
      for (int i = 0; i < 7; ++i) t._pad[i] = 0;
      kp.trades[env * kp.trade_cap + n_trades] = t;
    }
    ++n_trades;
    const int ptrader = static_cast<int>(o.st & 0xffu);
    if (ptrader > cfg.n_agents || m.trader > cfg.n_agents) err |= kErrBadTrader;
    if (ptrader > 0 && ptrader <= cfg.n_agents) apply_fill(ptrader - 1, price, qty, 1 - aside);
    if (m.trader > 0 && m.trader <= cfg.n_agents) apply_fill(m.trader - 1, price, qty, aside);
  }

  // book.hpp:169-187
  template <int S>
  __device__ void rest(const DevMsg& m, int32_t qty) {
    SideT& d = sd<S>();
    if (live<S>() == cfg.capacity) {
      int32_t lw = S == 0 ? INT_MAX : INT_MIN;
#pragma unroll
      for (int k = 0; k < SPL; ++k)
        if (d.Q(k) > 0) lw = S == 0 ? min(lw, d.P(k)) : max(lw, d.P(k));
      const int32_t worst =
          S == 0 ? __reduce_min_sync(FULLMASK, lw) : __reduce_max_sync(FULLMASK, lw);
      const bool better = S == 0 ? m.price > worst : m.price < worst;
      if (!better) return;
      const BestOrder ev = oldest_at<S>(worst);
      d.clear(ev.k, lane == ev.owner, empty_price<S>());
      --live<S>();
    }
    const uint32_t seq = next_seq++;
    if (seq >= kMaxSeq) err |= kErrSeqRange;
    int pk = -1, pl = 0;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const uint32_t b = __ballot_sync(FULLMASK, d.Q(k) == 0);
      if (pk < 0 && b) {
        pk = k;
        pl = __ffs(b) - 1;
      }
    }
    d.set(pk, lane == pl, m.price, qty, static_cast<uint32_t>(m.order_id),
          static_cast<uint32_t>(m.order_id >> 32),
          (seq << 8) | static_cast<uint32_t>(m.trader & 0xff));
    const int l = ++live<S>();
    best<S>() = l == 1 ? m.price : better_of<S>(best<S>(), m.price);
  }

  // book.hpp:150-167
  template <int S>
  __device__ void new_limit(const DevMsg& m) {
    if (m.qty <= 0) return;
    constexpr int O = 1 - S;
    SideT& od = sd<O>();
    int32_t rem = m.qty;
    while (rem > 0 && live<O>() > 0) {
      const int32_t bp = best<O>();
      const bool crosses = S == 0 ? bp <= m.price : bp >= m.price;
      if (!crosses) break;
      const BestOrder bo = oldest_at<O>(bp);
      const int32_t fill = min(rem, bo.q);
      const bool removed = fill == bo.q;
      if (removed)
        od.clear(bo.k, lane == bo.owner, empty_price<O>());
      else
        od.setq(bo.k, lane == bo.owner, bo.q - fill);
      rem -= fill;
      if (removed) {
        const int l = --live<O>();
        if (l > 0) best<O>() = side_best<O>();
      }
      emit_trade(bp, fill, m, bo, S);
    }
    if (rem > 0) rest<S>(m, rem);
  }

  // book.hpp:189-207 (reduce_order / remove_order); absent ids are no-ops.
  template <int S>
  __device__ void by_id(uint64_t id, int32_t by, bool remove) {
    SideT& d = sd<S>();
    const uint32_t lo = static_cast<uint32_t>(id), hi = static_cast<uint32_t>(id >> 32);
    int nm = 0, lk = 0;
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const bool c = d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi;
      lk = (c && nm == 0) ? k : lk;
      nm += c ? 1 : 0;
    }
    const uint32_t b = __ballot_sync(FULLMASK, nm > 0);
    if (b == 0) return;
    int owner;
    if (__popc(b) == 1 && __shfl_sync(FULLMASK, nm, __ffs(b) - 1) == 1) {
      owner = __ffs(b) - 1;
    } else {
      // Duplicate live ids: the reference takes the first match in storage
      // order (bids: lowest price then newest; asks: highest price then newest).
      int32_t kp_ = S == 0 ? INT_MAX : INT_MIN;
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const bool c = d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi;
        if (c) kp_ = S == 0 ? min(kp_, d.P(k)) : max(kp_, d.P(k));
      }
      const int32_t gp = S == 0 ? __reduce_min_sync(FULLMASK, kp_) : __reduce_max_sync(FULLMASK, kp_);
      uint32_t ms = 0;
      bool any = false;
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const bool c = d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi && d.P(k) == gp;
        if (c && (!any || d.ST(k) > ms)) {
          ms = d.ST(k);
          lk = k;
          any = true;
        }
      }
      const uint32_t gs = __reduce_max_sync(FULLMASK, any ? ms : 0u);
      owner = __ffs(__ballot_sync(FULLMASK, any && ms == gs)) - 1;
    }
    int32_t p, q;
    uint32_t l2, h2;
    d.get(lk, p, q, l2, h2);
    const int32_t op = __shfl_sync(FULLMASK, p, owner);
    const int32_t oq = __shfl_sync(FULLMASK, q, owner);
    const int32_t nq = remove ? 0 : oq - min(oq, by);
    if (nq == 0) {
      d.clear(lk, lane == owner, empty_price<S>());
      const int l = --live<S>();
      if (l > 0 && op == best<S>()) best<S>() = side_best<S>();
    } else {
      d.setq(lk, lane == owner, nq);
    }
  }

  // book.hpp:65-86 + env.hpp:223-235
  __device__ __forceinline__ void run_message(const DevMsg& m) {
    switch (m.kind) {
      case MLOB_NEW_LIMIT:
        if (m.side == MLOB_BID)
          new_limit<0>(m);
        else
          new_limit<1>(m);
        break;
      case MLOB_CANCEL_PARTIAL:
      case MLOB_EXECUTE_VISIBLE:
        if (m.side == MLOB_BID)
          by_id<0>(m.order_id, m.qty, false);
        else
          by_id<1>(m.order_id, m.qty, false);
        break;
      case MLOB_DELETE:
        if (m.side == MLOB_BID)
          by_id<0>(m.order_id, 0, true);
        else
          by_id<1>(m.order_id, 0, true);
        break;
      default:
        break;
    }
    update_mid();
    mid_sum += mid_half;
    ++mid_count;
    ++msgs;
    last_time = m.time;
  }

  // ---- agents (agents/actions.hpp, env.hpp:266-370) ----------------------
  __device__ __forceinline__ void effective_tops(const DevSpec& p, int64_t& bid, int64_t& ask) const {
    const int64_t mid_floor = mid_half >= 0 ? mid_half / 2 : (mid_half - 1) / 2;
    const int64_t mid_ceil = (mid_half + 1) / 2;
    bid = live0 > 0 ? static_cast<int64_t>(best0) : mid_floor - p.default_half_spread;
    ask = live1 > 0 ? static_cast<int64_t>(best1) : mid_ceil + p.default_half_spread;
    if (bid < 1) bid = 1;
    if (ask <= bid) ask = bid + 1;
  }

  struct Quotes {
    int n;
    int side[2];
    int64_t price[2], qty[2];
    __device__ void push(int s, int64_t p, int64_t q) {
      side[n] = s;
      price[n] = p;
      qty[n] = q;
      ++n;
    }
    __device__ void finish_two_sided() {  // actions.hpp:47-56
      for (int i = 0; i < n; ++i) price[i] = price[i] < 1 ? 1 : price[i];
      if (n == 2) {
        const int b = side[0] == MLOB_BID ? 0 : 1;
        const int a = side[0] == MLOB_ASK ? 0 : 1;
        if (price[b] >= price[a]) price[a] = price[b] + 1;
      }
    }
  };

  __device__ void decode(int a, int id, Quotes& q) {
    const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
    const AgentRec& st = sm.ag[a];
    int64_t bb, ba;
    effective_tops(sp, bb, ba);
    q.n = 0;
    if (sp.type == MLOB_EXECUTOR) {  // env.hpp:302-311, actions.hpp:193-224
      int64_t eb = bb, ea = ba;
      if (st.task_dir == MLOB_TASK_BUY && live1 == 0) ea = max(static_cast<int64_t>(2), last_ask + 1);
      if (st.task_dir == MLOB_TASK_SELL && live0 == 0) eb = max(static_cast<int64_t>(1), last_bid - 1);
      const int pi = id % 4, mi = id / 4;
      const int64_t spread = ea - eb;
      int64_t price;
      if (st.task_dir == MLOB_TASK_BUY)
        price = pi == 0 ? ea : pi == 1 ? eb : pi == 2 ? eb - 1 : eb + spread / 2;
      else
        price = pi == 0 ? eb : pi == 1 ? ea : pi == 2 ? ea + 1 : ea - spread / 2;
      int64_t qty = sp.order_size * (mi == 0 ? 1 : mi == 1 ? 2 : 5);
      if (qty > st.task_remaining) qty = st.task_remaining;
      if (qty > 0)
        q.push(st.task_dir == MLOB_TASK_BUY ? MLOB_BID : MLOB_ASK, price < 1 ? 1 : price, qty);
    } else if (sp.type == MLOB_DIRECTIONAL) {  // actions.hpp:227-235
      if (id == 1) q.push(MLOB_BID, bb < 1 ? 1 : bb, sp.order_size);
      if (id == 2) q.push(MLOB_ASK, ba < 1 ? 1 : ba, sp.order_size);
    } else if (sp.mm_space == MLOB_FIXED_QUANT) {  // actions.hpp:66-108
      const int64_t br = sp.fixed_quant_from_mid ? (bb + ba) / 2 : bb;
      const int64_t ar = sp.fixed_quant_from_mid ? (bb + ba + 1) / 2 : ba;
      const int64_t sz = sp.order_size;
      switch (id) {
        case 1: q.push(MLOB_BID, br - 2, sz); q.push(MLOB_ASK, ar + 2, sz); break;
        case 2: q.push(MLOB_BID, br - 4, sz); q.push(MLOB_ASK, ar + 4, sz); break;
        case 3: q.push(MLOB_BID, bb + 1, sz); q.push(MLOB_ASK, ba - 1, sz); break;
        case 4: q.push(MLOB_BID, br - 2, sz); q.push(MLOB_ASK, ba, sz); break;
        case 5: q.push(MLOB_BID, bb, sz); q.push(MLOB_ASK, ar + 2, sz); break;
        case 6: q.push(MLOB_BID, bb - 5, sz); q.push(MLOB_ASK, ba - 1, sz); break;
        case 7: q.push(MLOB_BID, bb + 1, sz); q.push(MLOB_ASK, ba + 5, sz); break;
        default: break;
      }
      q.finish_two_sided();
    } else if (sp.mm_space == MLOB_SPREAD_SKEW) {  // actions.hpp:128-140
      const int64_t hs = sp.ss_half[id], sk = sp.ss_skew[id];
      const int64_t bh = mid_half - 2 * hs + 2 * sk;
      const int64_t ah = mid_half + 2 * hs + 2 * sk;
      q.push(MLOB_BID, bh >= 0 ? bh / 2 : (bh - 1) / 2, sp.order_size);
      q.push(MLOB_ASK, (ah + 1) / 2, sp.order_size);
      q.finish_two_sided();
    } else {  // AvSt, actions.hpp:151-178
      const double gamma = sp.gamma[id];
      const double rem = sp.horizon - static_cast<double>(step);
      const double ttg = 0.0 < rem ? rem : 0.0;
      const double mid_ticks = static_cast<double>(mid_half) / 2.0;
      const double reservation =
          mid_ticks - static_cast<double>(st.inventory) * gamma * sp.sigma * sp.sigma * ttg;
      const double half_spread = 0.5 * (gamma * sp.sigma * sp.sigma * ttg + sp.avst_term[id]);
      q.push(MLOB_BID, static_cast<int64_t>(floor(reservation - half_spread)), sp.order_size);
      q.push(MLOB_ASK, static_cast<int64_t>(ceil(reservation + half_spread)), sp.order_size);
      q.finish_two_sided();
    }
  }

  // env.hpp:285-370: quotes -> Delete for stale active orders, NewLimit for
  // quotes not already resting at the same (side, price).
  __device__ void convert_action(int a, int64_t step_time, int& n_amsg) {
    const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
    AgentRec& st = sm.ag[a];
    Quotes q;
    q.n = 0;
    if (kp.action_mode == kActDirect) {
      const mlob_agent_action& da = kp.action_direct[env * cfg.n_agents + a];
      if (da.direct) {
        q.n = da.n_quotes;
        for (int i = 0; i < q.n; ++i) {
          q.side[i] = da.quotes[i].side;
          q.price[i] = da.quotes[i].price;
          q.qty[i] = da.quotes[i].quantity;
        }
        if (sp.type == MLOB_EXECUTOR) {
          for (int i = 0; i < q.n; ++i)
            if (q.qty[i] > st.task_remaining) q.qty[i] = st.task_remaining;
          if (q.n == 1 && q.qty[0] <= 0) q.n = 0;
        }
      } else {
        decode(a, da.id, q);
      }
    } else {
      int id;
      if (kp.action_mode == kActBench) {  // bench.hpp:57-60
        Rng r{key_fold(key_fold(key_fold(splitmix64(kp.bench_seed), kRngBenchAction), genv),
                       kp.global_step)};
        // one draw per agent, in agent order
        for (int b = 0; b < a; ++b) r.next();
        id = static_cast<int>(r.below(static_cast<uint64_t>(sp.arity)));
      } else {
        id = kp.action_ids[env * cfg.n_agents + a];
        if (id < 0 || id >= sp.arity) {
          err |= kErrBadAction;
          id = 0;
        }
      }
      decode(a, id, q);
    }
    bool kept[2] = {false, false};
    const int na = st.n_active;
    for (int i = 0; i < na; ++i) {
      const ActiveRec ar = sm.act[a * kMaxActive + i];
      const int side = static_cast<int>(ar.qty_side >> 31);
      bool reused = false;
      for (int j = 0; j < q.n; ++j)
        if (q.side[j] == side && q.price[j] == ar.price) {
          reused = true;
          kept[j] = true;
        }
      if (reused) continue;
      if (lane == 0) {
        DevMsg m;
        m.time = step_time;
        m.order_id = ar.order_id;
        m.price = 0;
        m.qty = 0;
        m.kind = MLOB_DELETE;
        m.side = static_cast<uint8_t>(side);
        m._pad = 0;
        m.trader = a + 1;
        sm.amsg[n_amsg] = m;
      }
      ++n_amsg;
    }
    uint64_t nonce = st.nonce;
    for (int j = 0; j < q.n; ++j) {
      if (kept[j]) continue;
      if (q.price[j] > INT_MAX - 1 || q.price[j] < INT_MIN + 1 || q.qty[j] > INT_MAX ||
          q.qty[j] < INT_MIN)
        err |= kErrPriceRange;
      if (lane == 0) {
        DevMsg m;
        m.time = step_time;
        m.order_id = cfg.agent_id_base + static_cast<uint64_t>(a) * cfg.agent_id_range + nonce;
        m.price = static_cast<int32_t>(q.price[j]);
        m.qty = static_cast<int32_t>(q.qty[j]);
        m.kind = MLOB_NEW_LIMIT;
        m.side = static_cast<uint8_t>(q.side[j]);
        m._pad = 0;
        m.trader = a + 1;
        sm.amsg[n_amsg] = m;
      }
      ++nonce;
      ++n_amsg;
    }
    if (lane == 0) st.nonce = nonce;
  }

  // ---- step outcomes -------------------------------------------------------
  // Top-D aggregated levels per side, best-first (book.hpp:109-120, 209-220).
  template <int S>
  __device__ int l2_levels(L2Lvl* out) {
    SideT& d = sd<S>();
    const int D = cfg.obs_depth;
    int n = 0;
    int32_t prev = 0;
    for (; n < D; ++n) {
      int32_t lb = empty_price<S>();
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const bool ok = d.Q(k) > 0 && (n == 0 || (S == 0 ? d.P(k) < prev : d.P(k) > prev));
        if (ok) lb = better_of<S>(lb, d.P(k));
      }
      const int32_t lvl = redux_best<S>(lb);
      if (lvl == empty_price<S>()) break;
      // per-lane sum < SPL * 2^31: reduce it as two 16-bit-split halves so the
      // 32-bit redux.sync add cannot overflow
      uint64_t s64 = 0;
#pragma unroll
      for (int k = 0; k < SPL; ++k)
        if (d.P(k) == lvl) s64 += static_cast<uint32_t>(d.Q(k));
      const uint32_t lo = __reduce_add_sync(FULLMASK, static_cast<uint32_t>(s64 & 0xffffu));
      const uint32_t hi = __reduce_add_sync(FULLMASK, static_cast<uint32_t>(s64 >> 16));
      const int64_t tot = static_cast<int64_t>(lo) + (static_cast<int64_t>(hi) << 16);
      if (lane == 0) out[n] = L2Lvl{lvl, 0, tot};
      prev = lvl;
    }
    __syncwarp();
    return n;
  }

  // env.hpp:398-407: active orders per agent, book storage order.
  __device__ void rebuild_active() {
    const int A = cfg.n_agents;
    for (int a = 0; a < A; ++a) sm.ag[a].n_active = 0;  // uniform write by all lanes (same value)
    __syncwarp();
    rebuild_side<0>();
    rebuild_side<1>();
  }
  template <int S>
  __device__ void rebuild_side() {
    SideT& d = sd<S>();
    uint32_t taken = 0;  // per-lane bitmask of consumed slots
    int cnt = 0;
#pragma unroll
    for (int k = 0; k < SPL; ++k) cnt += (d.Q(k) > 0 && (d.ST(k) & 0xffu) != 0) ? 1 : 0;
    const int total = __reduce_add_sync(FULLMASK, static_cast<uint32_t>(cnt));
    for (int i = 0; i < total; ++i) {
      // first in storage order: bids lowest price, asks highest; then newest seq
      int32_t lp = S == 0 ? INT_MAX : INT_MIN;
#pragma unroll
      for (int k = 0; k < SPL; ++k)
        if (d.Q(k) > 0 && (d.ST(k) & 0xffu) != 0 && !((taken >> k) & 1u))
          lp = S == 0 ? min(lp, d.P(k)) : max(lp, d.P(k));
      const int32_t gp = S == 0 ? __reduce_min_sync(FULLMASK, lp) : __reduce_max_sync(FULLMASK, lp);
      uint32_t ms = 0;
      int lk = 0;
      bool any = false;
#pragma unroll
      for (int k = 0; k < SPL; ++k) {
        const bool c = d.Q(k) > 0 && (d.ST(k) & 0xffu) != 0 && !((taken >> k) & 1u) && d.P(k) == gp;
        if (c && (!any || d.ST(k) > ms)) {
          ms = d.ST(k);
          lk = k;
          any = true;
        }
      }
      const uint32_t gs = __reduce_max_sync(FULLMASK, any ? ms : 0u);
      const int owner = __ffs(__ballot_sync(FULLMASK, any && ms == gs)) - 1;
      if (lane == owner) taken |= 1u << lk;
      int32_t p, q;
      uint32_t lo, hi;
      d.get(lk, p, q, lo, hi);
      q = __shfl_sync(FULLMASK, q, owner);
      lo = __shfl_sync(FULLMASK, lo, owner);
      hi = __shfl_sync(FULLMASK, hi, owner);
      const int a = static_cast<int>(gs & 0xffu) - 1;
      if (a >= cfg.n_agents) {
        err |= kErrBadTrader;
        continue;
      }
      const int n = sm.ag[a].n_active;
      if (n >= kMaxActive) {
        err |= kErrActiveOverflow;
        continue;
      }
      if (lane == 0) {
        sm.act[a * kMaxActive + n] =
            ActiveRec{(static_cast<uint64_t>(hi) << 32) | lo, gp,
                      static_cast<uint32_t>(q) | (static_cast<uint32_t>(S) << 31)};
        sm.ag[a].n_active = n + 1;
      }
      __syncwarp();
    }
  }

  // env.hpp:435-443
  __device__ double reference_price(const DevSpec& sp, const AgentRec& st) const {
    if (sp.ref_price == MLOB_REF_MID || st.inventory == 0) return static_cast<double>(mid_half) / 2.0;
    if (st.inventory > 0) return static_cast<double>(live0 > 0 ? static_cast<int64_t>(best0) : last_bid);
    return static_cast<double>(live1 > 0 ? static_cast<int64_t>(best1) : last_ask);
  }

  // env.hpp:445-464 (also accumulates slippage_total); lane 0 writes.
  __device__ void fill_info(int a) {
    const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
    AgentRec& st = sm.ag[a];
    const StepAcc& ac = sm.acc[a];
    mlob_agent_info info;
    info.inventory = st.inventory;
    info.cash = st.cash;
    info.portfolio_value =
        static_cast<double>(st.inventory) * reference_price(sp, st) + static_cast<double>(st.cash);
    info.slippage_step = sp.type == MLOB_EXECUTOR ? ac.slip : 0.0;
    const double total = st.slippage_total + info.slippage_step;
    info.slippage_total = total;
    info.task_remaining = st.task_remaining;
    info.step_filled = ac.filled;
    info.step_fill_count = ac.count;
    info._pad = 0;
    __syncwarp();
    if (lane == 0) {
      st.slippage_total = total;
      kp.infos[env * cfg.n_agents + a] = info;
    }
    __syncwarp();
  }

  // env.hpp:409-433 + rewards.hpp
  __device__ double compute_reward(int a) {
    const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
    const AgentRec& st = sm.ag[a];
    const StepAcc& ac = sm.acc[a];
    double r = 0.0;
    if (sp.reward == MLOB_REWARD_EXEC) {
      r = -ac.slip;
      if (terminal && st.task_remaining > 0)
        r -= sp.unfilled_penalty_coef * static_cast<double>(st.task_remaining) * st.p_init;
    } else {
      double pb = 0.0, ps = 0.0;
      if (!fill_overflow) {
        for (int i = 0; i < n_fills; ++i) {
          const FillEnt f = sm.fills[i];
          if (f.agent == a && f.side == MLOB_BID)
            pb += (mbar - static_cast<double>(f.price)) * static_cast<double>(f.qty);
        }
        for (int i = 0; i < n_fills; ++i) {
          const FillEnt f = sm.fills[i];
          if (f.agent == a && f.side == MLOB_ASK)
            ps += (static_cast<double>(f.price) - mbar) * static_cast<double>(f.qty);
        }
      } else {
        // exact-rational fallback beyond kFillLog fills in one env-step
        pb = mbar * static_cast<double>(ac.sq[0]) - static_cast<double>(ac.spq[0]);
        ps = static_cast<double>(ac.spq[1]) - mbar * static_cast<double>(ac.sq[1]);
      }
      if (sp.reward == MLOB_REWARD_BUYSELL) {
        r = pb + ps;
      } else {
        const double mid = static_cast<double>(mid_half) / 2.0;
        const double prev = static_cast<double>(prev_mid_half) / 2.0;
        const double psi_inv = static_cast<double>(st.inventory) * (mid - prev);
        r = pb + ps + psi_inv - (1.0 - sp.lambda) * (0.0 < psi_inv ? psi_inv : 0.0);
      }
      if (sp.quadratic_penalty) {
        const double frac = static_cast<double>(st.inventory) / static_cast<double>(sp.inventory_cap);
        r -= sp.rho * frac * frac;
      }
    }
    return r * sp.reward_scale;
  }

  // env.hpp:466-503, observations.hpp:42-148; features staged in smem then
  // written by lanes (coalesced).
  __device__ void build_observation(int a, const L2Lvl* l2b, int nb, const L2Lvl* l2a, int na) {
    const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
    const AgentRec& st = sm.ag[a];
    const int64_t bb = live0 > 0 ? best0 : -1;
    const int64_t ba = live1 > 0 ? best1 : -1;
    const double time_frac = static_cast<double>(step) / static_cast<double>(cfg.steps_per_episode);
    int64_t bq = 0, aq = 0;
    for (int i = 0; i < nb; ++i) bq += l2b[i].qty;
    for (int i = 0; i < na; ++i) aq += l2a[i].qty;
    const double imb = bq + aq == 0 ? 0.0 : static_cast<double>(bq - aq) / static_cast<double>(bq + aq);
    const double spread = (bb < 0 || ba < 0) ? 0.0 : fmin_ref(32.0, static_cast<double>(ba - bb));
    int64_t own_bid = -1, own_ask = -1;
    for (int i = 0; i < st.n_active; ++i) {
      const ActiveRec ar = sm.act[a * kMaxActive + i];
      if ((ar.qty_side >> 31) == 0)
        own_bid = own_bid < 0 ? ar.price : max(own_bid, static_cast<int64_t>(ar.price));
      else
        own_ask = own_ask < 0 ? ar.price : min(own_ask, static_cast<int64_t>(ar.price));
    }
    const double dmid = static_cast<double>(mid_half - prev_mid_half) / 2.0;
    double* out = sm.obs;
    const int dim = sp.obs_dim;
    if (lane == 0) {
      if (sp.type == MLOB_EXECUTOR) {
        const int dir = st.task_dir == MLOB_TASK_BUY ? 1 : -1;
        out[0] = static_cast<double>(st.task_remaining) /
                 static_cast<double>(sp.task_size > 1 ? sp.task_size : 1);
        out[1] = time_frac;
        out[2] = static_cast<double>(dir);
        out[3] = spread;
        out[4] = dmid;
        out[5] = static_cast<double>(mid_half) / 2.0 - st.p_init;
        out[6] = imb;
        out[7] = nb > 0 ? qty_feature(l2b[0].qty, sp.order_size) : 0.0;
        out[8] = na > 0 ? qty_feature(l2a[0].qty, sp.order_size) : 0.0;
        const bool buy = dir > 0;
        out[9] = offset_feature(buy ? own_bid : own_ask, buy ? bb : ba, buy);
        for (int j = 10; j < dim; ++j) out[j] = 0.0;  // MMFull-sized executor obs
      } else {
        const int64_t cs = sp.inventory_cap * static_cast<int64_t>(st.p_init);
        out[0] = static_cast<double>(st.inventory) / static_cast<double>(sp.inventory_cap);
        out[1] = static_cast<double>(st.cash) / static_cast<double>(cs > 1 ? cs : 1);
        out[2] = spread;
        out[3] = dmid;
        out[4] = imb;
        out[5] = time_frac;
        out[6] = offset_feature(own_bid, bb, true);
        out[7] = offset_feature(own_ask, ba, false);
        if (sp.obs_space == MLOB_OBS_MM_FULL) {
          int k = 8;
          const int levels = (dim - 8) / 4;
          for (int d = 0; d < levels; ++d) {
            const bool hb = d < nb, ha = d < na;
            out[k++] = hb ? fmin_ref(32.0, static_cast<double>(bb - l2b[d].price)) : -1.0;
            out[k++] = hb ? qty_feature(l2b[d].qty, sp.order_size) : 0.0;
            out[k++] = ha ? fmin_ref(32.0, static_cast<double>(l2a[d].price - ba)) : -1.0;
            out[k++] = ha ? qty_feature(l2a[d].qty, sp.order_size) : 0.0;
          }
        } else if (sp.obs_space == MLOB_OBS_EXEC) {
          out[8] = 0.0;  // the reference leaves these two zero-initialised
          out[9] = 0.0;
        }
      }
    }
    __syncwarp();
    const int t = cfg.flat_spec[a];
    const int kk = a - cfg.specs[t].flat_offset;
    double* dst = kp.obs[t] + (env * static_cast<uint64_t>(cfg.specs[t].count) + kk) * dim;
    for (int j = lane; j < dim; j += kWarp) dst[j] = out[j];
    __syncwarp();
  }

  __device__ static double fmin_ref(double a, double x) { return x < a ? x : a; }  // std::min(a, x)
  __device__ static double qty_feature(int64_t q, int64_t order_size) {
    return static_cast<double>(q) / static_cast<double>(q + (order_size > 1 ? order_size : 1));
  }
  __device__ static double offset_feature(int64_t own, int64_t touch, bool bid_side) {
    if (own < 0 || touch < 0) return -1.0;
    const double off = static_cast<double>(bid_side ? touch - own : own - touch);
    const double lo = -16.0 < off ? off : -16.0;
    return lo < 16.0 ? lo : 16.0;
  }

  __device__ void outcomes(bool write_rewards) {
    L2Lvl* l2b = sm.l2;
    L2Lvl* l2a = sm.l2 + cfg.obs_depth;
    const int nb = l2_levels<0>(l2b);
    const int na = l2_levels<1>(l2a);
    for (int a = 0; a < cfg.n_agents; ++a) {
      if (write_rewards) {
        const double r = compute_reward(a);
        if (lane == 0) {
          kp.rewards[env * cfg.n_agents + a] = r;
          kp.dones[env * cfg.n_agents + a] = terminal ? 1 : 0;
        }
      }
      fill_info(a);
      build_observation(a, l2b, nb, l2a, na);
    }
  }

  __device__ void clear_step_acc() {
    const int A = cfg.n_agents;
    for (int i = lane; i < A; i += kWarp) sm.acc[i] = StepAcc{0.0, 0, {0, 0}, {0, 0}, 0, 0};
    n_fills = 0;
    fill_overflow = false;
    __syncwarp();
  }

  // ---- reset (env.hpp:143-192, book.hpp:41-60) ---------------------------
  __device__ bool reset(uint64_t ep, bool write_rewards) {
    const EpState es = kp.ep_state[ep];
    if (!es.valid) {
      err |= kErrMissingState;
      return false;
    }
    if (static_cast<int>(es.nb) > cfg.capacity || static_cast<int>(es.na) > cfg.capacity) {
      err |= kErrTooDeep;
      return false;
    }
    episode = ep;
    const DevLevel* lv = kp.levels + es.level_offset;
    init_side<0>(lv, es.nb, cfg.synth_id_base, 0);
    init_side<1>(lv + es.nb, es.na, cfg.synth_id_base + es.nb, es.nb);
    next_seq = es.nb + es.na;
    live0 = static_cast<int>(es.nb);
    live1 = static_cast<int>(es.na);
    best0 = es.nb ? lv[0].price : 0;
    best1 = es.na ? lv[es.nb].price : 0;
    mid_half = cfg.fallback_mid_half;
    update_mid();
    prev_mid_half = mid_half;
    mbar = static_cast<double>(mid_half) / 2.0;
    last_bid = live0 > 0 ? static_cast<int64_t>(best0) : mid_half / 2 - 1;
    last_ask = live1 > 0 ? static_cast<int64_t>(best1) : (mid_half + 1) / 2 + 1;
    step = 0;
    terminal = false;
    n_trades = 0;
    const int A = cfg.n_agents;
    for (int a = 0; a < A; ++a) {
      const DevSpec& sp = cfg.specs[cfg.flat_spec[a]];
      AgentRec st;
      st.inventory = 0;
      st.cash = 0;
      st.filled_total = 0;
      st.slippage_total = 0.0;
      st.nonce = 0;
      st.n_active = 0;
      st.p_init = static_cast<double>(mid_half) / 2.0;
      st.task_dir = sm.ag[a].task_dir;
      if (sp.type == MLOB_EXECUTOR) {
        uint64_t h = splitmix64(seed);
        h = key_fold(h, genv);
        h = key_fold(h, ep);
        h = key_fold(h, 0);
        h = key_fold(h, kRngTaskDir);
        h = key_fold(h, static_cast<uint64_t>(a));
        Rng r{h};
        st.task_dir = r.coin() ? MLOB_TASK_BUY : MLOB_TASK_SELL;
        st.task_remaining = sp.task_size;
      } else {
        st.task_remaining = 0;
      }
      __syncwarp();
      if (lane == 0) sm.ag[a] = st;
    }
    __syncwarp();
    clear_step_acc();
    for (int a = 0; a < A && write_rewards; ++a)
      if (lane == 0) {
        kp.rewards[env * A + a] = 0.0;
        kp.dones[env * A + a] = 0;
      }
    outcomes(false);
    return true;
  }

  template <int S>
  __device__ void init_side(const DevLevel* lv, uint32_t n, uint64_t id_base, uint32_t seq_base) {
    SideT& d = sd<S>();
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
      const uint32_t i = static_cast<uint32_t>(k * kWarp + lane);
      if (i < n) {
        const uint64_t id = id_base + i;
        d.put(k, lv[i].price, lv[i].qty, static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32),
              (seq_base + i) << 8);
      } else {
        d.put(k, empty_price<S>(), 0, 0, 0, kEmptySt);
      }
    }
  }

  __device__ uint64_t episode_for(uint64_t k) const {  // rollout.hpp:286-288
    const uint64_t i = (genv + k * kp.n_envs_global) % kp.pool_len;
    return kp.pool ? kp.pool[i] : i;
  }
};

// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void mbar_expect_copy(uint64_t* bar, void* dst, const void* src,
                                                 uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__host__ __device__ inline size_t warp_smem_bytes(const DevCfg& c) {
  const int chunk = c.mps < kChunk ? c.mps : kChunk;
  const int nbuf = c.mps > kChunk ? 2 : 1;
  size_t b = 0;
  b += static_cast<size_t>(nbuf) * chunk * sizeof(DevMsg);
  b += 16;  // mbarriers
  b += static_cast<size_t>(4 * c.n_agents + 4) * sizeof(DevMsg);
  b += static_cast<size_t>(c.n_agents) * sizeof(AgentRec);
  b += static_cast<size_t>(c.n_agents) * kMaxActive * sizeof(ActiveRec);
  b += static_cast<size_t>(c.n_agents) * sizeof(StepAcc);
  b += kFillLog * sizeof(FillEnt);
  b += static_cast<size_t>(2 * c.obs_depth) * sizeof(L2Lvl);
  b += static_cast<size_t>(c.max_obs_dim + 1) * sizeof(double);
  return (b + 127) / 128 * 128;
}

__device__ WarpSmem carve(char* base, const DevCfg& c) {
  WarpSmem s;
  const int chunk = c.mps < kChunk ? c.mps : kChunk;
  const int nbuf = c.mps > kChunk ? 2 : 1;
  char* p = base;
  s.chunk[0] = reinterpret_cast<DevMsg*>(p);
  s.chunk[1] = nbuf == 2 ? s.chunk[0] + chunk : s.chunk[0];
  p += static_cast<size_t>(nbuf) * chunk * sizeof(DevMsg);
  s.bar = reinterpret_cast<uint64_t*>(p);
  p += 16;
  s.amsg = reinterpret_cast<DevMsg*>(p);
  p += static_cast<size_t>(4 * c.n_agents + 4) * sizeof(DevMsg);
  s.ag = reinterpret_cast<AgentRec*>(p);
  p += static_cast<size_t>(c.n_agents) * sizeof(AgentRec);
  s.act = reinterpret_cast<ActiveRec*>(p);
  p += static_cast<size_t>(c.n_agents) * kMaxActive * sizeof(ActiveRec);
  s.acc = reinterpret_cast<StepAcc*>(p);
  p += static_cast<size_t>(c.n_agents) * sizeof(StepAcc);
  s.fills = reinterpret_cast<FillEnt*>(p);
  p += kFillLog * sizeof(FillEnt);
  s.l2 = reinterpret_cast<L2Lvl*>(p);
  p += static_cast<size_t>(2 * c.obs_depth) * sizeof(L2Lvl);
  s.obs = reinterpret_cast<double*>(p);
  return s;
}

constexpr int kWarpsPerBlock = 4;

// K1+K2: one environment step per warp (MarketEnv::step, env.hpp:194-254,
// + MarketVecEnv::step_one auto-reset, rollout.hpp:290-318).
template <int SPL>
__global__ void __launch_bounds__(kWarpsPerBlock * kWarp)
    step_kernel(const __grid_constant__ KParams kp) {
  extern __shared__ __align__(128) char smem[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const uint64_t env = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + warp;
  if (env >= kp.n_envs) return;
  const DevCfg& cfg = kp.cfg;
  WarpSmem sm = carve(smem + warp * warp_smem_bytes(cfg), cfg);
  WarpEnv<SPL> w(kp, sm, env, lane);
  w.load_hdr();

  const int mps = cfg.mps;
  const DevMsg* slice = kp.msgs + kp.ep_start[w.episode] + static_cast<uint64_t>(w.step) * mps;
  const int n_chunks = (mps + kChunk - 1) / kChunk;
  if (mps > 0 && lane == 0) {
    mbar_init(&sm.bar[0]);
    mbar_init(&sm.bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int c = 0; c < 2 && c < n_chunks; ++c) {
      const int n = min(kChunk, mps - c * kChunk);
      mbar_expect_copy(&sm.bar[c], sm.chunk[c], slice + c * kChunk, n * sizeof(DevMsg));
    }
  }
  w.load_book();
  w.load_agents();
  w.clear_step_acc();
  const int64_t step_time = mps > 0 ? slice[0].time : w.last_time + 1;

  // (1) actions -> agent messages, (2) Fisher-Yates (rng.hpp:63-71)
  int n_amsg = 0;
  for (int a = 0; a < cfg.n_agents; ++a) w.convert_action(a, step_time, n_amsg);
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
        const DevMsg t = sm.amsg[i];
        sm.amsg[i] = sm.amsg[j];
        sm.amsg[j] = t;
      }
    }
  }
  __syncwarp();

  // (3) + (4): agent messages, then the replay slice
  w.prev_mid_half = w.mid_half;
  w.mid_sum = 0;
  w.mid_count = 0;
  w.n_trades = 0;
  for (int i = 0; i < n_amsg; ++i) {
    const DevMsg m = sm.amsg[i];
    w.run_message(m);
  }
  for (int c = 0; c < n_chunks; ++c) {
    const int b = c & 1;
    mbar_wait(&sm.bar[b], static_cast<uint32_t>((c >> 1) & 1));
    const int n = min(kChunk, mps - c * kChunk);
    const DevMsg* buf = sm.chunk[b];
    for (int i = 0; i < n; ++i) {
      const DevMsg m = buf[i];
      w.run_message(m);
    }
    if (c + 2 < n_chunks) {
      __syncwarp();
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int n2 = min(kChunk, mps - (c + 2) * kChunk);
        mbar_expect_copy(&sm.bar[b], sm.chunk[b], slice + (c + 2) * kChunk, n2 * sizeof(DevMsg));
      }
    }
  }
  if (w.live0 > 0) w.last_bid = w.best0;
  if (w.live1 > 0) w.last_ask = w.best1;

  // (5) outcomes
  w.mbar = w.mid_count > 0 ? static_cast<double>(w.mid_sum) / (2.0 * static_cast<double>(w.mid_count))
                           : static_cast<double>(w.prev_mid_half) / 2.0;
  if (w.fill_overflow && lane == 0) atomicAdd(kp.fill_overflow, 1ull);
  w.rebuild_active();
  ++w.step;
  w.terminal = w.step >= cfg.steps_per_episode;
  w.outcomes(true);

  uint8_t just_reset = 0;
  if (w.terminal && (kp.flags & MLOB_VENV_AUTO_RESET)) {
    const int A = cfg.n_agents;
    for (int a = 0; a < A; ++a) {  // rollout.hpp:300-313
      if (lane == 0) {
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
    }
    ++w.ep_finished;
    const uint64_t ep = w.episode_for(w.cursor);
    ++w.cursor;
    if (w.reset(ep, false)) just_reset = 1;
  }
  w.store_all(just_reset);
}

// K3: MarketEnv::reset for every env (reset_all / reset_envs).
template <int SPL>
__global__ void __launch_bounds__(kWarpsPerBlock * kWarp)
    reset_kernel(const __grid_constant__ KParams kp) {
  extern __shared__ __align__(128) char smem[];
  const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
  const uint64_t env = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + warp;
  if (env >= kp.n_envs) return;
  const DevCfg& cfg = kp.cfg;
  WarpSmem sm = carve(smem + warp * warp_smem_bytes(cfg), cfg);
  WarpEnv<SPL> w(kp, sm, env, lane);
  w.load_hdr();  // keeps last_time / messages_processed / cursor across resets
  w.load_agents();
  w.reset(kp.reset_episodes[env], true);
  w.cursor = 1;
  w.store_all(1);
}

// K4: per-type episode-stat sums over this handle's envs (for the NCCL
// all-reduce), 5 doubles per type: pv, slip, completion, inv², episodes.
__global__ void stats_kernel(const __grid_constant__ KParams kp, double* out) {
  const int t = blockIdx.y;
  const DevCfg& cfg = kp.cfg;
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

__global__ void clear_finished_kernel(EnvHdr* hdr, uint64_t n) {
  for (uint64_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    hdr[e].episodes_finished = 0;
}

// ---------------------------------------------------------------------------
// host-side launchers

static unsigned grid_for(uint64_t n) {
  const uint64_t b = (n + 255) / 256;
  return static_cast<unsigned>(b < 1184 ? (b > 0 ? b : 1) : 1184);
}

cudaError_t launch_sum_msgs(const EnvHdr* hdr, uint64_t n, unsigned long long* out, cudaStream_t s) {
  sum_msgs_kernel<<<grid_for(n), 256, 0, s>>>(hdr, n, out);
  return cudaGetLastError();
}

cudaError_t launch_clear_finished(EnvHdr* hdr, uint64_t n, cudaStream_t s) {
  clear_finished_kernel<<<grid_for(n), 256, 0, s>>>(hdr, n);
  return cudaGetLastError();
}

size_t step_smem_bytes(const DevCfg& c) { return warp_smem_bytes(c) * kWarpsPerBlock; }

template <int SPL>
static cudaError_t launch_step_t(const KParams& kp, cudaStream_t s) {
  const size_t sm = step_smem_bytes(kp.cfg);
  cudaError_t e = cudaFuncSetAttribute(step_kernel<SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm));
  if (e != cudaSuccess) return e;
  const unsigned blocks = static_cast<unsigned>((kp.n_envs + kWarpsPerBlock - 1) / kWarpsPerBlock);
  step_kernel<SPL><<<blocks, kWarpsPerBlock * kWarp, sm, s>>>(kp);
  return cudaGetLastError();
}

template <int SPL>
static cudaError_t launch_reset_t(const KParams& kp, cudaStream_t s) {
  const size_t sm = step_smem_bytes(kp.cfg);
  cudaError_t e = cudaFuncSetAttribute(reset_kernel<SPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(sm));
  if (e != cudaSuccess) return e;
  const unsigned blocks = static_cast<unsigned>((kp.n_envs + kWarpsPerBlock - 1) / kWarpsPerBlock);
  reset_kernel<SPL><<<blocks, kWarpsPerBlock * kWarp, sm, s>>>(kp);
  return cudaGetLastError();
}

int slots_per_lane(int capacity) {
  const int need = (capacity + kWarp - 1) / kWarp;
  if (need <= 1) return 1;
  if (need <= 2) return 2;
  if (need <= 4) return 4;
  if (need <= 8) return 8;
  return -1;
}

cudaError_t launch_step(const KParams& kp, int spl, cudaStream_t s) {
  switch (spl) {
    case 1: return launch_step_t<1>(kp, s);
    case 2: return launch_step_t<2>(kp, s);
    case 4: return launch_step_t<4>(kp, s);
    case 8: return launch_step_t<8>(kp, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_reset(const KParams& kp, int spl, cudaStream_t s) {
  switch (spl) {
    case 1: return launch_reset_t<1>(kp, s);
    case 2: return launch_reset_t<2>(kp, s);
    case 4: return launch_reset_t<4>(kp, s);
    case 8: return launch_reset_t<8>(kp, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_stats(const KParams& kp, double* out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double) * 5 * kp.cfg.n_specs, s);
  if (e != cudaSuccess) return e;
  const uint64_t nb = (kp.n_envs + 255) / 256;
  const unsigned bx = static_cast<unsigned>(nb < 1184 ? nb : 1184);
  stats_kernel<<<dim3(bx > 0 ? bx : 1, kp.cfg.n_specs), 256, 0, s>>>(kp, out);
  return cudaGetLastError();
}

}  // namespace mlob
