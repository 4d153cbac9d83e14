// mlob_step.cuh — the warp-per-environment book state machine (book_kernel,
// stages (3)+(4) of MarketEnv::step; the thread-per-env stages live in
// mlob_thread.cuh).
//
// One warp owns one environment for a whole step:
//   * the env's book is loaded from HBM into registers (SoA rows of 32 slots,
//     lane l owns slots l, l+32, ...; C <= 256) or, for deep books, bulk-copied
//     into shared memory in the HBM layout (4-word slots, C <= 1024);
//   * the step's replay slice is staged global->shared with cp.async.bulk
//     (TMA bulk copy, mbarrier completion), overlapped with the book load;
//   * every book operation is warp-cooperative: best price / oldest order by
//     redux.sync min/max, order-id lookup by match counting, free-slot search
//     by ballot;
//   * the handlers are specialised on the message's side (one dispatch per
//     message) and the trade log is a template parameter: the message loop is
//     bound by instruction issue and fetch, and its register budget (72 at 28
//     warps per SM) decides its speed;
//   * agent fills are appended to the env's fill log in fill order for the
//     outcome kernel; the L2 summary, active orders and header go back to HBM.
// Reference semantics followed (paths under /root/reference/proj/include/marlob):
//   lob/book.hpp:65-220, env/env.hpp:143-503, agents/*.hpp, core/rng.hpp,
//   ippo/rollout.hpp:290-318, bench/bench.hpp:53-70.
// Compiled with --fmad=false so every double expression rounds exactly like
// the reference's x86-64 build (no FMA contraction).
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <type_traits>

#include "mlob_dev.h"

// Crossing orders walk a whole price level by a warp prefix sum over the
// resting quantities (walk_level_t).  Bit-exact (40 GPU parity tests) but
// 2.5x slower on C / E than one fill per iteration (2.07e9 vs 5.12e9 on C):
// a crossing order fills ~2.4 orders, so the compaction, rank and update
// passes cost more than they save, and the extra code pushes the 72-register
// message loop into spills (470 B vs 288 B).  Off by default; DESIGN.md §4.
#ifndef MLOB_PREFIX_WALK
#define MLOB_PREFIX_WALK 0
#endif
#ifndef MLOB_EXPECT  // branch-probability hints on the rare paths of the message loop (+0.7 % on C)
#define MLOB_EXPECT 1
#endif
#if MLOB_EXPECT
#define MLOB_LIKELY(x) __builtin_expect(!!(x), 1)
#define MLOB_UNLIKELY(x) __builtin_expect(!!(x), 0)
#else
#define MLOB_LIKELY(x) (x)
#define MLOB_UNLIKELY(x) (x)
#endif

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
  // next() % n, computed without the 64-bit modulo subroutine call when n < 2^16:
  // x mod n = ((hi mod n) * (2^32 mod n) + lo mod n) mod n, all in 32 bits.
  __device__ __forceinline__ uint64_t below(uint64_t n) {
    const uint64_t x = next();
    if (n <= 0xffffu) {
      const uint32_t m = static_cast<uint32_t>(n);
      const uint32_t hi = static_cast<uint32_t>(x >> 32), lo = static_cast<uint32_t>(x);
      const uint32_t p32 = (0xffffffffu % m + 1u) % m;
      return ((hi % m) * p32 + lo % m) % m;
    }
    return x % n;
  }
  __device__ __forceinline__ bool coin() { return (next() & 1ull) != 0; }
};
enum : uint64_t { kRngShuffle = 1, kRngTaskDir = 2, kRngBenchAction = 7, kRngEpisodeDraw = 8 };

// ---------------------------------------------------------------------------
// Book side held in registers: SPL rows of 32 slots (lane-major).
// Empty slot: q == 0, p == side sentinel (bid INT_MIN, ask INT_MAX), st == ~0.
// st = arrival_seq << 8 | trader_id, so a u32 min over st is a min over seq.
template <int SPL>
struct RegSide {
  int32_t p_[SPL], q_[SPL];
  uint32_t st_[SPL];
  uint32_t lo_[SPL], hi_[SPL];
  __device__ __forceinline__ uint32_t LO(int k) const { return lo_[k]; }
  __device__ __forceinline__ uint32_t HI(int k) const { return hi_[k]; }
  __device__ __forceinline__ uint2 ID(int k) const { return make_uint2(lo_[k], hi_[k]); }
  __device__ __forceinline__ void put_id(int k, uint32_t lo, uint32_t hi) {
    lo_[k] = lo;
    hi_[k] = hi;
  }
  __device__ __forceinline__ int32_t P(int k) const { return p_[k]; }
  __device__ __forceinline__ int32_t Q(int k) const { return q_[k]; }
  __device__ __forceinline__ uint32_t ST(int k) const { return st_[k]; }
  __device__ __forceinline__ void put(int k, int32_t p, int32_t q, uint32_t lo, uint32_t hi,
                                      uint32_t st) {
    p_[k] = p;
    q_[k] = q;
    put_id(k, lo, hi);
    st_[k] = st;
  }
  // compile-time row K, runtime predicate.  The asm text differs per row
  // (the "row K" comment), so LLVM cannot merge the per-row branches of
  // insert_t into one runtime-indexed write (that demotes the book to local
  // memory).
#define MLOB_PUT_IF(K)                                                                          \
  asm volatile("{\n.reg .pred pp; // row " #K "\nsetp.ne.b32 pp, %5, 0;\n@pp mov.b32 %0, %6;\n"    \
               "@pp mov.b32 %1, %7;\n@pp mov.b32 %2, %8;\n@pp mov.b32 %3, %9;\n@pp mov.b32 %4, %10;\n}" \
               : "+r"(p_[K]), "+r"(q_[K]), "+r"(lo_[K]), "+r"(hi_[K]), "+r"(st_[K])                 \
               : "r"(static_cast<uint32_t>(pred)), "r"(p), "r"(q), "r"(lo), "r"(hi), "r"(st))
  template <int K>
  __device__ __forceinline__ void put_if(bool pred, int32_t p, int32_t q, uint32_t lo, uint32_t hi, uint32_t st) {
    static_assert(K < SPL && K < 8, "row");
    if constexpr (K == 0) MLOB_PUT_IF(0);
    else if constexpr (K == 1) MLOB_PUT_IF(1);
    else if constexpr (K == 2) MLOB_PUT_IF(2);
    else if constexpr (K == 3) MLOB_PUT_IF(3);
    else if constexpr (K == 4) MLOB_PUT_IF(4);
    else if constexpr (K == 5) MLOB_PUT_IF(5);
    else if constexpr (K == 6) MLOB_PUT_IF(6);
    else MLOB_PUT_IF(7);
  }
#undef MLOB_PUT_IF
  // first row K.. with a free lane (ballots b), warp-uniform branches
  template <int K>
  __device__ __forceinline__ void insert_rows(const uint32_t* b, int lane, int32_t p, int32_t q, uint32_t lo,
                                              uint32_t hi, uint32_t st) {
    if constexpr (K < SPL) {
      if (b[K])
        put_if<K>(lane == __ffs(b[K]) - 1, p, q, lo, hi, st);
      else
        insert_rows<K + 1>(b, lane, p, q, lo, hi, st);
    }
  }
  // compile-time row k, runtime predicate (no select chain over rows)
  // (st is left stale: every st query names a live order, st values are
  // never reused within an episode, and empty slots are excluded by their
  // sentinel price / zero quantity everywhere else)
  __device__ __forceinline__ void clear_row(int k, bool pred, int32_t empty_p) {
    if (pred) {
      p_[k] = empty_p;
      q_[k] = 0;
    }
  }
  __device__ __forceinline__ void setq_row(int k, bool pred, int32_t q) {
    if (pred) q_[k] = q;
  }
};

// Book side in shared memory (deep books, capacity > 256): same interface as
// RegSide.  Slots are laid out in groups of four rows: slot (row k, lane l)
// of an array at [(k / 4) * 128 + l * 4 + k % 4], so one 16-byte
// ld.shared.v4 brings a lane four consecutive rows and a warp's v4 load of a
// group is conflict-free; the row scans (best price, oldest at a price, id
// candidates, worst price) take SPL / 4 loads instead of SPL.
template <int SPL>
struct SmemSide {
  static_assert(SPL % 4 == 0, "rows in groups of four");
  // Four words per slot, in the HBM layout of one side of a deep book (so
  // whole arrays move with bulk copies): p[SPL*32]; qt = qty << 8 | trader;
  // lo = order id bits 0..31; hs = order id bits 32..43 << 20 | arrival_seq.
  // Four words instead of five is what fits a sixth 36.5 KB warp per SM at
  // C = 1000.  Limits (loud errors, kErrDeepRange): qty < 2^24, order ids
  // < 2^44, arrival_seq < 2^20 per episode.
  uint32_t* base_;
  int32_t* p_;
  uint32_t* qt_;
  uint32_t* lo_;
  uint32_t* hs_;
  uint32_t occ;  // this lane's occupied rows (bit k = row k), kept by every mutator
  // this lane's worst live price (bids: lowest, asks: highest; identity when
  // none), widened on inserts; a removal at that price marks it stale
  int32_t lw;
  uint32_t lw_stale;
  int side_;
  // word offset of row k from this lane's base (compile-time for unrolled k)
  __device__ __forceinline__ static int at(int k) { return (k >> 2) * 128 + (k & 3); }
  __device__ __forceinline__ int4 P4(int g) const { return *reinterpret_cast<const int4*>(p_ + g * 128); }
  __device__ __forceinline__ uint4 QT4(int g) const { return *reinterpret_cast<const uint4*>(qt_ + g * 128); }
  __device__ __forceinline__ uint4 LO4(int g) const { return *reinterpret_cast<const uint4*>(lo_ + g * 128); }
  __device__ __forceinline__ int32_t worse(int32_t a, int32_t b) const { return side_ ? max(a, b) : min(a, b); }
  __device__ __forceinline__ void occ_set(int k, bool on) {
    const uint32_t b = 1u << k;
    occ = on ? (occ | b) : (occ & ~b);
  }
  __device__ __forceinline__ uint32_t free_mask() const {
    return ~occ & (SPL >= 32 ? 0xffffffffu : ((1u << SPL) - 1u));
  }
  // this lane's worst live price, rescanned from the price rows under the
  // occupancy mask (a per-lane count at the worst price measured -30 % on D)
  __device__ __forceinline__ void refresh_lw() {
    lw = side_ ? INT_MIN : INT_MAX;
#pragma unroll
    for (int g = 0; g < SPL / 4; ++g) {
      const int4 p = P4(g);
      const uint32_t o = occ >> (4 * g);
      lw = (o & 1u) ? worse(lw, p.x) : lw;
      lw = (o & 2u) ? worse(lw, p.y) : lw;
      lw = (o & 4u) ? worse(lw, p.z) : lw;
      lw = (o & 8u) ? worse(lw, p.w) : lw;
    }
    lw_stale = 0;
  }
  // occupancy and worst price together, one pass (book load)
  __device__ __forceinline__ void recompute_occ() {
    occ = 0;
    lw = side_ ? INT_MIN : INT_MAX;
#pragma unroll
    for (int g = 0; g < SPL / 4; ++g) {
      const int4 p = P4(g);
      const uint4 qt = QT4(g);
      const int32_t pv[4] = {p.x, p.y, p.z, p.w};
      const uint32_t qv[4] = {qt.x, qt.y, qt.z, qt.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool live = (qv[j] >> 8) != 0;
        occ |= (live ? 1u : 0u) << (4 * g + j);
        lw = live ? worse(lw, pv[j]) : lw;
      }
    }
    lw_stale = 0;
  }
  __device__ __forceinline__ int32_t P(int k) const { return p_[at(k)]; }
  __device__ __forceinline__ int32_t Q(int k) const { return static_cast<int32_t>(qt_[at(k)] >> 8); }
  __device__ __forceinline__ uint32_t LO(int k) const { return lo_[at(k)]; }
  __device__ __forceinline__ uint32_t HI(int k) const { return hs_[at(k)] >> 20; }
  // the reference record's arrival word seq << 8 | trader (ordered like seq)
  __device__ __forceinline__ uint32_t ST(int k) const {
    return ((hs_[at(k)] & 0xfffffu) << 8) | (qt_[at(k)] & 0xffu);
  }
  __device__ __forceinline__ void put(int k, int32_t p, int32_t q, uint32_t lo, uint32_t hi,
                                      uint32_t st) {
    p_[at(k)] = p;
    qt_[at(k)] = (static_cast<uint32_t>(q) << 8) | (st & 0xffu);
    lo_[at(k)] = lo;
    hs_[at(k)] = (hi << 20) | ((st >> 8) & 0xfffffu);
    occ_set(k, q > 0);
    if (q > 0) lw = worse(lw, p);
  }
  __device__ __forceinline__ void get_pq(int k, int32_t& p, int32_t& q) const {
    p = p_[at(k)];
    q = Q(k);
  }
  __device__ __forceinline__ void get_qid(int k, int32_t& q, uint32_t& lo, uint32_t& hi) const {
    q = Q(k);
    lo = lo_[at(k)];
    hi = hs_[at(k)] >> 20;
  }
  __device__ __forceinline__ void set(int k, bool pred, int32_t p, int32_t q, uint32_t lo,
                                      uint32_t hi, uint32_t st) {
    if (pred) put(k, p, q, lo, hi, st);
  }
  __device__ __forceinline__ void set_u(int k, bool pred, int32_t p, int32_t q, uint32_t lo,
                                        uint32_t hi, uint32_t st) {
    set(k, pred, p, q, lo, hi, st);
  }
  __device__ __forceinline__ void setq(int k, bool pred, int32_t q) {
    if (pred) qt_[at(k)] = (static_cast<uint32_t>(q) << 8) | (qt_[at(k)] & 0xffu);
  }
  __device__ __forceinline__ void clear(int k, bool pred, int32_t empty_p) {
    if (pred) {
      if (p_[at(k)] == lw) lw_stale = 1;
      p_[at(k)] = empty_p;
      qt_[at(k)] = 0;
      occ_set(k, false);
    }
  }
  __device__ __forceinline__ void bind(uint32_t* base, int lane, int side) {  // 4 x SPL*32 words
    side_ = side;
    lw = side ? INT_MIN : INT_MAX;
    lw_stale = 1;
    occ = 0;
    base_ = base;
    p_ = reinterpret_cast<int32_t*>(base) + lane * 4;
    qt_ = base + SPL * 32 + lane * 4;
    lo_ = base + 2 * SPL * 32 + lane * 4;
    hs_ = base + 3 * SPL * 32 + lane * 4;
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

struct ActTmp {  // one agent-owned resting order, rebuild_active scratch (fits a DevMsg slot)
  int32_t price;
  uint32_t st;
  uint32_t lo, hi;
  int32_t qty;
  int32_t _pad;
};
static_assert(sizeof(ActTmp) <= sizeof(DevMsg), "ActTmp reuses the agent-message smem");

// Per-warp shared-memory regions.  The region offsets are the same for every
// warp of a block (they depend on the config only), so they live once in a
// block-shared table and a warp keeps only its base pointer: eleven 64-bit
// region pointers held in registers across the message loop forced spills
// at the 80-register cap.
struct SmemOff {
  uint32_t chunk0, chunk1, bar, amsg, act, nact, scal, l2, walk, _pad[3];
};
// One resting order of the price level being walked (walk_level_t).
struct WalkEnt {
  uint32_t st;
  int32_t q;
  int32_t fill;
  int32_t order;  // the entry filled at this priority rank
};
__shared__ __align__(16) SmemOff g_smem_off;  // written once per block by carve_block()
struct WarpSmem {
  char* base;
  __device__ __forceinline__ DevMsg* chunk0() const { return reinterpret_cast<DevMsg*>(base + g_smem_off.chunk0); }
  __device__ __forceinline__ DevMsg* chunk1() const { return reinterpret_cast<DevMsg*>(base + g_smem_off.chunk1); }
  __device__ __forceinline__ uint64_t* bar() const { return reinterpret_cast<uint64_t*>(base + g_smem_off.bar); }
  __device__ __forceinline__ DevMsg* amsg() const { return reinterpret_cast<DevMsg*>(base + g_smem_off.amsg); }
  __device__ __forceinline__ ActiveRec* act() const { return reinterpret_cast<ActiveRec*>(base + g_smem_off.act); }
  __device__ __forceinline__ int32_t* nact() const { return reinterpret_cast<int32_t*>(base + g_smem_off.nact); }
  __device__ __forceinline__ int32_t* scal() const { return reinterpret_cast<int32_t*>(base + g_smem_off.scal); }
  __device__ __forceinline__ L2Lvl* l2() const { return reinterpret_cast<L2Lvl*>(base + g_smem_off.l2); }
  __device__ __forceinline__ WalkEnt* walk() const { return reinterpret_cast<WalkEnt*>(base + g_smem_off.walk); }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 32-byte message record from shared memory (explicit ld.shared: the generic
// pointer would otherwise compile to a generic LD).
__device__ __forceinline__ DevMsg lds_msg(const DevMsg* p) {
  uint4 a, b;
  const uint32_t s = smem_u32(p);
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "r"(s));
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+16];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "r"(s));
  DevMsg m;
  m.time = static_cast<int64_t>((static_cast<uint64_t>(a.y) << 32) | a.x);
  m.order_id = (static_cast<uint64_t>(a.w) << 32) | a.z;
  m.price = static_cast<int32_t>(b.x);
  m.qty = static_cast<int32_t>(b.y);
  m.kind = static_cast<uint8_t>(b.z & 0xffu);
  m.side = static_cast<uint8_t>((b.z >> 8) & 0xffu);
  m._pad = 0;
  m.trader = static_cast<int32_t>(b.w);
  return m;
}

// A staged message in the loop: the hot fields (price, qty, kind, side,
// trader: one 16-byte ld.shared) live in registers; the order id and time are
// re-read from shared memory where they are used (rest, id lookup, trade
// record), which keeps four registers free across the fill loop.
struct MsgRef {
  uint32_t a;  // shared-window address of the record
  int32_t price, qty;
  int32_t kind, side;  // kind widened once at the load; side: nonzero = ask
  int32_t trader;
  __device__ __forceinline__ uint64_t order_id() const {
    uint32_t lo, hi;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2+8];" : "=r"(lo), "=r"(hi) : "r"(a) : "memory");
    return (static_cast<uint64_t>(hi) << 32) | lo;
  }
  __device__ __forceinline__ int64_t time() const {
    uint32_t lo, hi;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(a) : "memory");
    return static_cast<int64_t>((static_cast<uint64_t>(hi) << 32) | lo);
  }
};
__device__ __forceinline__ MsgRef lds_hot_a(uint32_t a) {
  MsgRef m;
  m.a = a;
  uint32_t x, y, z, w;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4+16];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(m.a));
  m.price = static_cast<int32_t>(x);
  m.qty = static_cast<int32_t>(y);
  m.kind = static_cast<int32_t>(z & 0xffu);
  m.side = static_cast<int32_t>(z & 0xff00u);  // only tested against zero (one LOP3 to a predicate)
  m.trader = static_cast<int32_t>(w);
  return m;
}
__device__ __forceinline__ MsgRef lds_hot(const DevMsg* p) { return lds_hot_a(smem_u32(p)); }

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

// bulk copy global -> shared completing on `bar` without an arrive (the
// caller arrives once with the total byte count)
__device__ __forceinline__ void bulk_load_tx(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// bulk copy shared -> global (bulk async-group)
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
#if MLOB_CHECKS  // a lost bulk copy would hang: trap after ~2^28 polls instead
  for (uint32_t spin = 0;; ++spin) {
    uint32_t done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    MLOB_CHECK(spin < (1u << 28));
  }
#endif
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// row loop over a side's SPL rows, unrolled kUnr at a time
#define MLOB_ROWS(k)                                        \
  _Pragma("unroll 1") for (int k##_g = 0; k##_g < SPL; k##_g += kUnr) \
  _Pragma("unroll") for (int k = k##_g; k < k##_g + kUnr; ++k)
// the shared-memory book's candidate-filter scans (id, oldest at a price,
// best price) with their own unroll width
#define MLOB_SCAN_ROWS(k)                                      \
  _Pragma("unroll 1") for (int k##_g = 0; k##_g < SPL; k##_g += kScanUnr) \
  _Pragma("unroll") for (int k = k##_g; k < k##_g + kScanUnr; ++k)
#ifndef MLOB_SCAN_UNR  // candidate-filter scans fully unrolled: 32 loads in flight
#define MLOB_SCAN_UNR 32
#endif
template <int SPL, bool REC, bool SMEM = (SPL > 8)>
struct WarpEnv {
  using SideT = typename std::conditional<SMEM, SmemSide<SPL>, RegSide<SPL>>::type;
  // rows per unrolled group: all rows for register books (a full unroll keeps
  // them in registers); for shared-memory books the candidate-filter scans
  // (id, oldest at a price, best price) unroll fully — 32 independent
  // ld.shared in flight, D +17 % over groups of 4 — and every other row loop
  // runs in groups of 4 (since the side-specialised handlers: +3 % on D over
  // groups of 2, 8 no better; 1 is -3 %).  An explicit `#pragma unroll N` on
  // the row loops changes the register-book code (measured -11% on config C),
  // hence the two-level loop below.
#ifndef MLOB_SMEM_UNR  // shared-memory books: rows per unrolled group (measured: 4)
#define MLOB_SMEM_UNR 4
#endif
  static constexpr int kUnr = (SMEM && SPL >= MLOB_SMEM_UNR) ? MLOB_SMEM_UNR : SPL;
  static constexpr int kScanUnr = (SMEM && SPL >= MLOB_SCAN_UNR) ? MLOB_SCAN_UNR : SPL;
  SideT bid, ask;
  const KParams& kp;
  const DevCfg& cfg;
  WarpSmem sm;
  int lane;
  uint64_t env;
  // uniform state (identical in every lane)
  int live0, live1;
  int32_t best0, best1;
  uint32_t next_seq;
  int64_t mid_half;
  int64_t mid_sum, mid_count;
  uint32_t n_trades;
  uint32_t n_fills, fill_head, fill_cur;  // agent-fill log (inline, then overflow chunks)
  uint32_t n_amsg;
  uint32_t err;
  // config words cached in registers (measured: reading them from the staged
  // shared-memory copy at each use is 4% slower)
  int capacity_, n_agents_;
  __device__ __forceinline__ int capacity() const { return capacity_; }
  // the trade log is a template parameter (a runtime flag in the fill loop
  // measured 5 % on config C: its register and branches)
  static __device__ __forceinline__ constexpr bool rec_trades() { return REC; }
  // register books: n_agents read from the staged config (only the rare
  // agent-fill path uses it) and an error met inside the message loop goes
  // straight to the handle's word — no register live across the loop for
  // either (C +2.5 %; the deep-book kernel keeps both: D -4 % otherwise)
  __device__ __forceinline__ int n_agents() const {
    if constexpr (SMEM)
      return n_agents_;
    else
      return cfg.n_agents;
  }
  __device__ __forceinline__ void loop_error(uint32_t bits) {
    if constexpr (SMEM) {
      err |= bits;
    } else if (lane == 0) {
      atomicOr(kp.error, bits);
    }
  }
  int nb_l2, na_l2;      // top-D level counts (snapshot)
  int64_t topq0, topq1;  // level-0 aggregated qty per side
  int64_t sumq0, sumq1;  // Σ qty over the top-D levels per side

  // book_smem: deep books only, [2 sides][5 arrays][SPL*32] words
  __device__ WarpEnv(const KParams& p, const DevCfg& c, const WarpSmem& s, uint64_t e, int ln,
                     uint32_t* book_smem)
      : kp(p), cfg(c), sm(s), lane(ln), env(e) {
    if constexpr (SMEM) {
      bid.bind(book_smem, ln, 0);
      ask.bind(book_smem + 4 * SPL * 32, ln, 1);
    }
    err = 0;
    capacity_ = c.capacity;
    n_agents_ = c.n_agents;
  }

  __device__ __forceinline__ void bind(uint64_t e) {
    MLOB_CHECK(e < kp.n_envs);
    env = e;
  }

  template <int S>
  __device__ __forceinline__ SideT& sd() {
    if constexpr (S == 0)
      return bid;
    else
      return ask;
  }

  // ---- HBM <-> registers --------------------------------------------------
  __device__ __forceinline__ size_t row_index(int s, int k) const {
    return ((env * 2 + static_cast<uint64_t>(s)) * SPL + static_cast<uint64_t>(k)) * kWarp + lane;
  }
  template <int S>
  __device__ __forceinline__ void load_side(int hwm) {
    SideT& d = sd<S>();
    MLOB_ROWS(k) {
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
    if constexpr (SMEM) {  // from the occupancy masks: one redux + one ballot
      const uint32_t rows = __reduce_or_sync(FULLMASK, d.occ);
      if (rows) {
        const int k = 31 - __clz(rows);
        hwm = k * kWarp + 32 - __clz(__ballot_sync(FULLMASK, (d.occ >> k) & 1u));
      }
    } else {
      MLOB_ROWS(k) {
        const uint32_t b = __ballot_sync(FULLMASK, d.Q(k) > 0);
        if (b) hwm = k * kWarp + 32 - __clz(b);
      }
    }
    if constexpr (SMEM) {  // rows below the high-water mark: four bulk stores
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // lanes' smem writes -> async proxy
      __syncwarp();
      // whole four-row groups (the grouped layout's contiguous prefix)
      const uint32_t rows = static_cast<uint32_t>((hwm + 4 * kWarp - 1) / (4 * kWarp) * 4);
      if (lane == 0 && rows) {
        const size_t g = (env * 2 + S) * SPL * kWarp;
        const uint32_t* b = d.base_;
        bulk_store(kp.bk_p + g, b, rows * kWarp * 4);
        bulk_store(kp.bk_q + g, b + SPL * kWarp, rows * kWarp * 4);
        bulk_store(reinterpret_cast<uint32_t*>(kp.bk_id) + g, b + 2 * SPL * kWarp, rows * kWarp * 4);
        bulk_store(kp.bk_st + g, b + 3 * SPL * kWarp, rows * kWarp * 4);
      }
    } else {
      MLOB_ROWS(k) {
        if (k * kWarp < hwm) {
          const size_t i = row_index(S, k);
          kp.bk_p[i] = d.P(k);
          kp.bk_q[i] = d.Q(k);
          if constexpr (SMEM)
            kp.bk_id[i] = make_uint2(d.LO(k), d.HI(k));
          else
            kp.bk_id[i] = d.ID(k);
          kp.bk_st[i] = d.ST(k);
        }
      }
    }
    return hwm;
  }

  // Only the state the message loop needs is held in registers; the rest of
  // the header is advanced in place after the loop (store_hdr).
  __device__ __forceinline__ void load_hdr() {
    EnvHdr& h = kp.hdr[env];
    mid_half = h.mid_half;
    next_seq = h.next_seq;
    live0 = h.live[0];
    live1 = h.live[1];
    best0 = h.best[0];
    best1 = h.best[1];
    n_amsg = h.n_amsg;
    __syncwarp();
    if (lane == 0) h.prev_mid_half = mid_half;  // env.hpp:220: the step's starting mid
  }
  __device__ __forceinline__ void load_book() {
    const EnvHdr& h = kp.hdr[env];
    load_side<0>(h.hwm[0]);
    load_side<1>(h.hwm[1]);
    if constexpr (SMEM) {
      bid.recompute_occ();
      ask.recompute_occ();
    }
  }
  int hwm0, hwm1;
  // chunk stager: copy #q goes to buffer q & 1 and completes phase (q >> 1) & 1
  // of that buffer's mbarrier.  Copies run ahead of consumption by <= 2.
  uint32_t q_issued = 0, q_consumed = 0;
  __device__ __forceinline__ void stage(const DevMsg* src, int n) {
    __syncwarp();
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const int b = q_issued & 1;
      bulk_copy(b ? sm.chunk1() : sm.chunk0(), src, static_cast<uint32_t>(n * sizeof(DevMsg)),
                b ? &sm.bar()[1] : &sm.bar()[0]);
    }
    ++q_issued;
  }
  __device__ __forceinline__ const DevMsg* staged() {
    const int b = q_consumed & 1;
    bar_wait(b ? &sm.bar()[1] : &sm.bar()[0], (q_consumed >> 1) & 1);
    ++q_consumed;
    return b ? sm.chunk1() : sm.chunk0();
  }
  // Shared-memory books: the rows below each side's high-water mark arrive by
  // bulk copies issued right after the header (they overlap the action
  // conversion); lanes fill the rows above with empty slots.  Register books
  // load at book_load_wait().
  uint32_t book_loads = 0;  // mbarrier [2] phase
  __device__ __forceinline__ void book_load_issue() {
    if constexpr (SMEM) {
      const EnvHdr& h = kp.hdr[env];
      // whole four-row groups below the high-water marks (stored / reset as groups)
      const int rows0 = (h.hwm[0] + 4 * kWarp - 1) / (4 * kWarp) * 4, rows1 = (h.hwm[1] + 4 * kWarp - 1) / (4 * kWarp) * 4;
      for (int k = rows0; k < SPL; ++k) bid.put(k, INT_MIN, 0, 0, 0, kEmptySt);
      for (int k = rows1; k < SPL; ++k) ask.put(k, INT_MAX, 0, 0, 0, kEmptySt);
      if (lane == 0) {
        bar_arrive_tx(&sm.bar()[2], static_cast<uint32_t>(rows0 + rows1) * kWarp * 16u);
#pragma unroll
        for (int S = 0; S < 2; ++S) {
          const uint32_t rows = static_cast<uint32_t>(S ? rows1 : rows0);
          if (rows == 0) continue;
          const size_t g = (env * 2 + S) * SPL * kWarp;
          uint32_t* b = S ? ask.base_ : bid.base_;
          bulk_load_tx(b, kp.bk_p + g, rows * kWarp * 4, &sm.bar()[2]);
          bulk_load_tx(b + SPL * kWarp, kp.bk_q + g, rows * kWarp * 4, &sm.bar()[2]);
          bulk_load_tx(b + 2 * SPL * kWarp, reinterpret_cast<const uint32_t*>(kp.bk_id) + g, rows * kWarp * 4,
                       &sm.bar()[2]);
          bulk_load_tx(b + 3 * SPL * kWarp, kp.bk_st + g, rows * kWarp * 4, &sm.bar()[2]);
        }
      }
    }
  }
  __device__ __forceinline__ void book_load_wait() {
    if constexpr (SMEM) {
      bar_wait(&sm.bar()[2], book_loads & 1);
      ++book_loads;
      __syncwarp();
      bid.recompute_occ();
      ask.recompute_occ();
    } else {
      load_book();
    }
  }
  __device__ __forceinline__ void store_book() {
    hwm0 = store_side<0>();
    hwm1 = store_side<1>();
    if constexpr (SMEM) {  // the bulk stores must have read the rows before they change
      if (lane == 0) {
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncwarp();
    }
  }
  __device__ __forceinline__ void book_store_drain() {  // before the kernel ends
    if constexpr (SMEM) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  }
  // The header fields the book kernel advances (the outcome kernel owns the
  // rest: episode bookkeeping, auto-reset): MarketEnv::step's tail after
  // the message loop (env.hpp:233-247).  `slice` is the step's replay slice.
  __device__ __forceinline__ void store_hdr(const DevMsg* slice) {
    const int h0 = hwm0, h1 = hwm1;
    if (lane == 0) {
      EnvHdr& h = kp.hdr[env];
      const int mps = cfg.mps;
      const int total = static_cast<int>(n_amsg) + mps;
      h.msgs_processed += static_cast<uint64_t>(total);
      if (total > 0) h.last_time = mps > 0 ? slice[mps - 1].time : lds_msg(sm.amsg() + n_amsg - 1).time;
      if (live0 > 0) h.last_bid = best0;  // env.hpp:238-239
      if (live1 > 0) h.last_ask = best1;
      h.mbar = mid_count > 0 ? static_cast<double>(mid_sum) / (2.0 * static_cast<double>(mid_count))
                             : static_cast<double>(h.prev_mid_half) / 2.0;  // env.hpp:242-244
      const int step = h.step + 1;
      h.step = step;
      h.terminal = step >= cfg.steps_per_episode ? 1 : 0;
      h.mid_half = mid_half;
      h.next_seq = next_seq;
      h.live[0] = static_cast<uint16_t>(live0);
      h.live[1] = static_cast<uint16_t>(live1);
      h.hwm[0] = static_cast<uint16_t>(h0);
      h.hwm[1] = static_cast<uint16_t>(h1);
      h.best[0] = best0;
      h.best[1] = best1;
      h.n_trades = REC ? n_trades : 0;  // counted only with the trade log (mlob_venv_read_trades)
      h.n_fills = n_fills;
      h.fill_head = fill_head;
    }
  }
  __device__ __forceinline__ void report_errors() {
    if (err && lane == 0) atomicOr(kp.error, err);
  }
  // this step's agent messages (act_kernel's hand-off) into shared memory
  __device__ __forceinline__ void load_agent_msgs() {
    MLOB_CHECK(n_amsg <= kp.amsg_cap);
    const uint4* src = reinterpret_cast<const uint4*>(kp.amsg + env * kp.amsg_cap);
    uint4* dst = reinterpret_cast<uint4*>(sm.amsg());
    for (uint32_t i = lane; i < 2 * n_amsg; i += kWarp) dst[i] = src[i];
    __syncwarp();
  }

  // ---- per-side scan primitives (the only side-specialised hot code) ------
  template <int S>
  __device__ __forceinline__ int32_t side_best_t() {
    SideT& d = sd<S>();
    int32_t b = empty_price<S>();
    if constexpr (SMEM) {  // four rows per 16-byte load
#pragma unroll
      for (int g = 0; g < SPL / 4; ++g) {
        const int4 v = d.P4(g);
        b = better_of<S>(better_of<S>(b, v.x), better_of<S>(v.y, better_of<S>(v.z, v.w)));
      }
    } else {
      MLOB_SCAN_ROWS(k) b = better_of<S>(b, d.P(k));
    }
    return redux_best<S>(b);
  }
  // lane-local oldest slot (min st) at `price`
  template <int S>
  __device__ __forceinline__ void scan_oldest_t(int32_t price, uint32_t& m, int& lk) {
    SideT& d = sd<S>();
    m = kEmptySt;
    lk = 0;
    if constexpr (SMEM && SPL <= 32) {
      // shared-memory book: one load per row for the price, the arrival word
      // only for the (few) rows at that price
      uint32_t cand = 0;
#pragma unroll
      for (int g = 0; g < SPL / 4; ++g) {
        const int4 v = d.P4(g);
        cand |= ((v.x == price ? 1u : 0u) | (v.y == price ? 2u : 0u) | (v.z == price ? 4u : 0u) |
                 (v.w == price ? 8u : 0u)) << (4 * g);
      }
      while (cand) {
        const int k = __ffs(cand) - 1;
        cand &= cand - 1;
        const uint32_t st = d.ST(k);
        if (st < m) {
          m = st;
          lk = k;
        }
      }
    } else {
      MLOB_ROWS(k) {
        const bool c = d.P(k) == price && d.ST(k) < m;
        m = c ? d.ST(k) : m;
        lk = c ? k : lk;
      }
    }
  }
  // lane-local id match: first matching row and match count
  template <int S>
  __device__ __forceinline__ void scan_id_t(uint32_t lo, uint32_t hi, int& nm, int& lk) {
    SideT& d = sd<S>();
    nm = 0;
    lk = 0;
    if constexpr (SMEM && SPL <= 32) {
      // shared-memory book: filter rows on the low id word (one load per row),
      // then check the high word and liveness of the candidates only
      uint32_t cand = 0;
#pragma unroll
      for (int g = 0; g < SPL / 4; ++g) {
        const uint4 v = d.LO4(g);
        cand |= ((v.x == lo ? 1u : 0u) | (v.y == lo ? 2u : 0u) | (v.z == lo ? 4u : 0u) | (v.w == lo ? 8u : 0u))
                << (4 * g);
      }
      while (cand) {
        const int k = __ffs(cand) - 1;
        cand &= cand - 1;
        if (d.HI(k) == hi && d.Q(k) > 0) {
          if (nm == 0) lk = k;
          ++nm;
        }
      }
    } else {
      MLOB_ROWS(k) {
        const bool c = d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi;
        lk = (c && nm == 0) ? k : lk;
        nm += c ? 1 : 0;
      }
    }
  }
  // lowest free position (row-major: row * 32 + lane) -> (row, lane), one
  // redux.min over each lane's lowest free row
  template <int S>
  __device__ __forceinline__ void free_slot_t(int& pk, int& pl) {
    SideT& d = sd<S>();
    uint32_t fm = 0;
    if constexpr (SMEM)
      fm = d.free_mask();  // maintained occupancy: no row scan
    else
      MLOB_ROWS(k) fm |= (d.Q(k) == 0 ? 1u : 0u) << k;
    const uint32_t key = fm ? (static_cast<uint32_t>(__ffs(fm) - 1) << 5) | static_cast<uint32_t>(lane)
                            : 0xffffffffu;
    const uint32_t g = __reduce_min_sync(FULLMASK, key);
    pk = static_cast<int>(g >> 5);
    pl = static_cast<int>(g & 31u);
  }
  __device__ __forceinline__ void slot_get_pq(int s, int k, int32_t& p, int32_t& q) const {
    if (s)
      ask.get_pq(k, p, q);
    else
      bid.get_pq(k, p, q);
  }
  __device__ __forceinline__ void slot_get_qid(int s, int k, int32_t& q, uint32_t& lo, uint32_t& hi) const {
    if (s)
      ask.get_qid(k, q, lo, hi);
    else
      bid.get_qid(k, q, lo, hi);
  }
  __device__ __forceinline__ void slot_setq(int s, int k, bool pred, int32_t q) {
    if (s)
      ask.setq(k, pred, q);
    else
      bid.setq(k, pred, q);
  }
  __device__ __forceinline__ void slot_clear(int s, int k, bool pred) {
    if (s)
      ask.clear(k, pred, INT_MAX);
    else
      bid.clear(k, pred, INT_MIN);
  }

  // Eviction on a full side (book.hpp:174-181): drop the newcomer unless it
  // improves on the worst price, else remove the oldest order at the worst.
  template <int S>
  __device__ __forceinline__ bool evict_t(int32_t price) {
    SideT& d = sd<S>();
    int32_t lw = S == 0 ? INT_MAX : INT_MIN;
    if constexpr (SMEM) {  // the side's cached per-lane worst, rescanned by stale lanes only
      if (__any_sync(FULLMASK, d.lw_stale)) {
        if (d.lw_stale) d.refresh_lw();
        __syncwarp();
      }
      lw = d.lw;
    } else {
      MLOB_ROWS(k) if (d.Q(k) > 0) lw = S == 0 ? min(lw, d.P(k)) : max(lw, d.P(k));
    }
    const int32_t worst = S == 0 ? __reduce_min_sync(FULLMASK, lw) : __reduce_max_sync(FULLMASK, lw);
    const bool better = S == 0 ? price > worst : price < worst;
    if (!better) return false;
    if constexpr (SMEM) {
      uint32_t m;
      int lk;
      scan_oldest_t<S>(worst, m, lk);
      const uint32_t g = __reduce_min_sync(FULLMASK, m);
      const int owner = __ffs(__ballot_sync(FULLMASK, m == g)) - 1;
      d.clear(lk, lane == owner, empty_price<S>());
    } else {  // register book: the oldest at the worst price by its arrival word
      clear_st_t<S>(oldest_st_t<S>(worst));
    }
    return true;
  }
  // Duplicate live ids: the reference takes the first match in storage order
  // (book.hpp:191-206; bids: lowest price then newest; asks: highest, newest).
  template <int S>
  __device__ __forceinline__ int dup_owner_t(uint32_t lo, uint32_t hi, int& lk) {
    SideT& d = sd<S>();
    int32_t kp_ = S == 0 ? INT_MAX : INT_MIN;
    MLOB_ROWS(k) {
      const bool c = d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi;
      if (c) kp_ = S == 0 ? min(kp_, d.P(k)) : max(kp_, d.P(k));
    }
    const int32_t gp = S == 0 ? __reduce_min_sync(FULLMASK, kp_) : __reduce_max_sync(FULLMASK, kp_);
    uint32_t ms = 0;
    bool any = false;
    MLOB_ROWS(k) {
      const bool c = d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi && d.P(k) == gp;
      if (c && (!any || d.ST(k) > ms)) {
        ms = d.ST(k);
        lk = k;
        any = true;
      }
    }
    const uint32_t gs = __reduce_max_sync(FULLMASK, any ? ms : 0u);
    return __ffs(__ballot_sync(FULLMASK, any && ms == gs)) - 1;
  }

  // ---- register books: slots addressed by content, not by (row, lane) ----
  // The arrival word `st` is unique within a book (one sequence counter for
  // both sides, book.hpp:183), so the oldest order at a price is named by its
  // st: a lane-local min, one redux.min, then the winner's fields gathered by
  // a one-hot redux.or and the slot updated where ST == st.  No row index,
  // owner ballot or shuffle sits on the fill chain.
  template <int S>
  __device__ __forceinline__ uint32_t oldest_st_t(int32_t price) {
    SideT& d = sd<S>();
    uint32_t m = kEmptySt;
    MLOB_ROWS(k) m = min(m, d.P(k) == price ? d.ST(k) : kEmptySt);
    return __reduce_min_sync(FULLMASK, m);
  }
  template <int S>
  __device__ __forceinline__ int32_t q_of_st_t(uint32_t st, bool ids, uint32_t& lo, uint32_t& hi) {
    SideT& d = sd<S>();
    uint32_t qv = 0;
    MLOB_ROWS(k) qv = d.ST(k) == st ? static_cast<uint32_t>(d.Q(k)) : qv;  // one-hot: a select chain
    if (MLOB_UNLIKELY(ids)) {  // the passive order's id (trade log only)
      uint32_t lv = 0, hv = 0;
      MLOB_ROWS(k) {
        const bool h = d.ST(k) == st;
        lv = h ? d.LO(k) : lv;
        hv = h ? d.HI(k) : hv;
      }
      lo = __reduce_or_sync(FULLMASK, lv);
      hi = __reduce_or_sync(FULLMASK, hv);
    }
    return static_cast<int32_t>(__reduce_or_sync(FULLMASK, qv));
  }
  template <int S>
  __device__ __forceinline__ void clear_st_t(uint32_t st) {
    SideT& d = sd<S>();
    MLOB_ROWS(k) d.clear_row(k, d.ST(k) == st, empty_price<S>());
  }
  template <int S>
  __device__ __forceinline__ void setq_st_t(uint32_t st, int32_t q) {
    SideT& d = sd<S>();
    MLOB_ROWS(k) d.setq_row(k, d.ST(k) == st, q);
  }
  // insert at the lowest free position (row-major), book.hpp:183-186 (any
  // free slot would do: priority is carried by st): one ballot per row, the
  // first row with a free lane taken by a warp-uniform branch, so only that
  // row's five registers are written (a runtime row index compiles to
  // selects over every row)
  template <int S>
  __device__ __forceinline__ void insert_t(int32_t p, int32_t q, uint32_t lo, uint32_t hi, uint32_t st) {
    SideT& d = sd<S>();
    uint32_t b[SPL];
    MLOB_ROWS(k) b[k] = __ballot_sync(FULLMASK, d.Q(k) == 0);
    d.template insert_rows<0>(b, lane, p, q, lo, hi, st);
  }
  // id lookup: live matches counted warp-wide; for a unique match its price,
  // quantity and st are gathered one-hot (duplicates take the slow path)
  template <int S>
  __device__ __forceinline__ uint32_t id_gather_t(uint32_t lo, uint32_t hi, int32_t& p, int32_t& q,
                                                  uint32_t& st) {
    SideT& d = sd<S>();
    uint32_t n = 0, pv = 0, qv = 0, sv = 0;
    MLOB_ROWS(k) {
      const bool c = d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi;
      n += c ? 1u : 0u;
      // select chains: the gathered values are used only when the match is
      // unique warp-wide (then one lane has exactly one matching row)
      pv = c ? static_cast<uint32_t>(d.P(k)) : pv;
      qv = c ? static_cast<uint32_t>(d.Q(k)) : qv;
      sv = c ? d.ST(k) : sv;
    }
    const uint32_t tot = __reduce_add_sync(FULLMASK, n);
    // gathered whenever there is a match (duplicates are re-resolved by the
    // caller): a two-way branch, where tot == 0 / 1 / > 1 compiled to a jump
    // table (BRX through the constant bank)
    if (tot != 0) {
      p = static_cast<int32_t>(__reduce_or_sync(FULLMASK, pv));
      q = static_cast<int32_t>(__reduce_or_sync(FULLMASK, qv));
      st = __reduce_or_sync(FULLMASK, sv);
    }
    return tot;
  }

  // The order walk of process_new_limit (book.hpp:154-165) over one whole
  // price level at once, by a warp prefix sum over the resting quantities in
  // priority order: the level's orders are compacted into shared memory, each
  // one's priority rank and the quantity resting ahead of it (Σ q of the
  // orders with a smaller arrival word) give its fill min(q, max(0, rem −
  // ahead)); the trades are then recorded in priority order and every slot
  // of the level is updated in place.  Returns the remaining quantity.
  template <int S>
  __device__ __forceinline__ int32_t walk_level_t(int32_t bp, int32_t rem, const MsgRef& m, int aside) {
    SideT& d = sd<S>();
    WalkEnt* w = sm.walk();
    const uint32_t lt = (1u << lane) - 1u;
    int n = 0;
    MLOB_ROWS(k) {
      const bool at = d.P(k) == bp;
      const uint32_t b = __ballot_sync(FULLMASK, at);
      if (at) {
        WalkEnt& e = w[n + __popc(b & lt)];
        e.st = d.ST(k);
        e.q = d.Q(k);
      }
      n += __popc(b);
    }
    __syncwarp();
    for (int i = lane; i < n; i += kWarp) {
      const WalkEnt e = w[i];
      int64_t ahead = 0;
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const WalkEnt f = w[j];
        const bool before = f.st < e.st;
        ahead += before ? f.q : 0;
        rank += before ? 1 : 0;
      }
      const int64_t left = static_cast<int64_t>(rem) - ahead;
      w[i].fill = left <= 0 ? 0 : static_cast<int32_t>(min(left, static_cast<int64_t>(e.q)));
      w[rank].order = i;
    }
    __syncwarp();
    // trades in priority order (env.hpp:226-229 attribution order)
    int32_t total = 0;
    for (int r = 0; r < n; ++r) {
      const WalkEnt e = w[w[r].order];
      if (e.fill == 0) break;
      total += e.fill;
      uint32_t idlo = 0, idhi = 0;
      if (MLOB_UNLIKELY(rec_trades())) q_of_st_t<S>(e.st, true, idlo, idhi);
      record_trade(bp, e.fill, m, idlo, idhi, e.st, aside);
    }
    // every slot of the level: quantity down by its fill, filled orders removed
    int base = 0, cleared = 0;
    MLOB_ROWS(k) {
      const bool at = d.P(k) == bp;
      const uint32_t b = __ballot_sync(FULLMASK, at);
      int32_t nq = 1;
      if (at) {
        nq = d.Q(k) - w[base + __popc(b & lt)].fill;
        if (nq == 0)
          d.clear_row(k, true, empty_price<S>());
        else
          d.setq_row(k, true, nq);
      }
      cleared += __popc(__ballot_sync(FULLMASK, at && nq == 0));
      base += __popc(b);
    }
    __syncwarp();  // the walk scratch is reused by the next level
    if (cleared) {
      moved = true;
      int& live = S ? live1 : live0;
      live -= cleared;
      if (cleared == n && live > 0) (S ? best1 : best0) = side_best_t<S>();
    }
    return rem - total;
  }

  // Duplicate live ids on a register book: the reference takes the first
  // match in storage order (book.hpp:191-206; bids: lowest price then newest,
  // asks: highest price then newest): the price by one reduction, then the
  // newest arrival word at that price by another.  Returns its st; p = price.
  template <int S>
  __device__ __forceinline__ uint32_t dup_st_t(uint32_t lo, uint32_t hi, int32_t& p) {
    SideT& d = sd<S>();
    int32_t kp_ = S == 0 ? INT_MAX : INT_MIN;
    MLOB_ROWS(k) {
      if (d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi) kp_ = S == 0 ? min(kp_, d.P(k)) : max(kp_, d.P(k));
    }
    p = S == 0 ? __reduce_min_sync(FULLMASK, kp_) : __reduce_max_sync(FULLMASK, kp_);
    uint32_t ms = 0;
    MLOB_ROWS(k) {
      if (d.Q(k) > 0 && d.LO(k) == lo && d.HI(k) == hi && d.P(k) == p) ms = max(ms, d.ST(k));
    }
    return __reduce_max_sync(FULLMASK, ms);
  }

  // ---- message handlers (runtime side) -------------------------------------
  __device__ __forceinline__ void record_trade(int32_t price, int32_t qty, const MsgRef& m,
                                               uint32_t lo, uint32_t hi, uint32_t st, int aside) {
    if (MLOB_UNLIKELY(rec_trades()) && lane == 0 && n_trades < kp.trade_cap) {
      mlob_trade t;
      t.price = price;
      t.quantity = qty;
      t.time = m.time();
      t.passive_order_id = (static_cast<uint64_t>(hi) << 32) | lo;
      t.aggressor_order_id = m.order_id();
      t.passive_trader_id = static_cast<int32_t>(st & 0xffu);
      t.aggressor_trader_id = m.trader;
      t.aggressor_side = static_cast<uint8_t>(aside);
#pragma unroll
      for (int i = 0; i < 7; ++i) t._pad[i] = 0;
      kp.trades[env * kp.trade_cap + n_trades] = t;
    }
    if constexpr (REC) ++n_trades;
    const uint32_t pt = st & 0xffu;
    if (MLOB_UNLIKELY(pt | static_cast<uint32_t>(m.trader))) {  // an agent may be involved: env.hpp:372-379 order
      // passive side, then the aggressor: one copy of the (cold) append code
      // per call site instead of two inside the message loop's code span
      // (C +1 %, E +1.8 %: the loop is instruction-fetch sensitive)
#pragma unroll 1
      for (int e = 0; e < 2; ++e) log_fill(price, qty, e ? m.trader : static_cast<int>(pt), e ? aside : 1 - aside);
    }
  }

  // Appends one agent-side fill to the env's log (inline entries, then
  // overflow chunks taken from the launch's pool).  Called by every lane with
  // the same arguments; lane 0 writes.
  __device__ __forceinline__ void log_fill(int32_t price, int32_t qty, int trader, int side) {
    if (trader <= 0 || trader > n_agents()) return;
    const uint32_t i = n_fills;
    FillEnt* dst;
    if (MLOB_LIKELY(i < static_cast<uint32_t>(kFillInline))) {
      dst = kp.fills + env * kFillInline + i;
    } else {
      const uint32_t k = i - kFillInline, off = k % (kFillChunk - 1) + 1;
      if (off == 1) {  // a new overflow chunk, linked from the previous one
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(kp.fill_pool_ctr, 1u);
        c = __shfl_sync(FULLMASK, c, 0);
        if (c >= kp.fill_pool_chunks) {
          loop_error(kErrFillPool);
          return;
        }
        if (k == 0)
          fill_head = c;
        else if (lane == 0)
          kp.fill_pool[static_cast<size_t>(fill_cur) * kFillChunk].price = static_cast<int32_t>(c);
        fill_cur = c;
      }
      MLOB_CHECK(fill_cur < kp.fill_pool_chunks && off < kFillChunk);
      dst = kp.fill_pool + static_cast<size_t>(fill_cur) * kFillChunk + off;
    }
    if (lane == 0) *dst = FillEnt{price, qty, trader - 1, side};
    n_fills = i + 1;
  }

  bool moved;  // a top (best price or side emptiness) changed: refresh the mid

  // side-specialised handlers: the message's side is dispatched once per
  // message (C +10.6 %, E +8.7 %, D +6 % over handlers branching on a runtime
  // side at every use)
  template <int S>
  __device__ __forceinline__ int& live_() {
    if constexpr (S == 0)
      return live0;
    else
      return live1;
  }
  template <int S>
  __device__ __forceinline__ int32_t& best_() {
    if constexpr (S == 0)
      return best0;
    else
      return best1;
  }
  // book.hpp:150-187 (process_new_limit + rest_order), S: the order's side
  template <int S>
  __device__ __forceinline__ void new_limit_t(const MsgRef& m) {
    constexpr int O = S ^ 1;
    int32_t rem = m.qty;
    const bool pass_ids = rec_trades();
    while (rem > 0) {
      const int32_t bp = best_<O>();
      // a buy crosses asks at or below its price, a sell bids at or above
      if (live_<O>() == 0 || (S == 0 ? bp > m.price : bp < m.price)) break;
      if constexpr (!SMEM) {
        const uint32_t gst = oldest_st_t<O>(bp);
        uint32_t idlo = 0, idhi = 0;
        const int32_t q = q_of_st_t<O>(gst, pass_ids, idlo, idhi);
        if (MLOB_PREFIX_WALK && q < rem) {  // the order walk goes past the level's oldest order
          rem = walk_level_t<O>(bp, rem, m, S);
          continue;
        }
        const int32_t fill = min(rem, q);
        rem -= fill;
        if (fill == q) {
          moved = true;
          clear_st_t<O>(gst);
          if (--live_<O>() > 0) best_<O>() = side_best_t<O>();
        } else {
          setq_st_t<O>(gst, q - fill);
        }
        record_trade(bp, fill, m, idlo, idhi, gst, S);
      } else {  // shared-memory (deep) books
        uint32_t lm;
        int lk;
        scan_oldest_t<O>(bp, lm, lk);
        const uint32_t gst = __reduce_min_sync(FULLMASK, lm);
        const int owner = __ffs(__ballot_sync(FULLMASK, lm == gst)) - 1;
        int32_t q;
        uint32_t idlo, idhi;
        slot_get_qid(O, lk, q, idlo, idhi);
        q = __shfl_sync(FULLMASK, q, owner);
        if (pass_ids) {
          idlo = __shfl_sync(FULLMASK, idlo, owner);
          idhi = __shfl_sync(FULLMASK, idhi, owner);
        }
        const int32_t fill = min(rem, q);
        const bool me = lane == owner;
        rem -= fill;
        if (fill == q) {
          slot_clear(O, lk, me);
          moved = true;
          if (--live_<O>() > 0) best_<O>() = side_best_t<O>();
        } else {
          slot_setq(O, lk, me, q - fill);
        }
        record_trade(bp, fill, m, idlo, idhi, gst, S);
      }
    }
    if (rem <= 0) return;
    // rest_order
    if (live_<S>() == capacity()) {
      if (!evict_t<S>(m.price)) return;  // newcomer dropped: no sequence number consumed
      moved = true;
      --live_<S>();
    }
    const uint32_t seq = next_seq++;  // range checked once after the loop (process_messages)
    const uint32_t st = (seq << 8) | static_cast<uint32_t>(m.trader & 0xff);
    const uint32_t ilo = static_cast<uint32_t>(m.order_id()), ihi = static_cast<uint32_t>(m.order_id() >> 32);
    if constexpr (!SMEM) {
      insert_t<S>(m.price, rem, ilo, ihi, st);
    } else {
      if (rem >= (1 << 24) || ihi >= (1u << 12) || seq >= (1u << 20)) loop_error(kErrDeepRange);  // 4-word slot
      int pk, pl;
      free_slot_t<S>(pk, pl);
      sd<S>().set_u(pk, lane == pl, m.price, rem, ilo, ihi, st);
    }
    if (++live_<S>() == 1 || (S == 0 ? m.price > best_<S>() : m.price < best_<S>())) {
      best_<S>() = m.price;
      moved = true;
    }
  }

  // book.hpp:189-207 (reduce_order / remove_order); absent ids are no-ops.
  template <int S>
  __device__ __forceinline__ bool by_id_t(const MsgRef& m, bool remove) {
    const uint32_t lo = static_cast<uint32_t>(m.order_id()), hi = static_cast<uint32_t>(m.order_id() >> 32);
    if constexpr (!SMEM) {
      int32_t p = 0, q = 0;
      uint32_t st = 0;
      const uint32_t tot = id_gather_t<S>(lo, hi, p, q, st);
      if (tot == 0) return false;
      if (MLOB_UNLIKELY(tot > 1)) {  // duplicate live ids: the first in storage order
        st = dup_st_t<S>(lo, hi, p);
        uint32_t ilo, ihi;
        q = q_of_st_t<S>(st, false, ilo, ihi);
      }
      const int32_t nq = remove ? 0 : q - min(q, m.qty);
      if (nq == 0) {
        clear_st_t<S>(st);
        if (--live_<S>() > 0 && p == best_<S>()) best_<S>() = side_best_t<S>();
        return true;
      }
      setq_st_t<S>(st, nq);
      return false;
    } else {  // shared-memory (deep) books
      int nm, lk;
      scan_id_t<S>(lo, hi, nm, lk);
      const uint32_t b = __ballot_sync(FULLMASK, nm > 0);
      if (b == 0) return false;
      int owner = __ffs(b) - 1;
      if (__reduce_add_sync(FULLMASK, static_cast<uint32_t>(nm)) != 1) owner = dup_owner_t<S>(lo, hi, lk);
      int32_t p, q;
      slot_get_pq(S, lk, p, q);
      p = __shfl_sync(FULLMASK, p, owner);
      q = __shfl_sync(FULLMASK, q, owner);
      const int32_t nq = remove ? 0 : q - min(q, m.qty);
      const bool me = lane == owner;
      if (nq == 0) {
        slot_clear(S, lk, me);
        if (--live_<S>() > 0 && p == best_<S>()) best_<S>() = side_best_t<S>();
        return true;
      }
      slot_setq(S, lk, me, nq);
      return false;
    }
  }

  // env.hpp:230: the mid follows the tops; it is refreshed only on the paths
  // that can move a top (any NewLimit, removals), not per message.
  // mid_sum (Σ of the mid after every message) is accumulated lazily: at a
  // mid change after message j (index within the step) the messages
  // mid_anchor..j-1 carried the old mid; the remainder is folded in after
  // the loop.  No per-message counter (a counter register was spilled: two
  // local loads and a store per message).
  // The fold state lives in shared memory (scal[2] anchor, scal[3] segment
  // base, scal[4..5] Σmid): it is touched only at mid changes, so it holds no
  // register across the loop.  m_a: the message record's shared address.
  __device__ __forceinline__ void refresh_mid(uint32_t m_a) {
    const int64_t b0 = best0, b1 = best1;
    const int64_t nm = live0 > 0 ? (live1 > 0 ? b0 + b1 : 2 * b0) : (live1 > 0 ? 2 * b1 : mid_half);
    if (nm != mid_half) {
      int32_t* sc = sm.scal();
      const int j = sc[3] + static_cast<int32_t>(m_a >> 5);  // sc[3]: segment base - (first record's address >> 5)
      int64_t& ms = *reinterpret_cast<int64_t*>(sc + 4);
      ms += mid_half * (j - sc[2]);
      sc[2] = j;
      mid_half = nm;
    }
  }

  // book.hpp:65-86 + env.hpp:223-235 (mid_count / last_time / messages are
  // derived once after the loop: they only depend on the message count).
  __device__ __forceinline__ void run_message(const MsgRef& m) {
    if (m.kind == MLOB_NEW_LIMIT) {
      if (m.qty > 0) {
        moved = false;
        if (m.side)
          new_limit_t<1>(m);
        else
          new_limit_t<0>(m);
        if (moved) refresh_mid(m.a);
      }
    } else if (m.kind <= MLOB_EXECUTE_VISIBLE) {
      const bool del = m.kind == MLOB_DELETE;
      if (m.side ? by_id_t<1>(m, del) : by_id_t<0>(m, del)) refresh_mid(m.a);
    }
  }

  // Agent messages, then the replay slice staged in smem chunks (env.hpp:236-237).
  // Chunk 0 (and 1) of this env were staged before the call; chunk c+2 is
  // staged once chunk c is consumed.
  __device__ __forceinline__ void process_messages(int n_amsg, const DevMsg* slice) {
    const int mps = cfg.mps;
    const int nch = (mps + kChunk - 1) / kChunk;
    {
      int32_t* sc = sm.scal();
      sc[2] = 0;
      sc[3] = 0;
      *reinterpret_cast<int64_t*>(sc + 4) = 0;
    }
    for (int seg = -1; seg < nch; ++seg) {
      const DevMsg* buf;
      int n;
      if (seg < 0) {
        buf = sm.amsg();
        n = n_amsg;
      } else {
        buf = staged();
        n = min(kChunk, mps - seg * kChunk);
        sm.scal()[3] = n_amsg + seg * kChunk;
      }
      // the loop runs over the records' shared-memory addresses (the index
      // refresh_mid needs is recovered from the address: C +2 % over a
      // counted loop, one register less across it)
      {
        const uint32_t a0 = smem_u32(buf);
        if (seg < 0) sm.scal()[3] = 0;
        sm.scal()[3] -= static_cast<int32_t>(a0 >> 5);
        for (uint32_t a = a0, e = a0 + 32u * static_cast<uint32_t>(n); a != e; a += 32u) run_message(lds_hot_a(a));
      }
      if (seg >= 0 && seg + 2 < nch) stage(slice + (seg + 2) * kChunk, min(kChunk, mps - (seg + 2) * kChunk));
    }
    __syncwarp();
    mid_sum = *reinterpret_cast<const int64_t*>(sm.scal() + 4) + mid_half * (n_amsg + mps - sm.scal()[2]);
    // next_seq only grows: some arrival sequence reached kMaxSeq iff it ends above it
    if (next_seq > kMaxSeq) err |= kErrSeqRange;
    mid_count = n_amsg + mps;
  }

  // ---- step outcomes -------------------------------------------------------
  // Top-D aggregated levels per side, best-first (book.hpp:109-120, 209-220).
  template <int S>
  __device__ __forceinline__ int l2_levels(L2Lvl* out) {
    SideT& d = sd<S>();
    const int D = cfg.obs_depth;
    int n = 0;
    int32_t prev = 0;
    for (; n < D; ++n) {
      int32_t lb = empty_price<S>();
      MLOB_ROWS(k) {
        const bool ok = d.Q(k) > 0 && (n == 0 || (S == 0 ? d.P(k) < prev : d.P(k) > prev));
        if (ok) lb = better_of<S>(lb, d.P(k));
      }
      const int32_t lvl = redux_best<S>(lb);
      if (lvl == empty_price<S>()) break;
      // per-lane sum < SPL * 2^31: reduce as 16-bit-split halves so the 32-bit
      // redux.sync add cannot overflow
      uint64_t s64 = 0;
      MLOB_ROWS(k)
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

  // env.hpp:398-407: active orders per agent, book storage order.  Agent
  // slots are compacted into smem by ballot rank, then lane 0 sorts the few
  // entries into storage order (bids worst->best, then asks) and deals them
  // out to the agents.
  __device__ __forceinline__ void rebuild_active() {
    const int A = cfg.n_agents;
    ActTmp* tmp = reinterpret_cast<ActTmp*>(sm.amsg());  // agent messages are consumed
    const int cap = static_cast<int>(kp.amsg_cap);      // DevMsg slots = ActTmp slots
    int base = 0;
    base = compact_side<0>(tmp, base, cap);
    const int nbid = base;
    base = compact_side<1>(tmp, base, cap);
    __syncwarp();
    if (lane == 0) {
      for (int a = 0; a < A; ++a) sm.nact()[a] = 0;
      const int total = base < cap ? base : cap;
      if (base > cap) err |= kErrActiveOverflow;
      // insertion sort each side into storage order: bids (price asc, seq desc),
      // asks (price desc, seq desc)
      for (int i = 1; i < total; ++i) {
        const ActTmp x = tmp[i];
        const bool bid = i < nbid;
        int j = i - 1;
        const int lo = bid ? 0 : nbid;
        while (j >= lo) {
          const ActTmp y = tmp[j];
          const bool after = y.price != x.price ? (bid ? y.price > x.price : y.price < x.price)
                                                : (y.st >> 8) < (x.st >> 8);
          if (!after) break;
          tmp[j + 1] = y;
          --j;
        }
        tmp[j + 1] = x;
      }
      for (int i = 0; i < total; ++i) {
        const ActTmp x = tmp[i];
        const int a = static_cast<int>(x.st & 0xffu) - 1;
        if (a >= A) {
          err |= kErrBadTrader;
          continue;
        }
        const int n = sm.nact()[a];
        if (n >= kMaxActive) {
          err |= kErrActiveOverflow;
          continue;
        }
        sm.act()[a * kMaxActive + n] =
            ActiveRec{(static_cast<uint64_t>(x.hi) << 32) | x.lo, x.price,
                      static_cast<uint32_t>(x.qty) | (static_cast<uint32_t>(i >= nbid) << 31)};
        sm.nact()[a] = n + 1;
      }
    }
    __syncwarp();
    // hand-off to the outcome kernel and the next step's act_kernel
    for (int a = lane; a < A; a += kWarp) kp.agents[env * A + a].n_active = sm.nact()[a];
    for (int i = lane; i < A * kMaxActive; i += kWarp)
      if (i % kMaxActive < sm.nact()[i / kMaxActive]) kp.active[env * A * kMaxActive + i] = sm.act()[i];
  }
  template <int S>
  __device__ __forceinline__ int compact_side(ActTmp* tmp, int base, int cap) {
    SideT& d = sd<S>();
    if constexpr (SMEM) {
      // shared-memory book: one pass over the arrival words (gated by the
      // occupancy mask) finds this lane's agent rows; only rows holding an
      // agent order in some lane take the ballot (same row-major order)
      uint32_t agm = 0;
      MLOB_SCAN_ROWS(k) agm |= (((d.occ >> k) & 1u) && (d.ST(k) & 0xffu) != 0 ? 1u : 0u) << k;
      uint32_t rows = __reduce_or_sync(FULLMASK, agm);
      while (rows) {
        const int k = __ffs(rows) - 1;
        rows &= rows - 1;
        const bool is_ag = (agm >> k) & 1u;
        const uint32_t b = __ballot_sync(FULLMASK, is_ag);
        const int pos = base + __popc(b & ((1u << lane) - 1u));
        if (is_ag && pos < cap) tmp[pos] = ActTmp{d.P(k), d.ST(k), d.LO(k), d.HI(k), d.Q(k), 0};
        base += __popc(b);
      }
    } else {
      MLOB_ROWS(k) {
        const bool is_ag = d.Q(k) > 0 && (d.ST(k) & 0xffu) != 0;
        const uint32_t b = __ballot_sync(FULLMASK, is_ag);
        if (b == 0) continue;
        const int pos = base + __popc(b & ((1u << lane) - 1u));
        if (is_ag && pos < cap) tmp[pos] = ActTmp{d.P(k), d.ST(k), d.LO(k), d.HI(k), d.Q(k), 0};
        base += __popc(b);
      }
    }
    return base;
  }

  // Book-dependent part of the step outcomes: L2 top-D into smem.  After this
  // (and rebuild_active) the book registers can be stored and released, so no
  // book register is live across the double-division / 64-bit-modulo
  // subroutine calls of the reward/observation code (they forced the book
  // through local memory in v1).
  __device__ __forceinline__ void snapshot() {
    if (cfg.full_l2 || !summarize_l2<0>() || !summarize_l2<1>()) {
      nb_l2 = l2_levels<0>(sm.l2());
      na_l2 = l2_levels<1>(sm.l2() + cfg.obs_depth);
      sumq0 = sumq1 = topq0 = topq1 = 0;
      for (int i = 0; i < nb_l2; ++i) sumq0 += sm.l2()[i].qty;
      for (int i = 0; i < na_l2; ++i) sumq1 += sm.l2()[cfg.obs_depth + i].qty;
      topq0 = nb_l2 > 0 ? sm.l2()[0].qty : 0;
      topq1 = na_l2 > 0 ? sm.l2()[cfg.obs_depth].qty : 0;
      if (cfg.full_l2) {  // the levels themselves, for MMFull observations
        const int D = cfg.obs_depth;
        L2Lvl* dst = kp.l2lv + env * 2 * D;
        for (int i = lane; i < 2 * D; i += kWarp)
          if ((i < D ? i < nb_l2 : i - D < na_l2)) dst[i] = sm.l2()[i];
      }
    }
    MLOB_CHECK(nb_l2 <= cfg.obs_depth && na_l2 <= cfg.obs_depth);
    MLOB_CHECK(live0 <= capacity() && live1 <= capacity() && live0 >= 0 && live1 >= 0);
    if (lane == 0) kp.l2sum[env] = L2Sum{nb_l2, na_l2, sumq0, sumq1, topq0, topq1, 0};
  }

  // Warp-sum of a per-lane value < 2^36 (16-bit split keeps redux.sync exact).
  __device__ __forceinline__ int64_t warp_sum64(uint64_t v) {
    const uint32_t lo = __reduce_add_sync(FULLMASK, static_cast<uint32_t>(v & 0xffffu));
    const uint32_t hi = __reduce_add_sync(FULLMASK, static_cast<uint32_t>(v >> 16));
    return static_cast<int64_t>(lo) + (static_cast<int64_t>(hi) << 16);
  }

  // Observation inputs without materialising the levels (MMBasic/Exec spaces):
  // the distinct prices within 32 ticks of the touch form one bitmask; if the
  // window holds the top D levels (or the whole side), the level count, the
  // top-D quantity and the touch quantity follow from two masked sums.
  template <int S>
  __device__ __forceinline__ bool summarize_l2() {
    SideT& d = sd<S>();
    const int live = S ? live1 : live0;
    const int32_t best = S ? best1 : best0;
    if (live == 0) {
      (S ? na_l2 : nb_l2) = 0;
      (S ? sumq1 : sumq0) = 0;
      (S ? topq1 : topq0) = 0;
      return true;
    }
    uint32_t m = 0;
    bool far = false;
    MLOB_ROWS(k) {
      if (d.Q(k) > 0) {
        const uint32_t off = static_cast<uint32_t>(S == 0 ? best - d.P(k) : d.P(k) - best);
        if (off < 32)
          m |= 1u << off;
        else
          far = true;
      }
    }
    const uint32_t mask = __reduce_or_sync(FULLMASK, m);
    const int D = cfg.obs_depth;
    const int nl = __popc(mask);
    if (nl < D && __any_sync(FULLMASK, far)) return false;  // levels beyond the window: slow path
    const int n = nl < D ? nl : D;
    uint32_t mm = mask;
    for (int i = 1; i < n; ++i) mm &= mm - 1;
    const uint32_t cut = static_cast<uint32_t>(__ffs(mm) - 1);  // offset of the n-th level
    uint64_t sa = 0, st = 0;
    MLOB_ROWS(k) {
      const uint32_t off = static_cast<uint32_t>(S == 0 ? best - d.P(k) : d.P(k) - best);
      const uint32_t q = d.Q(k) > 0 ? static_cast<uint32_t>(d.Q(k)) : 0u;
      sa += off <= cut ? q : 0u;
      st += off == 0 ? q : 0u;
    }
    (S ? na_l2 : nb_l2) = n;
    (S ? sumq1 : sumq0) = warp_sum64(sa);
    (S ? topq1 : topq0) = warp_sum64(st);
    return true;
  }

};

}  // namespace mlob
