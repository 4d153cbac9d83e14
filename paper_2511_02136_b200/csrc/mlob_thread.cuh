// mlob_thread.cuh — the per-environment scalar phases of the step, one THREAD
// per environment (kernels act_kernel and outcome_kernel, mlob_kernels.cu).
//
// The message loop needs a whole warp per env (book_kernel, mlob_step.cuh);
// everything around it is scalar per-env work — action decoding, the agent
// message list and its shuffle, fill accounting, rewards, infos,
// observations, episode statistics and the auto-reset.  Run by one lane of a
// warp-per-env kernel, that work cost ~28 % of the step's instructions
// (profiles/r2_*): here 32 envs share every warp instruction.
//
// Reference semantics followed (paths under /root/reference/proj/include/marlob):
//   env/env.hpp:143-192 (reset), :266-370 (effective_tops, convert_action),
//   :372-396 (fill attribution), :409-503 (rewards, infos, observations),
//   agents/actions.hpp, agents/rewards.hpp, agents/observations.hpp,
//   core/rng.hpp:63-71 (Fisher-Yates), ippo/rollout.hpp:290-318 (auto-reset),
//   baselines/twap.hpp:20-58, baselines/avst.hpp:19-32, bench/bench.hpp:53-70.
// Compiled with --fmad=false: double expressions round like the reference's
// x86-64 build.
#pragma once

#include "mlob_step.cuh"

namespace mlob {

__host__ __device__ inline int spl_of(int capacity) {
  const int need = (capacity + kWarp - 1) / kWarp;
  return need <= 1 ? 1 : need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : need <= 16 ? 16 : need <= 32 ? 32 : -1;
}

struct ThreadEnv {
  const KParams& kp;
  const DevCfg& cfg;
  uint64_t env, genv, seed;
  EnvHdr h;  // working copy of the env header
  uint32_t err = 0;

  __device__ ThreadEnv(const KParams& p, const DevCfg& c, uint64_t e) : kp(p), cfg(c), env(e) {
    MLOB_CHECK(e < kp.n_envs);
    genv = kp.env_index ? kp.env_index[e] : kp.env_index_base + e;
    seed = kp.env_seed ? kp.env_seed[e] : kp.seed;
    h = kp.hdr[e];
  }
  __device__ __forceinline__ int A() const { return cfg.n_agents; }
  __device__ __forceinline__ const DevSpec& spec(int a) const { return cfg.specs[cfg.flat_spec[a]]; }
  __device__ __forceinline__ void report_errors() const {
    if (err) atomicOr(kp.error, err);
  }

  // ---- actions (env.hpp:266-370, agents/actions.hpp) -----------------------
  __device__ void effective_tops(const DevSpec& p, int64_t& bid_, int64_t& ask_) const {
    const int64_t mh = h.mid_half;
    const int64_t mid_floor = mh >= 0 ? mh / 2 : (mh - 1) / 2;
    const int64_t mid_ceil = (mh + 1) / 2;
    bid_ = h.live[0] > 0 ? static_cast<int64_t>(h.best[0]) : mid_floor - p.default_half_spread;
    ask_ = h.live[1] > 0 ? static_cast<int64_t>(h.best[1]) : mid_ceil + p.default_half_spread;
    if (bid_ < 1) bid_ = 1;
    if (ask_ <= bid_) ask_ = bid_ + 1;
  }

  struct Quotes {  // agents::QuoteList (actions.hpp:24-40)
    int n;
    int s0, s1;
    int64_t p0, p1, q0, q1;
    __device__ void push(int s, int64_t p, int64_t q) {
      if (n == 0) {
        s0 = s;
        p0 = p;
        q0 = q;
      } else {
        s1 = s;
        p1 = p;
        q1 = q;
      }
      ++n;
    }
    __device__ void finish_two_sided() {  // actions.hpp:47-56
      if (n >= 1 && p0 < 1) p0 = 1;
      if (n >= 2 && p1 < 1) p1 = 1;
      if (n == 2) {
        const bool a0 = s0 == MLOB_ASK;
        const int64_t bp = s0 == MLOB_BID ? p0 : p1;
        const int64_t ap = a0 ? p0 : p1;
        if (bp >= ap) {
          if (a0)
            p0 = bp + 1;
          else
            p1 = bp + 1;
        }
      }
    }
  };

  // decode_avst (actions.hpp:164-178) over avst_quotes (actions.hpp:151-162);
  // avst_term = (2/gamma) log1p(gamma/kappa), evaluated on the host
  __device__ void avst(double gamma, double sigma, double horizon, double avst_term, int64_t inventory,
                       int64_t order_size, Quotes& q) const {
    const double rem = horizon - static_cast<double>(h.step);
    const double ttg = 0.0 < rem ? rem : 0.0;
    const double mid_ticks = static_cast<double>(h.mid_half) / 2.0;
    const double reservation = mid_ticks - static_cast<double>(inventory) * gamma * sigma * sigma * ttg;
    const double half_spread = 0.5 * (gamma * sigma * sigma * ttg + avst_term);
    q.push(MLOB_BID, static_cast<int64_t>(floor(reservation - half_spread)), order_size);
    q.push(MLOB_ASK, static_cast<int64_t>(ceil(reservation + half_spread)), order_size);
    q.finish_two_sided();
  }

  __device__ void decode(const DevSpec& sp, const AgentRec& st, int id, Quotes& q) const {
    int64_t bb, ba;
    effective_tops(sp, bb, ba);
    q.n = 0;
    if (sp.type == MLOB_EXECUTOR) {  // env.hpp:302-311, actions.hpp:193-224
      int64_t eb = bb, ea = ba;
      if (st.task_dir == MLOB_TASK_BUY && h.live[1] == 0) ea = max(static_cast<int64_t>(2), h.last_ask + 1);
      if (st.task_dir == MLOB_TASK_SELL && h.live[0] == 0) eb = max(static_cast<int64_t>(1), h.last_bid - 1);
      const int pi = id % 4, mi = id / 4;
      const int64_t spread = ea - eb;
      int64_t price;
      if (st.task_dir == MLOB_TASK_BUY)
        price = pi == 0 ? ea : pi == 1 ? eb : pi == 2 ? eb - 1 : eb + spread / 2;
      else
        price = pi == 0 ? eb : pi == 1 ? ea : pi == 2 ? ea + 1 : ea - spread / 2;
      int64_t qty = sp.order_size * (mi == 0 ? 1 : mi == 1 ? 2 : 5);
      if (qty > st.task_remaining) qty = st.task_remaining;
      if (qty > 0) q.push(st.task_dir == MLOB_TASK_BUY ? MLOB_BID : MLOB_ASK, price < 1 ? 1 : price, qty);
    } else if (sp.type == MLOB_DIRECTIONAL) {  // actions.hpp:227-235
      if (id == 1) q.push(MLOB_BID, bb < 1 ? 1 : bb, sp.order_size);
      if (id == 2) q.push(MLOB_ASK, ba < 1 ? 1 : ba, sp.order_size);
    } else if (sp.mm_space == MLOB_FIXED_QUANT) {  // actions.hpp:66-108
      const int64_t br = sp.fixed_quant_from_mid ? (bb + ba) / 2 : bb;
      const int64_t ar = sp.fixed_quant_from_mid ? (bb + ba + 1) / 2 : ba;
      const int64_t sz = sp.order_size;
      if (id != 0) {
        const int64_t pb = id == 1 ? br - 2 : id == 2 ? br - 4 : id == 3 ? bb + 1 : id == 4 ? br - 2
                         : id == 5 ? bb : id == 6 ? bb - 5 : bb + 1;
        const int64_t pa = id == 1 ? ar + 2 : id == 2 ? ar + 4 : id == 3 ? ba - 1 : id == 4 ? ba
                         : id == 5 ? ar + 2 : id == 6 ? ba - 1 : ba + 5;
        q.push(MLOB_BID, pb, sz);
        q.push(MLOB_ASK, pa, sz);
      }
      q.finish_two_sided();
    } else if (sp.mm_space == MLOB_SPREAD_SKEW) {  // actions.hpp:128-140
      const int64_t hs = sp.ss_half[id], sk = sp.ss_skew[id];
      const int64_t bh = h.mid_half - 2 * hs + 2 * sk;
      const int64_t ah = h.mid_half + 2 * hs + 2 * sk;
      q.push(MLOB_BID, bh >= 0 ? bh / 2 : (bh - 1) / 2, sp.order_size);
      q.push(MLOB_ASK, (ah + 1) / 2, sp.order_size);
      q.finish_two_sided();
    } else {  // AvSt, actions.hpp:151-178
      avst(sp.gamma[id], sp.sigma, sp.horizon, sp.avst_term[id], st.inventory, sp.order_size, q);
    }
  }

  // Scripted direct actions (evaluate.hpp:63-73): NoOp, twap_policy
  // (twap.hpp:37-58 over make_twap_plan, twap.hpp:21-33), avst_policy (avst.hpp:19-32).
  __device__ void scripted(const DevSpec& sp, const AgentRec& st, const DevPolicy& pol, Quotes& q) const {
    if (pol.kind == MLOB_POLICY_TWAP) {
      const int64_t S = cfg.steps_per_episode, T = sp.task_size, s = h.step;
      const int64_t sched = ((s + 1) * T) / S - (s * T) / S;
      const int64_t qty = s + 1 == S ? st.task_remaining : min(sched, st.task_remaining);
      if (qty <= 0) return;
      int64_t bb, ba;
      effective_tops(sp, bb, ba);
      const bool buy = st.task_dir == MLOB_TASK_BUY;
      const int64_t price = pol.twap_mode == MLOB_TWAP_AGGRESSIVE ? (buy ? ba : bb) : (buy ? bb : ba);
      q.push(buy ? MLOB_BID : MLOB_ASK, price, qty);
    } else if (pol.kind == MLOB_POLICY_AVST) {
      avst(pol.gamma, pol.sigma, pol.horizon, pol.avst_term, st.inventory, sp.order_size, q);
    }
  }

  __device__ __forceinline__ void push_amsg(DevMsg* out, uint32_t& n, int64_t time, uint64_t id, int64_t price,
                                            int64_t qty, int kind, int side, int trader) {
    if (n >= kp.amsg_cap) {
      err |= kErrAmsgCap;
      return;
    }
    DevMsg m;
    m.time = time;
    m.order_id = id;
    m.price = static_cast<int32_t>(price);
    m.qty = static_cast<int32_t>(qty);
    m.kind = static_cast<uint8_t>(kind);
    m.side = static_cast<uint8_t>(side);
    m._pad = 0;
    m.trader = trader;
    out[n++] = m;
  }

  // env.hpp:285-370 for agent a: quotes -> Delete for each active order not
  // requoted at the same (side, price), NewLimit for each quote not kept.
  __device__ void convert_action(int a, int64_t step_time, DevMsg* out, uint32_t& n, Rng& bench_rng) {
    const DevSpec& sp = spec(a);
    const size_t slot = env * cfg.n_agents + a;
    const AgentRec st = kp.agents[slot];
    Quotes q;
    q.n = 0;
    q.s0 = q.s1 = 0;
    q.p0 = q.p1 = q.q0 = q.q1 = 0;
    const DevPolicy* pol =
        kp.action_mode == kActScripted ? &kp.policies[kp.env_policy[env * cfg.n_specs + cfg.flat_spec[a]]] : nullptr;
    const bool direct = pol ? pol->kind != MLOB_POLICY_RANDOM && pol->kind != MLOB_POLICY_LEARNED
                            : kp.action_mode == kActDirect && kp.action_direct[slot].direct;
    if (direct) {  // env.hpp:290-298
      if (pol) {
        scripted(sp, st, *pol, q);
      } else {
        const mlob_agent_action& da = kp.action_direct[slot];
        q.n = da.n_quotes;
        q.s0 = da.quotes[0].side;
        q.p0 = da.quotes[0].price;
        q.q0 = da.quotes[0].quantity;
        q.s1 = da.quotes[1].side;
        q.p1 = da.quotes[1].price;
        q.q1 = da.quotes[1].quantity;
      }
      if (sp.type == MLOB_EXECUTOR) {
        if (q.n >= 1 && q.q0 > st.task_remaining) q.q0 = st.task_remaining;
        if (q.n >= 2 && q.q1 > st.task_remaining) q.q1 = st.task_remaining;
        if (q.n == 1 && q.q0 <= 0) q.n = 0;
      }
    } else {
      int id;
      if (kp.action_mode == kActBench) {  // bench.hpp:57-60: one rng per env-step, one draw per agent
        if (a == 0)
          bench_rng.s = key_fold(key_fold(key_fold(splitmix64(kp.bench_seed), kRngBenchAction), genv),
                                 kp.global_step);
        id = static_cast<int>(bench_rng.below(static_cast<uint64_t>(sp.arity)));
      } else if (pol && pol->kind == MLOB_POLICY_LEARNED) {  // argmax id from the policy kernel
        id = kp.action_ids[slot];
      } else if (pol) {  // PolicyKind::Random, evaluate.hpp:74-79
        uint64_t hh = key_fold(key_fold(splitmix64(seed), kRngEpisodeDraw), kp.env_cell ? kp.env_cell[env] : 0);
        hh = key_fold(key_fold(key_fold(hh, h.episode), static_cast<uint64_t>(h.step)), static_cast<uint64_t>(a));
        Rng r{hh};
        id = static_cast<int>(r.below(static_cast<uint64_t>(sp.arity)));
      } else if (kp.action_mode == kActDirect) {
        id = kp.action_direct[slot].id;
      } else {
        id = kp.action_ids[slot];
      }
      if (id < 0 || id >= sp.arity) {
        err |= kErrBadAction;
        id = 0;
      }
      decode(sp, st, id, q);
    }
    bool kept0 = false, kept1 = false;
    const ActiveRec* act = kp.active + slot * kMaxActive;
    for (int i = 0; i < st.n_active; ++i) {
      const ActiveRec ar = act[i];
      const int side = static_cast<int>(ar.qty_side >> 31);
      const bool r0 = q.n >= 1 && q.s0 == side && q.p0 == ar.price;
      const bool r1 = q.n >= 2 && q.s1 == side && q.p1 == ar.price;
      kept0 |= r0;
      kept1 |= r1;
      if (r0 || r1) continue;
      push_amsg(out, n, step_time, ar.order_id, 0, 0, MLOB_DELETE, side, a + 1);
    }
    uint64_t nonce = st.nonce;
    const uint64_t id_base = cfg.agent_id_base + static_cast<uint64_t>(a) * cfg.agent_id_range;
    for (int j = 0; j < q.n; ++j) {
      if (j == 0 ? kept0 : kept1) continue;
      const int64_t pr = j == 0 ? q.p0 : q.p1, qt = j == 0 ? q.q0 : q.q1;
      if (pr > INT_MAX - 1 || pr < INT_MIN + 1 || qt > INT_MAX || qt < INT_MIN) err |= kErrPriceRange;
      push_amsg(out, n, step_time, id_base + nonce, pr, qt, MLOB_NEW_LIMIT, j == 0 ? q.s0 : q.s1, a + 1);
      ++nonce;
    }
    if (nonce != st.nonce) kp.agents[slot].nonce = nonce;
  }

  // MarketEnv::step stages (1)+(2) (env.hpp:205-215): the agent messages of
  // this step, shuffled with CounterRng(seed, env, episode, step, Shuffle).
  __device__ void actions() {
    const int mps = cfg.mps;
    const int64_t step_time =
        mps > 0 ? kp.msgs[kp.ep_start[h.episode] + static_cast<uint64_t>(h.step) * mps].time : h.last_time + 1;
    DevMsg* out = kp.amsg + env * kp.amsg_cap;
    uint32_t n = 0;
    Rng bench_rng{0};
    for (int a = 0; a < A(); ++a) convert_action(a, step_time, out, n, bench_rng);
    if (n >= 2) {  // rng.hpp:63-71
      uint64_t hh = splitmix64(seed);
      hh = key_fold(hh, genv);
      hh = key_fold(hh, h.episode);
      hh = key_fold(hh, static_cast<uint64_t>(h.step));
      hh = key_fold(hh, kRngShuffle);
      Rng r{hh};
      for (int i = static_cast<int>(n) - 1; i > 0; --i) {
        const int j = static_cast<int>(r.below(static_cast<uint64_t>(i + 1)));
        if (i != j) {
          const DevMsg t = out[i];
          out[i] = out[j];
          out[j] = t;
        }
      }
    }
    kp.hdr[env].n_amsg = n;
  }

  // ---- outcomes (env.hpp:372-503, agents/rewards.hpp, observations.hpp) ---
  // Step accumulators of one agent, rebuilt from the fill log in fill order.
  struct Acc {
    double slip;
    int64_t filled;
    int32_t count;
  };

  // entry i of the env's fill log (inline part, then the overflow chunks)
  struct FillCursor {
    const FillEnt* inl;
    const FillEnt* pool;
    uint32_t chunk;
    __device__ FillEnt at(uint32_t i) {
      if (i < kFillInline) return inl[i];
      const uint32_t k = i - kFillInline, off = k % (kFillChunk - 1) + 1;
      if (off == 1 && k > 0) chunk = static_cast<uint32_t>(pool[static_cast<size_t>(chunk) * kFillChunk].price);
      MLOB_CHECK(chunk != kNoChunk);
      return pool[static_cast<size_t>(chunk) * kFillChunk + off];
    }
  };
  __device__ FillCursor fills() const {
    return FillCursor{kp.fills + env * kFillInline, kp.fill_pool, h.fill_head};
  }

  // env.hpp:381-396 (apply_fill) over agent a's fills in order, plus the
  // MM Ψ sums against M̄ (rewards.hpp:22-36) in the same order.
  __device__ void apply_fills(int a, const DevSpec& sp, AgentRec& st, Acc& ac, double& pb, double& ps) const {
    ac = Acc{0.0, 0, 0};
    pb = ps = 0.0;
    FillCursor fc = fills();
    const double sign = st.task_dir == MLOB_TASK_BUY ? 1.0 : -1.0;
    for (uint32_t i = 0; i < h.n_fills; ++i) {
      const FillEnt f = fc.at(i);
      if (f.agent != a) continue;
      const int64_t pq = static_cast<int64_t>(f.price) * f.qty;
      if (f.side == MLOB_BID) {
        st.inventory += f.qty;
        st.cash -= pq;
        pb += (h.mbar - static_cast<double>(f.price)) * static_cast<double>(f.qty);
      } else {
        st.inventory -= f.qty;
        st.cash += pq;
        ps += (static_cast<double>(f.price) - h.mbar) * static_cast<double>(f.qty);
      }
      st.filled_total += f.qty;
      if (sp.type == MLOB_EXECUTOR) {
        const bool task_side = (st.task_dir == MLOB_TASK_BUY) == (f.side == MLOB_BID);
        if (task_side) st.task_remaining = max(static_cast<int64_t>(0), st.task_remaining - f.qty);
      }
      // slippage term, rewards.hpp:69-75: (sign * q) * (price - p_init)
      ac.slip += sign * static_cast<double>(f.qty) * (static_cast<double>(f.price) - st.p_init);
      ac.filled += f.qty;
      ac.count += 1;
    }
  }

  // env.hpp:409-433 + rewards.hpp
  __device__ double compute_reward(const DevSpec& sp, const AgentRec& st, const Acc& ac, double pb,
                                   double ps) const {
    double r = 0.0;
    if (sp.reward == MLOB_REWARD_EXEC) {
      r = -ac.slip;
      if (h.terminal && st.task_remaining > 0)
        r -= sp.unfilled_penalty_coef * static_cast<double>(st.task_remaining) * st.p_init;
    } else {
      if (sp.reward == MLOB_REWARD_BUYSELL) {
        r = pb + ps;
      } else {
        const double mid = static_cast<double>(h.mid_half) / 2.0;
        const double prev = static_cast<double>(h.prev_mid_half) / 2.0;
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

  // env.hpp:435-443
  __device__ double reference_price(const DevSpec& sp, const AgentRec& st) const {
    if (sp.ref_price == MLOB_REF_MID || st.inventory == 0) return static_cast<double>(h.mid_half) / 2.0;
    if (st.inventory > 0) return static_cast<double>(h.live[0] > 0 ? static_cast<int64_t>(h.best[0]) : h.last_bid);
    return static_cast<double>(h.live[1] > 0 ? static_cast<int64_t>(h.best[1]) : h.last_ask);
  }

  // env.hpp:445-464 (also accumulates slippage_total)
  __device__ mlob_agent_info fill_info(const DevSpec& sp, AgentRec& st, const Acc& ac) const {
    mlob_agent_info info;
    info.inventory = st.inventory;
    info.cash = st.cash;
    info.portfolio_value = static_cast<double>(st.inventory) * reference_price(sp, st) + static_cast<double>(st.cash);
    info.slippage_step = sp.type == MLOB_EXECUTOR ? ac.slip : 0.0;
    const double total = st.slippage_total + info.slippage_step;
    info.slippage_total = total;
    info.task_remaining = st.task_remaining;
    info.step_filled = ac.filled;
    info.step_fill_count = ac.count;
    info._pad = 0;
    st.slippage_total = total;
    return info;
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

  // env.hpp:466-503, observations.hpp:42-148, straight into the gather layout
  __device__ void build_observation(int a, const DevSpec& sp, const AgentRec& st, const L2Sum& l2) const {
    const int dim = sp.obs_dim;
    const int t = cfg.flat_spec[a];
    const int kk = a - sp.flat_offset;
    double* out = kp.obs[t] + (env * static_cast<uint64_t>(sp.count) + kk) * dim;
    const int64_t bb = h.live[0] > 0 ? h.best[0] : -1;
    const int64_t ba = h.live[1] > 0 ? h.best[1] : -1;
    const double time_frac = static_cast<double>(h.step) / static_cast<double>(cfg.steps_per_episode);
    const int64_t bq = l2.sumq0, aq = l2.sumq1;
    const double imb = bq + aq == 0 ? 0.0 : static_cast<double>(bq - aq) / static_cast<double>(bq + aq);
    const double spread = (bb < 0 || ba < 0) ? 0.0 : fmin_ref(32.0, static_cast<double>(ba - bb));
    int64_t own_bid = -1, own_ask = -1;
    const ActiveRec* act = kp.active + (env * cfg.n_agents + a) * kMaxActive;
    for (int i = 0; i < st.n_active; ++i) {
      const ActiveRec ar = act[i];
      if ((ar.qty_side >> 31) == 0)
        own_bid = own_bid < 0 ? ar.price : max(own_bid, static_cast<int64_t>(ar.price));
      else
        own_ask = own_ask < 0 ? ar.price : min(own_ask, static_cast<int64_t>(ar.price));
    }
    const double dmid = static_cast<double>(h.mid_half - h.prev_mid_half) / 2.0;
    if (sp.type == MLOB_EXECUTOR) {
      const int dir = st.task_dir == MLOB_TASK_BUY ? 1 : -1;
      out[0] = static_cast<double>(st.task_remaining) / static_cast<double>(sp.task_size > 1 ? sp.task_size : 1);
      out[1] = time_frac;
      out[2] = static_cast<double>(dir);
      out[3] = spread;
      out[4] = dmid;
      out[5] = static_cast<double>(h.mid_half) / 2.0 - st.p_init;
      out[6] = imb;
      out[7] = l2.nb > 0 ? qty_feature(l2.topq0, sp.order_size) : 0.0;
      out[8] = l2.na > 0 ? qty_feature(l2.topq1, sp.order_size) : 0.0;
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
        const L2Lvl* l2b = kp.l2lv + env * 2 * cfg.obs_depth;
        const L2Lvl* l2a = l2b + cfg.obs_depth;
        int k = 8;
        const int levels = (dim - 8) / 4;
        for (int d = 0; d < levels; ++d) {
          const bool hb = d < l2.nb, ha = d < l2.na;
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

  // ---- reset (env.hpp:143-192, book.hpp:41-60) ------------------------------
  // Writes the new episode's book straight into the HBM layout, one synthetic
  // order per L2 level, and the L2 summary of that book.
  __device__ void init_side(int S, const DevLevel* lv, uint32_t n, uint64_t id_base, uint32_t seq_base, int spl,
                            L2Lvl* l2out, int32_t& nl, int64_t& sumq, int64_t& topq) {
    const int32_t empty_p = S == 0 ? INT_MIN : INT_MAX;
    const uint32_t rows = (n + kWarp - 1) / kWarp;
    MLOB_CHECK(rows <= static_cast<uint32_t>(spl));
    const size_t base = (env * 2 + static_cast<uint64_t>(S)) * spl * kWarp;
    if (spl > 8) {  // deep book: 4-word slots (SmemSide): p, q << 8 | trader, id lo, id hi << 20 | seq,
                    // slot (row k, lane l) at (k / 4) * 128 + l * 4 + k % 4, written in whole four-row groups
      uint32_t* lo = reinterpret_cast<uint32_t*>(kp.bk_id);
      const uint32_t grows = (rows + 3) / 4 * 4;
      for (uint32_t i = 0; i < grows * kWarp; ++i) {
        const uint32_t k = i / kWarp, l = i % kWarp;
        const size_t x = base + (k >> 2) * 128 + l * 4 + (k & 3);
        const uint64_t id = id_base + i;
        const bool live = i < n;
        if (live && (lv[i].qty >= (1 << 24) || (id >> 44) != 0)) err |= kErrDeepRange;
        kp.bk_p[x] = live ? lv[i].price : empty_p;
        kp.bk_q[x] = live ? static_cast<int32_t>(static_cast<uint32_t>(lv[i].qty) << 8) : 0;
        lo[x] = live ? static_cast<uint32_t>(id) : 0u;
        kp.bk_st[x] = live ? (static_cast<uint32_t>(id >> 32) << 20) | (seq_base + i) : kEmptySt;
      }
    } else {
      for (uint32_t i = 0; i < rows * kWarp; ++i) {
        const size_t x = base + i;
        if (i < n) {
          const uint64_t id = id_base + i;
          kp.bk_p[x] = lv[i].price;
          kp.bk_q[x] = lv[i].qty;
          kp.bk_id[x] = make_uint2(static_cast<uint32_t>(id), static_cast<uint32_t>(id >> 32));
          kp.bk_st[x] = (seq_base + i) << 8;
        } else {
          kp.bk_p[x] = empty_p;
          kp.bk_q[x] = 0;
          kp.bk_id[x] = make_uint2(0u, 0u);
          kp.bk_st[x] = kEmptySt;
        }
      }
    }
    // aggregate_levels (book.hpp:209-220) over the new book, best-first:
    // the levels of a sampled snapshot (best-first, distinct prices)
    const int D = static_cast<int>(cfg.obs_depth);
    nl = 0;
    sumq = topq = 0;
    int32_t last = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const int32_t p = lv[i].price;
      if (nl > 0 && p == last) {
        if (l2out) l2out[nl - 1].qty += lv[i].qty;
        sumq += lv[i].qty;
        if (nl == 1) topq += lv[i].qty;
        continue;
      }
      if (nl == D) break;
      if (l2out) l2out[nl] = L2Lvl{p, 0, lv[i].qty};
      sumq += lv[i].qty;
      if (nl == 0) topq = lv[i].qty;
      last = p;
      ++nl;
    }
  }

  // MarketEnv::reset(episode); false (and an error bit) when the episode has
  // no usable book state.  Agent records come back through `recs`.
  __device__ bool reset(uint64_t ep, L2Sum& l2) {
    const EpState es = kp.ep_state[ep];
    if (!es.valid) {
      err |= kErrMissingState;
      return false;
    }
    if (static_cast<int>(es.nb) > cfg.capacity || static_cast<int>(es.na) > cfg.capacity) {
      err |= kErrTooDeep;
      return false;
    }
    const int spl = spl_of(cfg.capacity);
    const DevLevel* lv = kp.levels + es.level_offset;
    L2Lvl* l2b = kp.l2lv ? kp.l2lv + env * 2 * cfg.obs_depth : nullptr;
    int32_t nb, na;
    int64_t s0, s1, t0, t1;
    init_side(0, lv, es.nb, cfg.synth_id_base, 0, spl, l2b, nb, s0, t0);
    init_side(1, lv + es.nb, es.na, cfg.synth_id_base + es.nb, es.nb, spl, l2b ? l2b + cfg.obs_depth : nullptr, na,
              s1, t1);
    l2 = L2Sum{nb, na, s0, s1, t0, t1, 0};
    h.episode = ep;
    h.next_seq = es.nb + es.na;
    h.live[0] = static_cast<uint16_t>(es.nb);
    h.live[1] = static_cast<uint16_t>(es.na);
    h.hwm[0] = static_cast<uint16_t>(es.nb);
    h.hwm[1] = static_cast<uint16_t>(es.na);
    h.best[0] = es.nb ? lv[0].price : 0;
    h.best[1] = es.na ? lv[es.nb].price : 0;
    {
      const bool hb = es.nb > 0, ha = es.na > 0;
      const int64_t b0 = h.best[0], b1 = h.best[1];
      h.mid_half = hb ? (ha ? b0 + b1 : 2 * b0) : (ha ? 2 * b1 : cfg.fallback_mid_half);
    }
    h.prev_mid_half = h.mid_half;
    h.mbar = static_cast<double>(h.mid_half) / 2.0;
    h.last_bid = es.nb > 0 ? static_cast<int64_t>(h.best[0]) : h.mid_half / 2 - 1;
    h.last_ask = es.na > 0 ? static_cast<int64_t>(h.best[1]) : (h.mid_half + 1) / 2 + 1;
    h.step = 0;
    h.terminal = 0;
    h.n_trades = 0;
    h.n_fills = 0;
    h.fill_head = kNoChunk;
    for (int a = 0; a < A(); ++a) {
      const DevSpec& sp = spec(a);
      const size_t slot = env * cfg.n_agents + a;
      AgentRec st;
      st.inventory = 0;
      st.cash = 0;
      st.filled_total = 0;
      st.slippage_total = 0.0;
      st.nonce = 0;
      st.n_active = 0;
      st.p_init = static_cast<double>(h.mid_half) / 2.0;
      st.task_dir = kp.agents[slot].task_dir;
      if (sp.type == MLOB_EXECUTOR) {
        uint64_t hh = splitmix64(seed);
        hh = key_fold(hh, genv);
        hh = key_fold(hh, ep);
        hh = key_fold(hh, 0);
        hh = key_fold(hh, kRngTaskDir);
        hh = key_fold(hh, static_cast<uint64_t>(a));
        Rng r{hh};
        st.task_dir = r.coin() ? MLOB_TASK_BUY : MLOB_TASK_SELL;
        st.task_remaining = sp.task_size;
      } else {
        st.task_remaining = 0;
      }
      kp.agents[slot] = st;
    }
    return true;
  }

  // infos + observations of every agent for the current state with empty
  // step accumulators (after a reset)
  __device__ void fresh_outputs(const L2Sum& l2) {
    for (int a = 0; a < A(); ++a) {
      const DevSpec& sp = spec(a);
      const size_t slot = env * cfg.n_agents + a;
      AgentRec st = kp.agents[slot];
      const Acc ac{0.0, 0, 0};
      kp.infos[slot] = fill_info(sp, st, ac);
      kp.agents[slot].slippage_total = st.slippage_total;
      build_observation(a, sp, st, l2);
    }
  }

  // MarketEnv::step stage (5) after the message loop (env.hpp:242-253) and
  // MarketVecEnv::step_one's caches / auto-reset (rollout.hpp:290-318).
  __device__ void outcomes() {
    const L2Sum l2 = kp.l2sum[env];
    const bool auto_reset = h.terminal && (kp.flags & MLOB_VENV_AUTO_RESET);
    for (int a = 0; a < A(); ++a) {
      const DevSpec& sp = spec(a);
      const size_t slot = env * cfg.n_agents + a;
      AgentRec st = kp.agents[slot];
      Acc ac;
      double pb, ps;
      apply_fills(a, sp, st, ac, pb, ps);
      kp.rewards[slot] = compute_reward(sp, st, ac, pb, ps);
      kp.dones[slot] = h.terminal ? 1 : 0;
      const mlob_agent_info info = fill_info(sp, st, ac);
      kp.infos[slot] = info;
      build_observation(a, sp, st, l2);
      kp.agents[slot] = st;
      if (auto_reset) {  // rollout.hpp:300-313
        kp.t_pv[slot] += info.portfolio_value;
        kp.t_slip[slot] += info.slippage_total;
        kp.t_comp[slot] += sp.type == MLOB_EXECUTOR
                               ? 1.0 - static_cast<double>(info.task_remaining) / static_cast<double>(sp.task_size)
                               : 0.0;
        kp.t_rem[slot] += sp.type == MLOB_EXECUTOR ? info.task_remaining : 0;
        kp.t_inv[slot] += static_cast<double>(info.inventory) * static_cast<double>(info.inventory);
      }
    }
    uint8_t just_reset = 0;
    if (auto_reset) {
      ++h.episodes_finished;
      const uint64_t i = (genv + h.cursor * kp.n_envs_global) % kp.pool_len;  // rollout.hpp:286-288
      const uint64_t ep = kp.pool ? kp.pool[i] : i;
      ++h.cursor;
      L2Sum fresh;
      if (reset(ep, fresh)) {
        fresh_outputs(fresh);
        kp.l2sum[env] = fresh;
        just_reset = 1;
      }
    }
    h.just_reset = just_reset;
    kp.hdr[env] = h;
    kp.just_reset[env] = just_reset;
  }

  // K3 (reset_all / reset_envs): MarketEnv::reset + the fresh outputs,
  // rewards / dones zeroed; last_time and messages_processed carry over.
  __device__ void reset_env() {
    L2Sum fresh;
    const bool ok = reset(kp.reset_episodes[env], fresh);
    if (ok) {
      fresh_outputs(fresh);
      kp.l2sum[env] = fresh;
      for (int a = 0; a < A(); ++a) {
        kp.rewards[env * cfg.n_agents + a] = 0.0;
        kp.dones[env * cfg.n_agents + a] = 0;
      }
    }
    h.cursor = 1;
    h.just_reset = 1;
    kp.hdr[env] = h;
    kp.just_reset[env] = 1;
  }
};

}  // namespace mlob
