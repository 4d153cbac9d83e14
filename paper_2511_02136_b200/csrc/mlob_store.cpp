// mlob_store.cpp — host-side message-store builders:
// the deterministic synthetic MBO generator (data/synth.hpp:39-177), episode
// indexing (data/store.hpp:52-72) and the config validation of
// env/config.hpp:96-120.  Input preparation only: the environment step itself
// runs on the GPU (mlob_kernels.cu); nothing here is a fallback for it.
#include <algorithm>
#include <cstring>

#include "mlob_host.h"

int64_t mlob_host_store::state_before(uint64_t idx) const {
  const auto it = std::lower_bound(st_index.begin(), st_index.end(), idx);
  if (it == st_index.end() || *it != idx) return -1;
  return it - st_index.begin();
}

void mlob_host_store::push_state(uint64_t idx, const mlob_level* bids, uint32_t nb,
                                 const mlob_level* asks, uint32_t na) {
  if (st_offset.empty()) st_offset.push_back(0);
  st_index.push_back(idx);
  st_nb.push_back(nb);
  levels.insert(levels.end(), bids, bids + nb);
  levels.insert(levels.end(), asks, asks + na);
  st_offset.push_back(levels.size());
}

namespace mlob {
namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
inline uint64_t splitmix64(uint64_t z) {
  z += kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t make_key1(uint64_t seed, uint64_t w) {  // core/rng.hpp:18-27
  const uint64_t h = splitmix64(seed);
  return splitmix64(h ^ (w + kGamma + (h << 6) + (h >> 2)));
}
struct Rng {
  uint64_t s;
  uint64_t next() { return splitmix64(s += kGamma); }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return next() % n; }
  bool coin() { return (next() & 1ull) != 0; }
};

// Generator-side book: the synthetic stream needs a live book to pick cancel
// and execute targets.  Per side a worst-to-best sorted array (ties: newest
// first), the priority order of lob/book.hpp:16-19, capacity 2^15 per side.
struct GenOrder {
  int64_t price, qty;
  uint64_t id, seq;
};
struct GenBook {
  std::vector<GenOrder> side[2];
  uint64_t next_seq = 0;

  static bool before(int s, const GenOrder& a, const GenOrder& b) {
    if (a.price != b.price) return s == MLOB_BID ? a.price < b.price : a.price > b.price;
    return a.seq > b.seq;
  }
  static constexpr size_t kCapacity = 1u << 15;  // synth.hpp:48
  void rest(int s, int64_t price, int64_t qty, uint64_t id) {  // book.hpp:169-187
    auto& v = side[s];
    if (v.size() == kCapacity) {
      const int64_t worst = v.front().price;
      if (!(s == MLOB_BID ? price > worst : price < worst)) return;
      size_t ev = 0;
      while (ev + 1 < v.size() && v[ev + 1].price == worst) ++ev;
      v.erase(v.begin() + static_cast<std::ptrdiff_t>(ev));
    }
    GenOrder o{price, qty, id, next_seq++};
    auto pos = std::upper_bound(v.begin(), v.end(), o,
                                [s](const GenOrder& a, const GenOrder& b) { return before(s, a, b); });
    v.insert(pos, o);
  }
  void reduce(int s, uint64_t id, int64_t by, bool remove) {
    auto& v = side[s];
    for (auto it = v.begin(); it != v.end(); ++it) {
      if (it->id != id) continue;
      if (remove) {
        v.erase(it);
      } else {
        it->qty -= std::min(it->qty, by);
        if (it->qty == 0) v.erase(it);
      }
      return;
    }
  }
  void process(const mlob_message& m) {
    switch (m.kind) {
      case MLOB_NEW_LIMIT: {
        if (m.quantity <= 0) return;
        int64_t rem = m.quantity;
        auto& opp = side[1 - m.side];
        while (rem > 0 && !opp.empty()) {
          GenOrder& b = opp.back();
          const bool crosses = m.side == MLOB_BID ? b.price <= m.price : b.price >= m.price;
          if (!crosses) break;
          const int64_t q = std::min(rem, b.qty);
          b.qty -= q;
          rem -= q;
          if (b.qty == 0) opp.pop_back();
        }
        if (rem > 0) rest(m.side, m.price, rem, m.order_id);
        break;
      }
      case MLOB_CANCEL_PARTIAL:
      case MLOB_EXECUTE_VISIBLE: reduce(m.side, m.order_id, m.quantity, false); break;
      case MLOB_DELETE: reduce(m.side, m.order_id, 0, true); break;
      default: break;
    }
  }
  uint32_t levels(int s, uint64_t depth, mlob_level* out) const {  // book.hpp:209-220
    uint32_t n = 0;
    const auto& v = side[s];
    for (auto it = v.rbegin(); it != v.rend(); ++it) {
      if (n > 0 && out[n - 1].price == it->price) {
        out[n - 1].quantity += it->qty;
      } else {
        if (n == depth) break;
        out[n++] = mlob_level{it->price, it->qty};
      }
    }
    return n;
  }
};

}  // namespace

void synth_generate(const mlob_synth_config& cfg, uint64_t seed, mlob_host_store& st) {
  if (cfg.n_messages == 0) fail(MLOB_E_INVALID_ARGUMENT, "synth_generate: n_messages >= 1");
  if (cfg.initial_mid <= cfg.band + 1)
    fail(MLOB_E_INVALID_ARGUMENT, "synth_generate: initial_mid must exceed band + 1");
  if (cfg.state_sample_every == 0)
    fail(MLOB_E_INVALID_ARGUMENT, "synth_generate: state_sample_every >= 1");
  st = mlob_host_store{};
  st.msgs.reserve(cfg.n_messages);
  st.st_offset.push_back(0);
  GenBook book;
  std::vector<mlob_level> bl(cfg.state_depth + 1), al(cfg.state_depth + 1);
  Rng rng{make_key1(seed, 4 /* RngStream::Synth */)};
  int64_t ref = cfg.initial_mid, time = 0;
  uint64_t next_id = 1;
  const double band = static_cast<double>(cfg.band);

  auto emit = [&](const mlob_message& m) {  // synth.hpp:56-63
    if (st.msgs.size() % cfg.state_sample_every == 0) {
      const uint32_t nb = book.levels(MLOB_BID, cfg.state_depth, bl.data());
      const uint32_t na = book.levels(MLOB_ASK, cfg.state_depth, al.data());
      st.push_state(st.msgs.size(), bl.data(), nb, al.data(), na);
    }
    book.process(m);
    st.msgs.push_back(m);
  };
  auto blank = [&](int kind, int side) {
    mlob_message m;
    std::memset(&m, 0, sizeof m);
    m.time = time;
    m.kind = static_cast<uint8_t>(kind);
    m.side = static_cast<uint8_t>(side);
    return m;
  };
  auto passive_quote = [&](int side) {  // synth.hpp:65-77
    const double u = rng.uniform();
    const int64_t off = static_cast<int64_t>(u * u * band);
    mlob_message m = blank(MLOB_NEW_LIMIT, side);
    m.order_id = next_id++;
    m.quantity = 1 + static_cast<int64_t>(rng.below(static_cast<uint64_t>(cfg.max_qty)));
    m.price = side == MLOB_BID ? ref - off : ref + 1 + off;
    emit(m);
  };

  for (int level = 0; level < cfg.seed_levels && st.msgs.size() < cfg.n_messages; ++level) {
    for (int s = 0; s < 2; ++s) {
      if (st.msgs.size() >= cfg.n_messages) break;
      time += 1000;
      mlob_message m = blank(MLOB_NEW_LIMIT, s);
      m.order_id = next_id++;
      m.quantity = cfg.seed_qty;
      m.price = s == MLOB_BID ? ref - level : ref + 1 + level;
      emit(m);
    }
  }
  const double c1 = cfg.p_new_passive, c2 = c1 + cfg.p_new_cross;
  const double c3 = c2 + cfg.p_cancel, c4 = c3 + cfg.p_delete, c5 = c4 + cfg.p_execute;
  while (st.msgs.size() < cfg.n_messages) {  // synth.hpp:94-174
    time += 1 + static_cast<int64_t>(rng.below(2000));
    if (rng.uniform() < cfg.volatility) {
      ref += rng.coin() ? 1 : -1;
      if (ref <= cfg.band + 1) ref = cfg.band + 2;
    }
    if (book.side[MLOB_BID].empty()) {
      passive_quote(MLOB_BID);
      continue;
    }
    if (book.side[MLOB_ASK].empty()) {
      passive_quote(MLOB_ASK);
      continue;
    }
    const double u = rng.uniform();
    const int side = rng.coin() ? MLOB_BID : MLOB_ASK;
    if (u < c1) {
      passive_quote(side);
    } else if (u < c2) {
      mlob_message m = blank(MLOB_NEW_LIMIT, side);
      m.order_id = next_id++;
      m.quantity = 1 + static_cast<int64_t>(rng.below(static_cast<uint64_t>(cfg.max_qty)));
      m.price = side == MLOB_BID ? book.side[MLOB_ASK].back().price : book.side[MLOB_BID].back().price;
      emit(m);
    } else if (u < c4) {
      const bool partial = u < c3;
      const auto& bids = book.side[MLOB_BID];
      const auto& asks = book.side[MLOB_ASK];
      const uint64_t total = bids.size() + asks.size();
      if (total == 0) continue;
      const uint64_t pick = rng.below(total);
      const GenOrder& t = pick < bids.size() ? bids[pick] : asks[pick - bids.size()];
      mlob_message m = blank(partial ? MLOB_CANCEL_PARTIAL : MLOB_DELETE,
                             pick < bids.size() ? MLOB_BID : MLOB_ASK);
      m.order_id = t.id;
      m.price = t.price;
      m.quantity = partial ? 1 + static_cast<int64_t>(rng.below(static_cast<uint64_t>(t.qty))) : t.qty;
      emit(m);
    } else if (u < c5) {
      const auto& o = book.side[side];
      if (o.empty()) continue;
      const GenOrder& best = o.back();
      mlob_message m = blank(MLOB_EXECUTE_VISIBLE, side);
      m.order_id = best.id;
      m.price = best.price;
      m.quantity = 1 + static_cast<int64_t>(rng.below(static_cast<uint64_t>(best.qty)));
      emit(m);
    } else {
      const uint64_t k = rng.below(3);
      mlob_message m = blank(k == 0 ? MLOB_EXECUTE_HIDDEN : k == 1 ? MLOB_CROSS : MLOB_HALT, side);
      m.order_id = 0;
      m.price = ref;
      m.quantity = 1;
      emit(m);
    }
  }
}

std::vector<uint64_t> build_episode_index(uint64_t n_messages, int steps, int mps, int stride) {
  if (n_messages == 0) fail(MLOB_E_INVALID_ARGUMENT, "build_episode_index: empty store");
  if (steps < 1 || mps < 0 || stride < 1)
    fail(MLOB_E_INVALID_ARGUMENT, "build_episode_index: invalid episode parameters");
  std::vector<uint64_t> starts;
  const uint64_t length = static_cast<uint64_t>(steps) * static_cast<uint64_t>(mps);
  const uint64_t step = static_cast<uint64_t>(stride) * static_cast<uint64_t>(mps);
  if (length == 0) return {0};
  for (uint64_t s = 0; s + length <= n_messages; s += step) starts.push_back(s);
  return starts;
}

static int arity_of(const mlob_agent_spec& s) {
  switch (s.type) {
    case MLOB_EXECUTOR: return s.params.exec_complex ? 12 : 4;
    case MLOB_DIRECTIONAL: return 3;
    case MLOB_MARKET_MAKER:
      switch (s.mm_space) {
        case MLOB_SPREAD_SKEW: return s.params.n_spread_skew;
        case MLOB_FIXED_QUANT: return 8;
        case MLOB_AVST: return s.params.n_gamma;
      }
  }
  return 0;
}

void validate_config(const mlob_env_config& c) {  // env/config.hpp:96-120
  auto bad = [](const std::string& m) { fail(MLOB_E_INVALID_ARGUMENT, m); };
  if (c.steps_per_episode < 1) bad("env.steps_per_episode must be >= 1");
  if (c.messages_per_step < 0) bad("env.messages_per_step must be >= 0");
  if (c.start_stride_steps < 1) bad("env.start_stride_steps must be >= 1");
  if (c.book_capacity < 1) bad("env.book_capacity must be >= 1");
  if (c.obs_depth < 1) bad("env.obs_depth must be >= 1");
  if (c.n_specs < 0 || c.n_specs > MLOB_MAX_SPECS) bad("env: at most 8 agent specs");
  for (int i = 0; i < c.n_specs; ++i) {
    const mlob_agent_spec& s = c.specs[i];
    const std::string w = "env.agents[" + std::to_string(i) + "]";
    if (s.count < 1) bad(w + ".count must be >= 1");
    if (s.params.order_size < 1) bad(w + ".order_size must be >= 1");
    if (s.params.inventory_cap < 1) bad(w + ".inventory_cap must be >= 1");
    if (s.params.lambda < 0.0 || s.params.lambda > 1.0) bad(w + ".lambda must lie in [0, 1]");
    if (s.params.rho < 0.0) bad(w + ".rho must be >= 0");
    if (s.type == MLOB_EXECUTOR && s.params.task_size < 1) bad(w + ".task_size must be >= 1");
    if (s.params.n_spread_skew < 0 || s.params.n_spread_skew > MLOB_MAX_SPREAD_SKEW_ROWS)
      bad(w + ": spread-skew table larger than 32 rows");
    if (s.params.n_gamma < 0 || s.params.n_gamma > MLOB_MAX_GAMMA)
      bad(w + ": gamma grid larger than 16 entries");
    if (arity_of(s) < 1) bad(w + ": empty action space");
  }
}

}  // namespace mlob
