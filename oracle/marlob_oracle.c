/*
 * marlob_oracle.c — TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * A plain-C restatement of the reference's batched LOB environment step:
 * price-time book, counter RNG, synthetic MBO generator, agent decoders,
 * observations, rewards, MarketEnv reset/step, MarketVecEnv and the random-
 * policy throughput harness.  Every function cites the reference file:line
 * (relative to /root/reference/proj/include/marlob/) it follows.
 *
 * Pinned by: the reference's own known-answer tests re-hosted in
 * tests/test_oracle.py, the SURVEY §8(c) digests (tests/golden/), and
 * differential runs against the compiled reference (oracle/_ref).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may load it;
 * the product never links it.
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "oracle_api.h"

/* ------------------------------------------------------------------------ */
/* errors                                                                    */

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* orc_last_error(void) { return g_err; }

#define VEC(T)      \
  struct {          \
    T* v;           \
    uint64_t n;     \
    uint64_t cap;   \
  }
#define VEC_PUSH(vec, x)                                                          \
  do {                                                                            \
    if ((vec).n == (vec).cap) {                                                   \
      (vec).cap = (vec).cap ? 2 * (vec).cap : 16;                                 \
      (vec).v = realloc((vec).v, (vec).cap * sizeof(*(vec).v));                   \
    }                                                                             \
    (vec).v[(vec).n++] = (x);                                                     \
  } while (0)

/* ------------------------------------------------------------------------ */
/* core/rng.hpp:11-71                                                        */

#define GAMMA64 0x9E3779B97F4A7C15ull

static uint64_t splitmix64(uint64_t z) { /* rng.hpp:11-16 */
  z += GAMMA64;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t key_fold(uint64_t h, uint64_t w) { /* rng.hpp:18-20 */
  return splitmix64(h ^ (w + GAMMA64 + (h << 6) + (h >> 2)));
}

static uint64_t make_key(uint64_t seed, int n, const uint64_t* words) { /* rng.hpp:22-27 */
  uint64_t h = splitmix64(seed);
  for (int i = 0; i < n; ++i) h = key_fold(h, words[i]);
  return h;
}

enum { RNG_SHUFFLE = 1, RNG_TASKDIR = 2, RNG_SYNTH = 4, RNG_BENCH_ACTION = 7 }; /* rng.hpp:30-39 */

typedef struct { uint64_t state; } crng;                                       /* rng.hpp:41-61 */
static uint64_t crng_next(crng* r) { return splitmix64(r->state += GAMMA64); }
static double crng_uniform(crng* r) { return (double)(crng_next(r) >> 11) * 0x1.0p-53; }
static uint64_t crng_below(crng* r, uint64_t n) { return crng_next(r) % n; }
static int crng_coin(crng* r) { return (crng_next(r) & 1ull) != 0; }

/* ------------------------------------------------------------------------ */
/* lob/book.hpp:23-226 — sorted worst-to-best vectors per side               */

typedef VEC(mlob_trade) trade_vec;
typedef VEC(mlob_resting_order) order_vec;

typedef struct book {
  order_vec side[2];
  uint64_t capacity;
  uint64_t next_seq;
} book;

static void book_init(book* b, uint64_t capacity) {
  memset(b, 0, sizeof *b);
  b->capacity = capacity;
}
static void book_release(book* b) {
  free(b->side[0].v);
  free(b->side[1].v);
}
static void book_clear(book* b) { /* book.hpp:33-37 */
  b->side[0].n = b->side[1].n = 0;
  b->next_seq = 0;
}

/* book.hpp:41-60: one synthetic order per level, arrival_seq best-first */
static int book_init_from_l2(book* b, const mlob_level* bids, uint32_t nb,
                             const mlob_level* asks, uint32_t na, uint64_t id_base) {
  if (nb > b->capacity || na > b->capacity)
    return fail(MLOB_E_INVALID_ARGUMENT, "OrderBook: snapshot deeper than book capacity");
  b->side[0].n = b->side[1].n = 0;
  for (uint32_t i = nb; i-- > 0;) {
    mlob_resting_order o = {bids[i].price, bids[i].quantity, id_base + i, b->next_seq + i, 0, 0};
    VEC_PUSH(b->side[0], o);
  }
  b->next_seq += nb;
  const uint64_t ask_base = id_base + nb;
  for (uint32_t i = na; i-- > 0;) {
    mlob_resting_order o = {asks[i].price, asks[i].quantity, ask_base + i, b->next_seq + i, 0, 0};
    VEC_PUSH(b->side[1], o);
  }
  b->next_seq += na;
  return MLOB_OK;
}

static int book_has(const book* b, int s) { return b->side[s].n > 0; }
static int64_t book_best(const book* b, int s) { return b->side[s].v[b->side[s].n - 1].price; }

static int64_t book_mid_half(const book* b, int64_t fallback) { /* book.hpp:98-106 */
  const int hb = book_has(b, 0), ha = book_has(b, 1);
  if (hb && ha) return book_best(b, 0) + book_best(b, 1);
  if (hb) return 2 * book_best(b, 0);
  if (ha) return 2 * book_best(b, 1);
  return fallback;
}

/* "a strictly before b" in storage order, book.hpp:134-143 */
static int before(int s, const mlob_resting_order* a, const mlob_resting_order* o) {
  if (a->price != o->price) return s == MLOB_BID ? a->price < o->price : a->price > o->price;
  return a->arrival_seq > o->arrival_seq;
}

static void erase_at(order_vec* v, uint64_t i) {
  memmove(v->v + i, v->v + i + 1, (v->n - i - 1) * sizeof *v->v);
  v->n--;
}

/* book.hpp:169-187 */
static void rest_order(book* b, const mlob_message* m, int64_t qty) {
  order_vec* side = &b->side[m->side];
  mlob_resting_order in = {m->price, qty, m->order_id, b->next_seq, m->trader_id, 0};
  if (side->n == b->capacity) {
    const int64_t worst = side->v[0].price;
    const int better = m->side == MLOB_BID ? m->price > worst : m->price < worst;
    if (!better) return;
    uint64_t evict = 0;
    while (evict + 1 < side->n && side->v[evict + 1].price == worst) ++evict;
    erase_at(side, evict);
  }
  ++b->next_seq;
  /* upper_bound: first position whose element the incoming one is strictly before */
  uint64_t lo = 0, hi = side->n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (before(m->side, &in, &side->v[mid]))
      hi = mid;
    else
      lo = mid + 1;
  }
  VEC_PUSH(*side, in); /* grow */
  memmove(side->v + lo + 1, side->v + lo, (side->n - 1 - lo) * sizeof *side->v);
  side->v[lo] = in;
}

/* book.hpp:150-167 */
static void process_new_limit(book* b, const mlob_message* m, trade_vec* trades) {
  if (m->quantity <= 0) return;
  int64_t remaining = m->quantity;
  order_vec* opp = &b->side[1 - m->side];
  while (remaining > 0 && opp->n > 0) {
    mlob_resting_order* best = &opp->v[opp->n - 1];
    const int crosses = m->side == MLOB_BID ? best->price <= m->price : best->price >= m->price;
    if (!crosses) break;
    const int64_t q = remaining < best->quantity ? remaining : best->quantity;
    mlob_trade t;
    memset(&t, 0, sizeof t);
    t.price = best->price;
    t.quantity = q;
    t.time = m->time;
    t.passive_order_id = best->order_id;
    t.aggressor_order_id = m->order_id;
    t.passive_trader_id = best->trader_id;
    t.aggressor_trader_id = m->trader_id;
    t.aggressor_side = m->side;
    VEC_PUSH(*trades, t);
    best->quantity -= q;
    remaining -= q;
    if (best->quantity == 0) opp->n--;
  }
  if (remaining > 0) rest_order(b, m, remaining);
}

/* book.hpp:189-197 */
static void reduce_order(book* b, int s, uint64_t id, int64_t by) {
  order_vec* side = &b->side[s];
  for (uint64_t i = 0; i < side->n; ++i) {
    if (side->v[i].order_id != id) continue;
    const int64_t q = side->v[i].quantity;
    side->v[i].quantity -= q < by ? q : by;
    if (side->v[i].quantity == 0) erase_at(side, i);
    return;
  }
}

/* book.hpp:199-207 */
static void remove_order(book* b, int s, uint64_t id) {
  order_vec* side = &b->side[s];
  for (uint64_t i = 0; i < side->n; ++i)
    if (side->v[i].order_id == id) {
      erase_at(side, i);
      return;
    }
}

/* book.hpp:65-86 */
static void book_process(book* b, const mlob_message* m, trade_vec* trades) {
  switch (m->kind) {
    case MLOB_NEW_LIMIT: process_new_limit(b, m, trades); break;
    case MLOB_CANCEL_PARTIAL: reduce_order(b, m->side, m->order_id, m->quantity); break;
    case MLOB_DELETE: remove_order(b, m->side, m->order_id); break;
    case MLOB_EXECUTE_VISIBLE: reduce_order(b, m->side, m->order_id, m->quantity); break;
    default: break; /* ExecuteHidden / Cross / Halt */
  }
}

/* book.hpp:109-120, 209-220: top-`depth` aggregated levels, best-first */
static uint32_t aggregate_levels(const order_vec* side, uint64_t depth, mlob_level* out) {
  uint32_t n = 0;
  for (uint64_t k = side->n; k-- > 0;) {
    const mlob_resting_order* o = &side->v[k];
    if (n > 0 && out[n - 1].price == o->price) {
      out[n - 1].quantity += o->quantity;
    } else {
      if (n == depth) break;
      out[n].price = o->price;
      out[n].quantity = o->quantity;
      ++n;
    }
  }
  return n;
}

/* ------------------------------------------------------------------------ */
/* data/store.hpp, data/synth.hpp                                            */

typedef struct state_rec {
  uint64_t message_index;
  uint32_t nb, na;
  mlob_level* levels; /* bids then asks */
} state_rec;

typedef struct store {
  VEC(mlob_message) msgs;
  VEC(state_rec) states;
} store;

static void push_state(store* st, uint64_t idx, const mlob_level* bids, uint32_t nb,
                       const mlob_level* asks, uint32_t na) {
  state_rec r;
  r.message_index = idx;
  r.nb = nb;
  r.na = na;
  r.levels = malloc((nb + na + 1) * sizeof(mlob_level));
  memcpy(r.levels, bids, nb * sizeof(mlob_level));
  memcpy(r.levels + nb, asks, na * sizeof(mlob_level));
  VEC_PUSH(st->states, r);
}

/* store.hpp:29-36: exact-match lower_bound */
static const state_rec* state_before(const store* st, uint64_t idx) {
  uint64_t lo = 0, hi = st->states.n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (st->states.v[mid].message_index < idx)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo == st->states.n || st->states.v[lo].message_index != idx) return NULL;
  return &st->states.v[lo];
}

void orc_store_free(void* s) {
  store* st = s;
  if (!st) return;
  for (uint64_t i = 0; i < st->states.n; ++i) free(st->states.v[i].levels);
  free(st->states.v);
  free(st->msgs.v);
  free(st);
}

/* synth.hpp:39-177 */
typedef struct synth_ctx {
  const mlob_synth_config* cfg;
  store* st;
  book bk;
  trade_vec trades;
  mlob_level* scratch;
} synth_ctx;

static void synth_emit(synth_ctx* c, const mlob_message* m) { /* synth.hpp:56-63 */
  if (c->st->msgs.n % c->cfg->state_sample_every == 0) {
    const uint32_t nb = aggregate_levels(&c->bk.side[0], c->cfg->state_depth, c->scratch);
    const uint32_t na =
        aggregate_levels(&c->bk.side[1], c->cfg->state_depth, c->scratch + c->cfg->state_depth);
    push_state(c->st, c->st->msgs.n, c->scratch, nb, c->scratch + c->cfg->state_depth, na);
  }
  c->trades.n = 0;
  book_process(&c->bk, m, &c->trades);
  VEC_PUSH(c->st->msgs, *m);
}

void* orc_store_synth(const mlob_synth_config* cfg, uint64_t seed) {
  if (cfg->n_messages == 0) {
    fail(MLOB_E_INVALID_ARGUMENT, "synth_generate: n_messages >= 1");
    return NULL;
  }
  if (cfg->initial_mid <= cfg->band + 1) {
    fail(MLOB_E_INVALID_ARGUMENT, "synth_generate: initial_mid must exceed band + 1");
    return NULL;
  }
  synth_ctx c;
  memset(&c, 0, sizeof c);
  c.cfg = cfg;
  c.st = calloc(1, sizeof(store));
  c.st->msgs.cap = cfg->n_messages;
  c.st->msgs.v = malloc(cfg->n_messages * sizeof(mlob_message));
  book_init(&c.bk, 1u << 15);
  c.scratch = malloc((2 * cfg->state_depth + 1) * sizeof(mlob_level));
  const uint64_t w = RNG_SYNTH;
  crng rng = {make_key(seed, 1, &w)};
  int64_t ref = cfg->initial_mid;
  int64_t time = 0;
  uint64_t next_id = 1;
  const double band = (double)cfg->band;

#define PASSIVE_QUOTE(SIDE)                                                         \
  do {                                                                              \
    const double u_ = crng_uniform(&rng);                                           \
    const int64_t off_ = (int64_t)(u_ * u_ * band);                                 \
    mlob_message m_;                                                                \
    memset(&m_, 0, sizeof m_);                                                      \
    m_.time = time;                                                                 \
    m_.kind = MLOB_NEW_LIMIT;                                                       \
    m_.side = (SIDE);                                                               \
    m_.order_id = next_id++;                                                        \
    m_.quantity = 1 + (int64_t)crng_below(&rng, (uint64_t)cfg->max_qty);            \
    m_.price = (SIDE) == MLOB_BID ? ref - off_ : ref + 1 + off_;                    \
    synth_emit(&c, &m_);                                                            \
  } while (0)

  /* initial ladder, synth.hpp:78-92 */
  for (int level = 0; level < cfg->seed_levels && c.st->msgs.n < cfg->n_messages; ++level) {
    for (int s = 0; s < 2; ++s) {
      if (c.st->msgs.n >= cfg->n_messages) break;
      time += 1000;
      mlob_message m;
      memset(&m, 0, sizeof m);
      m.time = time;
      m.kind = MLOB_NEW_LIMIT;
      m.side = (uint8_t)s;
      m.order_id = next_id++;
      m.quantity = cfg->seed_qty;
      m.price = s == MLOB_BID ? ref - level : ref + 1 + level;
      synth_emit(&c, &m);
    }
  }

  const double p1 = cfg->p_new_passive, p2 = p1 + cfg->p_new_cross;
  while (c.st->msgs.n < cfg->n_messages) { /* synth.hpp:94-174 */
    time += 1 + (int64_t)crng_below(&rng, 2000);
    if (crng_uniform(&rng) < cfg->volatility) {
      ref += crng_coin(&rng) ? 1 : -1;
      if (ref <= cfg->band + 1) ref = cfg->band + 2;
    }
    if (!book_has(&c.bk, MLOB_BID)) {
      PASSIVE_QUOTE(MLOB_BID);
      continue;
    }
    if (!book_has(&c.bk, MLOB_ASK)) {
      PASSIVE_QUOTE(MLOB_ASK);
      continue;
    }
    const double u = crng_uniform(&rng);
    const int side = crng_coin(&rng) ? MLOB_BID : MLOB_ASK;
    if (u < cfg->p_new_passive) {
      PASSIVE_QUOTE(side);
    } else if (u < p2) {
      mlob_message m;
      memset(&m, 0, sizeof m);
      m.time = time;
      m.kind = MLOB_NEW_LIMIT;
      m.side = (uint8_t)side;
      m.order_id = next_id++;
      m.quantity = 1 + (int64_t)crng_below(&rng, (uint64_t)cfg->max_qty);
      m.price = side == MLOB_BID ? book_best(&c.bk, MLOB_ASK) : book_best(&c.bk, MLOB_BID);
      synth_emit(&c, &m);
    } else if (u < p2 + cfg->p_cancel + cfg->p_delete) {
      const int partial = u < p2 + cfg->p_cancel;
      const uint64_t nb = c.bk.side[0].n, na = c.bk.side[1].n;
      const uint64_t total = nb + na;
      if (total == 0) continue;
      const uint64_t pick = crng_below(&rng, total);
      const mlob_resting_order* t = pick < nb ? &c.bk.side[0].v[pick] : &c.bk.side[1].v[pick - nb];
      mlob_message m;
      memset(&m, 0, sizeof m);
      m.time = time;
      m.kind = partial ? MLOB_CANCEL_PARTIAL : MLOB_DELETE;
      m.side = pick < nb ? MLOB_BID : MLOB_ASK;
      m.order_id = t->order_id;
      m.price = t->price;
      m.quantity = partial ? 1 + (int64_t)crng_below(&rng, (uint64_t)t->quantity) : t->quantity;
      synth_emit(&c, &m);
    } else if (u < p2 + cfg->p_cancel + cfg->p_delete + cfg->p_execute) {
      const order_vec* o = &c.bk.side[side];
      if (o->n == 0) continue;
      const mlob_resting_order* best = &o->v[o->n - 1];
      mlob_message m;
      memset(&m, 0, sizeof m);
      m.time = time;
      m.kind = MLOB_EXECUTE_VISIBLE;
      m.side = (uint8_t)side;
      m.order_id = best->order_id;
      m.price = best->price;
      m.quantity = 1 + (int64_t)crng_below(&rng, (uint64_t)best->quantity);
      synth_emit(&c, &m);
    } else {
      const uint64_t k = crng_below(&rng, 3);
      mlob_message m;
      memset(&m, 0, sizeof m);
      m.time = time;
      m.kind = k == 0 ? MLOB_EXECUTE_HIDDEN : k == 1 ? MLOB_CROSS : MLOB_HALT;
      m.side = (uint8_t)side;
      m.order_id = 0;
      m.price = ref;
      m.quantity = 1;
      synth_emit(&c, &m);
    }
  }
#undef PASSIVE_QUOTE
  book_release(&c.bk);
  free(c.trades.v);
  free(c.scratch);
  return c.st;
}

void* orc_store_create(const mlob_message* msgs, uint64_t n, const mlob_book_states* s) {
  store* st = calloc(1, sizeof(store));
  for (uint64_t i = 0; i < n; ++i) VEC_PUSH(st->msgs, msgs[i]);
  if (s)
    for (uint64_t i = 0; i < s->n_states; ++i) {
      const uint64_t off = s->level_offset[i];
      const uint32_t nb = s->n_bids[i];
      const uint32_t na = (uint32_t)(s->level_offset[i + 1] - off) - nb;
      push_state(st, s->message_index[i], s->levels + off, nb, s->levels + off + nb, na);
    }
  return st;
}

uint64_t orc_store_n_messages(void* s) { return ((store*)s)->msgs.n; }
const mlob_message* orc_store_messages(void* s) { return ((store*)s)->msgs.v; }
uint64_t orc_store_n_states(void* s) { return ((store*)s)->states.n; }
int orc_store_state(void* s, uint64_t i, uint64_t* msg_index, mlob_level* bids, uint32_t* nb,
                    mlob_level* asks, uint32_t* na, uint32_t cap) {
  const store* st = s;
  if (i >= st->states.n) return fail(MLOB_E_OUT_OF_RANGE, "state index");
  const state_rec* r = &st->states.v[i];
  *msg_index = r->message_index;
  *nb = r->nb;
  *na = r->na;
  if (r->nb > cap || r->na > cap) return MLOB_E_OUT_OF_RANGE;
  memcpy(bids, r->levels, r->nb * sizeof(mlob_level));
  memcpy(asks, r->levels + r->nb, r->na * sizeof(mlob_level));
  return MLOB_OK;
}

/* store.hpp:52-72 */
static int build_episode_index(const store* st, int steps, int mps, int stride, uint64_t** starts,
                               uint64_t* n) {
  if (st->msgs.n == 0) return fail(MLOB_E_INVALID_ARGUMENT, "build_episode_index: empty store");
  if (steps < 1 || mps < 0 || stride < 1)
    return fail(MLOB_E_INVALID_ARGUMENT, "build_episode_index: invalid episode parameters");
  const uint64_t length = (uint64_t)steps * (uint64_t)mps;
  const uint64_t step = (uint64_t)stride * (uint64_t)mps;
  *n = 0;
  *starts = NULL;
  if (length == 0) {
    *starts = malloc(sizeof(uint64_t));
    (*starts)[0] = 0;
    *n = 1;
    return MLOB_OK;
  }
  uint64_t cap = 0;
  for (uint64_t s = 0; s + length <= st->msgs.n; s += step) {
    if (*n == cap) {
      cap = cap ? 2 * cap : 64;
      *starts = realloc(*starts, cap * sizeof(uint64_t));
    }
    (*starts)[(*n)++] = s;
  }
  return MLOB_OK;
}

/* ------------------------------------------------------------------------ */
/* book handle API                                                           */

void* orc_book_create(uint64_t capacity) {
  if (capacity == 0) {
    fail(MLOB_E_INVALID_ARGUMENT, "OrderBook: capacity must be >= 1");
    return NULL;
  }
  book* b = malloc(sizeof(book));
  book_init(b, capacity);
  return b;
}
int orc_book_init_from_l2(void* b, const mlob_level* bids, uint32_t nb, const mlob_level* asks,
                          uint32_t na, uint64_t id_base) {
  return book_init_from_l2(b, bids, nb, asks, na, id_base);
}
uint64_t orc_book_process(void* b, const mlob_message* m, mlob_trade* out, uint64_t cap) {
  trade_vec t = {0};
  book_process(b, m, &t);
  for (uint64_t i = 0; i < t.n && i < cap; ++i) out[i] = t.v[i];
  const uint64_t n = t.n;
  free(t.v);
  return n;
}
uint64_t orc_book_orders(void* b, int side, mlob_resting_order* out, uint64_t cap) {
  const order_vec* v = &((book*)b)->side[side];
  for (uint64_t i = 0; i < v->n && i < cap; ++i) out[i] = v->v[i];
  return v->n;
}
uint64_t orc_book_next_seq(void* b) { return ((book*)b)->next_seq; }
int64_t orc_book_mid_half(void* b, int64_t fallback) { return book_mid_half(b, fallback); }
void orc_book_l2(void* b, uint64_t depth, mlob_level* bids, uint32_t* nb, mlob_level* asks,
                 uint32_t* na) {
  *nb = aggregate_levels(&((book*)b)->side[0], depth, bids);
  *na = aggregate_levels(&((book*)b)->side[1], depth, asks);
}
void orc_book_free(void* b) {
  if (!b) return;
  book_release(b);
  free(b);
}

/* ------------------------------------------------------------------------ */
/* agents/actions.hpp                                                        */

typedef struct quote_list {
  mlob_quote q[2];
  int n;
} quote_list;

static void ql_push(quote_list* l, int side, int64_t price, int64_t qty) {
  memset(&l->q[l->n], 0, sizeof(mlob_quote));
  l->q[l->n].side = (uint8_t)side;
  l->q[l->n].price = price;
  l->q[l->n].quantity = qty;
  l->n++;
}

static int64_t clamp_price(int64_t p) { return p < 1 ? 1 : p; } /* actions.hpp:45 */

static void finish_two_sided(quote_list* l) { /* actions.hpp:47-56 */
  for (int i = 0; i < l->n; ++i) l->q[i].price = clamp_price(l->q[i].price);
  if (l->n == 2) {
    mlob_quote* bid = l->q[0].side == MLOB_BID ? &l->q[0] : &l->q[1];
    mlob_quote* ask = l->q[0].side == MLOB_ASK ? &l->q[0] : &l->q[1];
    if (bid->price >= ask->price) ask->price = bid->price + 1;
  }
}

static int decode_fixed_quant(int id, int64_t bb, int64_t ba, int64_t sz, int from_mid,
                              quote_list* q) { /* actions.hpp:66-108 */
  if (id < 0 || id >= 8) return fail(MLOB_E_OUT_OF_RANGE, "decode_fixed_quant: action id %d", id);
  const int64_t bid_ref = from_mid ? (bb + ba) / 2 : bb;
  const int64_t ask_ref = from_mid ? (bb + ba + 1) / 2 : ba;
  q->n = 0;
  switch (id) {
    case 0: break;
    case 1: ql_push(q, MLOB_BID, bid_ref - 2, sz); ql_push(q, MLOB_ASK, ask_ref + 2, sz); break;
    case 2: ql_push(q, MLOB_BID, bid_ref - 4, sz); ql_push(q, MLOB_ASK, ask_ref + 4, sz); break;
    case 3: ql_push(q, MLOB_BID, bb + 1, sz); ql_push(q, MLOB_ASK, ba - 1, sz); break;
    case 4: ql_push(q, MLOB_BID, bid_ref - 2, sz); ql_push(q, MLOB_ASK, ba, sz); break;
    case 5: ql_push(q, MLOB_BID, bb, sz); ql_push(q, MLOB_ASK, ask_ref + 2, sz); break;
    case 6: ql_push(q, MLOB_BID, bb - 5, sz); ql_push(q, MLOB_ASK, ba - 1, sz); break;
    case 7: ql_push(q, MLOB_BID, bb + 1, sz); ql_push(q, MLOB_ASK, ba + 5, sz); break;
  }
  finish_two_sided(q);
  return MLOB_OK;
}

static int decode_spread_skew(int id, int64_t mid_half, const mlob_agent_params* p, int64_t sz,
                              quote_list* q) { /* actions.hpp:128-140 */
  if (id < 0 || id >= p->n_spread_skew)
    return fail(MLOB_E_OUT_OF_RANGE, "decode_spread_skew: action id %d", id);
  const int64_t hs = p->spread_skew_half[id], sk = p->spread_skew_skew[id];
  const int64_t bid_half = mid_half - 2 * hs + 2 * sk;
  const int64_t ask_half = mid_half + 2 * hs + 2 * sk;
  q->n = 0;
  ql_push(q, MLOB_BID, bid_half >= 0 ? bid_half / 2 : (bid_half - 1) / 2, sz);
  ql_push(q, MLOB_ASK, (ask_half + 1) / 2, sz);
  finish_two_sided(q);
  return MLOB_OK;
}

static int decode_avst(int id, int64_t mid_half, int64_t inventory, int step,
                       const mlob_agent_params* p, int64_t sz, quote_list* q) {
  /* actions.hpp:151-178 */
  if (id < 0 || id >= p->n_gamma) return fail(MLOB_E_OUT_OF_RANGE, "decode_avst: action id %d", id);
  const double gamma = p->gamma_grid[id];
  const double rem = p->horizon - (double)step;
  const double ttg = 0.0 < rem ? rem : 0.0; /* std::max(0.0, rem) */
  const double mid_ticks = (double)mid_half / 2.0;
  const double reservation = mid_ticks - (double)inventory * gamma * p->sigma * p->sigma * ttg;
  const double half_spread =
      0.5 * (gamma * p->sigma * p->sigma * ttg + (2.0 / gamma) * log1p(gamma / p->kappa));
  q->n = 0;
  ql_push(q, MLOB_BID, (int64_t)floor(reservation - half_spread), sz);
  ql_push(q, MLOB_ASK, (int64_t)ceil(reservation + half_spread), sz);
  finish_two_sided(q);
  return MLOB_OK;
}

static int decode_exec(int id, int64_t bb, int64_t ba, int64_t base, int complex_space, int dir,
                       int64_t task_remaining, quote_list* q) { /* actions.hpp:193-224 */
  const int arity = complex_space ? 12 : 4;
  if (id < 0 || id >= arity) return fail(MLOB_E_OUT_OF_RANGE, "decode_exec: action id %d", id);
  static const int64_t mult[3] = {1, 2, 5};
  const int price_idx = id % 4, mult_idx = id / 4;
  const int64_t spread = ba - bb;
  int64_t price = 0;
  if (dir == MLOB_TASK_BUY) {
    switch (price_idx) {
      case 0: price = ba; break;
      case 1: price = bb; break;
      case 2: price = bb - 1; break;
      case 3: price = bb + spread / 2; break;
    }
  } else {
    switch (price_idx) {
      case 0: price = bb; break;
      case 1: price = ba; break;
      case 2: price = ba + 1; break;
      case 3: price = ba - spread / 2; break;
    }
  }
  int64_t qty = base * mult[mult_idx];
  if (qty > task_remaining) qty = task_remaining;
  q->n = 0;
  if (qty > 0) ql_push(q, dir == MLOB_TASK_BUY ? MLOB_BID : MLOB_ASK, clamp_price(price), qty);
  return MLOB_OK;
}

static int decode_directional(int id, int64_t bb, int64_t ba, int64_t sz, quote_list* q) {
  /* actions.hpp:227-235 */
  if (id < 0 || id >= 3) return fail(MLOB_E_OUT_OF_RANGE, "decode_directional: action id %d", id);
  q->n = 0;
  if (id == 1) ql_push(q, MLOB_BID, clamp_price(bb), sz);
  if (id == 2) ql_push(q, MLOB_ASK, clamp_price(ba), sz);
  return MLOB_OK;
}

/* ------------------------------------------------------------------------ */
/* env/config.hpp                                                            */

static int action_arity(const mlob_agent_spec* s) { /* config.hpp:73-90 */
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

static uint64_t observation_size(int id, uint64_t depth) { /* observations.hpp:69-76 */
  switch (id) {
    case MLOB_OBS_MM_BASIC: return 8;
    case MLOB_OBS_MM_FULL: return 8 + 4 * depth;
    case MLOB_OBS_EXEC: return 10;
  }
  return 0;
}

static int validate(const mlob_env_config* c) { /* config.hpp:96-120 */
  if (c->steps_per_episode < 1) return fail(1, "env.steps_per_episode must be >= 1");
  if (c->messages_per_step < 0) return fail(1, "env.messages_per_step must be >= 0");
  if (c->start_stride_steps < 1) return fail(1, "env.start_stride_steps must be >= 1");
  if (c->book_capacity < 1) return fail(1, "env.book_capacity must be >= 1");
  if (c->obs_depth < 1) return fail(1, "env.obs_depth must be >= 1");
  for (int i = 0; i < c->n_specs; ++i) {
    const mlob_agent_spec* s = &c->specs[i];
    if (s->count < 1) return fail(1, "env.agents[%d].count must be >= 1", i);
    if (s->params.order_size < 1) return fail(1, "env.agents[%d].order_size must be >= 1", i);
    if (s->params.inventory_cap < 1) return fail(1, "env.agents[%d].inventory_cap must be >= 1", i);
    if (s->params.lambda < 0.0 || s->params.lambda > 1.0)
      return fail(1, "env.agents[%d].lambda must lie in [0, 1]", i);
    if (s->params.rho < 0.0) return fail(1, "env.agents[%d].rho must be >= 0", i);
    if (s->type == MLOB_EXECUTOR && s->params.task_size < 1)
      return fail(1, "env.agents[%d].task_size must be >= 1", i);
    if (action_arity(s) < 1) return fail(1, "env.agents[%d]: empty action space", i);
  }
  return MLOB_OK;
}

/* ------------------------------------------------------------------------ */
/* env/env.hpp MarketEnv                                                     */

typedef struct fill { /* rewards.hpp:15-19 */
  double price;
  int64_t quantity;
  int side;
} fill;

typedef struct agent_state { /* env.hpp:29-46 */
  int64_t inventory, cash;
  VEC(mlob_active_order) active;
  int64_t task_remaining;
  int task_dir;
  double p_init;
  uint64_t order_nonce;
  int64_t filled_total;
  double slippage_total;
  VEC(fill) fills;
  double* obs;
  uint64_t obs_n;
  double reward;
  uint8_t done;
  mlob_agent_info info;
} agent_state;

typedef struct env {
  const store* st;
  uint64_t* starts;
  uint64_t n_episodes;
  mlob_env_config cfg;
  uint64_t seed;
  int env_index;
  book bk;
  int n_agents;
  int flat_spec[MLOB_MAX_AGENTS];
  agent_state ag[MLOB_MAX_AGENTS];
  uint64_t episode;
  int step;
  int terminal;
  int64_t mid_half, prev_mid_half;
  double mbar;
  int64_t last_bid, last_ask, last_time;
  uint64_t messages_processed;
  VEC(mlob_message) agent_msgs;
  trade_vec trades;
  trade_vec step_trades;
  mlob_level* l2;
  uint32_t l2_nb, l2_na;
} env;

static const mlob_agent_spec* spec_of(const env* e, int a) { return &e->cfg.specs[e->flat_spec[a]]; }

void* orc_env_create(void* store_, const mlob_env_config* cfg, uint64_t seed, int env_index,
                     int* status) { /* env.hpp:100-122 */
  *status = validate(cfg);
  if (*status != MLOB_OK) return NULL;
  env* e = calloc(1, sizeof(env));
  e->st = store_;
  e->cfg = *cfg;
  e->seed = seed;
  e->env_index = env_index;
  *status = build_episode_index(e->st, cfg->steps_per_episode, cfg->messages_per_step,
                                cfg->start_stride_steps, &e->starts, &e->n_episodes);
  if (*status != MLOB_OK) {
    free(e);
    return NULL;
  }
  book_init(&e->bk, cfg->book_capacity);
  for (int s = 0; s < cfg->n_specs; ++s)
    for (int k = 0; k < cfg->specs[s].count; ++k) e->flat_spec[e->n_agents++] = s;
  for (int a = 0; a < e->n_agents; ++a) {
    e->ag[a].obs_n = observation_size(spec_of(e, a)->obs_space, cfg->obs_depth);
    /* >= 10: the reference writes the 10 executor features whatever the obs
     * space (env.hpp:115 vs 499-500; UB there for Executor+MMBasic). */
    e->ag[a].obs = calloc(e->ag[a].obs_n > 10 ? e->ag[a].obs_n : 10, sizeof(double));
  }
  e->terminal = 1;
  e->l2 = malloc(2 * (cfg->obs_depth + 1) * sizeof(mlob_level));
  return e;
}

uint64_t orc_env_n_episodes(void* e) { return ((env*)e)->n_episodes; }
uint64_t orc_env_episode_start(void* e, uint64_t ep) { return ((env*)e)->starts[ep]; }
int orc_env_n_agents(void* e) { return ((env*)e)->n_agents; }

static void l2_snapshot(env* e) { /* book.hpp:109-114 */
  e->l2_nb = aggregate_levels(&e->bk.side[0], e->cfg.obs_depth, e->l2);
  e->l2_na = aggregate_levels(&e->bk.side[1], e->cfg.obs_depth, e->l2 + e->cfg.obs_depth);
}

static double reference_price(const env* e, int a) { /* env.hpp:435-443 */
  const agent_state* st = &e->ag[a];
  if (spec_of(e, a)->params.ref_price == MLOB_REF_MID || st->inventory == 0)
    return (double)e->mid_half / 2.0;
  if (st->inventory > 0)
    return (double)(book_has(&e->bk, 0) ? book_best(&e->bk, 0) : e->last_bid);
  return (double)(book_has(&e->bk, 1) ? book_best(&e->bk, 1) : e->last_ask);
}

static double slippage(const agent_state* st) { /* rewards.hpp:69-75 */
  const double sign = st->task_dir == MLOB_TASK_BUY ? 1.0 : -1.0;
  double total = 0.0;
  for (uint64_t i = 0; i < st->fills.n; ++i)
    total += sign * (double)st->fills.v[i].quantity * (st->fills.v[i].price - st->p_init);
  return total;
}

static void fill_info(env* e, int a) { /* env.hpp:445-464 */
  agent_state* st = &e->ag[a];
  mlob_agent_info* info = &st->info;
  memset(info, 0, sizeof *info);
  info->inventory = st->inventory;
  info->cash = st->cash;
  info->portfolio_value = (double)st->inventory * reference_price(e, a) + (double)st->cash;
  info->slippage_step = spec_of(e, a)->type == MLOB_EXECUTOR ? slippage(st) : 0.0;
  st->slippage_total += info->slippage_step;
  info->slippage_total = st->slippage_total;
  info->task_remaining = st->task_remaining;
  int64_t filled = 0;
  for (uint64_t i = 0; i < st->fills.n; ++i) filled += st->fills.v[i].quantity;
  info->step_filled = filled;
  info->step_fill_count = (int32_t)st->fills.n;
}

/* observations.hpp:42-65 */
static double imbalance(const env* e) {
  int64_t bq = 0, aq = 0;
  for (uint32_t i = 0; i < e->l2_nb; ++i) bq += e->l2[i].quantity;
  for (uint32_t i = 0; i < e->l2_na; ++i) aq += e->l2[e->cfg.obs_depth + i].quantity;
  if (bq + aq == 0) return 0.0;
  return (double)(bq - aq) / (double)(bq + aq);
}
static double spread_ticks(int64_t bb, int64_t ba) {
  if (bb < 0 || ba < 0) return 0.0;
  const double s = (double)(ba - bb);
  return s < 32.0 ? s : 32.0;
}
static double qty_feature(int64_t q, int64_t order_size) {
  return (double)q / (double)(q + (order_size > 1 ? order_size : 1));
}
static double offset_feature(int64_t own, int64_t touch, int bid_side) {
  if (own < 0 || touch < 0) return -1.0;
  const double off = (double)(bid_side ? touch - own : own - touch);
  const double lo = -16.0 < off ? off : -16.0; /* std::max(-16.0, off) */
  return lo < 16.0 ? lo : 16.0;                 /* std::min(16.0, .) */
}
static double min32(double x) { return x < 32.0 ? x : 32.0; }

static void build_observation(env* e, int a) { /* env.hpp:466-503 */
  const mlob_agent_spec* sp = spec_of(e, a);
  const mlob_agent_params* p = &sp->params;
  agent_state* st = &e->ag[a];
  l2_snapshot(e);
  const int64_t bb = book_has(&e->bk, 0) ? book_best(&e->bk, 0) : -1;
  const int64_t ba = book_has(&e->bk, 1) ? book_best(&e->bk, 1) : -1;
  const double time_frac = (double)e->step / (double)e->cfg.steps_per_episode;
  const int64_t cash_scale_raw = p->inventory_cap * (int64_t)st->p_init;
  const int64_t cash_scale = cash_scale_raw > 1 ? cash_scale_raw : 1;
  int64_t own_bid = -1, own_ask = -1;
  for (uint64_t i = 0; i < st->active.n; ++i) {
    const mlob_active_order* o = &st->active.v[i];
    if (o->side == MLOB_BID)
      own_bid = own_bid < 0 ? o->price : (own_bid > o->price ? own_bid : o->price);
    else
      own_ask = own_ask < 0 ? o->price : (own_ask < o->price ? own_ask : o->price);
  }
  double* out = st->obs;
  const double dmid = (double)(e->mid_half - e->prev_mid_half) / 2.0;
  if (sp->type == MLOB_EXECUTOR) { /* observations.hpp:131-148 */
    const int direction = st->task_dir == MLOB_TASK_BUY ? 1 : -1;
    out[0] = (double)st->task_remaining / (double)(p->task_size > 1 ? p->task_size : 1);
    out[1] = time_frac;
    out[2] = (double)direction;
    out[3] = spread_ticks(bb, ba);
    out[4] = dmid;
    out[5] = (double)e->mid_half / 2.0 - st->p_init;
    out[6] = imbalance(e);
    out[7] = e->l2_nb > 0 ? qty_feature(e->l2[0].quantity, p->order_size) : 0.0;
    out[8] = e->l2_na > 0 ? qty_feature(e->l2[e->cfg.obs_depth].quantity, p->order_size) : 0.0;
    const int buy = direction > 0;
    out[9] = offset_feature(buy ? own_bid : own_ask, buy ? bb : ba, buy);
    return;
  }
  /* observations.hpp:105-129 */
  out[0] = (double)st->inventory / (double)p->inventory_cap;
  out[1] = (double)st->cash / (double)cash_scale;
  out[2] = spread_ticks(bb, ba);
  out[3] = dmid;
  out[4] = imbalance(e);
  out[5] = time_frac;
  out[6] = offset_feature(own_bid, bb, 1);
  out[7] = offset_feature(own_ask, ba, 0);
  if (sp->obs_space == MLOB_OBS_MM_BASIC) return;
  uint64_t k = 8;
  const uint64_t levels = (st->obs_n - 8) / 4;
  for (uint64_t d = 0; d < levels; ++d) {
    const int has_bid = d < e->l2_nb, has_ask = d < e->l2_na;
    const mlob_level* bl = &e->l2[d];
    const mlob_level* al = &e->l2[e->cfg.obs_depth + d];
    out[k++] = has_bid ? min32((double)(bb - bl->price)) : -1.0;
    out[k++] = has_bid ? qty_feature(bl->quantity, p->order_size) : 0.0;
    out[k++] = has_ask ? min32((double)(al->price - ba)) : -1.0;
    out[k++] = has_ask ? qty_feature(al->quantity, p->order_size) : 0.0;
  }
}

int orc_env_reset(void* e_, uint64_t episode) { /* env.hpp:143-192 */
  env* e = e_;
  if (episode >= e->n_episodes)
    return fail(MLOB_E_OUT_OF_RANGE, "MarketEnv::reset: episode %llu out of range (count %llu)",
                (unsigned long long)episode, (unsigned long long)e->n_episodes);
  const uint64_t start = e->starts[episode];
  const state_rec* snap = state_before(e->st, start);
  if (!snap)
    return fail(MLOB_E_RUNTIME,
                "MarketEnv::reset: no book state sampled at episode start offset %llu; reload "
                "the data with a matching sample stride",
                (unsigned long long)start);
  e->episode = episode;
  book_clear(&e->bk);
  int rc = book_init_from_l2(&e->bk, snap->levels, snap->nb, snap->levels + snap->nb, snap->na,
                             e->cfg.synthetic_init_id_base);
  if (rc != MLOB_OK) return rc;
  e->mid_half = book_mid_half(&e->bk, e->cfg.fallback_mid_half);
  e->prev_mid_half = e->mid_half;
  e->mbar = (double)e->mid_half / 2.0;
  e->last_bid = book_has(&e->bk, 0) ? book_best(&e->bk, 0) : e->mid_half / 2 - 1;
  e->last_ask = book_has(&e->bk, 1) ? book_best(&e->bk, 1) : (e->mid_half + 1) / 2 + 1;
  e->step = 0;
  e->terminal = 0;
  for (int a = 0; a < e->n_agents; ++a) {
    agent_state* st = &e->ag[a];
    st->inventory = 0;
    st->cash = 0;
    st->active.n = 0;
    st->order_nonce = 0;
    st->filled_total = 0;
    st->slippage_total = 0.0;
    st->p_init = (double)e->mid_half / 2.0;
    const mlob_agent_spec* sp = spec_of(e, a);
    if (sp->type == MLOB_EXECUTOR) {
      const uint64_t w[5] = {(uint64_t)(int64_t)e->env_index, episode, 0, RNG_TASKDIR, (uint64_t)a};
      crng r = {make_key(e->seed, 5, w)};
      st->task_dir = crng_coin(&r) ? MLOB_TASK_BUY : MLOB_TASK_SELL;
      st->task_remaining = sp->params.task_size;
    } else {
      st->task_remaining = 0;
    }
    st->fills.n = 0;
  }
  e->step_trades.n = 0;
  for (int a = 0; a < e->n_agents; ++a) {
    e->ag[a].reward = 0.0;
    e->ag[a].done = 0;
    fill_info(e, a);
    build_observation(e, a);
  }
  return MLOB_OK;
}

static void effective_tops(const env* e, int a, int64_t* bid, int64_t* ask) { /* env.hpp:266-275 */
  const mlob_agent_params* p = &spec_of(e, a)->params;
  const int64_t mid_floor = e->mid_half >= 0 ? e->mid_half / 2 : (e->mid_half - 1) / 2;
  const int64_t mid_ceil = (e->mid_half + 1) / 2;
  int64_t b = book_has(&e->bk, 0) ? book_best(&e->bk, 0) : mid_floor - p->default_half_spread;
  int64_t k = book_has(&e->bk, 1) ? book_best(&e->bk, 1) : mid_ceil + p->default_half_spread;
  if (b < 1) b = 1;
  if (k <= b) k = b + 1;
  *bid = b;
  *ask = k;
}

static int convert_action(env* e, int a, const mlob_agent_action* action, int64_t step_time) {
  /* env.hpp:285-370 */
  const mlob_agent_spec* sp = spec_of(e, a);
  const mlob_agent_params* p = &sp->params;
  agent_state* st = &e->ag[a];
  quote_list q;
  memset(&q, 0, sizeof q);
  int rc = MLOB_OK;
  if (action->direct) {
    q.n = action->n_quotes;
    for (int i = 0; i < q.n; ++i) q.q[i] = action->quotes[i];
    if (sp->type == MLOB_EXECUTOR) {
      for (int i = 0; i < q.n; ++i)
        if (q.q[i].quantity > st->task_remaining) q.q[i].quantity = st->task_remaining;
      if (q.n == 1 && q.q[0].quantity <= 0) q.n = 0;
    }
  } else {
    int64_t bid, ask;
    effective_tops(e, a, &bid, &ask);
    switch (sp->type) {
      case MLOB_EXECUTOR: {
        int64_t eb = bid, ea = ask;
        if (st->task_dir == MLOB_TASK_BUY && !book_has(&e->bk, 1))
          ea = e->last_ask + 1 > 2 ? e->last_ask + 1 : 2;
        if (st->task_dir == MLOB_TASK_SELL && !book_has(&e->bk, 0))
          eb = e->last_bid - 1 > 1 ? e->last_bid - 1 : 1;
        rc = decode_exec(action->id, eb, ea, p->order_size, p->exec_complex, st->task_dir,
                         st->task_remaining, &q);
        break;
      }
      case MLOB_DIRECTIONAL:
        rc = decode_directional(action->id, bid, ask, p->order_size, &q);
        break;
      case MLOB_MARKET_MAKER:
        switch (sp->mm_space) {
          case MLOB_FIXED_QUANT:
            rc = decode_fixed_quant(action->id, bid, ask, p->order_size, p->fixed_quant_from_mid, &q);
            break;
          case MLOB_SPREAD_SKEW:
            rc = decode_spread_skew(action->id, e->mid_half, p, p->order_size, &q);
            break;
          case MLOB_AVST:
            rc = decode_avst(action->id, e->mid_half, st->inventory, e->step, p, p->order_size, &q);
            break;
        }
        break;
    }
    if (rc != MLOB_OK) return rc;
  }
  int kept[2] = {0, 0};
  for (uint64_t i = 0; i < st->active.n; ++i) {
    const mlob_active_order* o = &st->active.v[i];
    int reused = 0;
    for (int k = 0; k < q.n; ++k)
      if (q.q[k].side == o->side && q.q[k].price == o->price) {
        reused = 1;
        kept[k] = 1;
      }
    if (reused) continue;
    mlob_message m;
    memset(&m, 0, sizeof m);
    m.time = step_time;
    m.kind = MLOB_DELETE;
    m.side = o->side;
    m.order_id = o->order_id;
    m.trader_id = a + 1;
    VEC_PUSH(e->agent_msgs, m);
  }
  for (int k = 0; k < q.n; ++k) {
    if (kept[k]) continue;
    mlob_message m;
    memset(&m, 0, sizeof m);
    m.time = step_time;
    m.kind = MLOB_NEW_LIMIT;
    m.side = q.q[k].side;
    m.price = q.q[k].price;
    m.quantity = q.q[k].quantity;
    m.order_id = e->cfg.agent_id_base + (uint64_t)a * e->cfg.agent_id_range + st->order_nonce++;
    m.trader_id = a + 1;
    VEC_PUSH(e->agent_msgs, m);
  }
  return MLOB_OK;
}

static void apply_fill(env* e, int a, int64_t price, int64_t qty, int side) { /* env.hpp:381-396 */
  agent_state* st = &e->ag[a];
  if (side == MLOB_BID) {
    st->inventory += qty;
    st->cash -= price * qty;
  } else {
    st->inventory -= qty;
    st->cash += price * qty;
  }
  const fill f = {(double)price, qty, side};
  VEC_PUSH(st->fills, f);
  st->filled_total += qty;
  if (spec_of(e, a)->type == MLOB_EXECUTOR) {
    const int task_side = (st->task_dir == MLOB_TASK_BUY) == (side == MLOB_BID);
    if (task_side) {
      const int64_t r = st->task_remaining - qty;
      st->task_remaining = r > 0 ? r : 0;
    }
  }
}

static void run_message(env* e, const mlob_message* m, int64_t* mid_sum, int64_t* mid_count) {
  /* env.hpp:223-235 */
  e->trades.n = 0;
  book_process(&e->bk, m, &e->trades);
  for (uint64_t i = 0; i < e->trades.n; ++i) {
    const mlob_trade* t = &e->trades.v[i];
    VEC_PUSH(e->step_trades, *t);
    if (t->passive_trader_id > 0) /* env.hpp:372-379 */
      apply_fill(e, t->passive_trader_id - 1, t->price, t->quantity, 1 - t->aggressor_side);
    if (t->aggressor_trader_id > 0)
      apply_fill(e, t->aggressor_trader_id - 1, t->price, t->quantity, t->aggressor_side);
  }
  e->mid_half = book_mid_half(&e->bk, e->mid_half);
  *mid_sum += e->mid_half;
  ++*mid_count;
  ++e->messages_processed;
  e->last_time = m->time;
}

static void rebuild_active_orders(env* e) { /* env.hpp:398-407 */
  for (int a = 0; a < e->n_agents; ++a) e->ag[a].active.n = 0;
  for (int s = 0; s < 2; ++s)
    for (uint64_t i = 0; i < e->bk.side[s].n; ++i) {
      const mlob_resting_order* o = &e->bk.side[s].v[i];
      if (o->trader_id <= 0) continue;
      mlob_active_order ao;
      memset(&ao, 0, sizeof ao);
      ao.order_id = o->order_id;
      ao.price = o->price;
      ao.quantity = o->quantity;
      ao.side = (uint8_t)s;
      VEC_PUSH(e->ag[o->trader_id - 1].active, ao);
    }
}

static double compute_reward(const env* e, int a) { /* env.hpp:409-433, rewards.hpp */
  const mlob_agent_spec* sp = spec_of(e, a);
  const mlob_agent_params* p = &sp->params;
  const agent_state* st = &e->ag[a];
  const double mid_ticks = (double)e->mid_half / 2.0;
  const double prev_ticks = (double)e->prev_mid_half / 2.0;
  double r = 0.0;
  double psi_buy = 0.0, psi_sell = 0.0;
  if (sp->reward != MLOB_REWARD_EXEC) {
    for (uint64_t i = 0; i < st->fills.n; ++i) /* rewards.hpp:22-28 */
      if (st->fills.v[i].side == MLOB_BID)
        psi_buy += (e->mbar - st->fills.v[i].price) * (double)st->fills.v[i].quantity;
    for (uint64_t i = 0; i < st->fills.n; ++i) /* rewards.hpp:30-36 */
      if (st->fills.v[i].side == MLOB_ASK)
        psi_sell += (st->fills.v[i].price - e->mbar) * (double)st->fills.v[i].quantity;
  }
  switch (sp->reward) {
    case MLOB_REWARD_BUYSELL: r = psi_buy + psi_sell; break; /* rewards.hpp:38-40 */
    case MLOB_REWARD_SPOONER: {                              /* rewards.hpp:45-53 */
      const double psi_inv = (double)st->inventory * (mid_ticks - prev_ticks);
      r = psi_buy + psi_sell + psi_inv - (1.0 - p->lambda) * (0.0 < psi_inv ? psi_inv : 0.0);
      break;
    }
    case MLOB_REWARD_EXEC: /* rewards.hpp:81-89 */
      r = -slippage(st);
      if (e->terminal && st->task_remaining > 0)
        r -= p->unfilled_penalty_coef * (double)st->task_remaining * st->p_init;
      break;
  }
  if (sp->reward != MLOB_REWARD_EXEC && p->quadratic_penalty) { /* rewards.hpp:55-61 */
    const double frac = (double)st->inventory / (double)p->inventory_cap;
    r -= p->rho * frac * frac;
  }
  return r * p->reward_scale;
}

int orc_env_step(void* e_, const mlob_agent_action* actions, uint64_t n) { /* env.hpp:194-254 */
  env* e = e_;
  if (e->terminal) return fail(MLOB_E_LOGIC, "MarketEnv::step: episode is terminal; reset first");
  if (n != (uint64_t)e->n_agents)
    return fail(MLOB_E_INVALID_ARGUMENT, "MarketEnv::step: expected %d actions, got %llu",
                e->n_agents, (unsigned long long)n);
  const uint64_t mps = (uint64_t)e->cfg.messages_per_step;
  const mlob_message* slice = NULL;
  if (mps > 0) /* store.hpp:75-89 */
    slice = e->st->msgs.v + e->starts[e->episode] + (uint64_t)e->step * mps;
  const int64_t step_time = mps == 0 ? e->last_time + 1 : slice[0].time;

  e->agent_msgs.n = 0; /* (1) */
  for (int a = 0; a < e->n_agents; ++a) {
    const int rc = convert_action(e, a, &actions[a], step_time);
    if (rc != MLOB_OK) return rc;
  }
  /* (2) rng.hpp:63-71 */
  const uint64_t w[4] = {(uint64_t)(int64_t)e->env_index, e->episode, (uint64_t)e->step, RNG_SHUFFLE};
  crng r = {make_key(e->seed, 4, w)};
  if (e->agent_msgs.n >= 2)
    for (uint64_t i = e->agent_msgs.n - 1; i > 0; --i) {
      const uint64_t j = crng_below(&r, i + 1);
      if (i != j) {
        const mlob_message t = e->agent_msgs.v[i];
        e->agent_msgs.v[i] = e->agent_msgs.v[j];
        e->agent_msgs.v[j] = t;
      }
    }
  /* (3) + (4) */
  e->prev_mid_half = e->mid_half;
  int64_t mid_sum = 0, mid_count = 0;
  e->step_trades.n = 0;
  for (int a = 0; a < e->n_agents; ++a) e->ag[a].fills.n = 0;
  for (uint64_t i = 0; i < e->agent_msgs.n; ++i)
    run_message(e, &e->agent_msgs.v[i], &mid_sum, &mid_count);
  for (uint64_t i = 0; i < mps; ++i) run_message(e, &slice[i], &mid_sum, &mid_count);
  if (book_has(&e->bk, 0)) e->last_bid = book_best(&e->bk, 0);
  if (book_has(&e->bk, 1)) e->last_ask = book_best(&e->bk, 1);
  /* (5) */
  e->mbar = mid_count > 0 ? (double)mid_sum / (2.0 * (double)mid_count)
                          : (double)e->prev_mid_half / 2.0;
  rebuild_active_orders(e);
  ++e->step;
  e->terminal = e->step >= e->cfg.steps_per_episode;
  for (int a = 0; a < e->n_agents; ++a) {
    e->ag[a].reward = compute_reward(e, a);
    e->ag[a].done = e->terminal ? 1 : 0;
    fill_info(e, a);
    build_observation(e, a);
  }
  return MLOB_OK;
}

int orc_env_step_ids(void* e, const int32_t* ids, uint64_t n) { /* env.hpp:256-263 */
  mlob_agent_action* acts = calloc(n ? n : 1, sizeof(mlob_agent_action));
  for (uint64_t i = 0; i < n; ++i) acts[i].id = ids[i];
  const int rc = orc_env_step(e, acts, n);
  free(acts);
  return rc;
}

void orc_env_scalars(void* e_, mlob_env_scalars* o) {
  const env* e = e_;
  memset(o, 0, sizeof *o);
  o->step = e->step;
  o->terminal = e->terminal;
  o->episode = e->episode;
  o->mid_half = e->mid_half;
  o->prev_mid_half = e->prev_mid_half;
  o->mean_mid_ticks = e->mbar;
  o->last_bid = e->last_bid;
  o->last_ask = e->last_ask;
  o->last_time = e->last_time;
  o->messages_processed = e->messages_processed;
  o->next_seq = e->bk.next_seq;
  o->live_bid = e->bk.side[0].n;
  o->live_ask = e->bk.side[1].n;
}

uint64_t orc_env_book(void* e, int side, mlob_resting_order* out, uint64_t cap) {
  return orc_book_orders(&((env*)e)->bk, side, out, cap);
}

void orc_env_agent(void* e_, int a, mlob_agent_state* o) {
  const agent_state* s = &((env*)e_)->ag[a];
  memset(o, 0, sizeof *o);
  o->inventory = s->inventory;
  o->cash = s->cash;
  o->task_remaining = s->task_remaining;
  o->task_dir = s->task_dir;
  o->p_init = s->p_init;
  o->order_nonce = s->order_nonce;
  o->filled_total = s->filled_total;
  o->slippage_total = s->slippage_total;
  o->n_active = (int32_t)s->active.n;
  for (uint64_t i = 0; i < s->active.n && i < MLOB_MAX_ACTIVE; ++i) o->active[i] = s->active.v[i];
}

void orc_env_info(void* e, int a, mlob_agent_info* o) { *o = ((env*)e)->ag[a].info; }
double orc_env_reward(void* e, int a) { return ((env*)e)->ag[a].reward; }
int orc_env_done(void* e, int a) { return ((env*)e)->ag[a].done; }
uint64_t orc_env_obs(void* e, int a, double* out, uint64_t cap) {
  const agent_state* s = &((env*)e)->ag[a];
  for (uint64_t i = 0; i < s->obs_n && i < cap; ++i) out[i] = s->obs[i];
  return s->obs_n;
}
uint64_t orc_env_trades(void* e_, mlob_trade* out, uint64_t cap) {
  const env* e = e_;
  for (uint64_t i = 0; i < e->step_trades.n && i < cap; ++i) out[i] = e->step_trades.v[i];
  return e->step_trades.n;
}

void orc_env_free(void* e_) {
  env* e = e_;
  if (!e) return;
  for (int a = 0; a < e->n_agents; ++a) {
    free(e->ag[a].active.v);
    free(e->ag[a].fills.v);
    free(e->ag[a].obs);
  }
  book_release(&e->bk);
  free(e->agent_msgs.v);
  free(e->trades.v);
  free(e->step_trades.v);
  free(e->l2);
  free(e->starts);
  free(e);
}

/* ------------------------------------------------------------------------ */
/* ippo/rollout.hpp:151-336 MarketVecEnv (single-threaded: results do not
 * depend on worker count, thread_pool.hpp:11-14)                           */

typedef struct venv {
  mlob_env_config cfg;
  uint64_t* pool;
  uint64_t pool_len;
  int n_envs;
  env** envs;
  uint64_t* cursor;
  int type_offset[MLOB_MAX_SPECS];
  int agents_per_env;
  mlob_agent_action* actions;
  uint8_t* just_reset;
  double* rewards;
  uint8_t* dones;
  int64_t* episodes_finished;
  double *t_pv, *t_slip, *t_comp, *t_inv;
  struct rollout_state* roll; /* collect_rollout state (below) */
} venv;
static void rollout_free(struct rollout_state* r);

void* orc_venv_create(void* st, const mlob_env_config* cfg, const uint64_t* pool,
                      uint64_t pool_len, uint64_t seed, int n_envs, int workers, int* status) {
  (void)workers;
  if (n_envs < 1) {
    *status = fail(MLOB_E_INVALID_ARGUMENT, "MarketVecEnv: n_envs >= 1");
    return NULL;
  }
  venv* v = calloc(1, sizeof(venv));
  v->cfg = *cfg;
  v->n_envs = n_envs;
  v->envs = calloc((size_t)n_envs, sizeof(env*));
  for (int e = 0; e < n_envs; ++e) {
    v->envs[e] = orc_env_create(st, cfg, seed, e, status);
    if (*status != MLOB_OK) return NULL;
  }
  if (pool) {
    v->pool_len = pool_len;
    v->pool = malloc(pool_len * sizeof(uint64_t));
    memcpy(v->pool, pool, pool_len * sizeof(uint64_t));
  } else {
    v->pool_len = v->envs[0]->n_episodes;
    v->pool = malloc((v->pool_len + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < v->pool_len; ++i) v->pool[i] = i;
  }
  if (v->pool_len == 0) {
    *status = fail(MLOB_E_INVALID_ARGUMENT, "MarketVecEnv: empty episode pool");
    return NULL;
  }
  int off = 0;
  for (int s = 0; s < cfg->n_specs; ++s) {
    v->type_offset[s] = off;
    off += cfg->specs[s].count;
  }
  v->agents_per_env = off;
  const size_t na = (size_t)n_envs * (size_t)(off ? off : 1);
  v->cursor = calloc((size_t)n_envs, sizeof(uint64_t));
  v->actions = calloc(na, sizeof(mlob_agent_action));
  v->just_reset = malloc((size_t)n_envs);
  memset(v->just_reset, 1, (size_t)n_envs);
  v->rewards = calloc(na, sizeof(double));
  v->dones = calloc(na, 1);
  v->episodes_finished = calloc((size_t)n_envs, sizeof(int64_t));
  v->t_pv = calloc(na, sizeof(double));
  v->t_slip = calloc(na, sizeof(double));
  v->t_comp = calloc(na, sizeof(double));
  v->t_inv = calloc(na, sizeof(double));
  *status = MLOB_OK;
  return v;
}

static uint64_t episode_for(const venv* v, uint64_t e, uint64_t k) { /* rollout.hpp:286-288 */
  return v->pool[(e + k * (uint64_t)v->n_envs) % v->pool_len];
}

int orc_venv_reset_all(void* v_) { /* rollout.hpp:194-200 */
  venv* v = v_;
  for (int e = 0; e < v->n_envs; ++e) {
    const int rc = orc_env_reset(v->envs[e], episode_for(v, (uint64_t)e, 0));
    if (rc != MLOB_OK) return rc;
    v->cursor[e] = 1;
    v->just_reset[e] = 1;
  }
  return MLOB_OK;
}

int orc_venv_set_action(void* v_, int type, uint64_t stream, int action) { /* rollout.hpp:215-222 */
  venv* v = v_;
  const uint64_t count = (uint64_t)v->cfg.specs[type].count;
  const uint64_t e = stream / count, k = stream % count;
  mlob_agent_action* slot = &v->actions[e * (uint64_t)v->agents_per_env + (uint64_t)v->type_offset[type] + k];
  memset(slot, 0, sizeof *slot);
  slot->id = action;
  return MLOB_OK;
}

int orc_venv_step_all(void* v_) { /* rollout.hpp:224-234 -> step_one 290-318 */
  venv* v = v_;
  const int A = v->agents_per_env;
  for (int e = 0; e < v->n_envs; ++e) {
    env* en = v->envs[e];
    int rc = orc_env_step(en, v->actions + (size_t)e * (size_t)A, (uint64_t)A);
    if (rc != MLOB_OK) return rc;
    for (int a = 0; a < A; ++a) {
      v->rewards[e * A + a] = en->ag[a].reward;
      v->dones[e * A + a] = en->ag[a].done;
    }
    v->just_reset[e] = 0;
    if (en->terminal) {
      for (int a = 0; a < A; ++a) {
        const mlob_agent_info* info = &en->ag[a].info;
        const size_t slot = (size_t)e * (size_t)A + (size_t)a;
        v->t_pv[slot] += info->portfolio_value;
        v->t_slip[slot] += info->slippage_total;
        const mlob_agent_spec* sp = spec_of(en, a);
        v->t_comp[slot] += sp->type == MLOB_EXECUTOR
                               ? 1.0 - (double)info->task_remaining / (double)sp->params.task_size
                               : 0.0;
        v->t_inv[slot] += (double)info->inventory * (double)info->inventory;
      }
      ++v->episodes_finished[e];
      rc = orc_env_reset(en, episode_for(v, (uint64_t)e, v->cursor[e]++));
      if (rc != MLOB_OK) return rc;
      v->just_reset[e] = 1;
    }
  }
  return MLOB_OK;
}

void orc_venv_gather(void* v_, int type, double* obs, uint8_t* resets) { /* rollout.hpp:202-213 */
  venv* v = v_;
  const int count = v->cfg.specs[type].count, off = v->type_offset[type];
  const uint64_t dim = observation_size(v->cfg.specs[type].obs_space, v->cfg.obs_depth);
  for (int e = 0; e < v->n_envs; ++e)
    for (int k = 0; k < count; ++k) {
      const agent_state* st = &v->envs[e]->ag[off + k];
      if (obs) memcpy(obs + ((uint64_t)e * count + k) * dim, st->obs, dim * sizeof(double));
      if (resets) resets[e * count + k] = v->just_reset[e];
    }
}

double orc_venv_reward(void* v_, int type, uint64_t stream) {
  venv* v = v_;
  const uint64_t count = (uint64_t)v->cfg.specs[type].count;
  return v->rewards[(stream / count) * v->agents_per_env + v->type_offset[type] + stream % count];
}
int orc_venv_done(void* v_, int type, uint64_t stream) {
  venv* v = v_;
  const uint64_t count = (uint64_t)v->cfg.specs[type].count;
  return v->dones[(stream / count) * v->agents_per_env + v->type_offset[type] + stream % count] != 0;
}

void orc_venv_episode_stats(void* v_, int type, mlob_episode_stats* out) { /* rollout.hpp:255-270 */
  venv* v = v_;
  memset(out, 0, sizeof *out);
  const int count = v->cfg.specs[type].count, off = v->type_offset[type];
  for (int e = 0; e < v->n_envs; ++e) {
    for (int k = 0; k < count; ++k) {
      const size_t slot = (size_t)e * v->agents_per_env + off + k;
      out->pv_sum += v->t_pv[slot];
      out->slippage_sum += v->t_slip[slot];
      out->completion_sum += v->t_comp[slot];
      out->inventory_sq_sum += v->t_inv[slot];
    }
    out->episodes += v->episodes_finished[e];
  }
}

void orc_venv_clear_episode_stats(void* v_) { /* rollout.hpp:272-278 */
  venv* v = v_;
  const size_t na = (size_t)v->n_envs * (size_t)(v->agents_per_env ? v->agents_per_env : 1);
  memset(v->t_pv, 0, na * sizeof(double));
  memset(v->t_slip, 0, na * sizeof(double));
  memset(v->t_comp, 0, na * sizeof(double));
  memset(v->t_inv, 0, na * sizeof(double));
  memset(v->episodes_finished, 0, (size_t)v->n_envs * sizeof(int64_t));
}

void* orc_venv_instance(void* v, uint64_t e) { return ((venv*)v)->envs[e]; }

void orc_venv_free(void* v_) {
  venv* v = v_;
  if (!v) return;
  rollout_free(v->roll);
  for (int e = 0; e < v->n_envs; ++e) orc_env_free(v->envs[e]);
  free(v->envs);
  free(v->pool);
  free(v->cursor);
  free(v->actions);
  free(v->just_reset);
  free(v->rewards);
  free(v->dones);
  free(v->episodes_finished);
  free(v->t_pv);
  free(v->t_slip);
  free(v->t_comp);
  free(v->t_inv);
  free(v);
}

/* ------------------------------------------------------------------------ */
/* bench/bench.hpp:98-160, one (messages, agents) grid cell, one worker      */

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int orc_bench_run(void* st, const mlob_env_config* base, int n_envs, int n_steps, int warmup,
                  int workers, uint64_t seed, int messages_per_step, int agents_per_type,
                  orc_bench_row* out) {
  (void)workers;
  mlob_env_config cfg = *base; /* bench.hpp:84-90 */
  cfg.messages_per_step = messages_per_step;
  for (int s = 0; s < cfg.n_specs; ++s) cfg.specs[s].count = agents_per_type;
  int status = MLOB_OK;
  env** envs = calloc((size_t)n_envs, sizeof(env*));
  for (int e = 0; e < n_envs; ++e) {
    envs[e] = orc_env_create(st, &cfg, seed, e, &status);
    if (status != MLOB_OK) return status;
  }
  const uint64_t n_ep = envs[0]->n_episodes;
  if (n_ep == 0) return fail(MLOB_E_RUNTIME, "run_throughput: store too short for the episode shape");
  const int A = envs[0]->n_agents;
  int arity[MLOB_MAX_AGENTS];
  for (int a = 0; a < A; ++a) arity[a] = action_arity(spec_of(envs[0], a));
  uint64_t* cursor = calloc((size_t)n_envs, sizeof(uint64_t));
  for (int e = 0; e < n_envs; ++e) {
    if ((status = orc_env_reset(envs[e], (uint64_t)e % n_ep)) != MLOB_OK) return status;
    cursor[e] = 1;
  }
  int32_t ids[MLOB_MAX_AGENTS];
  uint64_t global_step = 0, before = 0, after = 0;
  double t0 = 0.0;
  for (int s = 0; s < warmup + n_steps; ++s) {
    if (s == warmup) {
      for (int e = 0; e < n_envs; ++e) before += envs[e]->messages_processed;
      t0 = now_s();
    }
    for (int e = 0; e < n_envs; ++e) { /* bench.hpp:53-70 */
      const uint64_t w[3] = {RNG_BENCH_ACTION, (uint64_t)e, global_step};
      crng r = {make_key(seed, 3, w)};
      for (int a = 0; a < A; ++a) ids[a] = (int32_t)crng_below(&r, (uint64_t)arity[a]);
      if ((status = orc_env_step_ids(envs[e], ids, (uint64_t)A)) != MLOB_OK) return status;
      if (envs[e]->terminal) {
        status = orc_env_reset(envs[e], ((uint64_t)e + cursor[e] * (uint64_t)n_envs) % n_ep);
        if (status != MLOB_OK) return status;
        ++cursor[e];
      }
    }
    ++global_step;
  }
  const double wall = now_s() - t0;
  for (int e = 0; e < n_envs; ++e) after += envs[e]->messages_processed;
  memset(out, 0, sizeof *out);
  out->messages_per_step = messages_per_step;
  out->agents_per_type = agents_per_type;
  out->workers = 1;
  out->env_steps = (uint64_t)n_envs * (uint64_t)n_steps;
  out->messages = after - before;
  out->wall_seconds = wall;
  out->steps_per_sec = (double)out->env_steps / wall;
  out->messages_per_sec = (double)out->messages / wall;
  out->worker_utilization = 1.0;
  for (int e = 0; e < n_envs; ++e) orc_env_free(envs[e]);
  free(envs);
  free(cursor);
  return MLOB_OK;
}

/* ------------------------------------------------------------------------ */
/* RNG exports and tests/reference/random_messages.hpp:30-119 restated       */

uint64_t orc_splitmix64(uint64_t z) { return splitmix64(z); }
uint64_t orc_make_key(uint64_t seed, int n, const uint64_t* words) { return make_key(seed, n, words); }
void orc_crng_draws(uint64_t key, uint64_t n, uint64_t* out) {
  crng r = {key};
  for (uint64_t i = 0; i < n; ++i) out[i] = crng_next(&r);
}

void orc_random_stream(const orc_stream_config* cfg, uint64_t seed, mlob_message* out) {
  enum { kRecent = 512 };
  const uint64_t w = 0x5eedu;
  crng rng = {make_key(seed, 1, &w)};
  int64_t ref = cfg->initial_ref, time = 0;
  uint64_t next_id = 1, recent_n = 0, recent_pos = 0;
  uint64_t recent_id[kRecent];
  int recent_side[kRecent];
  for (uint64_t i = 0; i < cfg->n_messages; ++i) {
    time += 1 + (int64_t)crng_below(&rng, 1000);
    if (crng_uniform(&rng) < 0.02) ref += crng_coin(&rng) ? 1 : -1;
    if (ref < cfg->band + 2) ref = cfg->band + 2;
    mlob_message m;
    memset(&m, 0, sizeof m);
    m.time = time;
    const double u = crng_uniform(&rng);
    const int side = crng_coin(&rng) ? MLOB_BID : MLOB_ASK;
    m.side = (uint8_t)side;
    const double c1 = cfg->p_new, c2 = c1 + cfg->p_cancel, c3 = c2 + cfg->p_delete,
                 c4 = c3 + cfg->p_execute;
    if (u < c1) {
      m.kind = MLOB_NEW_LIMIT;
      m.order_id = next_id++;
      m.quantity = 1 + (int64_t)crng_below(&rng, (uint64_t)cfg->max_qty);
      const int64_t off = (int64_t)crng_below(&rng, (uint64_t)cfg->band);
      if (crng_uniform(&rng) < cfg->p_marketable)
        m.price = side == MLOB_BID ? ref + 1 + off / 4 : ref - off / 4;
      else
        m.price = side == MLOB_BID ? ref - off : ref + 1 + off;
      if (m.price < 1) m.price = 1;
      if (recent_n < kRecent) { /* remember() */
        recent_id[recent_n] = m.order_id;
        recent_side[recent_n++] = side;
      } else {
        recent_id[recent_pos % kRecent] = m.order_id;
        recent_side[recent_pos++ % kRecent] = side;
      }
    } else if (u < c4) {
      m.kind = u < c2 ? MLOB_CANCEL_PARTIAL : u < c3 ? MLOB_DELETE : MLOB_EXECUTE_VISIBLE;
      /* pick_target() */
      if (recent_n == 0 || crng_uniform(&rng) < cfg->p_absent) {
        m.order_id = next_id + 1000000;
        m.side = crng_coin(&rng) ? MLOB_BID : MLOB_ASK;
      } else {
        const uint64_t k = crng_below(&rng, recent_n);
        m.order_id = recent_id[k];
        m.side = (uint8_t)recent_side[k];
      }
      m.quantity = m.kind == MLOB_DELETE ? 0 : 1 + (int64_t)crng_below(&rng, (uint64_t)cfg->max_qty);
    } else {
      const uint64_t k = crng_below(&rng, 3);
      m.kind = k == 0 ? MLOB_EXECUTE_HIDDEN : k == 1 ? MLOB_CROSS : MLOB_HALT;
      m.order_id = 0;
      m.quantity = 1;
      m.price = ref;
    }
    out[i] = m;
  }
}

/* ------------------------------------------------------------------------ */
/* baselines/twap.hpp, baselines/avst.hpp, ippo/evaluate.hpp (scripted)      */

static void quotes_to_action(const quote_list* q, mlob_agent_action* act) {
  memset(act, 0, sizeof *act);
  act->direct = 1;
  act->n_quotes = q->n;
  for (int i = 0; i < q->n; ++i) act->quotes[i] = q->q[i];
}

/* twap_policy (twap.hpp:37-58) over make_twap_plan(task_size, steps) (twap.hpp:21-33) */
static void twap_action(const env* e, int a, int mode, int step, mlob_agent_action* act) {
  const agent_state* st = &e->ag[a];
  const int64_t T = spec_of(e, a)->params.task_size, S = e->cfg.steps_per_episode;
  const int64_t sched = ((int64_t)(step + 1) * T) / S - ((int64_t)step * T) / S;
  const int last = step + 1 == S;
  const int64_t qty = last ? st->task_remaining : (sched < st->task_remaining ? sched : st->task_remaining);
  quote_list q = {.n = 0};
  if (qty > 0) {
    int64_t bid, ask;
    effective_tops(e, a, &bid, &ask);
    const int buy = st->task_dir == MLOB_TASK_BUY;
    const int64_t price = mode == MLOB_TWAP_AGGRESSIVE ? (buy ? ask : bid) : (buy ? bid : ask);
    ql_push(&q, buy ? MLOB_BID : MLOB_ASK, price, qty);
  }
  quotes_to_action(&q, act);
}

/* avst_policy (avst.hpp:19-32): decode_avst with the baseline's parameters */
static int avst_action(const env* e, int a, const mlob_policy* p, mlob_agent_action* act) {
  if (p->avst_gamma_index < 0 || p->avst_gamma_index >= p->n_gamma)
    return fail(MLOB_E_OUT_OF_RANGE, "avst_policy: gamma_index out of range");
  mlob_agent_params prm;
  memset(&prm, 0, sizeof prm);
  prm.n_gamma = p->n_gamma;
  memcpy(prm.gamma_grid, p->gamma_grid, sizeof prm.gamma_grid);
  prm.kappa = p->kappa;
  prm.sigma = p->sigma;
  prm.horizon = p->horizon;
  quote_list q = {.n = 0};
  const int rc = decode_avst(p->avst_gamma_index, e->mid_half, e->ag[a].inventory, e->step, &prm,
                             spec_of(e, a)->params.order_size, &q);
  if (rc != MLOB_OK) return rc;
  quotes_to_action(&q, act);
  return MLOB_OK;
}

/* detail::choose_action (evaluate.hpp:56-99) for the scripted kinds */
static int choose_action(const env* e, int a, const mlob_policy* p, int step, uint64_t seed,
                         uint64_t cell_id, uint64_t episode, mlob_agent_action* act) {
  memset(act, 0, sizeof *act);
  switch (p->kind) {
    case MLOB_POLICY_NOOP: act->direct = 1; return MLOB_OK;
    case MLOB_POLICY_TWAP: twap_action(e, a, p->twap_mode, step, act); return MLOB_OK;
    case MLOB_POLICY_AVST: return avst_action(e, a, p, act);
    case MLOB_POLICY_RANDOM: {
      const uint64_t w[5] = {8 /* EpisodeDraw */, cell_id, episode, (uint64_t)step, (uint64_t)a};
      crng r = {make_key(seed, 5, w)};
      act->id = (int)crng_below(&r, (uint64_t)action_arity(spec_of(e, a)));
      return MLOB_OK;
    }
  }
  return fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: learned policy without a network");
}

int orc_choose_action(void* e, int a, const mlob_policy* p, int step, uint64_t seed, uint64_t cell_id,
                      uint64_t episode, mlob_agent_action* out) {
  return choose_action((const env*)e, a, p, step, seed, cell_id, episode, out);
}

static void policy_forward(const mlob_policy_net* net, const double* obs, const double* hidden,
                           const uint8_t* reset_mask, uint64_t batch, double* logits, double* values,
                           double* hidden_out);

static void mean_stderr(const double* xs, uint64_t n, double* mean, double* se) { /* evaluate.hpp:188-197 */
  const double k = (double)n;
  double m = 0.0;
  for (uint64_t i = 0; i < n; ++i) m += xs[i];
  m /= k;
  double var = 0.0;
  for (uint64_t i = 0; i < n; ++i) var += (xs[i] - m) * (xs[i] - m);
  *mean = m;
  *se = n > 1 ? sqrt(var / (k - 1.0) / k) : 0.0;
}

int orc_evaluate_matrix(void* store_, const mlob_env_config* cfg, const uint64_t* episodes, uint64_t n_eps,
                        const mlob_policy* t0, int n0, const mlob_policy* t1, int n1, uint64_t seed,
                        mlob_cell_stats* out) { /* evaluate.hpp:104-217 */
  if (cfg->n_specs != 2)
    return fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: exactly two agent types required");
  if (n_eps == 0) return fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: empty episode set");
  for (int i = 0; i < n0 + n1; ++i)
    if ((i < n0 ? t0[i] : t1[i - n0]).kind == MLOB_POLICY_LEARNED && !(i < n0 ? t0[i] : t1[i - n0]).net)
      return fail(MLOB_E_INVALID_ARGUMENT, "evaluate_matrix: learned policy without a network");
  int status = MLOB_OK;
  double* hidden[MLOB_MAX_AGENTS] = {0};
  double* hidden_scratch[MLOB_MAX_AGENTS] = {0};
  double logits[64];
  env* e = orc_env_create(store_, cfg, seed, 0, &status);
  if (!e) return status;
  const int A = e->n_agents;
  double* pv[2] = {malloc(n_eps * sizeof(double)), malloc(n_eps * sizeof(double))};
  double* slip[2] = {malloc(n_eps * sizeof(double)), malloc(n_eps * sizeof(double))};
  mlob_agent_action acts[MLOB_MAX_AGENTS];
  for (int row = 0; row < n0 && status == MLOB_OK; ++row)
    for (int col = 0; col < n1 && status == MLOB_OK; ++col) {
      const mlob_policy* choice[2] = {&t0[row], &t1[col]};
      const uint64_t cell_id = (uint64_t)row * 1000 + (uint64_t)col;
      double completion_sum[2] = {0.0, 0.0};
      int64_t filled[2] = {0, 0};
      for (uint64_t k = 0; k < n_eps && status == MLOB_OK; ++k) {
        const uint64_t ep = episodes[k];
        if ((status = orc_env_reset(e, ep)) != MLOB_OK) break;
        for (int a = 0; a < A; ++a) { /* evaluate.hpp:151-154: hidden zeroed per episode */
          const mlob_policy* p = choice[e->flat_spec[a]];
          if (p->kind != MLOB_POLICY_LEARNED) continue;
          free(hidden[a]);
          free(hidden_scratch[a]);
          hidden[a] = calloc((size_t)p->net->hidden, 8);
          hidden_scratch[a] = calloc((size_t)p->net->hidden, 8);
        }
        for (int step = 0; !e->terminal && status == MLOB_OK; ++step) {
          for (int a = 0; a < A && status == MLOB_OK; ++a) {
            const mlob_policy* p = choice[e->flat_spec[a]];
            if (p->kind == MLOB_POLICY_LEARNED) { /* evaluate.hpp:80-90 */
              const uint8_t reset = 0;
              double value = 0.0;
              memset(&acts[a], 0, sizeof acts[a]);
              policy_forward(p->net, e->ag[a].obs, hidden[a], &reset, 1, logits, &value, hidden_scratch[a]);
              double* tmp = hidden[a];
              hidden[a] = hidden_scratch[a];
              hidden_scratch[a] = tmp;
              int best = 0; /* argmax_action, ppo.hpp:100-105 */
              for (int i = 1; i < p->net->n_actions; ++i)
                if (logits[i] > logits[best]) best = i;
              acts[a].id = best;
              continue;
            }
            status = choose_action(e, a, p, step, seed, cell_id, ep, &acts[a]);
          }
          if (status == MLOB_OK) status = orc_env_step(e, acts, (uint64_t)A);
        }
        if (status != MLOB_OK) break;
        double ep_pv[2] = {0.0, 0.0}, ep_slip[2] = {0.0, 0.0};
        int type_agents[2] = {0, 0};
        for (int a = 0; a < A; ++a) {
          const int tau = e->flat_spec[a];
          const mlob_agent_info* info = &e->ag[a].info;
          ep_pv[tau] += info->portfolio_value;
          ep_slip[tau] += info->slippage_total;
          ++type_agents[tau];
          filled[tau] += e->ag[a].filled_total;
          const mlob_agent_spec* sp = spec_of(e, a);
          if (sp->type == MLOB_EXECUTOR)
            completion_sum[tau] += 1.0 - (double)info->task_remaining / (double)sp->params.task_size;
          else
            completion_sum[tau] += 0.0;
        }
        for (int tau = 0; tau < 2; ++tau) {
          pv[tau][k] = ep_pv[tau] / type_agents[tau];
          slip[tau][k] = ep_slip[tau] / type_agents[tau];
        }
      }
      if (status != MLOB_OK) break;
      mlob_cell_stats* cs = &out[row * n1 + col];
      memset(cs, 0, sizeof *cs);
      cs->episodes = (int64_t)n_eps;
      for (int tau = 0; tau < 2; ++tau) {
        mlob_type_cell_stats* t = &cs->per_type[tau];
        mean_stderr(pv[tau], n_eps, &t->pv_mean, &t->pv_stderr);
        t->filled_total = filled[tau];
        t->no_fills = filled[tau] == 0;
        if (!t->no_fills) mean_stderr(slip[tau], n_eps, &t->slippage_mean, &t->slippage_stderr);
        t->completion_mean = completion_sum[tau] / ((double)n_eps * (double)cfg->specs[tau].count);
      }
    }
  for (int tau = 0; tau < 2; ++tau) {
    free(pv[tau]);
    free(slip[tau]);
  }
  for (int a = 0; a < MLOB_MAX_AGENTS; ++a) {
    free(hidden[a]);
    free(hidden_scratch[a]);
  }
  orc_env_free(e);
  return status;
}

/* ------------------------------------------------------------------------ */
/* ippo/net.hpp PolicyNet, ppo.hpp sample_categorical, gae.hpp, rollout.hpp   */
/* collect_rollout                                                           */

int orc_make_policy_net(int D, int H, int A, uint64_t seed, double* out) { /* net.hpp:80-104 */
  if (D < 1 || H < 1 || A < 1) return fail(MLOB_E_INVALID_ARGUMENT, "make_policy_net: dimensions must be >= 1");
  if (H > 512) return fail(MLOB_E_INVALID_ARGUMENT, "make_policy_net: hidden size capped at 512");
  const uint64_t w[4] = {5 /* ParamInit */, (uint64_t)D, (uint64_t)H, (uint64_t)A};
  crng r = {make_key(seed, 4, w)};
  double* p = out;
#define INIT(n, fan_in, fan_out)                                        \
  do {                                                                  \
    const double bound = sqrt(6.0 / (double)((fan_in) + (fan_out)));    \
    for (size_t i_ = 0; i_ < (size_t)(n); ++i_)                         \
      p[i_] = -bound + (bound - -bound) * crng_uniform(&r);             \
  } while (0)
  INIT(3 * H * D, D, H); /* w_ih */
  p += 3 * H * D;
  INIT(3 * H * H, H, H); /* w_hh */
  p += 3 * H * H;
  for (int i = 0; i < 6 * H; ++i) *p++ = 0.0; /* b_ih, b_hh */
  INIT(A * H, H, A); /* w_actor, then scaled (net.hpp:97-98) */
  for (int i = 0; i < A * H; ++i) p[i] *= 0.01;
  p += A * H;
  for (int i = 0; i < A; ++i) *p++ = 0.0; /* b_actor */
  INIT(H, H, 1); /* w_critic */
  p += H;
  *p = 0.0; /* b_critic */
#undef INIT
  return MLOB_OK;
}

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); } /* net.hpp:107 */

/* policy_forward (net.hpp:120-188) without the backward cache */
static void policy_forward(const mlob_policy_net* net, const double* obs, const double* hidden,
                           const uint8_t* reset_mask, uint64_t batch, double* logits, double* values,
                           double* hidden_out) {
  const uint64_t H = (uint64_t)net->hidden, D = (uint64_t)net->obs_dim, A = (uint64_t)net->n_actions;
  for (uint64_t b = 0; b < batch; ++b) {
    const double* x = obs + b * D;
    const double* h_prev = hidden + b * H;
    const int reset = reset_mask[b] != 0;
    for (uint64_t i = 0; i < H; ++i) {
      double acc_r = net->b_ih[i] + net->b_hh[i];
      double acc_z = net->b_ih[H + i] + net->b_hh[H + i];
      double acc_n = net->b_ih[2 * H + i];
      double acc_hn = net->b_hh[2 * H + i];
      for (uint64_t d = 0; d < D; ++d) {
        acc_r += net->w_ih[i * D + d] * x[d];
        acc_z += net->w_ih[(H + i) * D + d] * x[d];
        acc_n += net->w_ih[(2 * H + i) * D + d] * x[d];
      }
      if (!reset) {
        for (uint64_t j = 0; j < H; ++j) {
          const double hj = h_prev[j];
          acc_r += net->w_hh[i * H + j] * hj;
          acc_z += net->w_hh[(H + i) * H + j] * hj;
          acc_hn += net->w_hh[(2 * H + i) * H + j] * hj;
        }
      }
      const double r = sigmoid(acc_r);
      const double z = sigmoid(acc_z);
      const double n = tanh(acc_n + r * acc_hn);
      const double h_old = reset ? 0.0 : h_prev[i];
      hidden_out[b * H + i] = (1.0 - z) * n + z * h_old;
    }
    const double* h = hidden_out + b * H;
    for (uint64_t a = 0; a < A; ++a) {
      double acc = net->b_actor[a];
      for (uint64_t j = 0; j < H; ++j) acc += net->w_actor[a * H + j] * h[j];
      logits[b * A + a] = acc;
    }
    double v = net->b_critic;
    for (uint64_t j = 0; j < H; ++j) v += net->w_critic[j] * h[j];
    values[b] = v;
  }
}

static int sample_categorical(const double* logits, int n, double u, double* logp) { /* ppo.hpp:80-98 */
  double max_l = logits[0];
  for (int a = 0; a < n; ++a) max_l = max_l < logits[a] ? logits[a] : max_l;
  double z = 0.0;
  for (int a = 0; a < n; ++a) z += exp(logits[a] - max_l);
  const double target = u * z;
  double cum = 0.0;
  int action = n - 1;
  for (int a = 0; a < n; ++a) {
    cum += exp(logits[a] - max_l);
    if (cum > target) {
      action = a;
      break;
    }
  }
  *logp = logits[action] - max_l - log(z);
  return action;
}

static void compute_gae(const double* rewards, const double* values, const uint8_t* dones, uint64_t T,
                        uint64_t B, double discount, double gae_lambda, double* adv, double* ret) { /* gae.hpp:14-32 */
  for (uint64_t b = 0; b < B; ++b) {
    double carry = 0.0;
    for (uint64_t t = T; t-- > 0;) {
      const double not_done = dones[t * B + b] ? 0.0 : 1.0;
      const double delta = rewards[t * B + b] + discount * values[(t + 1) * B + b] * not_done - values[t * B + b];
      carry = delta + discount * gae_lambda * not_done * carry;
      adv[t * B + b] = carry;
      ret[t * B + b] = carry + values[t * B + b];
    }
  }
}

typedef struct rbatch { /* RolloutBatch, ppo.hpp:33-66 */
  uint64_t T, B, D, H;
  double *obs, *log_probs, *values, *rewards, *h0, *adv, *ret;
  int32_t* actions;
  uint8_t *dones, *resets;
} rbatch;

struct rollout_state {
  int n_types;
  double* hidden[MLOB_MAX_SPECS];
  rbatch b[MLOB_MAX_SPECS];
};

static void rbatch_free(rbatch* b) {
  free(b->obs); free(b->log_probs); free(b->values); free(b->rewards); free(b->h0);
  free(b->adv); free(b->ret); free(b->actions); free(b->dones); free(b->resets);
  memset(b, 0, sizeof *b);
}

static void rollout_free(struct rollout_state* r) {
  if (!r) return;
  for (int t = 0; t < r->n_types; ++t) {
    free(r->hidden[t]);
    rbatch_free(&r->b[t]);
  }
  free(r);
}

static void rbatch_resize(rbatch* b, uint64_t T, uint64_t B, uint64_t D, uint64_t H) { /* ppo.hpp:50-63 */
  rbatch_free(b);
  b->T = T; b->B = B; b->D = D; b->H = H;
  b->obs = calloc(T * B * D + 1, 8);
  b->actions = calloc(T * B + 1, 4);
  b->log_probs = calloc(T * B + 1, 8);
  b->values = calloc((T + 1) * B + 1, 8);
  b->rewards = calloc(T * B + 1, 8);
  b->dones = calloc(T * B + 1, 1);
  b->resets = calloc(T * B + 1, 1);
  b->h0 = calloc(B * H + 1, 8);
  b->adv = calloc(T * B + 1, 8);
  b->ret = calloc(T * B + 1, 8);
}

int orc_venv_collect_rollout(void* v_, const mlob_policy_net* nets, const mlob_rollout_config* cfg,
                             uint64_t update_index) { /* rollout.hpp:41-124 */
  venv* v = v_;
  const int NT = v->cfg.n_specs;
  if (!v->roll) { /* train_loop: zero hidden per type (rollout.hpp:132-135) */
    v->roll = calloc(1, sizeof(struct rollout_state));
    v->roll->n_types = NT;
    for (int t = 0; t < NT; ++t)
      v->roll->hidden[t] = calloc((uint64_t)v->n_envs * v->cfg.specs[t].count * nets[t].hidden + 1, 8);
  }
  struct rollout_state* rs = v->roll;
  const uint64_t T = (uint64_t)cfg->rollout_len;
  double* logits[MLOB_MAX_SPECS];
  double* hidden_next[MLOB_MAX_SPECS];
  for (int t = 0; t < NT; ++t) {
    const uint64_t B = (uint64_t)v->n_envs * v->cfg.specs[t].count, H = (uint64_t)nets[t].hidden;
    rbatch* b = &rs->b[t];
    if (b->T != T || b->B != B)
      rbatch_resize(b, T, B, observation_size(v->cfg.specs[t].obs_space, v->cfg.obs_depth), H);
    logits[t] = calloc(B * nets[t].n_actions + 1, 8);
    hidden_next[t] = calloc(B * H + 1, 8);
    memcpy(b->h0, rs->hidden[t], B * H * 8);
  }
  int status = MLOB_OK;
  for (uint64_t step = 0; step < T && status == MLOB_OK; ++step) {
    for (int t = 0; t < NT; ++t) {
      rbatch* b = &rs->b[t];
      const uint64_t B = b->B, D = b->D, A = (uint64_t)nets[t].n_actions;
      orc_venv_gather(v, t, b->obs + step * B * D, b->resets + step * B);
      policy_forward(&nets[t], b->obs + step * B * D, rs->hidden[t], b->resets + step * B, B, logits[t],
                     b->values + step * B, hidden_next[t]);
      double* tmp = rs->hidden[t];
      rs->hidden[t] = hidden_next[t];
      hidden_next[t] = tmp;
      for (uint64_t s = 0; s < B; ++s) {
        const uint64_t w[5] = {3 /* ActionSample */, (uint64_t)t, update_index, step, s};
        crng r = {make_key(cfg->seed, 5, w)};
        double logp = 0.0;
        const int action = sample_categorical(logits[t] + s * A, (int)A, crng_uniform(&r), &logp);
        b->actions[step * B + s] = action;
        b->log_probs[step * B + s] = logp;
        orc_venv_set_action(v, t, s, action);
      }
    }
    status = orc_venv_step_all(v);
    for (int t = 0; t < NT && status == MLOB_OK; ++t) {
      rbatch* b = &rs->b[t];
      for (uint64_t s = 0; s < b->B; ++s) {
        b->rewards[step * b->B + s] = orc_venv_reward(v, t, s);
        b->dones[step * b->B + s] = orc_venv_done(v, t, s) ? 1 : 0;
      }
    }
  }
  for (int t = 0; t < NT && status == MLOB_OK; ++t) { /* bootstrap + GAE (rollout.hpp:105-123) */
    rbatch* b = &rs->b[t];
    double* boot_obs = calloc(b->B * b->D + 1, 8);
    uint8_t* boot_reset = calloc(b->B + 1, 1);
    double* scratch = calloc(b->B * b->H + 1, 8);
    orc_venv_gather(v, t, boot_obs, boot_reset);
    policy_forward(&nets[t], boot_obs, rs->hidden[t], boot_reset, b->B, logits[t], b->values + T * b->B, scratch);
    compute_gae(b->rewards, b->values, b->dones, T, b->B, cfg->discount, cfg->gae_lambda, b->adv, b->ret);
    free(boot_obs);
    free(boot_reset);
    free(scratch);
  }
  for (int t = 0; t < NT; ++t) {
    free(logits[t]);
    free(hidden_next[t]);
  }
  return status;
}

uint64_t orc_venv_rollout_field(void* v_, int type, int field, void* out, uint64_t cap) {
  venv* v = v_;
  if (!v->roll) return 0;
  const rbatch* b = &v->roll->b[type];
  const uint64_t TB = b->T * b->B;
  const void* src = NULL;
  uint64_t bytes = 0;
  switch (field) {
    case MLOB_RB_OBS: src = b->obs; bytes = TB * b->D * 8; break;
    case MLOB_RB_ACTIONS: src = b->actions; bytes = TB * 4; break;
    case MLOB_RB_LOG_PROBS: src = b->log_probs; bytes = TB * 8; break;
    case MLOB_RB_VALUES: src = b->values; bytes = (TB + b->B) * 8; break;
    case MLOB_RB_REWARDS: src = b->rewards; bytes = TB * 8; break;
    case MLOB_RB_DONES: src = b->dones; bytes = TB; break;
    case MLOB_RB_RESETS: src = b->resets; bytes = TB; break;
    case MLOB_RB_H0: src = b->h0; bytes = b->B * b->H * 8; break;
    case MLOB_RB_ADVANTAGES: src = b->adv; bytes = TB * 8; break;
    case MLOB_RB_RETURNS: src = b->ret; bytes = TB * 8; break;
    case MLOB_RB_HIDDEN: src = v->roll->hidden[type]; bytes = b->B * b->H * 8; break;
  }
  if (src && bytes <= cap) memcpy(out, src, bytes);
  return bytes;
}

/* ------------------------------------------------------------------------ */
/* data/lobster.hpp load_lobster                                              */

typedef struct linebuf { /* std::getline over a whole file */
  char* data;
  size_t size, pos;
} linebuf;

static int lb_open(linebuf* b, const char* path) {
  FILE* f = fopen(path, "rb");
  if (!f) return 0;
  fseek(f, 0, SEEK_END);
  const long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  b->size = n > 0 ? (size_t)n : 0;
  b->data = malloc(b->size + 1);
  b->pos = 0;
  if (b->size && fread(b->data, 1, b->size, f) != b->size) {
    fclose(f);
    free(b->data);
    return 0;
  }
  fclose(f);
  return 1;
}

/* next line [*s, *s + *n) without '\n'; 0 at EOF (getline semantics) */
static int lb_next(linebuf* b, const char** s, size_t* n) {
  if (b->pos >= b->size) return 0;
  const char* p = b->data + b->pos;
  const char* nl = memchr(p, '\n', b->size - b->pos);
  const size_t len = nl ? (size_t)(nl - p) : b->size - b->pos;
  b->pos += len + (nl ? 1 : 0);
  *s = p;
  *n = len;
  return 1;
}

static void strip_cr(const char* s, size_t* n) { /* lobster.hpp:72-75 */
  if (*n > 0 && s[*n - 1] == '\r') --*n;
}

/* lobster.hpp:26-37: std::from_chars after leading blanks, whole field */
static int lob_parse_int(const char* s, size_t n, int64_t* out) {
  size_t i = 0;
  while (i < n && (s[i] == ' ' || s[i] == '\t')) ++i;
  int neg = 0;
  if (i < n && s[i] == '-') {
    neg = 1;
    ++i;
  }
  if (i >= n) return 0;
  uint64_t mag = 0;
  const uint64_t lim = neg ? (1ull << 63) : (1ull << 63) - 1;
  for (; i < n; ++i) {
    if (s[i] < '0' || s[i] > '9') return 0;
    const uint64_t d = (uint64_t)(s[i] - '0');
    if (mag > (lim - d) / 10) return 0;
    mag = mag * 10 + d;
  }
  *out = neg ? (int64_t)(0 - mag) : (int64_t)mag;
  return 1;
}

#define LOB_FIELD(buf, s, n) snprintf(buf, sizeof buf, "%.*s", (int)(n), s)

static int lob_int(const char* s, size_t n, const char* what, uint64_t row, int64_t* out) {
  if (lob_parse_int(s, n, out)) return MLOB_OK;
  char f[512];
  LOB_FIELD(f, s, n);
  return fail(MLOB_E_RUNTIME, "lobster: row %llu: malformed %s field '%s'", (unsigned long long)(row + 1), what, f);
}

static int lob_time(const char* s, size_t n, uint64_t row, int64_t* t) { /* lobster.hpp:41-57 */
  const char* dot = memchr(s, '.', n);
  const size_t sec_n = dot ? (size_t)(dot - s) : n;
  int64_t sec = 0, frac = 0;
  int rc = lob_int(s, sec_n, "time", row, &sec);
  if (rc != MLOB_OK) return rc;
  if (dot) {
    size_t digits = n - sec_n - 1;
    if (digits > 9) digits = 9;
    if (digits == 0)
      return fail(MLOB_E_RUNTIME, "lobster: row %llu: malformed time field", (unsigned long long)(row + 1));
    rc = lob_int(dot + 1, digits, "time fraction", row, &frac);
    if (rc != MLOB_OK) return rc;
    for (size_t i = digits; i < 9; ++i) frac *= 10;
  }
  *t = (int64_t)((uint64_t)sec * 1000000000ull + (uint64_t)frac);
  return MLOB_OK;
}

static int lob_ticks(int64_t units, int64_t upt, uint64_t row, int64_t* out) { /* lobster.hpp:77-84 */
  if (units % upt != 0)
    return fail(MLOB_E_RUNTIME, "lobster: row %llu: price %lld not divisible by tick size %lld",
                (unsigned long long)(row + 1), (long long)units, (long long)upt);
  *out = units / upt;
  return MLOB_OK;
}

/* split on ',' (lobster.hpp:59-70): up to cap fields, returns the count */
static size_t lob_split(const char* s, size_t n, const char** fs, size_t* fn, size_t cap) {
  size_t k = 0, b = 0;
  for (size_t i = 0; i <= n; ++i)
    if (i == n || s[i] == ',') {
      if (k < cap) {
        fs[k] = s + b;
        fn[k] = i - b;
      }
      ++k;
      b = i + 1;
    }
  return k;
}

static int lob_book_row(const char* s, size_t n, int64_t upt, uint64_t row, mlob_level** bids, uint32_t* nb,
                        mlob_level** asks, uint32_t* na) { /* lobster.hpp:86-103 */
  const size_t nf = lob_split(s, n, NULL, NULL, 0);
  if (nf % 4 != 0)
    return fail(MLOB_E_RUNTIME, "lobster: orderbook row %llu: column count %zu is not a multiple of 4",
                (unsigned long long)(row + 1), nf);
  const char** fs = malloc(nf * sizeof(char*));
  size_t* fn = malloc(nf * sizeof(size_t));
  lob_split(s, n, fs, fn, nf);
  *bids = malloc((nf / 4 + 1) * sizeof(mlob_level));
  *asks = malloc((nf / 4 + 1) * sizeof(mlob_level));
  *nb = *na = 0;
  static const char* names[4] = {"ask price", "ask size", "bid price", "bid size"};
  int rc = MLOB_OK;
  for (size_t level = 0; level * 4 < nf && rc == MLOB_OK; ++level) {
    int64_t v[4];
    for (int c = 0; c < 4 && rc == MLOB_OK; ++c) rc = lob_int(fs[level * 4 + c], fn[level * 4 + c], names[c], row, &v[c]);
    if (rc != MLOB_OK) break;
    if (v[1] > 0 && v[0] > 0 && v[0] < 9999999999ll) {
      int64_t p = 0;
      if ((rc = lob_ticks(v[0], upt, row, &p)) != MLOB_OK) break;
      (*asks)[(*na)++] = (mlob_level){p, v[1]};
    }
    if (v[3] > 0 && v[2] > 0) {
      int64_t p = 0;
      if ((rc = lob_ticks(v[2], upt, row, &p)) != MLOB_OK) break;
      (*bids)[(*nb)++] = (mlob_level){p, v[3]};
    }
  }
  free(fs);
  free(fn);
  return rc;
}

void* orc_load_lobster(const char* msg_path, const char* book_path, int64_t upt, uint64_t sample_every,
                       int* status) { /* lobster.hpp:119-193 */
  if (upt < 1) {
    *status = fail(MLOB_E_INVALID_ARGUMENT, "load_lobster: units_per_tick >= 1");
    return NULL;
  }
  if (sample_every == 0) {
    *status = fail(MLOB_E_INVALID_ARGUMENT, "load_lobster: sample_every >= 1");
    return NULL;
  }
  linebuf mf, bf;
  if (!lb_open(&mf, msg_path)) {
    *status = fail(MLOB_E_RUNTIME, "load_lobster: cannot open %s", msg_path);
    return NULL;
  }
  if (!lb_open(&bf, book_path)) {
    free(mf.data);
    *status = fail(MLOB_E_RUNTIME, "load_lobster: cannot open %s", book_path);
    return NULL;
  }
  store* st = calloc(1, sizeof(store));
  push_state(st, 0, NULL, 0, NULL, 0);
  int rc = MLOB_OK;
  uint64_t row = 0;
  int64_t prev_time = -1;
  const char *ml, *bl;
  size_t mn, bn;
  static const int kinds[7] = {MLOB_NEW_LIMIT, MLOB_CANCEL_PARTIAL, MLOB_DELETE, MLOB_EXECUTE_VISIBLE,
                               MLOB_EXECUTE_HIDDEN, MLOB_CROSS, MLOB_HALT};
  while (rc == MLOB_OK && lb_next(&mf, &ml, &mn)) {
    strip_cr(ml, &mn);
    if (mn == 0) continue;
    if (!lb_next(&bf, &bl, &bn)) {
      rc = fail(MLOB_E_RUNTIME, "load_lobster: orderbook file has fewer rows than %s", msg_path);
      break;
    }
    const char* fs[6];
    size_t fn[6];
    const size_t nf = lob_split(ml, mn, fs, fn, 6);
    if (nf != 6) {
      rc = fail(MLOB_E_RUNTIME, "lobster: row %llu: expected 6 fields, got %zu", (unsigned long long)(row + 1), nf);
      break;
    }
    mlob_message m;
    memset(&m, 0, sizeof m);
    if ((rc = lob_time(fs[0], fn[0], row, &m.time)) != MLOB_OK) break;
    if (m.time < prev_time) {
      rc = fail(MLOB_E_RUNTIME, "lobster: row %llu: non-monotone time", (unsigned long long)(row + 1));
      break;
    }
    prev_time = m.time;
    int64_t type, id, dir, pu;
    if ((rc = lob_int(fs[1], fn[1], "type", row, &type)) != MLOB_OK) break;
    if (type < 1 || type > 7) {
      rc = fail(MLOB_E_RUNTIME, "lobster: row %llu: unknown event type %lld", (unsigned long long)(row + 1),
                (long long)type);
      break;
    }
    m.kind = (uint8_t)kinds[type - 1];
    if ((rc = lob_int(fs[2], fn[2], "order id", row, &id)) != MLOB_OK) break;
    m.order_id = (uint64_t)id;
    if ((rc = lob_int(fs[3], fn[3], "size", row, &m.quantity)) != MLOB_OK) break;
    if (m.quantity < 0) {
      rc = fail(MLOB_E_RUNTIME, "lobster: row %llu: negative size", (unsigned long long)(row + 1));
      break;
    }
    if ((rc = lob_int(fs[4], fn[4], "price", row, &pu)) != MLOB_OK) break;
    if ((rc = lob_ticks(pu, upt, row, &m.price)) != MLOB_OK) break;
    if ((rc = lob_int(fs[5], fn[5], "direction", row, &dir)) != MLOB_OK) break;
    if (dir != 1 && dir != -1) {
      rc = fail(MLOB_E_RUNTIME, "lobster: row %llu: direction must be +1 or -1", (unsigned long long)(row + 1));
      break;
    }
    m.side = dir == 1 ? MLOB_BID : MLOB_ASK;
    m.trader_id = 0;
    VEC_PUSH(st->msgs, m);
    if ((row + 1) % sample_every == 0) {
      strip_cr(bl, &bn);
      mlob_level *b = NULL, *a = NULL;
      uint32_t nb = 0, na = 0;
      rc = lob_book_row(bl, bn, upt, row, &b, &nb, &a, &na);
      if (rc == MLOB_OK) push_state(st, row + 1, b, nb, a, na);
      free(b);
      free(a);
      if (rc != MLOB_OK) break;
    }
    ++row;
  }
  while (rc == MLOB_OK && lb_next(&bf, &bl, &bn)) {
    strip_cr(bl, &bn);
    if (bn != 0) rc = fail(MLOB_E_RUNTIME, "load_lobster: message file has fewer rows than %s", book_path);
  }
  free(mf.data);
  free(bf.data);
  if (rc != MLOB_OK) {
    orc_store_free(st);
    *status = rc;
    return NULL;
  }
  if (st->states.n > 1 && st->states.v[st->states.n - 1].message_index == st->msgs.n) {
    free(st->states.v[st->states.n - 1].levels);
    --st->states.n;
  }
  *status = MLOB_OK;
  return st;
}
