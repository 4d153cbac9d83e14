// mlob_lobster.cuh — LOBSTER row parsing shared by the device loader (every
// row, one thread each) and the host (the first failing row only, to format
// the reference's error text).  Restates data/lobster.hpp:24-117 and the
// per-row checks of load_lobster (lobster.hpp:125-190) as error codes.
#pragma once

#include <cstdint>

namespace mlob {
namespace lobster {

// First failing check of a message row, in the reference's order.
enum Err : int32_t {
  kOk = 0,
  kBookMissing = 1,  // orderbook file has fewer rows (lobster.hpp:145-147)
  kFields = 2,       // expected 6 fields, aux = count
  kTimeSec = 3,      // malformed time field (integer part)
  kTimeEmptyFrac = 4,
  kTimeFrac = 5,     // malformed time fraction field
  kMonotone = 6,     // non-monotone time (checked across rows)
  kTypeParse = 7,
  kTypeRange = 8,    // aux = type
  kIdParse = 9,
  kSizeParse = 10,
  kSizeNeg = 11,
  kPriceParse = 12,
  kPriceTick = 13,   // aux = price units
  kDirParse = 14,
  kDirRange = 15,
  kBookCols = 16,    // sampled orderbook row: column count, aux = count
  kBookField = 17,   // aux = level * 4 + column
  kBookTick = 18,    // aux = price units
};

// std::from_chars<int64_t> over [p, p+n) after skipping leading spaces/tabs,
// and requiring the whole rest to be consumed (lobster.hpp:26-37).
__host__ __device__ inline bool parse_int(const char* p, int n, int64_t& out) {
  int i = 0;
  while (i < n && (p[i] == ' ' || p[i] == '\t')) ++i;
  bool neg = false;
  if (i < n && p[i] == '-') {
    neg = true;
    ++i;
  }
  if (i >= n) return false;
  uint64_t mag = 0;
  const uint64_t lim = neg ? (1ull << 63) : (1ull << 63) - 1;
  for (; i < n; ++i) {
    const char c = p[i];
    if (c < '0' || c > '9') return false;
    const uint64_t d = static_cast<uint64_t>(c - '0');
    if (mag > (lim - d) / 10) return false;  // result_out_of_range
    mag = mag * 10 + d;
  }
  out = neg ? static_cast<int64_t>(0 - mag) : static_cast<int64_t>(mag);
  return true;
}

struct Field {
  int begin, len;
};

// Splits on ',' into at most `cap` fields; returns the total field count.
__host__ __device__ inline int split(const char* line, int len, Field* f, int cap) {
  int n = 0, b = 0;
  for (int i = 0; i <= len; ++i) {
    if (i == len || line[i] == ',') {
      if (n < cap) f[n] = Field{b, i - b};
      ++n;
      b = i + 1;
    }
  }
  return n;
}

struct MsgRow {
  int64_t time, order_id, qty, price;
  int32_t kind, side;
};

// parse_time_ns (lobster.hpp:41-57)
__host__ __device__ inline int32_t parse_time(const char* p, int n, int64_t& t) {
  int dot = -1;
  for (int i = 0; i < n; ++i)
    if (p[i] == '.') {
      dot = i;
      break;
    }
  int64_t sec = 0;
  if (!parse_int(p, dot < 0 ? n : dot, sec)) return kTimeSec;
  int64_t frac = 0;
  if (dot >= 0) {
    int digits = n - dot - 1;
    if (digits > 9) digits = 9;
    if (digits == 0) return kTimeEmptyFrac;
    if (!parse_int(p + dot + 1, digits, frac)) return kTimeFrac;
    for (int i = digits; i < 9; ++i) frac *= 10;
  }
  t = static_cast<int64_t>(static_cast<uint64_t>(sec) * 1000000000ull + static_cast<uint64_t>(frac));
  return kOk;
}

// One message row (lobster.hpp:148-179) minus the cross-row checks.
// `bad` receives the failing field index (for the error text).
__host__ __device__ inline int32_t parse_msg(const char* line, int len, int64_t upt, MsgRow& m, int64_t& aux,
                                             int& bad) {
  Field f[6];
  const int nf = split(line, len, f, 6);
  if (nf != 6) {
    aux = nf;
    return kFields;
  }
  bad = 0;
  int32_t e = parse_time(line + f[0].begin, f[0].len, m.time);
  if (e != kOk) return e;
  int64_t type = 0;
  bad = 1;
  if (!parse_int(line + f[1].begin, f[1].len, type)) return kTypeParse;
  if (type < 1 || type > 7) {
    aux = type;
    return kTypeRange;
  }
  m.kind = static_cast<int32_t>(type - 1);  // kKinds: NewLimit .. Halt in order
  bad = 2;
  if (!parse_int(line + f[2].begin, f[2].len, m.order_id)) return kIdParse;
  bad = 3;
  if (!parse_int(line + f[3].begin, f[3].len, m.qty)) return kSizeParse;
  if (m.qty < 0) return kSizeNeg;
  bad = 4;
  int64_t pu = 0;
  if (!parse_int(line + f[4].begin, f[4].len, pu)) return kPriceParse;
  if (pu % upt != 0) {
    aux = pu;
    return kPriceTick;
  }
  m.price = pu / upt;
  bad = 5;
  int64_t dir = 0;
  if (!parse_int(line + f[5].begin, f[5].len, dir)) return kDirParse;
  if (dir != 1 && dir != -1) return kDirRange;
  m.side = dir == 1 ? 0 : 1;
  return kOk;
}

// parse_book_row (lobster.hpp:81-103): validates and counts (levels == nullptr)
// or writes the kept levels, bids then asks, best-first.  Columns of one level
// are parsed ask price, ask size, bid price, bid size, then the ticks checked.
template <class LevelT>
__host__ __device__ inline int32_t parse_book(const char* line, int len, int64_t upt, int& nb, int& na,
                                              LevelT* bids, LevelT* asks, int64_t& aux) {
  nb = na = 0;
  int ncol = 0;
  for (int i = 0; i <= len; ++i)
    if (i == len || line[i] == ',') ++ncol;
  if (ncol % 4 != 0) {
    aux = ncol;
    return kBookCols;
  }
  int b = 0, col = 0;
  int64_t v[4];
  for (int i = 0; i <= len; ++i) {
    if (i == len || line[i] == ',') {
      if (!parse_int(line + b, i - b, v[col % 4])) {
        aux = col;
        return kBookField;
      }
      b = i + 1;
      if (col % 4 == 3) {  // ask price, ask size, bid price, bid size
        if (v[1] > 0 && v[0] > 0 && v[0] < 9999999999ll) {
          if (v[0] % upt != 0) {
            aux = v[0];
            return kBookTick;
          }
          if (asks) asks[na] = LevelT{v[0] / upt, v[1]};
          ++na;
        }
        if (v[3] > 0 && v[2] > 0) {
          if (v[2] % upt != 0) {
            aux = v[2];
            return kBookTick;
          }
          if (bids) bids[nb] = LevelT{v[2] / upt, v[3]};
          ++nb;
        }
      }
      ++col;
    }
  }
  return kOk;
}

}  // namespace lobster
}  // namespace mlob
