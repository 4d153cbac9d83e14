// mlob_lobster.cu — LOBSTER message/orderbook CSV pair → device message store
// (data/lobster.hpp:119-193 load_lobster, then the 40 B →
// 32 B DevMsg repack of mlob_store_upload).  The files are read once, their
// bytes copied to HBM, and parsed there: line ends by a device select, one
// thread per message row writing its DevMsg directly, sampled orderbook rows
// parsed by a count pass and a write pass.  The first failing row (the
// reference's sequential order) is found by a min-reduction; the host then
// re-parses that one row with the same code (mlob_lobster.cuh) to format the
// reference's error text.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>
#include <chrono>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "mlob_dev.h"
#include "mlob_lobster.cuh"
#include "mlob_lobster.h"

namespace mlob {
namespace lobster {
namespace {

// line j = [start, end): starts after the previous '\n'; a final line without
// '\n' exists when non-empty (std::getline)
__device__ __forceinline__ void line_of(const uint64_t* nl, uint64_t n_nl, uint64_t size, uint64_t j,
                                        uint64_t& b, uint64_t& e) {
  b = j == 0 ? 0 : nl[j - 1] + 1;
  e = j < n_nl ? nl[j] : size;
}
__device__ __forceinline__ int strip_len(const char* p, uint64_t b, uint64_t e) {  // strip_cr
  int n = static_cast<int>(e - b);
  if (n > 0 && p[b + n - 1] == '\r') --n;
  return n;
}

struct NonEmptyLine {
  const char* b;
  const uint64_t* nl;
  uint64_t n_nl, size;
  __device__ bool operator()(uint64_t j) const {
    uint64_t s, e;
    line_of(nl, n_nl, size, j, s, e);
    return strip_len(b, s, e) > 0;
  }
};

struct L64 {
  int64_t p, q;
};

struct RowArgs {
  const char* msg;
  const uint64_t* msg_nl;
  uint64_t msg_nl_n, msg_size;
  const uint64_t* rows;  // message line index of row k
  uint64_t n_rows;
  const char* book;
  const uint64_t* book_nl;
  uint64_t book_nl_n, book_size, book_lines;
  int64_t upt;
  uint64_t sample_every;
  DevMsg* out;
  int64_t* time;
  int32_t* err;           // per row: first failing check
  uint32_t* n_bid;        // per sampled state (row k with (k+1) % sample_every == 0)
  uint32_t* n_ask;
  unsigned long long* first_bad;  // min row index with an error
  unsigned long long* first_range;  // min row index whose message exceeds the device int32 layout
};

__global__ void parse_rows_kernel(RowArgs a) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < a.n_rows;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    int32_t e = kOk;
    if (k >= a.book_lines) e = kBookMissing;
    MsgRow m{};
    int64_t aux = 0;
    int bad = 0;
    if (e == kOk) {
      uint64_t s, t;
      line_of(a.msg_nl, a.msg_nl_n, a.msg_size, a.rows[k], s, t);
      e = parse_msg(a.msg + s, strip_len(a.msg, s, t), a.upt, m, aux, bad);
    }
    a.time[k] = m.time;
    const bool sampled = (k + 1) % a.sample_every == 0;
    if (e == kOk && sampled) {
      uint64_t s, t;
      line_of(a.book_nl, a.book_nl_n, a.book_size, k, s, t);
      int nb = 0, na = 0;
      e = parse_book<L64>(a.book + s, strip_len(a.book, s, t), a.upt, nb, na, nullptr, nullptr, aux);
      const uint64_t st = (k + 1) / a.sample_every - 1;
      a.n_bid[st] = static_cast<uint32_t>(nb);
      a.n_ask[st] = static_cast<uint32_t>(na);
    }
    a.err[k] = e;
    // DevMsg (mlob_store_upload's repack): NewLimit keeps price / qty when
    // qty > 0, Cancel / ExecuteVisible keep min(qty, INT32_MAX), others zero
    DevMsg d{};
    d.time = m.time;
    d.order_id = static_cast<uint64_t>(m.order_id);
    d.kind = static_cast<uint8_t>(m.kind);
    d.side = static_cast<uint8_t>(m.side);
    d.trader = 0;
    bool range_bad = false;
    if (m.kind == MLOB_NEW_LIMIT && m.qty > 0) {
      range_bad = m.price <= INT32_MIN || m.price >= INT32_MAX || m.qty >= INT32_MAX;
      d.price = static_cast<int32_t>(m.price);
      d.qty = static_cast<int32_t>(m.qty);
    } else if (m.kind == MLOB_CANCEL_PARTIAL || m.kind == MLOB_EXECUTE_VISIBLE) {
      d.qty = static_cast<int32_t>(m.qty < INT32_MAX ? m.qty : INT32_MAX);
    }
    a.out[k] = d;
    if (e != kOk) atomicMin(a.first_bad, static_cast<unsigned long long>(k));
    if (e == kOk && range_bad) atomicMin(a.first_range, static_cast<unsigned long long>(k));
  }
}

// non-monotone time (lobster.hpp:152-155): a row whose own checks pass up to
// the time field fails here when its time is below the previous row's
__global__ void monotone_kernel(const int64_t* time, int32_t* err, uint64_t n, unsigned long long* first_bad) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int32_t e = err[k];
    const int64_t prev = k == 0 ? -1 : time[k - 1];  // prev_time starts at -1 (lobster.hpp:135)
    if ((e == kOk || e > kMonotone) && time[k] < prev) {
      err[k] = kMonotone;
      atomicMin(first_bad, static_cast<unsigned long long>(k));
    }
  }
}

// trailing orderbook lines past the last message row must be empty
__global__ void extra_book_kernel(const char* book, const uint64_t* nl, uint64_t n_nl, uint64_t size,
                                  uint64_t first, uint64_t lines, unsigned int* flag) {
  for (uint64_t j = first + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < lines;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t s, e;
    line_of(nl, n_nl, size, j, s, e);
    if (strip_len(book, s, e) > 0) atomicOr(flag, 1u);
  }
}

// write pass of the sampled orderbook rows: kept levels, bids then asks
__global__ void write_levels_kernel(RowArgs a, const uint64_t* lv_off, uint64_t n_states, DevLevel* levels,
                                    unsigned int* level_bad) {
  for (uint64_t st = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; st < n_states;
       st += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t k = (st + 1) * a.sample_every - 1;
    uint64_t s, t;
    line_of(a.book_nl, a.book_nl_n, a.book_size, k, s, t);
    const int len = strip_len(a.book, s, t);
    const uint32_t nb = a.n_bid[st], na = a.n_ask[st];
    DevLevel* out = levels + lv_off[st];
    // re-walk the row: levels arrive interleaved per LOBSTER level (ask, bid)
    int bi = 0, ai = 0, b = 0, col = 0;
    int64_t v[4];
    for (int i = 0; i <= len; ++i) {
      if (i == len || a.book[s + i] == ',') {
        parse_int(a.book + s + b, i - b, v[col % 4]);
        b = i + 1;
        if (col % 4 == 3) {
          if (v[1] > 0 && v[0] > 0 && v[0] < 9999999999ll) {
            const int64_t p = v[0] / a.upt;
            if (p <= INT32_MIN || p >= INT32_MAX || v[1] >= INT32_MAX) atomicOr(level_bad, 1u);
            out[nb + ai++] = DevLevel{static_cast<int32_t>(p), static_cast<int32_t>(v[1])};
          }
          if (v[3] > 0 && v[2] > 0) {
            const int64_t p = v[2] / a.upt;
            if (p <= INT32_MIN || p >= INT32_MAX || v[3] >= INT32_MAX) atomicOr(level_bad, 1u);
            out[bi++] = DevLevel{static_cast<int32_t>(p), static_cast<int32_t>(v[3])};
          }
        }
        ++col;
      }
    }
    (void)na;
  }
}

unsigned grid_of(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 8192) b = 8192;
  return static_cast<unsigned>(b);
}

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw LobsterError(std::string("CUDA ") + what + ": " + cudaGetErrorString(e), 5);
}

// newline positions of a device buffer, in order: pass 1 counts '\n' per
// block segment (16-byte loads, SWAR byte compare), an exclusive scan gives
// each segment's output offset, pass 2 re-reads the segment tile by tile and
// writes positions with a block scan.  Two streaming reads of the buffer.
constexpr int kNlThreads = 256;
constexpr int kNlBlocks = 2048;
__device__ __forceinline__ uint32_t nl_mask(uint32_t w) {  // high bit of each '\n' byte
  const uint32_t x = w ^ 0x0A0A0A0Au;
  return (x - 0x01010101u) & ~x & 0x80808080u;
}
__device__ __forceinline__ int nl_count16(const uint4& v) {
  return __popc(nl_mask(v.x)) + __popc(nl_mask(v.y)) + __popc(nl_mask(v.z)) + __popc(nl_mask(v.w));
}
__device__ __forceinline__ uint4 load16(const char* b, uint64_t size, uint64_t off) {
  if (off + 16 <= size) return *reinterpret_cast<const uint4*>(b + off);
  uint32_t w[4] = {0, 0, 0, 0};
  for (uint64_t i = off; i < size; ++i) w[(i - off) / 4] |= static_cast<uint32_t>(static_cast<uint8_t>(b[i])) << (8 * ((i - off) % 4));
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__global__ void nl_count_kernel(const char* b, uint64_t size, uint64_t seg, unsigned long long* counts) {
  const uint64_t lo = blockIdx.x * seg, hi = min(size, lo + seg);
  unsigned long long c = 0;
  for (uint64_t off = lo + threadIdx.x * 16ull; off < hi; off += kNlThreads * 16ull) c += nl_count16(load16(b, size, off));
  typedef cub::BlockReduce<unsigned long long, kNlThreads> R;
  __shared__ typename R::TempStorage tmp;
  const unsigned long long t = R(tmp).Sum(c);
  if (threadIdx.x == 0) counts[blockIdx.x] = t;
}
__global__ void nl_write_kernel(const char* b, uint64_t size, uint64_t seg, const unsigned long long* offs,
                                uint64_t* out) {
  typedef cub::BlockScan<unsigned int, kNlThreads> S;
  __shared__ typename S::TempStorage tmp;
  __shared__ unsigned long long base;
  const uint64_t lo = blockIdx.x * seg, hi = min(size, lo + seg);
  if (threadIdx.x == 0) base = offs[blockIdx.x];
  __syncthreads();
  for (uint64_t tile = lo; tile < hi; tile += kNlThreads * 16ull) {
    const uint64_t off = tile + threadIdx.x * 16ull;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (off < hi) v = load16(b, size, off);
    const unsigned int c = off < hi ? static_cast<unsigned int>(nl_count16(v)) : 0u;
    unsigned int pre = 0, tot = 0;
    S(tmp).ExclusiveSum(c, pre, tot);
    if (c) {
      uint64_t o = base + pre;
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
      for (int i = 0; i < 16; ++i)
        if (static_cast<uint8_t>(w[i / 4] >> (8 * (i % 4))) == '\n') out[o++] = off + i;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
}

uint64_t newlines(const char* d_buf, uint64_t size, uint64_t** d_nl, void** tmp, size_t* tmp_bytes,
                  cudaStream_t s) {
  *d_nl = nullptr;
  if (size == 0) {
    check(cudaMallocAsync(reinterpret_cast<void**>(d_nl), 8, s), "alloc nl");
    return 0;
  }
  const uint64_t seg = ((size + kNlBlocks - 1) / kNlBlocks + 15) / 16 * 16;
  const unsigned blocks = static_cast<unsigned>((size + seg - 1) / seg);
  unsigned long long* cnt = nullptr;
  check(cudaMallocAsync(reinterpret_cast<void**>(&cnt), (blocks + 1) * 8, s), "alloc");
  nl_count_kernel<<<blocks, kNlThreads, 0, s>>>(d_buf, size, seg, cnt);
  check(cudaGetLastError(), "newline count");
  size_t need = 0;
  check(cub::DeviceScan::ExclusiveSum(nullptr, need, cnt, cnt, blocks + 1, s), "scan");
  if (need > *tmp_bytes) {
    if (*tmp) check(cudaFreeAsync(*tmp, s), "free");
    check(cudaMallocAsync(tmp, need, s), "alloc tmp");
    *tmp_bytes = need;
  }
  check(cudaMemsetAsync(cnt + blocks, 0, 8, s), "memset");
  check(cub::DeviceScan::ExclusiveSum(*tmp, need, cnt, cnt, blocks + 1, s), "scan");
  unsigned long long n = 0;
  check(cudaMemcpyAsync(&n, cnt + blocks, 8, cudaMemcpyDeviceToHost, s), "D2H");
  check(cudaStreamSynchronize(s), "sync");
  check(cudaMallocAsync(reinterpret_cast<void**>(d_nl), (n + 1) * 8, s), "alloc nl");
  nl_write_kernel<<<blocks, kNlThreads, 0, s>>>(d_buf, size, seg, cnt, *d_nl);
  check(cudaGetLastError(), "newline write");
  check(cudaFreeAsync(cnt, s), "free");
  return n;
}

// Streams a file into device memory through two page-locked chunk buffers:
// the read of chunk i+1 overlaps the copy of chunk i.  Returns the size;
// `last` = the final byte (for std::getline's tail-line rule).
constexpr size_t kChunkBytes = size_t(16) << 20;
constexpr int kReaders = 4;  // page-cache reads are memcpy-bound: a few threads in parallel
struct PinnedPool {
  char* buf[kReaders][2] = {};
  cudaEvent_t ev[kReaders][2] = {};
};
PinnedPool& pinned_pool() {  // process-lifetime staging buffers (page-locking is slow)
  static PinnedPool p;
  static std::once_flag once;
  std::call_once(once, [] {
    for (int r = 0; r < kReaders; ++r)
      for (int i = 0; i < 2; ++i) {
        check(cudaHostAlloc(reinterpret_cast<void**>(&p.buf[r][i]), kChunkBytes, cudaHostAllocDefault), "pinned");
        check(cudaEventCreateWithFlags(&p.ev[r][i], cudaEventDisableTiming), "event");
      }
  });
  return p;
}
uint64_t file_size(const std::string& path) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw LobsterError("load_lobster: cannot open " + path, 4);
  std::fseek(f, 0, SEEK_END);
  const long n = std::ftell(f);
  std::fclose(f);
  return n > 0 ? static_cast<uint64_t>(n) : 0;
}
// Reader r takes chunks r, r + kReaders, ...: pread into one of its two
// page-locked buffers while the other's copy is in flight on stream s.
void stream_file(const std::string& path, char* d_dst, uint64_t size, char& last, cudaStream_t s) {
  last = '\n';
  if (size == 0) return;
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) throw LobsterError("load_lobster: cannot open " + path, 4);
  PinnedPool& pp = pinned_pool();
  const uint64_t n_chunks = (size + kChunkBytes - 1) / kChunkBytes;
  std::atomic<bool> failed{false};
  std::vector<std::thread> th;
  for (int r = 0; r < kReaders; ++r)
    th.emplace_back([&, r] {
      int i = 0;
      for (uint64_t c = r; c < n_chunks && !failed; c += kReaders, i ^= 1) {
        if (cudaEventSynchronize(pp.ev[r][i]) != cudaSuccess) {
          failed = true;
          return;
        }
        const uint64_t off = c * kChunkBytes;
        const size_t n = static_cast<size_t>(std::min<uint64_t>(kChunkBytes, size - off));
        size_t got = 0;
        while (got < n) {
          const ssize_t k = ::pread(fd, pp.buf[r][i] + got, n - got, static_cast<off_t>(off + got));
          if (k <= 0) {
            failed = true;
            return;
          }
          got += static_cast<size_t>(k);
        }
        if (off + n == size) last = pp.buf[r][i][n - 1];
        if (cudaMemcpyAsync(d_dst + off, pp.buf[r][i], n, cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaEventRecord(pp.ev[r][i], s) != cudaSuccess)
          failed = true;
      }
    });
  for (auto& t : th) t.join();
  ::close(fd);
  if (failed) throw LobsterError("load_lobster: cannot open " + path, 4);
}

// text of line j of a device buffer (strip_cr applied), for error messages
std::string device_line(const char* d_buf, uint64_t size, const uint64_t* d_nl, uint64_t n_nl, uint64_t j) {
  uint64_t b = 0, e = size;
  if (j > 0) {
    check(cudaMemcpy(&b, d_nl + j - 1, 8, cudaMemcpyDeviceToHost), "D2H");
    ++b;
  }
  if (j < n_nl) check(cudaMemcpy(&e, d_nl + j, 8, cudaMemcpyDeviceToHost), "D2H");
  std::string t(e - b, '\0');
  if (e > b) check(cudaMemcpy(&t[0], d_buf + b, e - b, cudaMemcpyDeviceToHost), "D2H");
  if (!t.empty() && t.back() == '\r') t.pop_back();
  return t;
}

}  // namespace

// Host formatting of the first failing row: the same parser, the reference's text.
static std::string format_row_error(const std::string& line, const std::string* book_line, uint64_t row,
                                    int64_t upt, bool sampled, int32_t dev_code, const std::string& msg_path) {
  const std::string r = "lobster: row " + std::to_string(row + 1) + ": ";
  if (dev_code == kBookMissing) return "load_lobster: orderbook file has fewer rows than " + msg_path;
  if (dev_code == kMonotone) return r + "non-monotone time";
  MsgRow m{};
  int64_t aux = 0;
  int bad = 0;
  int32_t e = parse_msg(line.data(), static_cast<int>(line.size()), upt, m, aux, bad);
  Field f[6];
  split(line.data(), static_cast<int>(line.size()), f, 6);
  const auto field = [&](int i) { return line.substr(f[i].begin, f[i].len); };
  static const char* names[6] = {"time", "type", "order id", "size", "price", "direction"};
  switch (e) {
    case kFields: return r + "expected 6 fields, got " + std::to_string(aux);
    case kTimeSec: {
      const std::string t = field(0);
      const size_t dot = t.find('.');
      return r + "malformed time field '" + (dot == std::string::npos ? t : t.substr(0, dot)) + "'";
    }
    case kTimeEmptyFrac: return r + "malformed time field";
    case kTimeFrac: {
      const std::string t = field(0);
      std::string frac = t.substr(t.find('.') + 1);
      if (frac.size() > 9) frac = frac.substr(0, 9);
      return r + "malformed time fraction field '" + frac + "'";
    }
    case kTypeParse:
    case kIdParse:
    case kSizeParse:
    case kPriceParse:
    case kDirParse: return r + "malformed " + names[bad] + " field '" + field(bad) + "'";
    case kTypeRange: return r + "unknown event type " + std::to_string(aux);
    case kSizeNeg: return r + "negative size";
    case kPriceTick:
      return r + "price " + std::to_string(aux) + " not divisible by tick size " + std::to_string(upt);
    case kDirRange: return r + "direction must be +1 or -1";
    default: break;
  }
  if (sampled && book_line) {
    int nb = 0, na = 0;
    e = parse_book<L64>(book_line->data(), static_cast<int>(book_line->size()), upt, nb, na, nullptr, nullptr,
                        aux);
    if (e == kBookCols)
      return "lobster: orderbook row " + std::to_string(row + 1) + ": column count " + std::to_string(aux) +
             " is not a multiple of 4";
    if (e == kBookField) {
      static const char* cols[4] = {"ask price", "ask size", "bid price", "bid size"};
      std::vector<std::string> parts;
      size_t b = 0;
      for (size_t i = 0; i <= book_line->size(); ++i)
        if (i == book_line->size() || (*book_line)[i] == ',') {
          parts.push_back(book_line->substr(b, i - b));
          b = i + 1;
        }
      return r + "malformed " + cols[aux % 4] + " field '" + parts[static_cast<size_t>(aux)] + "'";
    }
    if (e == kBookTick)
      return r + "price " + std::to_string(aux) + " not divisible by tick size " + std::to_string(upt);
  }
  return r + "malformed row";
}

void load(const std::string& msg_path, const std::string& book_path, int64_t upt, uint64_t sample_every,
          cudaStream_t s, LobsterStore& out) {
  if (upt < 1) throw LobsterError("load_lobster: units_per_tick >= 1", 1);
  if (sample_every == 0) throw LobsterError("load_lobster: sample_every >= 1", 1);
  const uint64_t ms = file_size(msg_path), bs = file_size(book_path);
  const bool timing = std::getenv("MLOB_LOBSTER_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  const auto mark = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "lobster %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };

  char *d_msg = nullptr, *d_book = nullptr;
  uint64_t *m_nl = nullptr, *b_nl = nullptr, *rows = nullptr, *d_cnt = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int64_t* d_time = nullptr;
  int32_t* d_err = nullptr;
  uint32_t *d_nb = nullptr, *d_na = nullptr;
  unsigned long long* d_flags = nullptr;  // [first_bad, first_range, extra_book|level_bad]
  uint64_t* d_lvoff = nullptr;
  std::vector<void*> owned;
  const auto cleanup = [&] {  // idempotent: the error paths reach it twice
    for (void* p : owned)
      if (p) cudaFreeAsync(p, s);
    owned.clear();
    if (tmp) cudaFreeAsync(tmp, s);
    tmp = nullptr;
    cudaStreamSynchronize(s);
    cudaGetLastError();  // no stale (non-sticky) error left for the next call
  };
  try {
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_msg), ms + 1, s), "alloc");
    owned.push_back(d_msg);
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_book), bs + 1, s), "alloc");
    owned.push_back(d_book);
    char m_last = '\n', b_last = '\n';
    stream_file(msg_path, d_msg, ms, m_last, s);
    stream_file(book_path, d_book, bs, b_last, s);
    mark("read+H2D");
    const uint64_t m_nl_n = newlines(d_msg, ms, &m_nl, &tmp, &tmp_bytes, s);
    owned.push_back(m_nl);
    const uint64_t b_nl_n = newlines(d_book, bs, &b_nl, &tmp, &tmp_bytes, s);
    owned.push_back(b_nl);
    mark("newlines");
    // std::getline line counts: a tail without '\n' counts when non-empty
    const uint64_t m_lines = m_nl_n + ((ms > 0 && m_last != '\n') ? 1 : 0);
    const uint64_t b_lines = b_nl_n + ((bs > 0 && b_last != '\n') ? 1 : 0);
    // non-empty message lines = message rows
    check(cudaMallocAsync(reinterpret_cast<void**>(&rows), (m_lines + 1) * sizeof(uint64_t), s), "alloc");
    owned.push_back(rows);
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_cnt), sizeof(uint64_t), s), "alloc");
    owned.push_back(d_cnt);
    thrust::counting_iterator<uint64_t> it(0);
    size_t need = 0;
    const NonEmptyLine pred{d_msg, m_nl, m_nl_n, ms};
    check(cub::DeviceSelect::If(nullptr, need, it, rows, d_cnt, m_lines, pred, s), "select");
    if (need > tmp_bytes) {
      if (tmp) check(cudaFreeAsync(tmp, s), "free");
      check(cudaMallocAsync(&tmp, need, s), "alloc");
      tmp_bytes = need;
    }
    check(cub::DeviceSelect::If(tmp, need, it, rows, d_cnt, m_lines, pred, s), "select");
    uint64_t n = 0;
    check(cudaMemcpyAsync(&n, d_cnt, sizeof n, cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");

    const uint64_t n_states = n / sample_every;  // sampled rows k with (k+1) % sample_every == 0
    DevMsg* d_out = nullptr;
    check(cudaMalloc(reinterpret_cast<void**>(&d_out), std::max<uint64_t>(n, 1) * sizeof(DevMsg)), "alloc store");
    out.d_msgs = d_out;
    out.n_msgs = n;
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_time), (n + 1) * 8, s), "alloc");
    owned.push_back(d_time);
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_err), (n + 1) * 4, s), "alloc");
    owned.push_back(d_err);
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_nb), (n_states + 1) * 4, s), "alloc");
    owned.push_back(d_nb);
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_na), (n_states + 1) * 4, s), "alloc");
    owned.push_back(d_na);
    check(cudaMallocAsync(reinterpret_cast<void**>(&d_flags), 4 * sizeof(unsigned long long), s), "alloc");
    owned.push_back(d_flags);
    const unsigned long long init[4] = {~0ull, ~0ull, 0, 0};
    check(cudaMemcpyAsync(d_flags, init, sizeof init, cudaMemcpyHostToDevice, s), "H2D");
    RowArgs a{};
    a.msg = d_msg;
    a.msg_nl = m_nl;
    a.msg_nl_n = m_nl_n;
    a.msg_size = ms;
    a.rows = rows;
    a.n_rows = n;
    a.book = d_book;
    a.book_nl = b_nl;
    a.book_nl_n = b_nl_n;
    a.book_size = bs;
    a.book_lines = b_lines;
    a.upt = upt;
    a.sample_every = sample_every;
    a.out = d_out;
    a.time = d_time;
    a.err = d_err;
    a.n_bid = d_nb;
    a.n_ask = d_na;
    a.first_bad = d_flags;
    a.first_range = d_flags + 1;
    if (n) {
      parse_rows_kernel<<<grid_of(n), 256, 0, s>>>(a);
      check(cudaGetLastError(), "parse kernel");
      monotone_kernel<<<grid_of(n), 256, 0, s>>>(d_time, d_err, n, d_flags);
      check(cudaGetLastError(), "monotone kernel");
    }
    if (b_lines > n) {
      extra_book_kernel<<<grid_of(b_lines - n), 256, 0, s>>>(d_book, b_nl, b_nl_n, bs, n, b_lines,
                                                           reinterpret_cast<unsigned int*>(d_flags + 2));
      check(cudaGetLastError(), "extra rows kernel");
    }
    unsigned long long flags[4];
    check(cudaMemcpyAsync(flags, d_flags, sizeof flags, cudaMemcpyDeviceToHost, s), "D2H");
    check(cudaStreamSynchronize(s), "sync");
    mark("rows+parse");
    out.n_lines_msg = m_lines;
    if (flags[0] != ~0ull) {  // the reference throws at this row
      const uint64_t k = flags[0];
      int32_t code = 0;
      uint64_t line_idx = 0;
      check(cudaMemcpy(&code, d_err + k, 4, cudaMemcpyDeviceToHost), "D2H");
      check(cudaMemcpy(&line_idx, rows + k, 8, cudaMemcpyDeviceToHost), "D2H");
      const std::string line = device_line(d_msg, ms, m_nl, m_nl_n, line_idx);
      std::string bl;
      const bool have_book = k < b_lines;
      if (have_book) bl = device_line(d_book, bs, b_nl, b_nl_n, k);
      cleanup();
      throw LobsterError(format_row_error(line, have_book ? &bl : nullptr, k, upt, (k + 1) % sample_every == 0,
                                          code, msg_path),
                         4);
    }
    if (flags[2]) {
      cleanup();
      throw LobsterError("load_lobster: message file has fewer rows than " + book_path, 4);
    }
    if (flags[1] != ~0ull) {
      cleanup();
      throw LobsterError("NewLimit price or quantity outside the device int32 range", 1);
    }
    // book states: offset 0 = empty book, then every sampled row k -> offset k + 1
    std::vector<uint32_t> nb(n_states), na(n_states);
    if (n_states) {
      check(cudaMemcpyAsync(nb.data(), d_nb, n_states * 4, cudaMemcpyDeviceToHost, s), "D2H");
      check(cudaMemcpyAsync(na.data(), d_na, n_states * 4, cudaMemcpyDeviceToHost, s), "D2H");
      check(cudaStreamSynchronize(s), "sync");
    }
    out.st_index.assign(1, 0);
    out.st_offset.assign(2, 0);  // state 0: [0, 0)
    out.st_nb.assign(1, 0);
    std::vector<uint64_t> lvoff(n_states);
    uint64_t total = 0;
    for (uint64_t st = 0; st < n_states; ++st) {
      lvoff[st] = total;
      out.st_index.push_back((st + 1) * sample_every);
      out.st_nb.push_back(nb[st]);
      total += nb[st] + na[st];
      out.st_offset.push_back(total);
    }
    // a state keyed one past the last message can never seed an episode (lobster.hpp:186-189)
    if (out.st_index.back() == n && out.st_index.size() > 1) {
      out.st_index.pop_back();
      out.st_nb.pop_back();
      out.st_offset.pop_back();
      total = out.st_offset.back();
    }
    DevLevel* d_levels = nullptr;
    check(cudaMalloc(reinterpret_cast<void**>(&d_levels), std::max<uint64_t>(total, 1) * sizeof(DevLevel)),
          "alloc levels");
    out.d_levels = d_levels;
    out.n_levels = total;
    const uint64_t write_states = out.st_index.size() - 1;
    if (write_states) {
      check(cudaMallocAsync(reinterpret_cast<void**>(&d_lvoff), write_states * 8, s), "alloc");
      owned.push_back(d_lvoff);
      check(cudaMemcpyAsync(d_lvoff, lvoff.data(), write_states * 8, cudaMemcpyHostToDevice, s), "H2D");
      write_levels_kernel<<<grid_of(write_states), 256, 0, s>>>(a, d_lvoff, write_states, d_levels,
                                                               reinterpret_cast<unsigned int*>(d_flags + 3));
      check(cudaGetLastError(), "levels kernel");
      check(cudaMemcpyAsync(flags, d_flags, sizeof flags, cudaMemcpyDeviceToHost, s), "D2H");
      check(cudaStreamSynchronize(s), "sync");
      if (flags[3]) {
        cleanup();
        throw LobsterError("book-state price or quantity outside the device int32 range", 1);
      }
    }
    mark("states");
    cleanup();
  } catch (...) {
    cleanup();
    cudaFree(out.d_msgs);
    cudaFree(out.d_levels);
    out.d_msgs = nullptr;
    out.d_levels = nullptr;
    throw;
  }
}

}  // namespace lobster
}  // namespace mlob
