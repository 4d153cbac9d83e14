// mlob_lobster.h — host interface of the device LOBSTER loader (mlob_lobster.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mlob_dev.h"

namespace mlob {
namespace lobster {

// status: the mlob_status the ABI returns (1 invalid_argument, 4 runtime, 5 CUDA)
struct LobsterError : std::runtime_error {
  int status;
  LobsterError(const std::string& m, int st) : std::runtime_error(m), status(st) {}
};

// The device store parts: DevMsg / DevLevel arrays (cudaMalloc, owned by the
// caller on success) and the host-side book-state table.
struct LobsterStore {
  DevMsg* d_msgs = nullptr;
  uint64_t n_msgs = 0;
  DevLevel* d_levels = nullptr;
  uint64_t n_levels = 0;
  uint64_t n_lines_msg = 0;
  std::vector<uint64_t> st_index, st_offset;
  std::vector<uint32_t> st_nb;
};

void load(const std::string& msg_path, const std::string& book_path, int64_t units_per_tick, uint64_t sample_every,
          cudaStream_t s, LobsterStore& out);

}  // namespace lobster
}  // namespace mlob
