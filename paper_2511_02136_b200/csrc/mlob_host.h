// mlob_host.h — internal host-side declarations shared by the runtime
// translation units (C ABI in mlob_runtime.cu, store builders in mlob_store.cpp).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mlob.h"

struct mlob_host_store {
  std::vector<mlob_message> msgs;
  std::vector<uint64_t> st_index;   // message_index per state, increasing
  std::vector<uint64_t> st_offset;  // [n_states + 1] into levels
  std::vector<uint32_t> st_nb;      // bid levels per state
  std::vector<mlob_level> levels;   // per state: bids then asks, best-first

  const mlob_level* state_levels(uint64_t i) const { return levels.data() + st_offset[i]; }
  uint32_t state_na(uint64_t i) const {
    return static_cast<uint32_t>(st_offset[i + 1] - st_offset[i]) - st_nb[i];
  }
  // data::MessageStore::state_before (store.hpp:29-36): exact index match or -1
  int64_t state_before(uint64_t message_index) const;
  void push_state(uint64_t idx, const mlob_level* bids, uint32_t nb, const mlob_level* asks,
                  uint32_t na);
};

namespace mlob {

// Exceptions mapped onto mlob_status at the C boundary.
struct Error : std::runtime_error {
  mlob_status code;
  Error(mlob_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(mlob_status c, const std::string& m) { throw Error(c, m); }

void synth_generate(const mlob_synth_config& cfg, uint64_t seed, mlob_host_store& out);
std::vector<uint64_t> build_episode_index(uint64_t n_messages, int steps, int mps, int stride);
void validate_config(const mlob_env_config& c);

}  // namespace mlob
