// mlob_policy.h — device-side recurrent actor-critic (ippo::PolicyNet,
// net.hpp:18-30) and the per-launch arguments of the rollout kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mlob {

constexpr int kPolicyWarps = 8;         // streams per block
constexpr int kPolicyMaxObs = 8 + 4 * 64;  // MMFull at obs_depth 64 (observations.hpp:69-76)
constexpr int kPolicyMaxHidden = 512;   // make_policy_net cap (net.hpp:86-87)
constexpr int kPolicyMaxActions = 32;   // largest action arity (spread-skew table rows)

// A PolicyNet in HBM.  Input-side matrices are stored transposed so the lanes
// of a warp (one hidden unit each) read consecutive addresses:
//   w_ihT[d * 3H + g * H + i] = w_ih[(g * H + i) * D + d]
//   w_hhT[j * 3H + g * H + i] = w_hh[(g * H + i) * H + j]
//   w_actorT[j * A + a]       = w_actor[a * H + j]
struct DevNet {
  int32_t D, H, A, _pad;
  const double* w_ihT;
  const double* w_hhT;
  const double* b_ih;
  const double* b_hh;
  const double* w_actorT;
  const double* b_actor;
  const double* w_critic;
  double b_critic;
  const double* b_critic_dev;  // non-null: b_critic read from device memory (kept current by ppo_update)
};

struct PolicyArgs {
  DevNet net;
  uint64_t B;                 // streams of this type (n_envs * count)
  int32_t count, offset, agents_per_env, type;
  int32_t row;                // batch row written (t, or T for the bootstrap value)
  int32_t prev_row;           // row whose rewards / dones are filed (-1: none)
  int32_t sample;             // 1: draw an action (rollout step); 0: value only (bootstrap)
  int32_t argmax;             // 1: argmax_action into env_actions only (evaluate.hpp:80-90)
  // argmax mode: only envs whose type-`type` policy index equals `filter`
  const uint8_t* env_policy;  // [env * n_specs + type]
  int32_t n_specs, filter;
  uint64_t seed, update_index;
  const uint64_t* seed_update;  // non-null: {seed, update_index} read from device memory (graph replays)
  // env side
  const double* obs_env;      // the type's observation buffer, [s * D]
  const uint8_t* just_reset;  // [env]; null = no reset (evaluate.hpp:83)
  const double* env_rewards;  // [env * agents_per_env + a]
  const uint8_t* env_dones;
  int32_t* env_actions;       // the step kernel's action ids
  // recurrent state
  const double* hidden_in;    // [s * H]
  double* hidden_out;         // [s * H] or null
  double* h0_out;             // rollout start: batch.h0, else null
  // RolloutBatch (ppo.hpp:33-48), time-major
  double* obs_out;            // row t of batch.obs or null
  int32_t* actions;
  double* log_probs;
  double* values;             // (T + 1, B)
  double* rewards;
  uint8_t* dones;
  uint8_t* resets;
};

cudaError_t launch_policy(const PolicyArgs& pa, cudaStream_t s);
cudaError_t launch_gae(const double* rewards, const double* values, const uint8_t* dones, uint64_t T, uint64_t B,
                       double discount, double gae_lambda, double* adv, double* ret, cudaStream_t s);

}  // namespace mlob
