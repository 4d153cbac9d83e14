// mlob_policy.cu — on-device recurrent actor-critic inference and the rollout
// bookkeeping around the env step:
//   policy_forward      net.hpp:120-188  (GRU cell, actor + critic heads, fp64)
//   sample_categorical  ppo.hpp:80-98    (CounterRng ActionSample key, rollout.hpp:90-93)
//   compute_gae         gae.hpp:14-32
// collect_rollout (rollout.hpp:41-124) is driven from mlob_runtime.cu: per
// step one policy launch per agent type, then the env step kernel.
//
// One warp per stream; lane l owns hidden units l, l+32, ...  Every dot
// product runs sequentially in the reference's order, built with
// --fmad=false, so sums are bit-identical to the host; exp / tanh / log are
// the device libm (<= 1-2 ulp from glibc), hence the 1e-12-relative parity bar
// on logits / values / log-probs in the tests.
#include <cuda_runtime.h>

#include <cstdint>

#include "mlob_dev.h"
#include "mlob_policy.h"

namespace mlob {

namespace {

__device__ __forceinline__ uint64_t pol_splitmix64(uint64_t z) {  // rng.hpp:11-16
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t pol_fold(uint64_t h, uint64_t w) {  // rng.hpp:18-20
  return pol_splitmix64(h ^ (w + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2)));
}
__device__ __forceinline__ double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }  // net.hpp:107

}  // namespace

// Per stream: GRU step + heads; then (kSample) the categorical draw written into
// the rollout batch and the env's action buffer, or (bootstrap) the value only.
// Also files the rewards / dones of the previous env step (rollout.hpp:94-100).
__global__ void __launch_bounds__(kPolicyWarps * 32) policy_kernel(const PolicyArgs pa) {
  extern __shared__ double psm[];  // per warp: x[D], h_prev[H], h_new[H], logits[A]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * kPolicyWarps + warp;
  if (s >= pa.B) return;
  const DevNet& nt = pa.net;
  const int D = nt.D, H = nt.H, A = nt.A, H3 = 3 * nt.H;
  double* const sx = psm + static_cast<size_t>(warp) * (D + 2 * H + A);
  double* const sh = sx + D;
  double* const sn = sh + H;
  double* const sl = sn + H;
  const uint64_t e = s / pa.count, slot = e * pa.agents_per_env + pa.offset + s % pa.count;
  const uint64_t B = pa.B;
  if (pa.argmax && pa.env_policy[e * pa.n_specs + pa.type] != pa.filter) return;
  // rewards / dones of the step just taken (row t - 1)
  if (pa.prev_row >= 0 && lane == 0) {
    pa.rewards[static_cast<uint64_t>(pa.prev_row) * B + s] = pa.env_rewards[slot];
    pa.dones[static_cast<uint64_t>(pa.prev_row) * B + s] = pa.env_dones[slot];
  }
  const uint8_t reset = pa.just_reset ? pa.just_reset[e] : 0;  // gather's reset flag (rollout.hpp:210)
  const double* x = pa.obs_env + s * D;
  for (int d = lane; d < D; d += 32) {
    sx[d] = x[d];
    if (pa.obs_out) pa.obs_out[s * D + d] = x[d];
  }
  const double* hp = pa.hidden_in + s * H;
  for (int j = lane; j < H; j += 32) {
    sh[j] = hp[j];
    if (pa.h0_out) pa.h0_out[s * H + j] = hp[j];
  }
  __syncwarp();
  for (int i = lane; i < H; i += 32) {  // net.hpp:141-172
    double acc_r = nt.b_ih[i] + nt.b_hh[i];
    double acc_z = nt.b_ih[H + i] + nt.b_hh[H + i];
    double acc_n = nt.b_ih[2 * H + i];
    double acc_hn = nt.b_hh[2 * H + i];
    for (int d = 0; d < D; ++d) {
      const double xd = sx[d];
      const double* w = nt.w_ihT + static_cast<size_t>(d) * H3;
      acc_r += w[i] * xd;
      acc_z += w[H + i] * xd;
      acc_n += w[2 * H + i] * xd;
    }
    if (!reset) {
      for (int j = 0; j < H; ++j) {
        const double hj = sh[j];
        const double* w = nt.w_hhT + static_cast<size_t>(j) * H3;
        acc_r += w[i] * hj;
        acc_z += w[H + i] * hj;
        acc_hn += w[2 * H + i] * hj;
      }
    }
    const double r = sigmoid(acc_r);
    const double z = sigmoid(acc_z);
    const double n = tanh(acc_n + r * acc_hn);
    const double h_old = reset ? 0.0 : sh[i];
    const double h_new = (1.0 - z) * n + z * h_old;
    sn[i] = h_new;
    if (pa.hidden_out) pa.hidden_out[s * H + i] = h_new;
  }
  __syncwarp();
  for (int a = lane; a < A; a += 32) {  // actor head, net.hpp:175-179
    double acc = nt.b_actor[a];
    for (int j = 0; j < H; ++j) acc += nt.w_actorT[static_cast<size_t>(j) * A + a] * sn[j];
    sl[a] = acc;
  }
  __syncwarp();
  if (lane != 0) return;
  if (pa.argmax) {  // argmax_action (ppo.hpp:100-105): first maximum
    int best = 0;
    for (int a = 1; a < A; ++a)
      if (sl[a] > sl[best]) best = a;
    pa.env_actions[slot] = best;
    return;
  }
  double v = nt.b_critic_dev ? *nt.b_critic_dev : nt.b_critic;  // critic head, net.hpp:180-182
  for (int j = 0; j < H; ++j) v += nt.w_critic[j] * sn[j];
  pa.values[static_cast<uint64_t>(pa.row) * B + s] = v;
  if (!pa.sample) return;
  pa.resets[static_cast<uint64_t>(pa.row) * B + s] = reset;
  // sample_categorical (ppo.hpp:80-98), u = CounterRng(make_key(seed, ActionSample,
  // tau, update, t, s)).uniform() (rollout.hpp:88-93)
  const uint64_t seed = pa.seed_update ? pa.seed_update[0] : pa.seed;
  const uint64_t update = pa.seed_update ? pa.seed_update[1] : pa.update_index;
  uint64_t key = pol_fold(pol_fold(pol_splitmix64(seed), 3), static_cast<uint64_t>(pa.type));
  key = pol_fold(pol_fold(pol_fold(key, update), static_cast<uint64_t>(pa.row)), s);
  const double u = static_cast<double>(pol_splitmix64(key + 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
  const double* lg = sl;
  double max_l = lg[0];
  for (int a = 0; a < A; ++a) max_l = max_l < lg[a] ? lg[a] : max_l;  // std::max(max_l, l)
  double zs = 0.0;
  for (int a = 0; a < A; ++a) zs += exp(lg[a] - max_l);
  const double target = u * zs;
  double cum = 0.0;
  int action = A - 1;
  for (int a = 0; a < A; ++a) {
    cum += exp(lg[a] - max_l);
    if (cum > target) {
      action = a;
      break;
    }
  }
  pa.actions[static_cast<uint64_t>(pa.row) * B + s] = action;
  pa.log_probs[static_cast<uint64_t>(pa.row) * B + s] = lg[action] - max_l - log(zs);
  pa.env_actions[slot] = action;
}

// compute_gae (gae.hpp:14-32), one thread per stream, same expression order.
__global__ void gae_kernel(const double* rewards, const double* values, const uint8_t* dones, uint64_t T,
                           uint64_t B, double discount, double gae_lambda, double* adv, double* ret) {
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < B;
       b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
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

cudaError_t launch_policy(const PolicyArgs& pa, cudaStream_t s) {
  if (pa.B == 0) return cudaSuccess;
  const unsigned blocks = static_cast<unsigned>((pa.B + kPolicyWarps - 1) / kPolicyWarps);
  const size_t smem = static_cast<size_t>(kPolicyWarps) * (pa.net.D + 2 * pa.net.H + pa.net.A) * sizeof(double);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(policy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  policy_kernel<<<blocks, kPolicyWarps * 32, smem, s>>>(pa);
  return cudaGetLastError();
}

cudaError_t launch_gae(const double* rewards, const double* values, const uint8_t* dones, uint64_t T, uint64_t B,
                       double discount, double gae_lambda, double* adv, double* ret, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  uint64_t blocks = (B + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  gae_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(rewards, values, dones, T, B, discount, gae_lambda, adv,
                                                           ret);
  return cudaGetLastError();
}

}  // namespace mlob
