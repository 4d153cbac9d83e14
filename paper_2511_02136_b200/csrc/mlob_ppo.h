// mlob_ppo.h — device PPO update (mlob_ppo.cu): kernel arguments and launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace mlob {

// One minibatch: S streams of the rollout batch (B streams, T steps); every
// per-row array is time-major over the minibatch, row k = t * S + s.
struct PpoArgs {
  int32_t D, H, A, _pad;
  uint64_t T, B, S;
  const int32_t* mb;  // [S] batch stream ids
  // rollout batch (ppo.hpp:33-48)
  const double* obs;
  const uint8_t* resets;
  const int32_t* actions;
  const double* logp_old;
  const double* returns;
  const double* h0;
  const double* adv;  // [K] gathered (and normalized) advantages
  // transposed copies for the forward's lane-coalesced reads (mlob_policy.h layout)
  const double* w_ihT;
  const double* w_hhT;
  const double* w_actorT;
  // parameters, reference layout (net.hpp:18-30)
  const double* w_ih;
  const double* w_hh;
  const double* b_ih;
  const double* b_hh;
  const double* w_actor;
  const double* b_actor;
  const double* w_critic;
  double b_critic;
  double clip_eps, vf_coef, ent_coef;
  // caches and gradients, [K][...]
  double *X, *Hin, *R, *Z, *N, *HN, *Hout, *dL, *dV, *terms, *dA, *dB;
};

cudaError_t launch_ppo_forward(const PpoArgs& a, cudaStream_t s);
cudaError_t launch_ppo_backward(const PpoArgs& a, cudaStream_t s);
cudaError_t launch_gather_adv(const double* adv, const int32_t* mb, uint64_t T, uint64_t B, uint64_t S, double* out,
                              bool normalize, cudaStream_t s);
cudaError_t launch_clip_adam(double* p, double* g, double* m, double* v, uint64_t n, double max_norm, double lr,
                             double c1, double c2, double* norm_out, cudaStream_t s);
cudaError_t launch_to_inference(const double* p, int D, int H, int A, double* w, cudaStream_t s);
cudaError_t launch_fill(double* x, uint64_t n, double v, cudaStream_t s);
// Parameter-gradient contractions over the K = T x S rows of a minibatch
// (hand-written split-K fp64 reductions, deterministic: per-block partials
// summed in block order).  out (R x C, row-major) = L^T (R x K) . M (K x C);
// M == nullptr: column sums of L.  `part` holds kGemmBlocks x R x C doubles.
constexpr int kGemmBlocks = 296;
cudaError_t gemm_tn(const double* L, const double* M, uint64_t K, int R, int C, double* out, double* part,
                    cudaStream_t s);
inline cudaError_t colsum(const double* L, uint64_t K, int R, double* out, double* part, cudaStream_t s) {
  return gemm_tn(L, nullptr, K, R, 1, out, part, s);
}

}  // namespace mlob
