// mlob_ppo.cu — ppo_update (ippo/ppo.hpp:263-310) for one agent type on the
// device, over the rollout batch collect_rollout left in HBM (SURVEY §8(f)
// row 4).  Per minibatch:
//   adv      gather + normalize_advantages (ppo.hpp:107-122)
//   forward  warp per stream, T steps of the GRU with every cache row kept
//            (net.hpp:120-188), then per element the clipped objective,
//            value loss and entropy bonus gradients (ppo.hpp:170-231)
//   backward warp per stream, t = T-1..0: head gradients into dh, the GRU cell
//            backward, the recurrent carry (net.hpp:193-277); gate gradients
//            stored per (t, stream)
//   weights  every parameter gradient is a sum over K = T x S rows: a
//            hand-written split-K fp64 contraction (gemm_tn: K-chunks staged
//            in shared memory, per-block partials summed in block order, so
//            the result is deterministic) straight into the PolicyGrad layout
//   step     global-norm clip + Adam (net.hpp:281-331), one block
// The reductions run in a different order than the reference's sequential
// loops, so parity is to a tolerance (tests: 1e-8 relative on parameters).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "mlob_ppo.h"

namespace mlob {

namespace {

constexpr int kWarps = 4;

// forward over the sequence + loss gradients, warp per minibatch stream
__global__ void __launch_bounds__(kWarps * 32) ppo_forward_kernel(const PpoArgs a) {
  extern __shared__ double fsm[];  // per warp: x[D], h[H] (+ A spare words)
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
  if (s >= a.S) return;
  const int D = a.D, H = a.H, A = a.A;
  double* sx = fsm + static_cast<size_t>(warp) * (D + H + A);
  double* sh = sx + D;
  const uint64_t b = static_cast<uint64_t>(a.mb[s]);
  const uint64_t S = a.S, B = a.B;
  for (int j = lane; j < H; j += 32) sh[j] = a.h0[b * H + j];
  const double n_elems = static_cast<double>(a.T * S);
  for (uint64_t t = 0; t < a.T; ++t) {
    const uint64_t k = t * S + s;  // minibatch row (time-major)
    const uint8_t reset = a.resets[t * B + b];
    for (int d = lane; d < D; d += 32) {
      const double v = a.obs[(t * B + b) * D + d];
      sx[d] = v;
      a.X[k * D + d] = v;
    }
    __syncwarp();
    for (int i = lane; i < H; i += 32) {  // net.hpp:141-172 with the cache
      double acc_r = a.b_ih[i] + a.b_hh[i];
      double acc_z = a.b_ih[H + i] + a.b_hh[H + i];
      double acc_n = a.b_ih[2 * H + i];
      double acc_hn = a.b_hh[2 * H + i];
      const size_t H3 = 3 * static_cast<size_t>(H);
      for (int d = 0; d < D; ++d) {  // transposed weights: lanes read consecutive words
        const double xd = sx[d];
        const double* w = a.w_ihT + d * H3;
        acc_r += w[i] * xd;
        acc_z += w[H + i] * xd;
        acc_n += w[2 * H + i] * xd;
      }
      if (!reset)
        for (int j = 0; j < H; ++j) {
          const double hj = sh[j];
          const double* w = a.w_hhT + j * H3;
          acc_r += w[i] * hj;
          acc_z += w[H + i] * hj;
          acc_hn += w[2 * H + i] * hj;
        }
      const double r = 1.0 / (1.0 + exp(-acc_r));
      const double z = 1.0 / (1.0 + exp(-acc_z));
      const double n = tanh(acc_n + r * acc_hn);
      const double h_old = reset ? 0.0 : sh[i];
      a.Hin[k * H + i] = h_old;
      a.R[k * H + i] = r;
      a.Z[k * H + i] = z;
      a.N[k * H + i] = n;
      a.HN[k * H + i] = acc_hn;
      a.Hout[k * H + i] = (1.0 - z) * n + z * h_old;
    }
    __syncwarp();
    for (int j = lane; j < H; j += 32) sh[j] = a.Hout[k * H + j];
    __syncwarp();
    // ppo.hpp:170-231 for element (t, s), warp-parallel: lane q = action q
    // (A <= 32), lane j = hidden unit j for the critic
    double lq = -INFINITY;
    if (lane < A) {
      double acc = a.b_actor[lane];
      for (int j = 0; j < H; ++j) acc += a.w_actorT[static_cast<size_t>(j) * A + lane] * sh[j];
      lq = acc;
    }
    double vpart = 0.0;
    for (int j = lane; j < H; j += 32) vpart += a.w_critic[j] * sh[j];
    double max_l = lq;
    for (int o = 16; o > 0; o >>= 1) max_l = fmax(max_l, __shfl_xor_sync(0xffffffffu, max_l, o));
    const double eq = lane < A ? exp(lq - max_l) : 0.0;
    double zs = eq;
    for (int o = 16; o > 0; o >>= 1) {
      zs += __shfl_xor_sync(0xffffffffu, zs, o);
      vpart += __shfl_xor_sync(0xffffffffu, vpart, o);
    }
    const double v = a.b_critic + vpart;
    const double log_z = log(zs);
    const double p = eq / zs;
    double ent = (lane < A && p > 0.0) ? -p * (lq - max_l - log_z) : 0.0;
    for (int o = 16; o > 0; o >>= 1) ent += __shfl_xor_sync(0xffffffffu, ent, o);
    const int act = a.actions[t * B + b];
    const double l_act = __shfl_sync(0xffffffffu, lq, act);
    const double logp_new = l_act - max_l - log_z;
    const double log_ratio = logp_new - a.logp_old[t * B + b];
    const double ratio = exp(log_ratio);
    const double a_hat = a.adv[k];
    const double l_unclipped = -a_hat * ratio;
    const double cl = ratio < 1.0 - a.clip_eps ? 1.0 - a.clip_eps : (ratio > 1.0 + a.clip_eps ? 1.0 + a.clip_eps : ratio);
    const double l_clipped = -a_hat * cl;
    const bool unclipped_active = l_unclipped >= l_clipped;
    const double dlogp = unclipped_active ? -a_hat * ratio / n_elems : 0.0;
    if (lane < A) {
      double dl = dlogp * ((lane == act ? 1.0 : 0.0) - p);
      dl += a.ent_coef * p * ((lq - max_l - log_z) + ent) / n_elems;
      a.dL[k * A + lane] = dl;
    }
    if (lane == 0) {
      const double ret = a.returns[t * B + b];
      double* tm = a.terms + k * 5;
      tm[0] = l_unclipped > l_clipped ? l_unclipped : l_clipped;
      tm[1] = 0.5 * (v - ret) * (v - ret);
      tm[2] = ent;
      tm[3] = (ratio - 1.0) - log_ratio;
      tm[4] = fabs(ratio - 1.0) > a.clip_eps ? 1.0 : 0.0;
      a.dV[k] = a.vf_coef * (v - ret) / n_elems;
    }
    __syncwarp();
  }
}

// backward through time, warp per minibatch stream (net.hpp:193-277)
__global__ void __launch_bounds__(kWarps * 32) ppo_backward_kernel(const PpoArgs a) {
  extern __shared__ double bsm[];  // per warp: carry[H], dh[H], da_r[H], da_z[H], dhn[H]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * kWarps + warp;
  if (s >= a.S) return;
  const int H = a.H, A = a.A, H3 = 3 * a.H;
  double* carry = bsm + static_cast<size_t>(warp) * 5 * H;
  double* dh = carry + H;
  double* dr = dh + H;
  double* dz = dr + H;
  double* dn_ = dz + H;
  const uint64_t b = static_cast<uint64_t>(a.mb[s]);
  const uint64_t S = a.S, B = a.B;
  for (int j = lane; j < H; j += 32) carry[j] = 0.0;
  __syncwarp();
  for (uint64_t t = a.T; t-- > 0;) {
    const uint64_t k = t * S + s;
    const double dv = a.dV[k];
    for (int j = lane; j < H; j += 32) {  // head gradients into dh
      double g = carry[j];
      for (int q = 0; q < A; ++q) {
        const double dl = a.dL[k * A + q];
        if (dl == 0.0) continue;
        g += dl * a.w_actor[static_cast<size_t>(q) * H + j];
      }
      if (dv != 0.0) g += dv * a.w_critic[j];
      dh[j] = g;
    }
    __syncwarp();
    for (int i = lane; i < H; i += 32) {  // GRU cell backward
      const double r = a.R[k * H + i], z = a.Z[k * H + i], n = a.N[k * H + i];
      const double dn = dh[i] * (1.0 - z);
      const double dzz = dh[i] * (a.Hin[k * H + i] - n);
      const double dan = dn * (1.0 - n * n);
      const double dhn = dan * r;
      const double drr = dan * a.HN[k * H + i];
      const double da_r = drr * r * (1.0 - r);
      const double da_z = dzz * z * (1.0 - z);
      a.dA[k * H3 + i] = da_r;
      a.dA[k * H3 + H + i] = da_z;
      a.dA[k * H3 + 2 * H + i] = dan;
      a.dB[k * H3 + i] = da_r;
      a.dB[k * H3 + H + i] = da_z;
      a.dB[k * H3 + 2 * H + i] = dhn;
      dr[i] = da_r;
      dz[i] = da_z;
      dn_[i] = dhn;
    }
    __syncwarp();
    const bool reset = a.resets[t * B + b] != 0;
    for (int j = lane; j < H; j += 32) {  // recurrent carry (zero across a reset)
      double acc = 0.0;
      if (!reset) {
        acc = dh[j] * a.Z[k * H + j];
        for (int i = 0; i < H; ++i) {
          acc += dr[i] * a.w_hh[static_cast<size_t>(i) * H + j];
          acc += dz[i] * a.w_hh[static_cast<size_t>(H + i) * H + j];
          acc += dn_[i] * a.w_hh[static_cast<size_t>(2 * H + i) * H + j];
        }
      }
      carry[j] = acc;
    }
    __syncwarp();
  }
}

// advantages of the minibatch streams, time-major (ppo.hpp:148-155)
__global__ void gather_adv_kernel(const double* adv, const int32_t* mb, uint64_t T, uint64_t B, uint64_t S,
                                  double* out) {
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < T * S;
       k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[k] = adv[(k / S) * B + static_cast<uint64_t>(mb[k % S])];
}

// normalize_advantages (ppo.hpp:107-122): block-reduced mean / population std
__global__ void normalize_adv_kernel(double* adv, uint64_t n) {
  __shared__ double red[1024];
  __shared__ double mean_s, std_s;
  double acc = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) acc += adv[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) mean_s = red[0] / static_cast<double>(n);
  __syncthreads();
  const double mean = mean_s;
  acc = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) acc += (adv[i] - mean) * (adv[i] - mean);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) std_s = sqrt(red[0] / static_cast<double>(n));
  __syncthreads();
  const double sd = std_s;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) adv[i] = sd > 0.0 ? (adv[i] - mean) / sd : 0.0;
}

// clip_grad_norm + adam_step (net.hpp:281-331), one block over the flat parameters
__global__ void clip_adam_kernel(double* p, double* g, double* m, double* v, uint64_t n, double max_norm, double lr,
                                 double c1, double c2, double* norm_out) {
  __shared__ double red[1024];
  double acc = 0.0;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) acc += g[i] * g[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double norm = sqrt(red[0]);
  if (threadIdx.x == 0) *norm_out = norm;
  const bool clip = max_norm > 0.0 && norm > max_norm;
  const double scale = clip ? max_norm / norm : 1.0;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double gi = clip ? g[i] * scale : g[i];
    m[i] = b1 * m[i] + (1.0 - b1) * gi;
    v[i] = b2 * v[i] + (1.0 - b2) * gi * gi;
    p[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
  }
}

// canonical (reference) layout -> the policy kernel's transposed layout
__global__ void to_inference_kernel(const double* p, int D, int H, int A, double* w) {
  const size_t H3 = 3 * static_cast<size_t>(H);
  const size_t n_ih = H3 * D, n_hh = H3 * H;
  const double* w_ih = p;
  const double* w_hh = w_ih + n_ih;
  const double* b_ih = w_hh + n_hh;
  const double* b_hh = b_ih + H3;
  const double* w_a = b_hh + H3;
  const double* b_a = w_a + static_cast<size_t>(A) * H;
  const double* w_c = b_a + A;
  double* o_ihT = w;
  double* o_hhT = o_ihT + n_ih;
  double* o_bih = o_hhT + n_hh;
  double* o_bhh = o_bih + H3;
  double* o_aT = o_bhh + H3;
  double* o_ba = o_aT + static_cast<size_t>(A) * H;
  double* o_wc = o_ba + A;
  const size_t total = n_ih + n_hh + 2 * H3 + static_cast<size_t>(A) * H + A + H;
  for (size_t x = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (x < n_ih) {
      const size_t r = x / D, d = x % D;
      o_ihT[d * H3 + r] = w_ih[x];
    } else if (x < n_ih + n_hh) {
      const size_t y = x - n_ih, r = y / H, j = y % H;
      o_hhT[j * H3 + r] = w_hh[y];
    } else if (x < n_ih + n_hh + H3) {
      o_bih[x - n_ih - n_hh] = b_ih[x - n_ih - n_hh];
    } else if (x < n_ih + n_hh + 2 * H3) {
      o_bhh[x - n_ih - n_hh - H3] = b_hh[x - n_ih - n_hh - H3];
    } else if (x < n_ih + n_hh + 2 * H3 + static_cast<size_t>(A) * H) {
      const size_t y = x - n_ih - n_hh - 2 * H3, q = y / H, j = y % H;
      o_aT[j * A + q] = w_a[y];
    } else if (x < n_ih + n_hh + 2 * H3 + static_cast<size_t>(A) * H + A) {
      const size_t y = x - n_ih - n_hh - 2 * H3 - static_cast<size_t>(A) * H;
      o_ba[y] = b_a[y];
    } else {
      const size_t y = x - n_ih - n_hh - 2 * H3 - static_cast<size_t>(A) * H - A;
      o_wc[y] = w_c[y];
    }
  }
}

__global__ void fill_kernel(double* x, uint64_t n, double v) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    x[i] = v;
}

unsigned grid_of(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 8192) b = 8192;
  return static_cast<unsigned>(b);
}

}  // namespace

cudaError_t launch_ppo_forward(const PpoArgs& a, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(kWarps) * (a.D + a.H + a.A) * sizeof(double);
  ppo_forward_kernel<<<static_cast<unsigned>((a.S + kWarps - 1) / kWarps), kWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_ppo_backward(const PpoArgs& a, cudaStream_t s) {
  const size_t smem = static_cast<size_t>(kWarps) * 5 * a.H * sizeof(double);
  ppo_backward_kernel<<<static_cast<unsigned>((a.S + kWarps - 1) / kWarps), kWarps * 32, smem, s>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_gather_adv(const double* adv, const int32_t* mb, uint64_t T, uint64_t B, uint64_t S, double* out,
                              bool normalize, cudaStream_t s) {
  gather_adv_kernel<<<grid_of(T * S), 256, 0, s>>>(adv, mb, T, B, S, out);
  if (normalize) normalize_adv_kernel<<<1, 1024, 0, s>>>(out, T * S);
  return cudaGetLastError();
}
cudaError_t launch_clip_adam(double* p, double* g, double* m, double* v, uint64_t n, double max_norm, double lr,
                             double c1, double c2, double* norm_out, cudaStream_t s) {
  clip_adam_kernel<<<1, 1024, 0, s>>>(p, g, m, v, n, max_norm, lr, c1, c2, norm_out);
  return cudaGetLastError();
}
cudaError_t launch_to_inference(const double* p, int D, int H, int A, double* w, cudaStream_t s) {
  const uint64_t total = 3ull * H * D + 3ull * H * H + 6ull * H + static_cast<uint64_t>(A) * H + A + H;
  to_inference_kernel<<<grid_of(total), 256, 0, s>>>(p, D, H, A, w);
  return cudaGetLastError();
}
cudaError_t launch_fill(double* x, uint64_t n, double v, cudaStream_t s) {
  fill_kernel<<<grid_of(n), 256, 0, s>>>(x, n, v);
  return cudaGetLastError();
}

namespace {
// Thread work unit: one output column c and kGemmRB consecutive output rows
// r0.. (out[r][c] = sum_k L[k][r] M[k][c]): per staged row k, one M value and
// kGemmRB L values feed kGemmRB fused multiply-adds (explicit __fma_rn: the
// file is built with --fmad=false for the env kernels' bit-exactness; the
// learner is compared to 1e-8).
constexpr int kGemmThreads = 256, kGemmTK = 32, kGemmRB = 8;

// Block b sums rows [b * chunk, (b + 1) * chunk) for work units
// [u0, u0 + nu) into part[b * E + e].  Narrow outputs (fewer units than
// threads) split each staged tile's rows over `ks` = blockDim / nu thread
// groups whose accumulators are then added in group order (deterministic).
__global__ void __launch_bounds__(kGemmThreads) gemm_tn_partial_kernel(const double* __restrict__ L,
                                                                      const double* __restrict__ M, uint64_t K,
                                                                      int R, int C, uint64_t chunk, int u0, int nu,
                                                                      double* __restrict__ part) {
  extern __shared__ double gsm[];
  double* Ls = gsm;                  // [kGemmTK][R]
  double* Ms = gsm + kGemmTK * R;    // [kGemmTK][C]
  double* red = Ms + kGemmTK * C;    // [kGemmThreads][kGemmRB] group partials
  const int E = R * C;
  const int ks = kGemmThreads / nu;  // row groups
  const int grp = static_cast<int>(threadIdx.x) / nu, lu = static_cast<int>(threadIdx.x) % nu;
  const bool active = grp < ks;
  const int u = u0 + lu;
  const int c = u % C, r0 = (u / C) * kGemmRB;
  const uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * chunk;
  const uint64_t k1 = k0 + chunk < K ? k0 + chunk : K;
  double acc[kGemmRB];
#pragma unroll
  for (int j = 0; j < kGemmRB; ++j) acc[j] = 0.0;
  for (uint64_t kt = k0; kt < k1; kt += kGemmTK) {
    const int n = static_cast<int>(k1 - kt < kGemmTK ? k1 - kt : kGemmTK);
    for (int x = threadIdx.x; x < n * R; x += kGemmThreads) Ls[x] = L[kt * R + x];
    if (M)
      for (int x = threadIdx.x; x < n * C; x += kGemmThreads) Ms[x] = M[kt * C + x];
    __syncthreads();
    if (active) {
      for (int i = grp; i < n; i += ks) {
        const double mv = M ? Ms[i * C + c] : 1.0;
        const double* lr = Ls + i * R + r0;
#pragma unroll
        for (int j = 0; j < kGemmRB; ++j)
          if (r0 + j < R) acc[j] = __fma_rn(lr[j], mv, acc[j]);
      }
    }
    __syncthreads();
  }
  if (ks > 1) {  // fold the row groups, in group order
#pragma unroll
    for (int j = 0; j < kGemmRB; ++j) red[threadIdx.x * kGemmRB + j] = acc[j];
    __syncthreads();
    if (grp == 0) {
      for (int g = 1; g < ks; ++g)
#pragma unroll
        for (int j = 0; j < kGemmRB; ++j) acc[j] += red[(g * nu + lu) * kGemmRB + j];
    }
  }
  if (grp == 0) {
#pragma unroll
    for (int j = 0; j < kGemmRB; ++j)
      if (r0 + j < R) part[static_cast<size_t>(blockIdx.x) * E + (r0 + j) * C + c] = acc[j];
  }
}

__global__ void gemm_tn_sum_kernel(const double* __restrict__ part, int P, int E, double* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double s = 0.0;
  for (int b = 0; b < P; ++b) s += part[static_cast<size_t>(b) * E + e];
  out[e] = s;
}
}  // namespace

cudaError_t gemm_tn(const double* L, const double* M, uint64_t K, int R, int C, double* out, double* part,
                    cudaStream_t s) {
  const int E = R * C;
  if (E <= 0) return cudaSuccess;
  uint64_t chunk = (K + kGemmBlocks - 1) / kGemmBlocks;
  chunk = (chunk + kGemmTK - 1) / kGemmTK * kGemmTK;
  const int P = static_cast<int>(K == 0 ? 1 : (K + chunk - 1) / chunk);
  const size_t smem = (static_cast<size_t>(kGemmTK) * (R + C) + kGemmThreads * kGemmRB) * sizeof(double);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(gemm_tn_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int units = (R + kGemmRB - 1) / kGemmRB * C;
  if (K == 0) {
    const cudaError_t e = cudaMemsetAsync(part, 0, static_cast<size_t>(E) * sizeof(double), s);
    if (e != cudaSuccess) return e;
  }
  for (int u0 = 0; u0 < units && K > 0; u0 += kGemmThreads) {
    const int nu = units - u0 < kGemmThreads ? units - u0 : kGemmThreads;
    gemm_tn_partial_kernel<<<P, kGemmThreads, smem, s>>>(L, M, K, R, C, chunk, u0, nu, part);
  }
  gemm_tn_sum_kernel<<<(E + 255) / 256, 256, 0, s>>>(part, P, E, out);
  return cudaGetLastError();
}

}  // namespace mlob
