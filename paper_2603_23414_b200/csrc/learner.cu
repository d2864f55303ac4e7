// learner.cu — the update group's consumer on the GPU (include/srl_learner.h;
// SURVEY §8(f) N2; Eq. (1)-(3)).  The group is small next to
// a decode step (U trajectories x a few thousand tokens: a few MB), so these are
// latency-bound kernels: fp64 arithmetic on fp32 inputs (the B200's fp64 pipe is
// ample at this size), fixed reduction orders, no atomics on floating point.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "srl_learner.h"

namespace srl {
void set_error(const char* fmt, const char* a, long b);
}

namespace {

constexpr int kRedThreads = 1024;
constexpr int kGaeThreads = 256;
constexpr int kPpoThreads = 256;
constexpr int kPpoBlocks = 296;  // 2 per SM: the token loop is grid-strided

// Deterministic block sum: a fixed xor-shuffle tree per warp, then the warp
// totals added in warp order by every thread.
__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  return t;
}

// Eq. (3): A_i = (R_i - mu) / sigma, population sigma; sigma = 0 -> 0.
__global__ void __launch_bounds__(kRedThreads) reinforcepp_kernel(const float* __restrict__ R, int n,
                                                                  float* __restrict__ adv) {
  __shared__ double sh[kRedThreads / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += (double)R[i];
  const double mu = block_sum(s, sh) / n;
  double q = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = (double)R[i] - mu;
    q += d * d;
  }
  const double sigma = sqrt(block_sum(q, sh) / n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) adv[i] = sigma == 0.0 ? 0.f : (float)(((double)R[i] - mu) / sigma);
}

__global__ void expand_kernel(const float* __restrict__ v, const int64_t* __restrict__ off, float* __restrict__ out) {
  const int i = blockIdx.x;
  const float x = v[i];
  for (int64_t t = off[i] + threadIdx.x; t < off[i + 1]; t += blockDim.x) out[t] = x;
}

// Eq. (2) for trajectory blockIdx.x: A_t = delta_t + c A_{t+1} (c = gamma lambda,
// A_T = 0) is an affine map per token; thread j owns a contiguous chunk, reduces
// it to (L_j, m_j) = (A at the chunk start if A after it were 0, c^len), the
// chunk carries are chained from the end, and each chunk is re-walked from its
// carry.
__global__ void __launch_bounds__(kGaeThreads) gae_kernel(const float* __restrict__ r, const float* __restrict__ V,
                                                          const int64_t* __restrict__ off, double gamma, double lam,
                                                          float* __restrict__ adv) {
  __shared__ double L[kGaeThreads], Mul[kGaeThreads], cin[kGaeThreads];
  const int i = blockIdx.x;
  const int64_t base = off[i], T = off[i + 1] - off[i];
  const float* v = V + base + i;  // V(s_0 .. s_T) of this trajectory
  const double c = gamma * lam;
  const int64_t chunk = (T + kGaeThreads - 1) / kGaeThreads;
  const int64_t s = (int64_t)threadIdx.x * chunk, e = s + chunk < T ? s + chunk : T;
  double a = 0.0, m = 1.0;
  for (int64_t t = e - 1; t >= s; --t) {
    const double delta = (double)r[base + t] + gamma * (double)v[t + 1] - (double)v[t];
    a = delta + c * a;
    m *= c;
  }
  L[threadIdx.x] = a;
  Mul[threadIdx.x] = m;
  __syncthreads();
  if (threadIdx.x == 0) {  // carry into each chunk = A at its end (the next chunk's start)
    double carry = 0.0;
    for (int j = kGaeThreads - 1; j >= 0; --j) {
      cin[j] = carry;
      carry = L[j] + Mul[j] * carry;
    }
  }
  __syncthreads();
  a = cin[threadIdx.x];
  for (int64_t t = e - 1; t >= s; --t) {
    const double delta = (double)r[base + t] + gamma * (double)v[t + 1] - (double)v[t];
    a = delta + c * a;
    adv[base + t] = (float)a;
  }
}

// Eq. (1) per token + per-block partial sums of the terms (fixed token -> thread map).
__global__ void __launch_bounds__(kPpoThreads) ppo_kernel(const float* __restrict__ nw, const float* __restrict__ od,
                                                          const float* __restrict__ A, int64_t n, double lo, double hi,
                                                          float* __restrict__ ratio, float* __restrict__ dterm,
                                                          double* __restrict__ part) {
  __shared__ double sh[kPpoThreads / 32];
  double acc = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    const double rho = exp((double)nw[t] - (double)od[t]);
    const double a = (double)A[t];
    const double u = rho * a;
    const double cl = fmin(fmax(rho, lo), hi) * a;
    const bool unclipped = u <= cl;
    acc += unclipped ? u : cl;
    if (ratio) ratio[t] = (float)rho;
    if (dterm) dterm[t] = unclipped ? (float)(rho * a) : 0.f;
  }
  const double b = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void ppo_finish_kernel(const double* __restrict__ part, int nb, int64_t n, double* __restrict__ obj) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += part[b];
    *obj = n > 0 ? s / (double)n : 0.0;
  }
}

__global__ void staleness_kernel(const int32_t* __restrict__ ver, int64_t n, int v_update, int nbins, int32_t* hist) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    int d = v_update - ver[t];
    d = d < 0 ? 0 : (d >= nbins ? nbins - 1 : d);
    atomicAdd(hist + d, 1);
  }
}

int launch_rc(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return 0;
  srl::set_error("%s: launch failed (%ld)", what, (long)e);
  return -3;
}

int bad(const char* what) {
  srl::set_error("%s: bad arguments", what, 0);
  return -1;
}

}  // namespace

extern "C" {

int32_t srl_learner_reinforcepp(const float* rewards, int32_t n, float* adv, void* stream) {
  if (!rewards || !adv || n < 2 || n > 65536) return bad("srl_learner_reinforcepp");
  reinforcepp_kernel<<<1, kRedThreads, 0, (cudaStream_t)stream>>>(rewards, n, adv);
  return launch_rc("srl_learner_reinforcepp");
}

int32_t srl_learner_expand(const float* per_traj, const int64_t* tok_off, int32_t n, float* per_tok, void* stream) {
  if (!per_traj || !tok_off || !per_tok || n < 0) return bad("srl_learner_expand");
  if (n == 0) return 0;
  expand_kernel<<<n, 256, 0, (cudaStream_t)stream>>>(per_traj, tok_off, per_tok);
  return launch_rc("srl_learner_expand");
}

int32_t srl_learner_gae(const float* rewards, const float* values, const int64_t* tok_off, int32_t n, float gamma,
                        float lambda, float* adv, void* stream) {
  if (!rewards || !values || !tok_off || !adv || n < 0 || !(gamma >= 0.f && gamma <= 1.f) ||
      !(lambda >= 0.f && lambda <= 1.f))
    return bad("srl_learner_gae");
  if (n == 0) return 0;
  gae_kernel<<<n, kGaeThreads, 0, (cudaStream_t)stream>>>(rewards, values, tok_off, (double)gamma, (double)lambda, adv);
  return launch_rc("srl_learner_gae");
}

int64_t srl_learner_ppo_workspace(int64_t n) { return n < 0 ? -1 : (int64_t)kPpoBlocks * (int64_t)sizeof(double); }

int32_t srl_learner_ppo_objective(const float* new_lp, const float* old_lp, const float* adv, int64_t n,
                                  float eps_low, float eps_high, float* ratio, float* dterm, double* objective,
                                  void* workspace, void* stream) {
  if (!new_lp || !old_lp || !adv || !objective || !workspace || n < 0 || !(eps_low > 0.f) || !(eps_high > 0.f))
    return bad("srl_learner_ppo_objective");
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)workspace;
  ppo_kernel<<<kPpoBlocks, kPpoThreads, 0, st>>>(new_lp, old_lp, adv, n, 1.0 - (double)eps_low, 1.0 + (double)eps_high,
                                                 ratio, dterm, part);
  ppo_finish_kernel<<<1, 32, 0, st>>>(part, kPpoBlocks, n, objective);
  return launch_rc("srl_learner_ppo_objective");
}

int32_t srl_learner_staleness(const int32_t* versions, int64_t n, int32_t v_update, int32_t nbins, int32_t* hist,
                              void* stream) {
  if (!versions || !hist || n < 0 || nbins < 1) return bad("srl_learner_staleness");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(hist, 0, sizeof(int32_t) * nbins, st) != cudaSuccess) return launch_rc("srl_learner_staleness");
  if (n > 0) staleness_kernel<<<148 * 2, 256, 0, st>>>(versions, n, v_update, nbins, hist);
  return launch_rc("srl_learner_staleness");
}

}  // extern "C"
