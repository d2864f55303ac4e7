// layers.cu — the element-wise / row-wise steps of one decode layer that sit
// around the tcgen05 GEMMs (SURVEY §8(a) rows a3, a4, a5 epilogue, a7/a9
// residual, a8 SiLU-mul).  Definitions: DESIGN.md "Model" (LLaMA / Qwen
// pre-norm block, reading R19):
//   n(x) = x * rsqrt(mean(x^2) + eps) * w
//   RoPE rotate_half: (x_i, x_{i+dh/2}) -> (x_i c - x_{i+dh/2} s, x_{i+dh/2} c + x_i s),
//   angle = pos * theta^(-2i/dh)
// The K-split partial sums of the GEMM are reduced here in split order, so
// every output is bit-reproducible.
#include "common.cuh"
#include "layers.hpp"

namespace srl {

__device__ __forceinline__ float block_reduce_sum(float v) {
  __shared__ float red[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// ---------------------------------------------------------------- RoPE table (fp64 -> fp32)
__global__ void rope_table_kernel(float* cos_t, float* sin_t, int max_pos, int half, int dh, double theta) {
  const long long n = (long long)max_pos * half;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int pos = (int)(i / half), j = (int)(i % half);
    const double ang = (double)pos * pow(theta, -2.0 * (double)j / (double)dh);
    cos_t[i] = (float)cos(ang);
    sin_t[i] = (float)sin(ang);
  }
}

void rope_table(float* cos_t, float* sin_t, int max_pos, int dh, double theta, cudaStream_t st) {
  rope_table_kernel<<<296, 256, 0, st>>>(cos_t, sin_t, max_pos, dh / 2, dh, theta);
}

// ---------------------------------------------------------------- embedding + first RMSNorm
__global__ void embed_norm_kernel(const int* __restrict__ row_tok, const int* __restrict__ row_pos, int d,
                                  const __nv_bfloat16* __restrict__ embed, const __nv_bfloat16* __restrict__ w,
                                  float eps, float* __restrict__ x_res, __nv_bfloat16* __restrict__ xn) {
  const int m = blockIdx.x;
  float* x = x_res + (size_t)m * d;
  __nv_bfloat16* y = xn + (size_t)m * d;
  const bool active = row_pos[m] >= 0;
  const __nv_bfloat16* e = embed + (size_t)(active ? row_tok[m] : 0) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const float v = active ? __bfloat162float(e[i]) : 0.f;
    x[i] = v;
    ss += v * v;
  }
  ss = block_reduce_sum(ss);
  const float inv = rsqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    y[i] = __float2bfloat16(active ? x[i] * inv * __bfloat162float(w[i]) : 0.f);
}

void embed_norm(const int* row_tok, const int* row_pos, int M, int d, const __nv_bfloat16* embed,
                const __nv_bfloat16* w, float eps, float* x_res, __nv_bfloat16* xn, cudaStream_t st) {
  if (M > 0) embed_norm_kernel<<<M, 256, 0, st>>>(row_tok, row_pos, d, embed, w, eps, x_res, xn);
}

// ---------------------------------------------------------------- residual add + next RMSNorm
__global__ void resid_norm_kernel(const float* __restrict__ P, int S, int M, int d, const int* __restrict__ row_pos,
                                  float* __restrict__ x_res, const __nv_bfloat16* __restrict__ w, float eps,
                                  __nv_bfloat16* __restrict__ xn) {
  const int m = blockIdx.x;
  float* x = x_res + (size_t)m * d;
  __nv_bfloat16* y = xn + (size_t)m * d;
  const bool active = row_pos[m] >= 0;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < S; ++s) acc += P[((size_t)s * M + m) * d + i];
    const float v = active ? x[i] + acc : 0.f;
    x[i] = v;
    ss += v * v;
  }
  ss = block_reduce_sum(ss);
  const float inv = rsqrtf(ss / (float)d + eps);
  for (int i = threadIdx.x; i < d; i += blockDim.x)
    y[i] = __float2bfloat16(active ? x[i] * inv * __bfloat162float(w[i]) : 0.f);
}

void resid_norm(const float* P, int S, int M, int d, const int* row_pos, float* x_res, const __nv_bfloat16* w,
                float eps, __nv_bfloat16* xn, cudaStream_t st) {
  if (M > 0) resid_norm_kernel<<<M, 256, 0, st>>>(P, S, M, d, row_pos, x_res, w, eps, xn);
}

// ---------------------------------------------------------------- SiLU(gate) * up
__global__ void silu_mul_kernel(const float* __restrict__ P, int S, int M, int ff, __nv_bfloat16* __restrict__ act) {
  const long long n = (long long)M * ff;
  const long long N2 = 2LL * ff;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long m = i / ff, j = i % ff;
    float g = 0.f, u = 0.f;
    for (int s = 0; s < S; ++s) {
      const float* row = P + ((size_t)s * M + m) * N2;
      g += row[j];
      u += row[ff + j];
    }
    act[i] = __float2bfloat16(g / (1.f + expf(-g)) * u);
  }
}

void silu_mul(const float* P, int S, int M, int ff, __nv_bfloat16* act, cudaStream_t st) {
  if (M > 0) silu_mul_kernel<<<148 * 8, 256, 0, st>>>(P, S, M, ff, act);
}

// ---------------------------------------------------------------- split reduction (fp32 out)
__global__ void reduce_splits_kernel(const float* __restrict__ P, int S, long long n, float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float a = 0.f;
    for (int s = 0; s < S; ++s) a += P[(size_t)s * n + i];
    out[i] = a;
  }
}

void reduce_splits(const float* P, int S, long long n, float* out, cudaStream_t st) {
  if (n > 0) reduce_splits_kernel<<<148 * 4, 256, 0, st>>>(P, S, n, out);
}

// ---------------------------------------------------------------- QKV epilogue: bias + RoPE + KV append
template <typename KV, typename QT>
__global__ void qkv_epi_kernel(QkvEpiArgs a) {
  const int m = blockIdx.x;
  const int pos = a.row_pos[m];
  if (pos < 0) return;
  const int slot = a.row_slot[m];
  const int half = a.dh / 2;
  const int N = (a.Hq + 2 * a.Hkv) * a.dh;
  const int page = a.page_table[(size_t)slot * a.max_pages + pos / 64];
  const int prow = pos % 64;
  const float* cs = a.rope_cos + (size_t)pos * half;
  const float* sn = a.rope_sin + (size_t)pos * half;
  KV* kp = reinterpret_cast<KV*>(a.k_pool);
  KV* vp = reinterpret_cast<KV*>(a.v_pool);
  QT* qo = reinterpret_cast<QT*>(a.q_out) + (size_t)m * a.Hq * a.dh;
  auto val = [&](int n) {
    float acc = 0.f;
    for (int s = 0; s < a.S; ++s) acc += a.P[((size_t)s * a.M + m) * N + n];
    if (a.bias) acc += __bfloat162float(a.bias[n]);
    return acc;
  };
  const int n_rope = (a.Hq + a.Hkv) * half;  // rotated pairs (q heads then k heads)
  for (int i = threadIdx.x; i < n_rope + a.Hkv * a.dh; i += blockDim.x) {
    if (i < n_rope) {
      const int h = i / half, j = i % half;
      const int n0 = h * a.dh + j;
      const float x0 = val(n0), x1 = val(n0 + half);
      const float c = cs[j], s = sn[j];
      const float y0 = x0 * c - x1 * s, y1 = x1 * c + x0 * s;
      if (h < a.Hq) {
        qo[h * a.dh + j] = (QT)y0;
        qo[h * a.dh + j + half] = (QT)y1;
      } else {
        const int kh = h - a.Hq;
        const size_t base = (((size_t)page * a.Hkv + kh) * 64 + prow) * a.dh;
        kp[base + j] = (KV)y0;
        kp[base + j + half] = (KV)y1;
      }
    } else {
      const int i2 = i - n_rope;
      const int vh = i2 / a.dh, dd = i2 % a.dh;
      const float x = val((a.Hq + a.Hkv) * a.dh + i2);
      vp[(((size_t)page * a.Hkv + vh) * 64 + prow) * a.dh + dd] = (KV)x;
    }
  }
}

void qkv_epilogue(const QkvEpiArgs& a, bool kv_fp32, cudaStream_t st) {
  if (a.M <= 0) return;
  if (kv_fp32)
    qkv_epi_kernel<float, float><<<a.M, 256, 0, st>>>(a);
  else
    qkv_epi_kernel<__nv_bfloat16, __nv_bfloat16><<<a.M, 256, 0, st>>>(a);
}

}  // namespace srl
