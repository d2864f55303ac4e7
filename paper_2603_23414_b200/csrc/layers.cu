// layers.cu — the row-wise steps of one decode layer around the fused
// tcgen05 GEMMs (SURVEY §8(a) rows a3 embedding, a4 RMSNorm).  Definition
// (reading R19): n(x) = x * rsqrt(mean(x^2) + eps) * w,
// computed in fp32 from the fp32 residual stream, written as bf16 (the GEMM
// operand).  The residual adds, SiLU-mul, bias + RoPE + KV append run inside
// the GEMM epilogues (gemm_tc.cu).
#include "common.cuh"
#include "launch.hpp"
#include "layers.hpp"
#include "norm_row.cuh"

namespace srl {

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

// ---------------------------------------------------------------- RMSNorm: one CTA per row
// x fp32 [M][d] (d % 4 == 0, d <= 8192), w bf16 [d] -> y bf16 [M][d]; when `embed` is
// set, x is first overwritten with the fp32 embedding row of row_tok[m] (layer 0).
// The row arithmetic (norm_row.cuh) is the one the pair GEMM's norm prologue runs, so
// both give the same bits.  Every load of the row is issued before the reduction
// (the kernel is latency-bound otherwise).
constexpr int kNormThreads = kNormVT;  // one virtual thread per real thread
template <int VEC, int MAXS>
__global__ void __launch_bounds__(kNormThreads, 2) rmsnorm_kernel(NormRowArgs a) {
  __shared__ float red[kNormVT / 32];
  pdl_trigger();
  pdl_wait();
  norm_row<1, VEC, MAXS>(a, blockIdx.x, threadIdx.x, red, [] { __syncthreads(); });
}

// ---------------------------------------------------------------- QKV finish
// The QKV projection's split-K partials (EPI_PARTIAL, [nsplit][M][N] fp32) summed in
// split order, + bias, RoPE on the q / k heads at the row's position (rotate_half
// pairs (i, i + dh/2)), then q -> q_out [M][Hq][dh] and k / v -> the row's KV page
// (page_table[slot][pos / 64], row pos % 64) -- the EPI_QKV epilogue, after the
// GEMM instead of inside it.  One CTA per row; thread t owns a (head, i < dh/2) pair.
__global__ void __launch_bounds__(256) qkv_finish_kernel(QkvFinishArgs a) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const int pos = a.row_pos[m];
  if (pos < 0) return;
  const int half = a.dh / 2, H = a.Hq + 2 * a.Hkv, N = H * a.dh;
  const int page = a.page_table[(size_t)a.row_slot[m] * a.max_pages + pos / 64];
  const int quads = half / 4;  // 4 consecutive rotary pairs per thread step (vector loads)
  for (int t = threadIdx.x; t < H * quads; t += blockDim.x) {
    const int h = t / quads, i = (t % quads) * 4;
    const int n0 = h * a.dh + i, n1 = n0 + half;
    float4 q0[4], q1[4];
#pragma unroll
    for (int sp = 0; sp < 4; ++sp) {  // <= 4 splits, every load in flight before the adds
      const float* pp = a.part + sp * a.part_stride + (size_t)m * N;
      q0[sp] = sp < a.nsplit ? __ldcg(reinterpret_cast<const float4*>(pp + n0)) : make_float4(0.f, 0.f, 0.f, 0.f);
      q1[sp] = sp < a.nsplit ? __ldcg(reinterpret_cast<const float4*>(pp + n1)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float x0[4] = {q0[0].x, q0[0].y, q0[0].z, q0[0].w}, x1[4] = {q1[0].x, q1[0].y, q1[0].z, q1[0].w};
#pragma unroll
    for (int sp = 1; sp < 4; ++sp)
      if (sp < a.nsplit) {
        x0[0] += q0[sp].x; x0[1] += q0[sp].y; x0[2] += q0[sp].z; x0[3] += q0[sp].w;
        x1[0] += q1[sp].x; x1[1] += q1[sp].y; x1[2] += q1[sp].z; x1[3] += q1[sp].w;
      }
    if (a.bias) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x0[k] += __bfloat162float(a.bias[n0 + k]);
        x1[k] += __bfloat162float(a.bias[n1 + k]);
      }
    }
    float y0[4], y1[4];
    if (h < a.Hq + a.Hkv) {
      const float4 c = __ldg(reinterpret_cast<const float4*>(a.rope_cos + (size_t)pos * half + i));
      const float4 sn = __ldg(reinterpret_cast<const float4*>(a.rope_sin + (size_t)pos * half + i));
      const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {sn.x, sn.y, sn.z, sn.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        y0[k] = x0[k] * cc[k] - x1[k] * ss[k];
        y1[k] = x1[k] * cc[k] + x0[k] * ss[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        y0[k] = x0[k];
        y1[k] = x1[k];
      }
    }
    size_t off;
    void* base;
    if (h < a.Hq) {
      off = ((size_t)m * a.Hq + h) * a.dh;
      base = a.q_out;
    } else {
      const int kvh = h < a.Hq + a.Hkv ? h - a.Hq : h - a.Hq - a.Hkv;
      off = (((size_t)page * a.Hkv + kvh) * 64 + pos % 64) * a.dh;
      base = h < a.Hq + a.Hkv ? a.k_pool : a.v_pool;
    }
    if (a.kv_f32) {
      float* b = reinterpret_cast<float*>(base) + off;
      *reinterpret_cast<float4*>(b + i) = make_float4(y0[0], y0[1], y0[2], y0[3]);
      *reinterpret_cast<float4*>(b + i + half) = make_float4(y1[0], y1[1], y1[2], y1[3]);
    } else {
      __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(base) + off;
      *reinterpret_cast<uint2*>(b + i) = make_uint2(pack_bf16(y0[0], y0[1]), pack_bf16(y0[2], y0[3]));
      *reinterpret_cast<uint2*>(b + i + half) = make_uint2(pack_bf16(y1[0], y1[1]), pack_bf16(y1[2], y1[3]));
    }
  }
}

void qkv_finish(const QkvFinishArgs& a, int M, cudaStream_t st) {
  if (M > 0) launch_k(qkv_finish_kernel, dim3(M), dim3(256), 0, st, 1, a);
}

void rmsnorm(float* x_res, const int* row_tok, const int* row_pos, int M, int d, const __nv_bfloat16* embed,
             const __nv_bfloat16* w, float eps, __nv_bfloat16* y, cudaStream_t st, const float* part, int nsplit,
             size_t part_stride) {
  rmsnorm(norm_args(x_res, row_tok, row_pos, d, embed, w, eps, y, part, nsplit, part_stride), M, st);
}
void rmsnorm(const NormRowArgs& a, int M, cudaStream_t st) {
  if (M <= 0) return;
  if (a.d <= 4 * 2 * kNormVT && a.nsplit <= 4)  // the 8B decode shapes
    launch_k(rmsnorm_kernel<2, 4>, dim3(M), dim3(kNormThreads), 0, st, 1, a);
  else if (a.d <= 4 * 3 * kNormVT && a.nsplit <= 4)  // the 32B width (d = 5120)
    launch_k(rmsnorm_kernel<3, 4>, dim3(M), dim3(kNormThreads), 0, st, 1, a);
  else
    launch_k(rmsnorm_kernel<kNormVec, kNormMaxSplits>, dim3(M), dim3(kNormThreads), 0, st, 1, a);
}

}  // namespace srl
