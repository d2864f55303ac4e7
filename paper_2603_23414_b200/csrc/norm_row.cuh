// norm_row.cuh — the RMSNorm row arithmetic (DESIGN.md reading
// R19: n(x) = x * rsqrt(mean(x^2) + eps) * w in fp32, stored as bf16) of rmsnorm_kernel
// (layers.cu: 512 threads per row).  Written for any number of real threads per row
// (r02 also ran it as a 256-thread prologue inside the pair GEMM: measured slower,
// DESIGN.md §7, removed).
//
// One fixed order of fp32 operations, written with explicit _rn intrinsics (no FMA
// contraction left to the compiler), so every instantiation gives the same bits:
//   * 512 virtual threads; float4 i of the row belongs to virtual thread i % 512 and is
//     its (i / 512)-th element;
//   * x_i = x_res_i + (((p_0 + p_1) + p_2) + ...) over the split-K partials (split order),
//     or the embedding row (layer 0);
//   * a virtual thread's sum of squares: ss = fma(c, c, ss) over its elements in order,
//     components x, y, z, w;
//   * xor-shuffle tree 16, 8, 4, 2, 1 inside each 32-wide virtual warp, then the 16
//     virtual-warp sums added in warp order;
//   * inv = rsqrt(tot / d + eps);  y_i = bf16((x_i * inv) * w_i).
// A real thread hosts NV virtual threads t + j * (512 / NV), j < NV; real warp r then
// holds virtual warps r + j * (16 / NV) at the same lanes.
#pragma once
#include "common.cuh"
#include "layers.hpp"

namespace srl {

constexpr int kNormVT = 512;  // virtual threads per row
constexpr int kNormVec = 4;   // float4 per virtual thread: d <= 4 * 4 * 512 = 8192

struct NormRowArgs {
  float* x_res;                // [M][d] fp32 residual stream (updated when partials or embed are given)
  const int* row_tok;          // embed mode: token of each row
  const int* row_pos;          // [M] (< 0: inactive row -> zeros)
  const __nv_bfloat16* embed;  // nullable: layer-0 embedding gather
  const __nv_bfloat16* w;      // [d] norm weight
  float eps;
  __nv_bfloat16* y;            // [M][d] bf16 output (the next GEMM's operand)
  const float* part;           // nullable: nsplit fp32 partials [M][d], part_stride floats apart
  int nsplit;
  size_t part_stride;
  int d;
};

inline NormRowArgs norm_args(float* x_res, const int* row_tok, const int* row_pos, int d, const __nv_bfloat16* embed,
                             const __nv_bfloat16* w, float eps, __nv_bfloat16* y, const float* part, int nsplit,
                             size_t part_stride) {
  NormRowArgs a;
  a.x_res = x_res;
  a.row_tok = row_tok;
  a.row_pos = row_pos;
  a.embed = embed;
  a.w = w;
  a.eps = eps;
  a.y = y;
  a.part = nsplit > 1 ? part : nullptr;
  a.nsplit = nsplit > 1 ? nsplit : 0;
  a.part_stride = part_stride;
  a.d = d;
  return a;
}

// Row m by the real threads t in [0, 512 / NV); red: >= 16 floats of
// shared memory; sync(): a barrier over exactly these real threads.  VEC >= d / 2048
// float4 per virtual thread and MAXS >= nsplit bound the registers (compile time).
template <int NV, int VEC, int MAXS, typename Sync>
__device__ __forceinline__ void norm_row(const NormRowArgs& a, int m, int t, float* red, Sync sync) {
  constexpr int RT = kNormVT / NV;  // real threads
  const int d = a.d, nv = d >> 2;
  float* x = a.x_res + (size_t)m * d;
  const bool active = a.row_pos[m] >= 0;
  const __nv_bfloat16* e = a.embed ? a.embed + (size_t)(active ? a.row_tok[m] : 0) * d : nullptr;
  float4 v[NV][VEC];
  uint2 wr[NV][VEC];
  float ss[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    ss[j] = 0.f;
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const int i = t + j * RT + k * kNormVT;
      if (i < nv) {
        if (e) {
          const uint2 raw = __ldg(reinterpret_cast<const uint2*>(e) + i);
          v[j][k] = make_float4(bf16lo(raw.x), bf16hi(raw.x), bf16lo(raw.y), bf16hi(raw.y));
        } else {
          v[j][k] = reinterpret_cast<const float4*>(x)[i];
          if (a.part) {
            // every partial's load in flight before the adds (split order)
            float4 q[MAXS];
#pragma unroll
            for (int sp = 0; sp < MAXS; ++sp)
              if (sp < a.nsplit)
                q[sp] = __ldcg(reinterpret_cast<const float4*>(a.part + sp * a.part_stride + (size_t)m * d) + i);
            float4 acc = q[0];
#pragma unroll
            for (int sp = 1; sp < MAXS; ++sp)
              if (sp < a.nsplit) {
                acc.x = __fadd_rn(acc.x, q[sp].x);
                acc.y = __fadd_rn(acc.y, q[sp].y);
                acc.z = __fadd_rn(acc.z, q[sp].z);
                acc.w = __fadd_rn(acc.w, q[sp].w);
              }
            v[j][k].x = __fadd_rn(v[j][k].x, acc.x);
            v[j][k].y = __fadd_rn(v[j][k].y, acc.y);
            v[j][k].z = __fadd_rn(v[j][k].z, acc.z);
            v[j][k].w = __fadd_rn(v[j][k].w, acc.w);
          }
        }
        wr[j][k] = __ldg(reinterpret_cast<const uint2*>(a.w) + i);
      }
    }
  }
  // every load above is issued before the first store below (a store to x_res could
  // alias a later partial load, which would serialise the round trips)
#pragma unroll
  for (int j = 0; j < NV; ++j) {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const int i = t + j * RT + k * kNormVT;
      if (i < nv) {
        if (!active) v[j][k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e || a.part) reinterpret_cast<float4*>(x)[i] = v[j][k];
        ss[j] = __fmaf_rn(v[j][k].x, v[j][k].x, ss[j]);
        ss[j] = __fmaf_rn(v[j][k].y, v[j][k].y, ss[j]);
        ss[j] = __fmaf_rn(v[j][k].z, v[j][k].z, ss[j]);
        ss[j] = __fmaf_rn(v[j][k].w, v[j][k].w, ss[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NV; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss[j] = __fadd_rn(ss[j], __shfl_xor_sync(0xffffffffu, ss[j], o));
  }
  sync();  // the previous row's readers of red are done
  if ((t & 31) == 0) {
#pragma unroll
    for (int j = 0; j < NV; ++j) red[(t >> 5) + j * (RT / 32)] = ss[j];
  }
  sync();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < kNormVT / 32; ++i) tot = __fadd_rn(tot, red[i]);
  const float inv = active ? rsqrtf(__fadd_rn(__fdiv_rn(tot, (float)d), a.eps)) : 0.f;
  __nv_bfloat16* out = a.y + (size_t)m * d;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
      const int i = t + j * RT + k * kNormVT;
      if (i < nv) {
        const float4 s = v[j][k];
        uint2 o;
        o.x = pack_bf16(__fmul_rn(__fmul_rn(s.x, inv), bf16lo(wr[j][k].x)),
                        __fmul_rn(__fmul_rn(s.y, inv), bf16hi(wr[j][k].x)));
        o.y = pack_bf16(__fmul_rn(__fmul_rn(s.z, inv), bf16lo(wr[j][k].y)),
                        __fmul_rn(__fmul_rn(s.w, inv), bf16hi(wr[j][k].y)));
        reinterpret_cast<uint2*>(out)[i] = o;
      }
    }
  }
}

}  // namespace srl
