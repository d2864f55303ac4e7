// gumbel.cuh -- Philox4x32-10 and the RN-only msun logf behind the seeded
// Gumbel-max sampler (sampler.cu) and the LM-head GEMM's fused sampling
// epilogue (gemm_epi.cuh, EPI_SAMPLE).  One definition so both paths take the
// token decision with the same correctly rounded fp32 operations.
// The log_rn algorithm below follows FreeBSD msun e_logf.c, which carries:
//   Conversion to float by Ian Lance Taylor, Cygnus Support, ian@cygnus.com.
//   ====================================================
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this
//   software is freely granted, provided that this notice
//   is preserved.
//   ====================================================
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace srl {

static __device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// msun e_logf.c, transcribed with explicitly rounded fp32 operations.
static __device__ __noinline__ float log_rn(float x) {
  const float ln2_hi = __int_as_float(0x3f317180), ln2_lo = __int_as_float(0x3717f7d1);
  const float two25 = __int_as_float(0x4c000000);
  const float Lg1 = __int_as_float(0x3f2aaaaa), Lg2 = __int_as_float(0x3eccce13);
  const float Lg3 = __int_as_float(0x3e91e9ee), Lg4 = __int_as_float(0x3e789e26);
  const float third = __int_as_float(0x3eaaaaab);
  int ix = __float_as_int(x);
  int k = 0;
  if (ix < 0x00800000) {
    if ((ix & 0x7fffffff) == 0) return -INFINITY;
    if (ix < 0) return __int_as_float(0x7fc00000);
    k -= 25;
    x = __fmul_rn(x, two25);
    ix = __float_as_int(x);
  }
  if (ix >= 0x7f800000) return __fadd_rn(x, x);
  k += (ix >> 23) - 127;
  ix &= 0x007fffff;
  const int i = (ix + (0x95f64 << 3)) & 0x800000;
  x = __int_as_float(ix | (i ^ 0x3f800000));
  k += (i >> 23);
  const float f = __fsub_rn(x, 1.0f);
  const float dk = (float)k;
  if ((0x007fffff & (0x8000 + ix)) < 0xc000) {
    if (f == 0.0f) {
      if (k == 0) return 0.0f;
      return __fadd_rn(__fmul_rn(dk, ln2_hi), __fmul_rn(dk, ln2_lo));
    }
    const float R = __fmul_rn(__fmul_rn(f, f), __fsub_rn(0.5f, __fmul_rn(third, f)));
    if (k == 0) return __fsub_rn(f, R);
    return __fsub_rn(__fmul_rn(dk, ln2_hi), __fsub_rn(__fsub_rn(R, __fmul_rn(dk, ln2_lo)), f));
  }
  const float s = __fdiv_rn(f, __fadd_rn(2.0f, f));
  const float z = __fmul_rn(s, s);
  int i2 = ix - (0x6147a << 3);
  const float w = __fmul_rn(z, z);
  const int j = (0x6b851 << 3) - ix;
  const float t1 = __fmul_rn(w, __fadd_rn(Lg2, __fmul_rn(w, Lg4)));
  const float t2 = __fmul_rn(z, __fadd_rn(Lg1, __fmul_rn(w, Lg3)));
  i2 |= j;
  const float R = __fadd_rn(t2, t1);
  if (i2 > 0) {
    const float hfsq = __fmul_rn(__fmul_rn(0.5f, f), f);
    if (k == 0) return __fsub_rn(f, __fsub_rn(hfsq, __fmul_rn(s, __fadd_rn(hfsq, R))));
    return __fsub_rn(__fmul_rn(dk, ln2_hi),
                     __fsub_rn(__fsub_rn(hfsq, __fadd_rn(__fmul_rn(s, __fadd_rn(hfsq, R)), __fmul_rn(dk, ln2_lo))), f));
  }
  if (k == 0) return __fsub_rn(f, __fmul_rn(s, __fsub_rn(f, R)));
  return __fsub_rn(__fmul_rn(dk, ln2_hi), __fsub_rn(__fsub_rn(__fmul_rn(s, __fsub_rn(f, R)), __fmul_rn(dk, ln2_lo)), f));
}

static __device__ __forceinline__ float gumbel_from_bits(uint32_t x) {
  float u = __fmul_rn(__fadd_rn(__fmul_rn((float)(x >> 9), 2.0f), 1.0f), 5.9604644775390625e-08f);  // 2^-24
  return -log_rn(-log_rn(u));
}

// pruning bound (see sample_kernel): generous against the <= 1e-5 deviation
constexpr float kPrune = 1e-3f;
// The inner log needs CUDA's logf (<= 1 ulp): for u -> 1, t = -log u -> 6e-8 and an
// absolute-error log (__logf: 2^-21.4 on [0.5, 2]) would be far off exactly where the
// largest Gumbel values (the likely winners) are.  The outer one takes __logf (MUFU):
// |log t| <= 16.7, error <= 2^-21.4 absolute on [0.5, 2], <= 3 ulp elsewhere -- so
// |g_fast - g| < 1e-5 still (1 ulp of t -> 1.2e-7, + <= 5.7e-6), far inside kPrune.
static __device__ __forceinline__ float gumbel_fast(uint32_t x) {
  const float u = ((float)(x >> 9) * 2.0f + 1.0f) * 5.9604644775390625e-08f;  // exact (24-bit integer * 2^-24)
  return -__logf(-logf(u));
}

static __device__ __forceinline__ bool better(float s, int j, float bs, int bj) {
  return s > bs || (s == bs && j < bj);
}


}  // namespace srl
