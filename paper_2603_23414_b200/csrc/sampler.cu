// sampler.cu — seeded Gumbel-max sampling + behaviour log-probability
// ("the exact log probability value that was
// used to generate each token").  One CTA per decode row streams the fp32
// logits row once:
//   u_j  = Philox4x32-10(key = seed; counter = (j>>2, n, traj, restarts))[j&3]
//          -> float(2*(x>>9)+1) * 2^-24
//   g_j  = -LOG(-LOG(u_j))   (msun e_logf algorithm, every op IEEE RN, no FMA)
//   tok  = argmax_j (z_j*invT + g_j), ties -> lowest j
//   lp   = z_tok*invT - (m + log sum_j exp(z_j*invT - m))
// The token decision is bit-reproducible against the CPU oracle because every
// operation on its path is a correctly rounded fp32 op (__fmul_rn/__fadd_rn/
// __fdiv_rn) in the order the algorithm states; candidates that provably lose
// (a cheap logf-based bound) skip the exact evaluation.  The logprob uses a
// parallel reduction and is compared with a tolerance (reading R15).
#include "common.cuh"
#include "launch.hpp"
#include "layers.hpp"

namespace srl {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
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
__device__ __noinline__ float log_rn(float x) {
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

__device__ __forceinline__ float gumbel_from_bits(uint32_t x) {
  float u = __fmul_rn(__fadd_rn(__fmul_rn((float)(x >> 9), 2.0f), 1.0f), 5.9604644775390625e-08f);  // 2^-24
  return -log_rn(-log_rn(u));
}

// pruning bound (see sample_kernel): generous against the <= 1e-5 deviation
constexpr float kPrune = 1e-3f;
__device__ __forceinline__ float gumbel_fast(uint32_t x) {
  const float u = ((float)(x >> 9) * 2.0f + 1.0f) * 5.9604644775390625e-08f;  // exact (24-bit integer * 2^-24)
  return -logf(-logf(u));
}

__device__ __forceinline__ bool better(float s, int j, float bs, int bj) {
  return s > bs || (s == bs && j < bj);
}

constexpr int kSampThreads = 512;

__global__ void __launch_bounds__(kSampThreads) sample_kernel(SampleArgs a) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const int om = a.row_slot ? a.row_slot[m] : m;  // where this row's sample goes
  if (a.row_pos[m] < 0 || om < 0) {
    if (threadIdx.x == 0 && om >= 0) {
      a.tok_out[om] = -1;
      a.lp_out[om] = 0.f;
    }
    return;
  }
  const float* z = a.logits + (size_t)m * a.V;
  const uint32_t n = (uint32_t)a.row_n[m], traj = (uint32_t)a.row_traj[m], rs = (uint32_t)a.row_restarts[m];
  const uint2 key = make_uint2((uint32_t)(a.seed & 0xffffffffu), (uint32_t)(a.seed >> 32));
  const float invT = a.invT;
  float bs = -INFINITY;
  int bj = 0x7fffffff;
  float mx = -INFINITY, sum = 0.f;
  for (int j4 = threadIdx.x * 4; j4 < a.V; j4 += kSampThreads * 4) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)(j4 >> 2), n, traj, rs), key);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j4 + q;
      if (j < a.V) {
        const float zs = __fmul_rn(z[j], invT);
        // Exact score only where it could win: g_fast (CUDA logf, <= 1 ulp each)
        // is within 1e-5 of the RN msun value for u in [2^-24, 1 - 2^-24] (|g| <= 16.6),
        // so zs + g_fast + kPrune < bs proves exact(s) < bs.  The decision is
        // unchanged; most of the V - 1 losers skip the two RN-only logs.
        if (__fadd_rn(zs, gumbel_fast(ws[q])) + kPrune + 1e-6f * fabsf(bs) >= bs) {
          const float s = __fadd_rn(zs, gumbel_from_bits(ws[q]));
          if (better(s, j, bs, bj)) {
            bs = s;
            bj = j;
          }
        }
        if (zs > mx) {
          sum = sum * expf(mx - zs) + 1.f;
          mx = zs;
        } else {
          sum += expf(zs - mx);
        }
      }
    }
  }
  // block reduction: argmax (s, j) and log-sum-exp (mx, sum)
  __shared__ float r_bs[32], r_mx[32], r_sum[32];
  __shared__ int r_bj[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float os = __shfl_xor_sync(0xffffffffu, bs, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (better(os, oj, bs, bj)) {
      bs = os;
      bj = oj;
    }
    const float om = __shfl_xor_sync(0xffffffffu, mx, o);
    const float osum = __shfl_xor_sync(0xffffffffu, sum, o);
    const float nm = fmaxf(mx, om);
    sum = (mx == -INFINITY ? 0.f : sum * expf(mx - nm)) + (om == -INFINITY ? 0.f : osum * expf(om - nm));
    mx = nm;
  }
  if (lane == 0) {
    r_bs[wid] = bs;
    r_bj[wid] = bj;
    r_mx[wid] = mx;
    r_sum[wid] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kSampThreads / 32; ++i) {
      if (better(r_bs[i], r_bj[i], bs, bj)) {
        bs = r_bs[i];
        bj = r_bj[i];
      }
      const float nm = fmaxf(mx, r_mx[i]);
      sum = (mx == -INFINITY ? 0.f : sum * expf(mx - nm)) + (r_mx[i] == -INFINITY ? 0.f : r_sum[i] * expf(r_mx[i] - nm));
      mx = nm;
    }
    a.tok_out[om] = bj;
    a.lp_out[om] = __fmul_rn(z[bj], invT) - (mx + logf(sum));
  }
}

void sample(const SampleArgs& a, cudaStream_t st) {
  if (a.M > 0) launch_k(sample_kernel, dim3(a.M), dim3(kSampThreads), 0, st, 1, a);
}

}  // namespace srl
