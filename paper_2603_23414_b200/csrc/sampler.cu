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
#include "gumbel.cuh"
#include "launch.hpp"
#include "layers.hpp"

namespace srl {

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
          sum = sum * __expf(mx - zs) + 1.f;
          mx = zs;
        } else {
          sum += __expf(zs - mx);
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

// one CTA per row: the vocab-block partials in block order (ties -> lowest index is
// order-free; the LSE is combined in a fixed order: deterministic)
constexpr int kRedThreads = 256;
__global__ void __launch_bounds__(kRedThreads) sample_reduce_kernel(SampleArgs a, const float4* __restrict__ part,
                                                                    const int* __restrict__ part_j, int nblk) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x;
  const int om = a.row_slot ? a.row_slot[m] : m;
  if (a.row_pos[m] < 0 || om < 0) return;
  float bs = -INFINITY, bz = 0.f, mx = -INFINITY, sum = 0.f;
  int bj = 0x7fffffff;
  auto merge = [&](float os, int oj, float oz, float om_, float osum) {
    if (better(os, oj, bs, bj)) {
      bs = os;
      bj = oj;
      bz = oz;
    }
    const float nm = fmaxf(mx, om_);
    sum = (mx == -INFINITY ? 0.f : sum * expf(mx - nm)) + (om_ == -INFINITY ? 0.f : osum * expf(om_ - nm));
    mx = nm;
  };
  for (int b = threadIdx.x; b < nblk; b += kRedThreads) {
    const float4 v = part[(size_t)m * nblk + b];
    merge(v.x, part_j[(size_t)m * nblk + b], v.y, v.z, v.w);
  }
  __shared__ float r_bs[kRedThreads / 32], r_bz[kRedThreads / 32], r_mx[kRedThreads / 32], r_sum[kRedThreads / 32];
  __shared__ int r_bj[kRedThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const float os = __shfl_xor_sync(0xffffffffu, bs, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    const float oz = __shfl_xor_sync(0xffffffffu, bz, o);
    const float om_ = __shfl_xor_sync(0xffffffffu, mx, o);
    const float osum = __shfl_xor_sync(0xffffffffu, sum, o);
    merge(os, oj, oz, om_, osum);
  }
  if (lane == 0) {
    r_bs[wid] = bs;
    r_bj[wid] = bj;
    r_bz[wid] = bz;
    r_mx[wid] = mx;
    r_sum[wid] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kRedThreads / 32; ++i) merge(r_bs[i], r_bj[i], r_bz[i], r_mx[i], r_sum[i]);
    a.tok_out[om] = bj;
    a.lp_out[om] = __fmul_rn(bz, a.invT) - (mx + logf(sum));
  }
}

void sample_reduce(const SampleArgs& a, const float4* part, const int* part_j, int nblk, cudaStream_t st) {
  if (a.M > 0) launch_k(sample_reduce_kernel, dim3(a.M), dim3(kRedThreads), 0, st, 1, a, part, part_j, nblk);
}

void sample(const SampleArgs& a, cudaStream_t st) {
  if (a.M > 0) launch_k(sample_kernel, dim3(a.M), dim3(kSampThreads), 0, st, 1, a);
}

}  // namespace srl
