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
  // the logits of the next group of 4 are loaded one iteration ahead (float4 when the
  // row is 16-byte aligned): their latency overlaps this group's Philox and logs
  // instead of stalling every iteration
  const bool vec = (a.V & 3) == 0;
  auto load4 = [&](int j4) -> float4 {
    if (vec && j4 + 3 < a.V) return __ldg(reinterpret_cast<const float4*>(z + j4));
    float t[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) t[q] = j4 + q < a.V ? __ldg(z + j4 + q) : 0.f;
    return make_float4(t[0], t[1], t[2], t[3]);
  };
  float4 znext = threadIdx.x * 4 < a.V ? load4(threadIdx.x * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j4 = threadIdx.x * 4; j4 < a.V; j4 += kSampThreads * 4) {
    const float4 zc = znext;
    if (j4 + kSampThreads * 4 < a.V) znext = load4(j4 + kSampThreads * 4);
    const float zv[4] = {zc.x, zc.y, zc.z, zc.w};
    const uint4 w = philox4x32_10(make_uint4((uint32_t)(j4 >> 2), n, traj, rs), key);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j4 + q;
      if (j < a.V) {
        const float zs = __fmul_rn(zv[q], invT);
        // Exact score only where it could win: g_fast (CUDA logf inside, __logf
        // outside: gumbel.cuh) is within 1e-5 of the RN msun value for u in [2^-24, 1 - 2^-24] (|g| <= 16.6),
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

// ---------------------------------------------------------------- top-k / top-p
// One CTA per row.  The truncation set (oracle/sampler.py truncation_set): rank by
// (scaled logit desc, index asc); keep the first top_k; of those, keep the shortest
// ranked prefix whose mass under the top-k softmax reaches top_p.  Found without a
// sort by MSB-first radix selection on the order-preserving key of the fp32 logit
// (4 passes of 8 bits): counts for top-k; for top-p, masses as fixed-point integers
// w_j = round(exp(zs_j - max) * 2^44) summed with integer atomics -- exact and
// order-free, so the decision is deterministic (it differs from the oracle's fp64
// cumulative sum only when the cut lands within ~1e-8 of top_p: tests/test_gpu_ops).
// Elements whose key equals the threshold are taken in index order (a small
// shared-memory list, bitonic-sorted; a serial scan if it overflows).  Then the
// Gumbel-max and the log-sum-exp run over the kept set only.
constexpr int kTrThreads = 1024;
constexpr int kTrEq = 2048;  // equal-key list capacity
constexpr double kTrScale = 17592186044416.0;  // 2^44

__device__ __forceinline__ uint32_t zkey(float f) {
  if (f == 0.f) f = 0.f;  // -0 ranks as +0
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

struct TrSel {  // kept iff key > t, or key == t and its index rank among the equal ones < n_eq
  uint32_t t;
  int n_eq;     // -1: nothing at the threshold is excluded (no cut)
  int eq_lim;   // index bound: equal-key elements with index < eq_lim are the kept ones
};

__device__ __forceinline__ bool tr_in(const TrSel& s, uint32_t u, int j) {
  return s.n_eq < 0 || u > s.t || (u == s.t && j < s.eq_lim);
}

// Index bound of the n smallest indices among elements with key == t that pass `pre`.
template <class Pre>
__device__ int tr_eq_limit(const float* z, int V, float invT, uint32_t t, int n, Pre pre, int* lst, int* cnt) {
  if (threadIdx.x == 0) *cnt = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const uint32_t u = zkey(__fmul_rn(z[j], invT));
    if (u == t && pre(u, j)) {
      const int at = atomicAdd(cnt, 1);
      if (at < kTrEq) lst[at] = j;
    }
  }
  __syncthreads();
  const int c = *cnt;
  int lim;
  if (c <= kTrEq) {
    int N = 1;
    while (N < c) N <<= 1;
    for (int i = c + threadIdx.x; i < N; i += blockDim.x) lst[i] = 0x7fffffff;
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1)
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
          const int ixj = i ^ jj;
          if (ixj > i) {
            const int x = lst[i], y = lst[ixj];
            if ((x > y) == ((i & k) == 0)) {
              lst[i] = y;
              lst[ixj] = x;
            }
          }
        }
        __syncthreads();
      }
    lim = n <= 0 ? 0 : (n >= c ? 0x7fffffff : lst[n - 1] + 1);
  } else {  // degenerate row (thousands of equal logits): serial scan in index order
    __shared__ int sh_lim;
    if (threadIdx.x == 0) {
      int seen = 0, l = 0x7fffffff;
      for (int j = 0; j < V && seen < n; ++j) {
        const uint32_t u = zkey(__fmul_rn(z[j], invT));
        if (u == t && pre(u, j) && ++seen == n) l = j + 1;
      }
      sh_lim = n <= 0 ? 0 : l;
    }
    __syncthreads();
    lim = sh_lim;
  }
  __syncthreads();
  return lim;
}

__global__ void __launch_bounds__(kTrThreads, 1) sample_trunc_kernel(SampleArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ unsigned long long hist[256];
  __shared__ int lst[kTrEq];
  __shared__ int cnt;
  __shared__ uint32_t sh_digit;
  __shared__ unsigned long long sh_rem;
  __shared__ float r_f[32], r_g[32], r_h[32];
  __shared__ int r_i[32];
  const int m = blockIdx.x;
  const int om = a.row_slot ? a.row_slot[m] : m;
  if (a.row_pos[m] < 0 || om < 0) {
    if (threadIdx.x == 0 && om >= 0) {
      a.tok_out[om] = -1;
      a.lp_out[om] = 0.f;
    }
    return;
  }
  const float* z = a.logits + (size_t)m * a.V;
  const int V = a.V;
  const float invT = a.invT;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // radix descent: the key t where the running total (count or mass, from the top,
  // over elements passing `pre`) first reaches `target`; returns t and the amount
  // strictly above it
  auto descend = [&](auto weight, auto pre, unsigned long long target, uint32_t* t_out,
                     unsigned long long* above_out) {
    uint32_t prefix = 0, mask = 0;
    unsigned long long above = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
      __syncthreads();
      for (int j = threadIdx.x; j < V; j += blockDim.x) {
        const float zs = __fmul_rn(z[j], invT);
        const uint32_t u = zkey(zs);
        if ((u & mask) == prefix && pre(u, j)) atomicAdd(&hist[(u >> shift) & 255u], weight(zs));
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long cum = above;
        int d = 0;
        for (int b = 255; b >= 0; --b) {
          if (cum + hist[b] >= target) {
            d = b;
            break;
          }
          cum += hist[b];
        }
        sh_digit = (uint32_t)d;
        sh_rem = cum;
      }
      __syncthreads();
      prefix |= sh_digit << shift;
      mask |= 255u << shift;
      above = sh_rem;
      __syncthreads();
    }
    *t_out = prefix;
    *above_out = above;
  };
  // block max of the scaled logits (the top key is always kept)
  float mx = -INFINITY;
  for (int j = threadIdx.x; j < V; j += blockDim.x) mx = fmaxf(mx, __fmul_rn(z[j], invT));
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) r_f[wid] = mx;
  __syncthreads();
  mx = r_f[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, r_f[i]);
  __syncthreads();
  const auto all = [](uint32_t, int) { return true; };
  // ---- top-k
  TrSel K{0u, -1, 0};
  if (a.top_k > 0 && a.top_k < V) {
    uint32_t t;
    unsigned long long above;
    descend([](float) { return 1ull; }, all, (unsigned long long)a.top_k, &t, &above);
    K.t = t;
    K.n_eq = (int)((unsigned long long)a.top_k - above);
    K.eq_lim = tr_eq_limit(z, V, invT, t, K.n_eq, all, lst, &cnt);
  }
  const auto inK = [&](uint32_t u, int j) { return tr_in(K, u, j); };
  // ---- top-p over the top-k set
  TrSel P{0u, -1, 0};
  if (a.top_p < 1.f) {
    const double m64 = (double)mx;
    const auto wq = [&](float zs) { return (unsigned long long)__double2ull_rn(exp((double)zs - m64) * kTrScale); };
    unsigned long long tot = 0;
    for (int j = threadIdx.x; j < V; j += blockDim.x) {
      const float zs = __fmul_rn(z[j], invT);
      if (inK(zkey(zs), j)) tot += wq(zs);
    }
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    __shared__ unsigned long long r_t[32];
    if (lane == 0) r_t[wid] = tot;
    __syncthreads();
    tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tot += r_t[i];
    __syncthreads();
    unsigned long long target = (unsigned long long)ceil((double)a.top_p * (double)tot);
    if (target < 1) target = 1;
    uint32_t t;
    unsigned long long above;
    descend(wq, inK, target, &t, &above);
    // every element at the threshold key has the same weight
    const float zt = __uint_as_float((t & 0x80000000u) ? (t & 0x7fffffffu) : ~t);
    const unsigned long long we = wq(zt);
    const unsigned long long need = target - above;
    P.t = t;
    P.n_eq = we == 0 ? 1 : (int)((need + we - 1) / we);
    P.eq_lim = tr_eq_limit(z, V, invT, t, P.n_eq, inK, lst, &cnt);
  }
  // ---- Gumbel-max + log-sum-exp over the kept set
  const uint32_t n = (uint32_t)a.row_n[m], traj = (uint32_t)a.row_traj[m], rs = (uint32_t)a.row_restarts[m];
  const uint2 key = make_uint2((uint32_t)(a.seed & 0xffffffffu), (uint32_t)(a.seed >> 32));
  float bs = -INFINITY, bz = 0.f, lmx = -INFINITY, sum = 0.f;
  int bj = 0x7fffffff;
  for (int j4 = threadIdx.x * 4; j4 < V; j4 += blockDim.x * 4) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)(j4 >> 2), n, traj, rs), key);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j4 + q;
      if (j >= V) break;
      const float zs = __fmul_rn(z[j], invT);
      const uint32_t u = zkey(zs);
      if (!inK(u, j) || !tr_in(P, u, j)) continue;
      const float s = __fadd_rn(zs, gumbel_from_bits(ws[q]));
      if (better(s, j, bs, bj)) {
        bs = s;
        bj = j;
        bz = zs;
      }
      if (zs > lmx) {
        sum = sum * __expf(lmx - zs) + 1.f;
        lmx = zs;
      } else {
        sum += __expf(zs - lmx);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float os = __shfl_xor_sync(0xffffffffu, bs, o);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    const float oz = __shfl_xor_sync(0xffffffffu, bz, o);
    if (better(os, oj, bs, bj)) {
      bs = os;
      bj = oj;
      bz = oz;
    }
    const float om_ = __shfl_xor_sync(0xffffffffu, lmx, o);
    const float osum = __shfl_xor_sync(0xffffffffu, sum, o);
    const float nm = fmaxf(lmx, om_);
    sum = (lmx == -INFINITY ? 0.f : sum * expf(lmx - nm)) + (om_ == -INFINITY ? 0.f : osum * expf(om_ - nm));
    lmx = nm;
  }
  if (lane == 0) {
    r_f[wid] = bs;
    r_i[wid] = bj;
    r_g[wid] = lmx;
    r_h[wid] = sum;
    lst[wid] = __float_as_int(bz);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      if (better(r_f[i], r_i[i], bs, bj)) {
        bs = r_f[i];
        bj = r_i[i];
        bz = __int_as_float(lst[i]);
      }
      const float nm = fmaxf(lmx, r_g[i]);
      sum = (lmx == -INFINITY ? 0.f : sum * expf(lmx - nm)) + (r_g[i] == -INFINITY ? 0.f : r_h[i] * expf(r_g[i] - nm));
      lmx = nm;
    }
    a.tok_out[om] = bj;
    a.lp_out[om] = bz - (lmx + logf(sum));
  }
}

void sample(const SampleArgs& a, cudaStream_t st) {
  if (a.M <= 0) return;
  if (a.top_k > 0 || a.top_p < 1.f)
    launch_k(sample_trunc_kernel, dim3(a.M), dim3(kTrThreads), 0, st, 1, a);
  else
    launch_k(sample_kernel, dim3(a.M), dim3(kSampThreads), 0, st, 1, a);
}

}  // namespace srl
