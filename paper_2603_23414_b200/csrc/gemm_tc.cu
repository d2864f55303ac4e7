// gemm_tc.cu — weight-streaming decode GEMM on tcgen05 tensor cores (sm_100a)
// with fused epilogues and a deterministic stream-K fixup.
//
// Computes Y[m][n] = sum_k X[m][k] * W[n][k] for the projection / MLP /
// LM-head contractions of the decode step (SURVEY §8(a) rows a5, a7, a8, a9,
// a10; "throughput is primarily constrained by limited HBM
// bandwidth, due to frequent loading of model weights") and applies the
// consumer op in the epilogue:
//   EPI_F32   out[m][n] = Y                            (LM-head logits, op tests)
//   EPI_RESID x_res[m][n] += Y                          (O and down projections)
//   EPI_SILU  act[m][j] = silu(Yg[m][j]) * Yu[m][j]     (gate/up: the CTA owns the
//             gate tile j and the up tile ff+j, two TMEM accumulators)
//   EPI_QKV   (+bias), RoPE on q/k at the row's position, q -> q buffer, k/v ->
//             the paged KV cache (page_table[slot][pos/64], row pos%64)
//
// Swap-AB: 128 weight rows are the UMMA M side, the ragged decode batch
// (M_b <= 256 rows, multiple of 16) is the UMMA N side; the fp32 accumulator
// (128 lanes x M_b columns per weight tile) lives in TMEM.
// Persistent stream-K: the linear space (work unit, k-block) is cut into one
// contiguous range per CTA (grid = #SMs), so every SM streams the same number
// of weight bytes.  A unit whose k-range is split across CTAs is finished by
// the last arriving CTA, which sums the partials in CTA order (fixed order ->
// bit-reproducible) and runs the epilogue; nothing else is ever atomically
// accumulated.  Warp roles: w0 TMA producer, w1 TMEM allocator + MMA issuer,
// w2..w5 epilogue (tcgen05.ld -> fused op -> coalesced stores).  For one-tile
// units the TMEM accumulator is double-buffered so the epilogue of a segment
// overlaps the MMAs of the next.
#include "common.cuh"
#include "kernels.hpp"
#include "tma.hpp"

namespace srl {

struct GemmParams {
  int M, N, K;
  int m_blk, m_blocks, n_tiles, nt, tile2_off, kb;
  long long total;  // units * kb
  int stages, xstages, tmem_cols, acc_stages;
  int w_blocked;    // W stored tile-blocked: [N/128][K/64][128][64] (each TMA box contiguous)
  float* ws;        // [grid][2][nt][m_blk][128]
  int* counters;    // [units]
  GemmEpi epi;
  unsigned long long* dbg;  // optional [grid][16] globaltimer stamps (profiling builds)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DBG(slot)                                                  \
  do {                                                             \
    if (p.dbg) p.dbg[(size_t)blockIdx.x * 16 + (slot)] = gtimer(); \
  } while (0)

static constexpr int kStageA = 128 * 128;  // 128 weight rows x 64 bf16 (128 B)
static constexpr int kEpiThreads = 128;

__host__ __device__ __forceinline__ long long cta_start(long long total, int G, int c) {
  return (long long)c * total / G;
}
// CTA whose range contains linear index i
__host__ __device__ __forceinline__ int cta_of(long long i, long long total, int G) {
  int c = (int)((i * G) / total);
  while (c + 1 < G && cta_start(total, G, c + 1) <= i) ++c;
  while (c > 0 && cta_start(total, G, c) > i) --c;
  return c;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads)); }

// ---------------------------------------------------------------- fused epilogue
// v[t][j]: value of weight row (tile t, lane n) for batch row m0 + j, j < 16.
// xch: smem exchange buffer [128][17] (QKV only).
template <int NT>
__device__ __forceinline__ void apply_epilogue(const GemmParams& p, int unit_n0, int n, int m0, float (&v)[NT][16],
                                               float* xch) {
  const GemmEpi& e = p.epi;
  const int ng = unit_n0 + n;
  switch (e.kind) {
    case EPI_F32: {
      if (ng < p.N)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = m0 + j;
          if (m < p.M) e.out_f32[(size_t)m * e.ldo + ng] = v[0][j];
        }
      break;
    }
    case EPI_RESID: {
      // exactly one contribution per element per launch: a fire-and-forget
      // reduction (RED) is order-independent here and hides the read latency
      if (ng < p.N)
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = m0 + j;
          if (m < p.M) atomicAdd(e.x_res + (size_t)m * e.ldo + ng, v[0][j]);
        }
      break;
    }
    case EPI_SILU: {
      if (NT == 2) {  // gate tile / up tile held by the same thread
        if (ng < p.N)
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = m0 + j;
            if (m < p.M) {
              const float g = v[0][j], u = v[NT - 1][j];
              e.act[(size_t)m * e.ldo + ng] = __float2bfloat16(g / (1.f + expf(-g)) * u);
            }
          }
      } else {
        // 64-row interleave: tile rows [0,64) are gate rows, [64,128) the up rows of
        // the same 64 outputs; meet through shared memory, split columns 8/8
#pragma unroll
        for (int j = 0; j < 16; ++j) xch[n * 17 + j] = v[0][j];
        epi_bar();
        const int o = n & 63;                      // output within the tile
        const int out = (unit_n0 >> 1) + o;        // global output index
        const int jb = n < 64 ? 0 : 8;
        if (unit_n0 + o < p.N) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int j = jb + jj;
            const int m = m0 + j;
            if (m < p.M) {
              const float g = xch[o * 17 + j], u = xch[(o + 64) * 17 + j];
              e.act[(size_t)m * e.ldo + out] = __float2bfloat16(g / (1.f + expf(-g)) * u);
            }
          }
        }
        epi_bar();
      }
      break;
    }
    case EPI_QKV: {
      // exchange the 128 x 16 tile through shared memory so RoPE pairs meet;
      // the chunk's 16 (position, KV page) pairs are looked up once into smem
      int* spos = reinterpret_cast<int*>(xch + 128 * 17);
      int* spage = spos + 16;
#pragma unroll
      for (int j = 0; j < 16; ++j) xch[n * 17 + j] = v[0][j];
      if (n < 16) {
        const int m = m0 + n;
        const int pos = m < p.M ? __ldg(e.row_pos + m) : -1;
        spos[n] = pos;
        spage[n] = pos >= 0 ? __ldg(e.page_table + (size_t)__ldg(e.row_slot + m) * e.max_pages + pos / 64) : 0;
      }
      epi_bar();
      const int dh = e.dh, half = dh / 2;
      const int qd = e.Hq * dh, kd = e.Hkv * dh;
      const int i = ng % dh;            // dim within the head
      const int h = ng / dh;            // head index in [q heads | k heads | v heads]
      if (ng < qd + kd) {
        // rope pair (lo, lo+half); the lo-thread does columns 0..7, the hi-thread 8..15
        const int lo = i < half ? i : i - half;
        const int nlo = n - (i - lo), nhi = nlo + half;
        const int jb = i < half ? 0 : 8;
        const float blo = e.bias ? __bfloat162float(e.bias[ng - (i - lo)]) : 0.f;
        const float bhi = e.bias ? __bfloat162float(e.bias[ng - (i - lo) + half]) : 0.f;
        float cv[8], sv[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int pos = spos[jb + jj];
          cv[jj] = pos >= 0 ? __ldg(e.rope_cos + (size_t)pos * half + lo) : 0.f;
          sv[jj] = pos >= 0 ? __ldg(e.rope_sin + (size_t)pos * half + lo) : 0.f;
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = jb + jj;
          const int m = m0 + j;
          const int pos = spos[j];
          if (pos < 0) continue;
          const float x0 = xch[nlo * 17 + j] + blo, x1 = xch[nhi * 17 + j] + bhi;
          const float c = cv[jj], s = sv[jj];
          const float y0 = x0 * c - x1 * s, y1 = x1 * c + x0 * s;
          if (h < e.Hq) {
            const size_t qo = ((size_t)m * e.Hq + h) * dh;
            if (e.kv_f32) {
              float* q = reinterpret_cast<float*>(e.q_out);
              q[qo + lo] = y0;
              q[qo + lo + half] = y1;
            } else {
              __nv_bfloat16* q = reinterpret_cast<__nv_bfloat16*>(e.q_out);
              q[qo + lo] = __float2bfloat16(y0);
              q[qo + lo + half] = __float2bfloat16(y1);
            }
          } else {
            const int kh = h - e.Hq;
            const int page = spage[j];
            const size_t ko = (((size_t)page * e.Hkv + kh) * 64 + pos % 64) * dh;
            if (e.kv_f32) {
              float* k = reinterpret_cast<float*>(e.k_pool);
              k[ko + lo] = y0;
              k[ko + lo + half] = y1;
            } else {
              __nv_bfloat16* k = reinterpret_cast<__nv_bfloat16*>(e.k_pool);
              k[ko + lo] = __float2bfloat16(y0);
              k[ko + lo + half] = __float2bfloat16(y1);
            }
          }
        }
      } else if (ng < p.N) {
        const int vh = h - e.Hq - e.Hkv;
        const float b = e.bias ? __bfloat162float(e.bias[ng]) : 0.f;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int pos = spos[j];
          if (pos < 0) continue;
          const int page = spage[j];
          const size_t vo = (((size_t)page * e.Hkv + vh) * 64 + pos % 64) * dh + i;
          if (e.kv_f32)
            reinterpret_cast<float*>(e.v_pool)[vo] = xch[n * 17 + j] + b;
          else
            reinterpret_cast<__nv_bfloat16*>(e.v_pool)[vo] = __float2bfloat16(xch[n * 17 + j] + b);
        }
      }
      epi_bar();
      break;
    }
  }
}

// ---------------------------------------------------------------- kernel
// Warp roles: w0 weight (W) TMA producer, w6 activation (X) TMA producer, w1 TMEM
// allocator + MMA issuer, w2..w5 epilogue.  W and X have separate smem rings:
// the weights stream from HBM and need a deep ring, the activation k-slices are
// L2-resident and only need a short one.
constexpr int kGemmThreads = 224;

template <int NT>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                        GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_a = NT * kStageA;
  const int stage_b = p.m_blk * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + p.stages * stage_a;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + p.xstages * stage_b);
  uint64_t* empty = full + p.stages;
  uint64_t* xfull = empty + p.stages;
  uint64_t* xempty = xfull + p.xstages;
  uint64_t* tfull = xempty + p.xstages;  // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tholder = reinterpret_cast<uint32_t*>(tempty + 2);
  int* sh_flag = reinterpret_cast<int*>(tholder + 1);
  float* xch = reinterpret_cast<float*>(sh_flag + 4);  // [128][17]

  const int G = gridDim.x, c = blockIdx.x;
  const long long r0 = cta_start(p.total, G, c), r1 = cta_start(p.total, G, c + 1);
  const int w = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    DBG(0);
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < p.xstages; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
  }
  if (w == 1) tmem_alloc(tholder, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tholder;
  if (threadIdx.x == 0) DBG(1);
  if (r0 >= r1) {  // empty range
    tc_fence_before();
    __syncthreads();
    if (w == 1) tmem_dealloc(tbase, p.tmem_cols);
    return;
  }
  const int u_first = (int)(r0 / p.kb), u_last = (int)((r1 - 1) / p.kb);

  if (w == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
      int q = 0;
      for (int u = u_first; u <= u_last; ++u) {
        const long long ub = (long long)u * p.kb;
        const int k0 = (int)((r0 > ub ? r0 : ub) - ub), k1 = (int)((r1 < ub + p.kb ? r1 : ub + p.kb) - ub);
        const int t = u % p.n_tiles;
        for (int k = k0; k < k1; ++k, ++q) {
          const int s = q % p.stages;
          const uint32_t ph = (q / p.stages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], stage_a);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            if (p.w_blocked)
              tma_load_2d_hint(sA + s * stage_a + j * kStageA, &tmW, &full[s], 0, (t * p.kb + k) * 128, pol_w);
            else
              tma_load_2d_hint(sA + s * stage_a + j * kStageA, &tmW, &full[s], k * 64, t * 128 + j * p.tile2_off,
                               pol_w);
          }
          if (q == 0) DBG(2);
        }
      }
      DBG(3);
    }
  } else if (w == 6) {
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_last();  // activations: re-read by every tile
      int q = 0;
      for (int u = u_first; u <= u_last; ++u) {
        const long long ub = (long long)u * p.kb;
        const int k0 = (int)((r0 > ub ? r0 : ub) - ub), k1 = (int)((r1 < ub + p.kb ? r1 : ub + p.kb) - ub);
        const int mb = u / p.n_tiles;
        for (int k = k0; k < k1; ++k, ++q) {
          const int s = q % p.xstages;
          const uint32_t ph = (q / p.xstages) & 1;
          mbar_wait(&xempty[s], ph ^ 1);
          mbar_arrive_expect_tx(&xfull[s], stage_b);
          tma_load_2d_hint(sB + s * stage_b, &tmX, &xfull[s], k * 64, mb * p.m_blk, pol_x);
        }
      }
    }
  } else if (w == 1) {
    if (lane == 0) {
      int q = 0, seg = 0;
      for (int u = u_first; u <= u_last; ++u, ++seg) {
        const long long ub = (long long)u * p.kb;
        const int k0 = (int)((r0 > ub ? r0 : ub) - ub), k1 = (int)((r1 < ub + p.kb ? r1 : ub + p.kb) - ub);
        const int mb = u / p.n_tiles;
        int nmma = p.M - mb * p.m_blk;
        nmma = nmma > p.m_blk ? p.m_blk : nmma;
        nmma = (nmma + 15) & ~15;
        const uint32_t idesc = umma_idesc_bf16(128, nmma);
        const int a = seg % p.acc_stages;
        const uint32_t aph = (seg / p.acc_stages) & 1;
        mbar_wait(&tempty[a], aph ^ 1);
        tc_fence_after();
        for (int k = k0; k < k1; ++k, ++q) {
          const int s = q % p.stages;
          const uint32_t ph = (q / p.stages) & 1;
          const int sx = q % p.xstages;
          const uint32_t phx = (q / p.xstages) & 1;
          mbar_wait(&full[s], ph);
          mbar_wait(&xfull[sx], phx);
          tc_fence_after();
          if (q == 0) DBG(4);
          const uint32_t b = smem_u32(sB + sx * stage_b);
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            const uint32_t aa = smem_u32(sA + s * stage_a + j * kStageA);
            const uint32_t tacc = tbase + (uint32_t)((a * NT + j) * p.m_blk);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc_mma_bf16(tacc, umma_desc_sw128(aa + kk * 32), umma_desc_sw128(b + kk * 32), idesc,
                          (k > k0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[s]);
          tc_commit(&xempty[sx]);
        }
        tc_commit(&tfull[a]);
      }
      DBG(5);
    }
    __syncwarp();
  } else {
    // ------------------------------ epilogue warps
    const int qw = w & 3;                   // TMEM lane quarter of this warp
    const int n = qw * 32 + lane;            // weight row within the tile
    const int et = threadIdx.x - 64;         // 0..127 within the epilogue group
    int seg = 0;
    for (int u = u_first; u <= u_last; ++u, ++seg) {
      const long long ub = (long long)u * p.kb;
      const int k0 = (int)((r0 > ub ? r0 : ub) - ub), k1 = (int)((r1 < ub + p.kb ? r1 : ub + p.kb) - ub);
      const int mb = u / p.n_tiles, t = u % p.n_tiles;
      const int m_base = mb * p.m_blk;
      int mrows = p.M - m_base;
      mrows = mrows > p.m_blk ? p.m_blk : mrows;
      const int ncol = (mrows + 15) & ~15;
      const int a = seg % p.acc_stages;
      const uint32_t aph = (seg / p.acc_stages) & 1;
      mbar_wait(&tfull[a], aph);
      tc_fence_after();
      if (et == 0 && seg < 3) DBG(6 + seg);
      const uint32_t tl = tbase + ((uint32_t)(qw * 32) << 16);
      const bool full_unit = (k0 == 0 && k1 == p.kb);
      if (full_unit) {
        for (int cc = 0; cc < ncol; cc += 16) {
          float v[NT][16];
#pragma unroll
          for (int j = 0; j < NT; ++j) tmem_ld16(tl + (uint32_t)((a * NT + j) * p.m_blk + cc), v[j]);
          apply_epilogue<NT>(p, t * 128, n, m_base + cc, v, xch);
        }
      } else {
        // stream-K partial: publish; gemm_fixup_kernel reduces the unit in CTA order.
        // Layout per (slot, chunk, tile): [4 col quads][128 rows][4 cols], so each warp
        // store instruction writes 512 contiguous bytes.
        const int slot = (u == u_first) ? 0 : 1;
        float* my = p.ws + ((size_t)c * 2 + slot) * (size_t)NT * p.m_blk * 128;
        for (int cc = 0; cc < ncol; cc += 16) {
          float v[NT][16];
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            tmem_ld16(tl + (uint32_t)((a * NT + j) * p.m_blk + cc), v[j]);
            float4* dst = reinterpret_cast<float4*>(my + ((size_t)(cc >> 4) * NT + j) * 2048) + n;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              __stcg(dst + q4 * 128, make_float4(v[j][4 * q4], v[j][4 * q4 + 1], v[j][4 * q4 + 2], v[j][4 * q4 + 3]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
      if (et == 0 && seg < 3) DBG(9 + seg);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) DBG(12);
  if (w == 1) tmem_dealloc(tbase, p.tmem_cols);
}

// ---------------------------------------------------------------- stream-K fixup
// One CTA (128 threads = the 128 weight rows of a tile) per (split unit, group of
// kFixChunks 16-column chunks).  Sums the unit's partials in CTA (= k) order
// -- a fixed order, so results are bit-reproducible -- and runs the fused
// epilogue.  Every SM takes part, so no CTA serialises the reduction.
static constexpr int kFixChunks = 2;

template <int NT>
__global__ void __launch_bounds__(128) gemm_fixup_kernel(GemmParams p, int G) {
  __shared__ float xch[128 * 17 + 64];
  const int units = p.n_tiles * p.m_blocks;
  const int groups = (p.m_blk / 16 + kFixChunks - 1) / kFixChunks;
  const int u = blockIdx.x / groups, gi = blockIdx.x % groups;
  if (u >= units) return;
  const long long ub = (long long)u * p.kb;
  const int c_first = cta_of(ub, p.total, G), c_last = cta_of(ub + p.kb - 1, p.total, G);
  if (c_first == c_last) return;  // finished inside the GEMM
  const int mb = u / p.n_tiles, t = u % p.n_tiles;
  const int m_base = mb * p.m_blk;
  int mrows = p.M - m_base;
  mrows = mrows > p.m_blk ? p.m_blk : mrows;
  const int nchunk = ((mrows + 15) & ~15) >> 4;
  const int n = threadIdx.x;
  for (int ci = gi * kFixChunks; ci < nchunk && ci < (gi + 1) * kFixChunks; ++ci) {
    float v[NT][16];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) v[j][jj] = 0.f;
    // partials of up to 4 segments are loaded before they are summed (latency)
    for (int c0 = c_first; c0 <= c_last; c0 += 4) {
      float4 buf[4][NT][4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int cx = c0 + b;
        if (cx > c_last) break;
        const int s2 = (u == (int)(cta_start(p.total, G, cx) / p.kb)) ? 0 : 1;
        const float* src = p.ws + ((size_t)cx * 2 + s2) * (size_t)NT * p.m_blk * 128;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const float4* s4 = reinterpret_cast<const float4*>(src + ((size_t)ci * NT + j) * 2048) + n;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) buf[b][j][q4] = __ldcg(s4 + q4 * 128);
        }
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (c0 + b > c_last) break;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            v[j][4 * q4] += buf[b][j][q4].x;
            v[j][4 * q4 + 1] += buf[b][j][q4].y;
            v[j][4 * q4 + 2] += buf[b][j][q4].z;
            v[j][4 * q4 + 3] += buf[b][j][q4].w;
          }
      }
    }
    apply_epilogue<NT>(p, t * 128, n, m_base + ci * 16, v, xch);
  }
}

// debug hook: when set, the next gemm launch records per-CTA phase timestamps
static unsigned long long* g_dbg = nullptr;
static int g_dbg_target = 0, g_dbg_count = 0;
// record the stamps of the `target`-th launch after this call (0 = the next one)
void gemm_set_debug(unsigned long long* buf, int target) {
  g_dbg = buf;
  g_dbg_target = target;
  g_dbg_count = 0;
}

// ---------------------------------------------------------------- host side
static int pick_mblk(int M) {
  const int mb = M < 256 ? M : 256;
  return (mb + 15) & ~15;
}

size_t gemm_workspace_bytes(int M, int nt, int num_sms) {
  const int mblk = pick_mblk(M < 1 ? 1 : M);
  return (size_t)num_sms * 2 * nt * mblk * 128 * sizeof(float);
}
size_t gemm_counter_count(int M, int N_units_rows) {
  const int mblk = pick_mblk(M < 1 ? 1 : M);
  const int m_blocks = (M + mblk - 1) / mblk;
  return (size_t)m_blocks * ((N_units_rows + 127) / 128) + 64;
}

int gemm_bf16_fused(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, const GemmEpi& epi,
                    float* ws, int* counters, int num_sms, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return 0;
  if (K % 64 != 0) return -1;
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  p.m_blk = pick_mblk(M);
  p.m_blocks = (M + p.m_blk - 1) / p.m_blk;
  // EPI_SILU: W holds the interleaved gate/up rows (2 x outputs), N counts rows
  p.nt = 1;
  p.tile2_off = 0;
  if (epi.kind == EPI_SILU && N % 128 != 0) return -1;
  p.n_tiles = (N + 127) / 128;
  p.kb = K / 64;
  p.total = (long long)p.n_tiles * p.m_blocks * p.kb;
  p.epi = epi;
  p.ws = ws;
  p.counters = counters;
  p.dbg = (g_dbg && g_dbg_count++ == g_dbg_target) ? g_dbg : nullptr;
  // smem: a short ring of activation k-slices (L2-resident) and the rest for a deep
  // ring of weight k-slices streamed from HBM
  const int stage_a = p.nt * kStageA, stage_b = p.m_blk * 128;
  const int budget = 192 * 1024;
  int xstages = stage_b <= 8192 ? 4 : (stage_b <= 16384 ? 3 : 2);
  int stages = (budget - xstages * stage_b) / stage_a;
  if (stages > 12) stages = 12;
  p.stages = stages;
  p.xstages = xstages;
  const int stage_bytes = 0;
  (void)stage_bytes;
  p.acc_stages = (p.nt * p.m_blk * 2 <= 512) ? 2 : 1;
  int tc = 32;
  while (tc < p.nt * p.m_blk * p.acc_stages) tc <<= 1;
  p.tmem_cols = tc;
  CUtensorMap tmW, tmX;
  const int wrows = p.nt == 2 ? 2 * N : N;
  p.w_blocked = epi.w_blocked;
  if (p.w_blocked) {
    if (N % 128) return -1;
    if (tma_encode_2d(&tmW, W, (uint64_t)wrows * p.kb, 64, 128, 128, 64, 2, true)) return -2;
  } else if (tma_encode_2d(&tmW, W, wrows, K, (uint64_t)K * 2, 128, 64, 2, true)) {
    return -2;
  }
  if (tma_encode_2d(&tmX, X, M, K, (uint64_t)K * 2, p.m_blk, 64, 2, true)) return -2;
  const size_t smem = 1024 + (size_t)stages * stage_a + (size_t)xstages * stage_b + (2 * stages + 2 * xstages + 8) * 8 +
                      32 + 128 * 17 * 4 + 128;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(gemm_bf16_tc_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  int grid = num_sms;
  if (p.total < grid) grid = (int)p.total;
  if (p.nt == 2)
    gemm_bf16_tc_kernel<2><<<grid, kGemmThreads, smem, stream>>>(tmW, tmX, p);
  else
    gemm_bf16_tc_kernel<1><<<grid, kGemmThreads, smem, stream>>>(tmW, tmX, p);
  // units split across CTAs are finished by the parallel fixup kernel
  const int units = p.n_tiles * p.m_blocks;
  bool split = false;
  for (int u = 0; u < units && !split; ++u)
    split = cta_of((long long)u * p.kb, p.total, grid) != cta_of((long long)u * p.kb + p.kb - 1, p.total, grid);
  if (split) {
    const int groups = (p.m_blk / 16 + kFixChunks - 1) / kFixChunks;
    if (p.nt == 2)
      gemm_fixup_kernel<2><<<units * groups, 128, 0, stream>>>(p, grid);
    else
      gemm_fixup_kernel<1><<<units * groups, 128, 0, stream>>>(p, grid);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace srl
