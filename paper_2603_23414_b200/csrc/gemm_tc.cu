// gemm_tc.cu — weight-streaming decode GEMM on tcgen05 tensor cores (sm_100a)
// with fused epilogues.
//
// Computes Y[m][n] = sum_k X[m][k] * W[n][k] for the projection / MLP /
// LM-head contractions of the decode step (SURVEY §8(a) rows a5, a7, a8, a9,
// a10; "throughput is primarily constrained by limited HBM
// bandwidth, due to frequent loading of model weights") and applies the
// consumer op in the epilogue (gemm_epi.cuh):
//   EPI_F32   out[m][n] = Y                             (LM-head logits, op tests)
//   EPI_RESID x_res[m][n] += Y                           (O and down projections)
//   EPI_SILU  act[m][j] = silu(Yg[m][j]) * Yu[m][j]      (gate/up rows interleaved in
//             16-row blocks, so one 128-row tile -- one warp's 32 lanes -- holds both operands)
//   EPI_QKV   (+bias), RoPE on q/k at the row's position, q -> q buffer, k/v ->
//             the paged KV cache (page_table[slot][pos/64], row pos%64)
//
// Swap-AB: 128 weight rows are the UMMA M side, the ragged decode batch
// (M_b <= 256 rows, multiple of 16) is the UMMA N side; the fp32 accumulator
// (128 lanes x M_b columns) lives in TMEM.  Warp roles: w0 weight TMA producer
// (deep ring: streamed from HBM), w10 activation TMA producer (short ring: the
// k-slices are L2-resident), w1 TMEM allocator + single-thread MMA issuer,
// w2..w9 epilogue in two groups of four warps (each group covers the 128 TMEM
// lanes; the groups take alternate 16-column chunks).  A weight tile is H = 2 such
// halves (256 rows) when the batch is wide: the activation slice is then
// loaded once per 256 weight rows, which halves the L2->SM activation
// traffic (at M_b = 256 it is otherwise twice the weight traffic).
//
// Work decomposition (unit = one 128H-row weight tile x one <=256-row batch block):
//  * units >= #SMs (gate/up, LM head, prefill): persistent CTAs own whole units
//    round-robin; TMEM is double-buffered so a unit's epilogue overlaps the
//    next unit's MMAs.
//  * units < #SMs (QKV, O, down at decode): split-K over a thread-block cluster
//    of S CTAs.  Each CTA accumulates its k-range in TMEM, dumps it to its own
//    shared memory, and after a cluster barrier every CTA reduces a slice of the
//    columns by reading the S partials over DSMEM in rank (= k) order -- a fixed
//    order, so results are bit-reproducible -- then runs the fused epilogue.
//    No partials touch HBM and there is no second kernel.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "gumbel.cuh"
#include "kernels.hpp"
#include "launch.hpp"
#include "tma.hpp"

namespace srl {

struct GemmParams {
  int M, N, K;
  int m_blk, m_blocks, n_tiles, kb, units;
  int H;   // 128-row halves per weight tile (1 or 2): both multiply one activation slice
  int S;   // cluster split-K factor (1 = persistent whole-unit mode)
  int split_pairs;  // EPI_PARTIAL: the S splits of a unit are S independent CTA pairs (cluster of 2)
  int w_shared;  // pair kernel: several batch blocks stream the same weight tile (keep it in L2)
  int hp;  // SPLIT: tile halves reduced per DSMEM phase (what fits in the idle rings)
  int stages, xstages, tmem_cols, acc_stages;
  GemmEpi epi;
  const uint8_t* wp;  // packed weights (epi.w_packed), else null
  unsigned long long* dbg;  // optional [grid][16] globaltimer stamps (profiling builds)
  // stream-K (pair kernel, SPLIT == 2): partial slots, per-(unit, row half) arrival counters
  float* sk_ws;
  int* sk_cnt;
  long long sk_total;  // k-blocks of the stream-K space: (units - sk_unit0) * kb
  int sk_pairs;
  int sk_unit0;        // hybrid: units [0, sk_unit0) are whole, sk_full of them per pair, done AFTER
  int sk_full;         //         each pair's stream-K pieces of the remainder units (so their fix-ups overlap)
};

static constexpr int kStageA = 128 * 128;  // 128 weight rows x 64 bf16 (128 B)
static constexpr int kEpiThreads = 128;
constexpr int kGemmThreads = 352;  // w0 W TMA, w1 MMA, w2..9 epilogue (2 groups), w10 X TMA

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int kDbgSlots = 16;  // per CTA phase stamps
#define DBG(slot)                                                         \
  do {                                                                    \
    if (p.dbg) p.dbg[(size_t)blockIdx.x * kDbgSlots + (slot)] = gtimer(); \
  } while (0)

#include "gemm_epi.cuh"

// ---------------------------------------------------------------- cluster helpers
SRL_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SRL_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
SRL_DEV float4 ld_dsmem_f4(uint32_t local_addr, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local_addr), "r"(rank));
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(remote));
  return v;
}

// segment i of this CTA: unit and k-block range
struct Seg {
  int u, k0, k1;
  int ph = 0;  // fused MLP kernel: 0 = phase A (gate/up) unit, 1 = phase B (down) k-split
};
template <int SPLIT>
__device__ __forceinline__ int seg_count(const GemmParams& p) {
  if (SPLIT) return 1;
  return blockIdx.x < (unsigned)p.units ? (p.units - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
}
template <int SPLIT>
__device__ __forceinline__ Seg seg_at(const GemmParams& p, int i) {
  Seg s;
  if (SPLIT) {
    const int r = blockIdx.x % p.S;
    s.u = blockIdx.x / p.S;
    s.k0 = r * p.kb / p.S;
    s.k1 = (r + 1) * p.kb / p.S;
  } else {
    s.u = blockIdx.x + i * gridDim.x;
    s.k0 = 0;
    s.k1 = p.kb;
  }
  return s;
}
// 128-row halves of unit u's weight tile that hold real rows (the last tile may be half empty)
__device__ __forceinline__ int halves_valid(const GemmParams& p, int u) {
  const int row0 = (u % p.n_tiles) * 128 * p.H;
  const int h = (p.N - row0 + 127) / 128;
  return h < p.H ? h : p.H;
}
__device__ __forceinline__ int unit_cols(const GemmParams& p, int u) {
  int mrows = p.M - (u / p.n_tiles) * p.m_blk;
  mrows = mrows > p.m_blk ? p.m_blk : mrows;
  return (mrows + 15) & ~15;
}

// ---------------------------------------------------------------- kernel
template <int SPLIT>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                        GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned (SWIZZLE_128B); pointer arithmetic on the array keeps the
  // shared address space visible to the compiler (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stage_a = p.H * kStageA;
  const int stage_b = p.m_blk * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + p.stages * stage_a;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + p.xstages * stage_b);
  uint64_t* empty = full + p.stages;
  uint64_t* xfull = empty + p.stages;
  uint64_t* xempty = xfull + p.xstages;
  uint64_t* tfull = xempty + p.xstages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tholder = reinterpret_cast<uint32_t*>(tempty + 2);
  float* xch = reinterpret_cast<float*>(tholder + 4);  // [2 groups][kXchFloats]
  int* rtab = reinterpret_cast<int*>(xch + 2 * kXchFloats);  // [kRowTab] (QKV row table)
  float* red = reinterpret_cast<float*>(smem);         // SPLIT: this CTA's partial, reuses the rings

  const int w = warp_id(), lane = lane_id();
  const int nseg = seg_count<SPLIT>(p);
  pdl_trigger();
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
      mbar_init(&tempty[a], 8);
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
  // PDL: only the weight stream (constant during decode) may start before the
  // predecessor grid has completed; every other role reads or writes its data
  if (w != 0) pdl_wait();

  // The three issuing threads run lean loops: ring slot / phase counters are
  // advanced incrementally (no runtime division) and the shared-memory
  // descriptors are precomputed, so a k-block costs a few dozen instructions --
  // a single thread issuing 4 tcgen05.mma per k-block is otherwise the limit.
  if (w == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
      int s = 0;
      uint32_t ph = 1;  // producer waits on "empty" with the inverted phase
      bool first = true;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = seg_at<SPLIT>(p, i);
        const int row0 = (sg.u % p.n_tiles) * 128 * p.H;
        const uint8_t* src = p.wp ? p.wp + ((size_t)(row0 >> 7) * p.kb + sg.k0) * kStageA : nullptr;
        const size_t hstride = (size_t)p.kb * kStageA;
        for (int k = sg.k0; k < sg.k1; ++k) {
          mbar_wait(&empty[s], ph);
          mbar_arrive_expect_tx(&full[s], stage_a);  // rows past N are zero-filled and still counted
          uint8_t* dst = sA + s * stage_a;
          if (src) {
            // packed: each 128-row half is one contiguous, pre-swizzled 16 KB block
            bulk_g2s_hint(dst, src, kStageA, &full[s], pol_w);
            if (p.H == 2) bulk_g2s_hint(dst + kStageA, src + hstride, kStageA, &full[s], pol_w);
            src += kStageA;
          } else {
            tma_load_2d_hint(dst, &tmW, &full[s], k * 64, row0, pol_w);
          }
          if (first) {
            DBG(2);
            first = false;
          }
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
      DBG(3);
    }
  } else if (w == 10) {
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_last();  // activations: re-read by every tile
      int s = 0;
      uint32_t ph = 1;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = seg_at<SPLIT>(p, i);
        const int mrow = (sg.u / p.n_tiles) * p.m_blk;
        for (int k = sg.k0; k < sg.k1; ++k) {
          mbar_wait(&xempty[s], ph);
          mbar_arrive_expect_tx(&xfull[s], stage_b);
          tma_load_2d_hint(sB + s * stage_b, &tmX, &xfull[s], k * 64, mrow, pol_x);
          if (++s == p.xstages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (w == 1) {
    if (lane == 0) {
      // descriptor of slot 0; slot s / k-step kk / half h add (offset >> 4) to the
      // 14-bit start-address field (no carry: shared memory < 256 KB)
      const uint64_t da0 = umma_desc_sw128(smem_u32(sA)), db0 = umma_desc_sw128(smem_u32(sB));
      const uint32_t sa16 = (uint32_t)stage_a >> 4, sb16 = (uint32_t)stage_b >> 4;
      int s = 0, sx = 0;
      uint32_t ph = 0, phx = 0;
      bool first = true;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = seg_at<SPLIT>(p, i);
        const int nh = halves_valid(p, sg.u);
        const uint32_t idesc = umma_idesc_bf16(128, unit_cols(p, sg.u));
        const int a = i % p.acc_stages;
        mbar_wait(&tempty[a], ((i / p.acc_stages) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tacc = tbase + (uint32_t)(a * p.H * p.m_blk);
        const uint32_t tacc1 = tacc + (uint32_t)p.m_blk;
        uint32_t acc = 0;  // the unit's first MMA overwrites the accumulator
        for (int k = sg.k0; k < sg.k1; ++k) {
          mbar_wait(&full[s], ph);
          mbar_wait(&xfull[sx], phx);
          tc_fence_after();
          const uint64_t da = da0 + (uint64_t)(s * sa16), db = db0 + (uint64_t)(sx * sb16);
          tc_mma_bf16(tacc, da, db, idesc, acc);
          tc_mma_bf16(tacc, da + 2, db + 2, idesc, 1u);
          tc_mma_bf16(tacc, da + 4, db + 4, idesc, 1u);
          tc_mma_bf16(tacc, da + 6, db + 6, idesc, 1u);
          if (nh == 2) {  // second 128-row half: same activation slice
            const uint64_t dh = da + (kStageA >> 4);
            tc_mma_bf16(tacc1, dh, db, idesc, acc);
            tc_mma_bf16(tacc1, dh + 2, db + 2, idesc, 1u);
            tc_mma_bf16(tacc1, dh + 4, db + 4, idesc, 1u);
            tc_mma_bf16(tacc1, dh + 6, db + 6, idesc, 1u);
          }
          acc = 1;
          tc_commit(&empty[s]);  // frees the smem slots once these MMAs retire
          tc_commit(&xempty[sx]);
          if (first) {
            DBG(4);
            first = false;
          }
          if (++s == p.stages) {
            s = 0;
            ph ^= 1;
          }
          if (++sx == p.xstages) {
            sx = 0;
            phx ^= 1;
          }
        }
        tc_commit(&tfull[a]);
      }
      DBG(5);
    }
    __syncwarp();
  } else if (!SPLIT) {
    // ------------------------------ epilogue warps (2..9): TMEM -> fused op
    const int qw = w & 3;          // TMEM lane quarter this warp may access
    const int n = qw * 32 + lane;  // weight row within a 128-row half
    const int eg = (w - 2) >> 2;   // epilogue group: 16-column chunks eg, eg+2, ...
    float* xg = xch + eg * kXchFloats;
    for (int i = 0; i < nseg; ++i) {
      const Seg sg = seg_at<SPLIT>(p, i);
      const int t = sg.u % p.n_tiles, m_base = (sg.u / p.n_tiles) * p.m_blk;
      const int ncol = unit_cols(p, sg.u), nh = halves_valid(p, sg.u);
      const int a = i % p.acc_stages;
      fill_row_table(p, m_base, ncol, rtab, (int)threadIdx.x - 64);  // overlaps the MMAs
      mbar_wait(&tfull[a], (i / p.acc_stages) & 1);
      tc_fence_after();
      if (lane == 0 && qw == 0 && i < 3) DBG(6 + i);
      for (int h = 0; h < nh; ++h) {
        const uint32_t tl = tbase + ((uint32_t)(qw * 32) << 16) + (uint32_t)((a * p.H + h) * p.m_blk);
        for (int cc = eg * 16; cc < ncol; cc += 32) {
          float v[16];
          tmem_ld16(tl + cc, v);
          apply_epilogue(p, (t * p.H + h) * 128, n, m_base + cc, v, xg, 1 + eg, rtab + cc);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
      if (lane == 0 && qw == 0 && i < 3) DBG(9 + i);
    }
  }

  if (SPLIT && p.epi.kind == EPI_PARTIAL) {
    // ------------------------------ split k-range r's fp32 partial -> part[r] for the next
    // RMSNorm (independent CTAs: no exchange, no cluster barriers)
    const Seg sg = seg_at<SPLIT>(p, 0);
    const int t = sg.u % p.n_tiles, m_base = (sg.u / p.n_tiles) * p.m_blk;
    const int ncol = unit_cols(p, sg.u), nh = halves_valid(p, sg.u), nchunk = ncol >> 4;
    const int pi = blockIdx.x % p.S;
    if (w >= 2 && w <= 9) {
      const int qw = w & 3, n = qw * 32 + lane, eg = (w - 2) >> 2;
      mbar_wait(&tfull[0], 0);
      tc_fence_after();
      for (int h = 0; h < nh; ++h) {
        const int unit_n0 = (t * p.H + h) * 128;
        const uint32_t tl = tbase + ((uint32_t)(qw * 32) << 16) + (uint32_t)(h * p.m_blk);
        float* dst = p.epi.part + (size_t)pi * p.epi.part_stride + unit_n0 + n;
        const bool rok = unit_n0 + n < p.N;
        for (int c = eg; c < nchunk; c += 2) {
          float v[16];
          tmem_ld16(tl + (uint32_t)(c * 16), v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = m_base + c * 16 + j;
            if (rok && m < p.M) dst[(size_t)m * p.epi.ldo] = v[j];
          }
        }
      }
    }
  } else if (SPLIT) {
    // ------------------------------ cluster split-K reduction over DSMEM
    // Phase = the weight-tile halves whose partials fit in the (now idle) rings at once.
    const Seg sg = seg_at<SPLIT>(p, 0);
    const int t = sg.u % p.n_tiles, m_base = (sg.u / p.n_tiles) * p.m_blk;
    const int ncol = unit_cols(p, sg.u), nh = halves_valid(p, sg.u);
    const int nchunk = ncol >> 4, cmax = p.m_blk >> 4;
    const int r = (int)cluster_rank();
    const bool epi = w >= 2 && w <= 9;
    const int qw = w & 3, n = qw * 32 + lane, eg = (w - 2) >> 2;
    float* xg = xch + eg * kXchFloats;
    const uint32_t red_u32 = smem_u32(red);
    if (epi) {
      fill_row_table(p, m_base, ncol, rtab, (int)threadIdx.x - 64);
      mbar_wait(&tfull[0], 0);
      tc_fence_after();
      if (lane == 0 && qw == 0) DBG(6);
    }
    for (int h0 = 0; h0 < nh; h0 += p.hp) {
      const int hn = nh - h0 < p.hp ? nh - h0 : p.hp;
      if (epi) {
        // partial -> own smem, layout [half][chunk][4 col quads][128 rows][4 cols]
        for (int hl = 0; hl < hn; ++hl) {
          const uint32_t tl = tbase + ((uint32_t)(qw * 32) << 16) + (uint32_t)((h0 + hl) * p.m_blk);
          for (int cc = eg * 16; cc < ncol; cc += 32) {
            float v[16];
            tmem_ld16(tl + cc, v);
            float4* dst = reinterpret_cast<float4*>(red + (size_t)(hl * cmax + (cc >> 4)) * 2048) + n;
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
              dst[q4 * 128] = make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
          }
        }
      }
      cluster_sync_all();  // every partial of this phase is visible cluster-wide
      if (threadIdx.x == 0 && h0 == 0) DBG(13);
      if (epi) {
        const int tot = hn * nchunk, c0 = r * tot / p.S, c1 = (r + 1) * tot / p.S;
        for (int c = c0 + eg; c < c1; c += 2) {
          const int hl = c / nchunk, ci = c % nchunk;
          const uint32_t base = red_u32 + (uint32_t)(((hl * cmax + ci) * 512 + n) * 16);
          float v[16];
#pragma unroll
          for (int jj = 0; jj < 16; ++jj) v[jj] = 0.f;
          // rank order = k order: deterministic.  Remote loads are issued in
          // batches of four ranks before the first add: DSMEM latency is paid
          // once per batch.
          for (int r0 = 0; r0 < p.S; r0 += 4) {
            float4 x[4][4];
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
              if (r0 + rr < p.S)
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                  x[rr][q4] = ld_dsmem_f4(base + (uint32_t)(q4 * 2048), (uint32_t)(r0 + rr));
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
              if (r0 + rr < p.S)
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  v[4 * q4] += x[rr][q4].x;
                  v[4 * q4 + 1] += x[rr][q4].y;
                  v[4 * q4 + 2] += x[rr][q4].z;
                  v[4 * q4 + 3] += x[rr][q4].w;
                }
          }
          apply_epilogue(p, (t * p.H + h0 + hl) * 128, n, m_base + ci * 16, v, xg, 1 + eg, rtab + ci * 16);
        }
        if (w == 2 && lane == 0) DBG(14);
      }
      cluster_sync_all();  // nobody overwrites / leaves while a peer may still read its smem
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) DBG(12);
  if (w == 1) tmem_dealloc(tbase, p.tmem_cols);
}

#include "gemm_pair.cuh"

// debug hook: when set, the target-th gemm launch records per-CTA phase timestamps
static unsigned long long* g_dbg = nullptr;
static int g_dbg_target = 0, g_dbg_count = 0;
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

// co-resident clusters of `size` GEMM CTAs (1 CTA per SM), queried once per size
template <class Kern>
static int max_clusters_of(Kern kern, int size, int* cache) {
  if (cache[size] == 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(size * 64);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = 190 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = size;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 1;
    }
    cache[size] = n;
  }
  return cache[size];
}
static int max_clusters(int S) {
  static int cache[17] = {0};
  return max_clusters_of(gemm_bf16_tc_kernel<1>, S, cache);
}
static int max_clusters_pair(int size) {
  static int cache[17] = {0};
  return max_clusters_of(gemm_pair_kernel<1>, size, cache);
}

static int launch_cluster(void (*kern)(const CUtensorMap, const CUtensorMap, GemmParams), int grid, int csize,
                          size_t smem, cudaStream_t stream, const CUtensorMap& tmW, const CUtensorMap& tmX,
                          const GemmParams& p) {
  return launch_k(kern, dim3(grid), dim3(kGemmThreads), smem, stream, csize, tmW, tmX, p) == cudaSuccess ? 0 : -3;
}

// CTA-pair variant (gemm_pair.cuh) for wide batches; returns 1 when not applicable
// split factor of the single-CTA kernel's partial mode (1: it would not split)
static int single_partial_split(int units, int kb, int num_sms) {
  if (units >= num_sms) return 1;
  int S = num_sms / units;
  if (S > 4) S = 4;
  if (S > kb) S = kb;
  return S;
}

// fused-MLP split counters + exit counter, after the stream-K slots and counters
static size_t fuse_ctr_offset(int num_sms) {
  return (size_t)num_sms * 2 * kSkSlotBytes + (size_t)kSkMaxUnits * 2 * sizeof(int);
}
size_t gemm_workspace_bytes(int num_sms) { return fuse_ctr_offset(num_sms) + 64 * sizeof(int); }

static int gemm_pair_fused(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, const GemmEpi& epi,
                           int num_sms, cudaStream_t stream, int* plan_s = nullptr) {
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = N;
  p.K = K;
  const int pairs = num_sms / 2;
  p.n_tiles = (N + 255) / 256;  // pair tiles
  // Decomposition when whole pair units cannot occupy the pairs evenly (decode
  // QKV / O / down: 24 / 16 / 16 tiles, gate/up 112, on 74 pairs):
  //   1 (default) split-K over a cluster of S pairs with a DSMEM reduction;
  //   0 batch split -- each weight tile multiplied by nb = pairs/tiles batch blocks
  //     on nb pairs (UMMA N = M/nb), no partial sums.  Measured r01: slower -- the
  //     nb-fold weight re-reads are served at ~6.4 TB/s aggregate, HBM-like, not
  //     deduplicated by L2 (QKV 32 vs 30 us, down 72 vs 42 us per launch);
  //   2 stream-K with an L2 fix-up (gemm_pair.cuh).  Measured r01: slower (QKV
  //     53 us in the decode graph): 128 KB fp32 partials per piece through L2.
  const int mode = tuning().gemm_split;
  int mb = pick_mblk(M);
  bool bsplit = false;
  if (mode == 0 && M <= 256 && p.n_tiles < pairs) {
    const int nb = pairs / p.n_tiles;
    if (nb > 1) {
      int m = (M + nb - 1) / nb;
      m = (m + 15) & ~15;
      if (m < mb) {
        mb = m;
        bsplit = true;
      }
    }
  }
  p.m_blk = mb;
  p.m_blocks = (M + p.m_blk - 1) / p.m_blk;
  p.H = 1;
  p.w_shared = bsplit ? 1 : 0;
  p.kb = K / 64;
  p.units = p.n_tiles * p.m_blocks;
  p.epi = epi;
  p.dbg = (!plan_s && g_dbg && g_dbg_count++ == g_dbg_target) ? g_dbg : nullptr;
  // hybrid stream-K (mode 3): whole units round-robin plus the remainder units cut into
  // equal stream-K ranges, pieces first -- balances e.g. gate/up's 112 units on 74 pairs
  const bool hyb = mode == 3 && epi.ws && p.units > pairs && p.units % pairs != 0 && p.units < 4 * pairs &&
                   p.units <= kSkMaxUnits;
  const bool sk = (mode == 2 && epi.ws && p.units % pairs != 0 && p.units <= kSkMaxUnits) || hyb;
  int S = 1;
  // EPI_PARTIAL needs no exchange between the splits: they run as independent CTA
  // pairs, so S is not limited by how many (2S)-CTA clusters can be co-resident
  const bool part = epi.kind == EPI_PARTIAL;
  if (!sk && !bsplit && p.units < pairs) {
    S = pairs / p.units;
    if (S > 4) S = 4;
    if (S > p.kb) S = p.kb;
    while (!part && S > 1 && p.units > max_clusters_pair(2 * S)) --S;
  }
  p.S = S;
  p.split_pairs = part && S > 1;
  if (sk) {
    p.sk_full = hyb ? p.units / pairs : 0;
    p.sk_unit0 = p.sk_full * pairs;
    p.sk_total = (long long)(p.units - p.sk_unit0) * p.kb;
    p.sk_pairs = hyb ? pairs : (int)(p.sk_total < pairs ? p.sk_total : pairs);
    p.sk_ws = reinterpret_cast<float*>(epi.ws);
    p.sk_cnt = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(epi.ws) + (size_t)num_sms * 2 * kSkSlotBytes);
  }
  // H = 2 (whole units): 512-row pair units, two MMAs per k-step sharing the activation
  // slice (gemm_pair.cuh) -- when that at least halves the waves of 256-row units (a
  // 512-row unit takes ~1.8x as long, incl. its un-overlapped epilogue): gate/up's 112
  // units = 2 waves on 74 pairs -> 56 = 1 wave (measured r02: gate/up 2.41 -> 2.26 ms per
  // step); not the LM head (501 units = 7 waves -> 251 = 4: measured 0.228 -> 0.238 ms)
  if (tuning().pair_h2 && !sk && !bsplit && S == 1 && epi.kind != EPI_SAMPLE) {
    const int units2 = (N + 511) / 512 * p.m_blocks;
    const int w1 = (p.units + pairs - 1) / pairs, w2 = (units2 + pairs - 1) / pairs;
    if (w2 * 2 <= w1) {
      p.H = 2;
      p.n_tiles = (N + 511) / 512;
      p.units = units2;
    }
  }
  const int stage_b = (p.m_blk >> 1) * 128;
  const int budget = 200 * 1024;
  int xstages = stage_b <= 4096 ? 8 : (stage_b <= 8192 ? 6 : 4);
  int stages = (budget - xstages * stage_b) / (kStageA * p.H);
  if (stages > 12) stages = 12;
  p.stages = stages;
  p.xstages = xstages;
  const size_t rings = (size_t)stages * kStageA * p.H + (size_t)xstages * stage_b;
  if (S > 1 && !part) {
    const int cpr = ((p.m_blk >> 4) + S - 1) / S;
    if ((size_t)S * cpr * 8192 > rings) return 1;
  }
  if (plan_s) {  // dry run: report the split factor of the cluster split-K path
    *plan_s = (!sk && !bsplit && S > 1) ? S : 1;
    return 0;
  }
  if (epi.kind == EPI_PARTIAL && !(S > 1 && !sk && !bsplit)) return -1;  // caller must ask gemm_partial_split
  p.acc_stages = (S == 1 && 2 * p.H * p.m_blk <= 512) ? 2 : 1;
  int tc = 32;
  while (tc < p.H * p.m_blk * p.acc_stages) tc <<= 1;
  p.tmem_cols = tc;
  CUtensorMap tmW, tmX;
  if (epi.w_packed) {
    // the packed image viewed as [blocks * 128 rows, 64 cols]: one box = one 16 KB block
    p.wp = reinterpret_cast<const uint8_t*>(W);
    const uint64_t rows = (uint64_t)((N + 127) / 128) * p.kb * 128;
    if (tma_encode_2d(&tmW, W, rows, 64, 128, 128, 64, 2, false)) return -2;
  } else if (tma_encode_2d(&tmW, W, N, K, (uint64_t)K * 2, 128, 64, 2, true)) {
    return -2;
  }
  if (tma_encode_2d(&tmX, X, M, K, (uint64_t)K * 2, p.m_blk >> 1, 64, 2, true)) return -2;
  const size_t smem = 1024 + rings + (2 * stages + 2 * xstages + 4) * 8 + 16 + 2 * kXchFloats * 4 + kRowTab * 4;
  if (once_per_device(kOnceGemmPair)) {  // a per-device function attribute
    cudaFuncSetAttribute(gemm_pair_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(gemm_pair_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(gemm_pair_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  if (tuning().verbose)
    fprintf(stderr, "gemm(pair) M=%d N=%d K=%d H=%d units=%d S=%d sk=%d stages=%d/%d smem=%zu\n", M, N, K, p.H,
            p.units, S, (int)sk, stages, xstages, smem);
  int rc;
  if (sk) {
    rc = launch_cluster(gemm_pair_kernel<2>, 2 * p.sk_pairs, 2, smem, stream, tmW, tmX, p);
  } else if (S == 1) {
    const int np = p.units < pairs ? p.units : pairs;
    rc = launch_cluster(gemm_pair_kernel<0>, 2 * np, 2, smem, stream, tmW, tmX, p);
  } else {
    rc = launch_cluster(gemm_pair_kernel<1>, p.units * 2 * S, p.split_pairs ? 2 : 2 * S, smem, stream, tmW, tmX, p);
  }
  if (rc) cudaGetLastError();
  return rc;
}

// ---------------------------------------------------------------- fused MLP (SPLIT 3)
// Static per-pair work list: phase-A (gate/up) units round-robin, then every
// phase-B (down) k-split item, in split order, to the pair where it can start first
// (the later of the pair's finish time and the time its split's act columns are
// complete), costs in k-blocks -- a list-scheduling makespan model of the tensor /
// weight-stream-bound items.  Cached per shape.
struct FuseSched {
  bool ok = false;
  uint8_t n_items[kFuseMaxPairs];
  uint8_t items[kFuseMaxPairs][kFuseMaxItems];
};
static FuseSched fuse_schedule(int P, int nA, int nt2, int S2, int kbA, int kbB) {
  // engines of one process may launch from several host threads (SRL_COMM_LOCAL)
  static std::mutex mu;
  static std::vector<std::pair<std::vector<int>, FuseSched>> cache;
  const std::vector<int> key{P, nA, nt2, S2, kbA, kbB};
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& c : cache)
    if (c.first == key) return c.second;
  FuseSched f;
  memset(f.n_items, 0, sizeof(f.n_items));
  bool ok = P <= kFuseMaxPairs && nA % S2 == 0 && nA + S2 * nt2 <= 255;
  std::vector<long long> t(P, 0), avail(S2, 0);
  const int apS = ok ? nA / S2 : 1;
  for (int u = 0; ok && u < nA; ++u) {
    const int q = u % P;
    if (f.n_items[q] >= kFuseMaxItems) ok = false;
    else f.items[q][f.n_items[q]++] = (uint8_t)u;
    t[q] += kbA;
    avail[u / apS] = std::max(avail[u / apS], (long long)(u / P + 1) * kbA);
  }
  const int cB = kbB / S2;
  for (int j = 0; ok && j < S2 * nt2; ++j) {
    const long long av = avail[j / nt2];
    int best = -1;
    long long bs = 0;
    for (int q = 0; q < P; ++q) {
      if (f.n_items[q] >= kFuseMaxItems) continue;
      const long long st = std::max(t[q], av);
      if (best < 0 || st < bs) {
        best = q;
        bs = st;
      }
    }
    if (best < 0) {
      ok = false;
      break;
    }
    f.items[best][f.n_items[best]++] = (uint8_t)(nA + j);
    t[best] = bs + cB;
  }
  f.ok = ok;
  cache.emplace_back(key, f);
  return cache.back().second;
}

int gemm_mlp_fused(const __nv_bfloat16* X, int M, const void* Wgu, int ff, int d, __nv_bfloat16* act, const void* Wd,
                   float* part, size_t part_stride, int S2, void* ws, int num_sms, cudaStream_t stream) {
  const int pairs = num_sms / 2;
  if (M < 128 || M > 256 || !ws || S2 < 1 || ff % (S2 * 128) || (2 * ff) % 256 || d % 256 || d % 64 || ff % 64 ||
      pairs > kFuseMaxPairs)
    return 1;
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = 2 * ff;
  p.K = d;
  p.m_blk = pick_mblk(M);
  p.m_blocks = 1;
  p.H = 1;
  p.kb = d / 64;
  p.n_tiles = p.N / 256;
  p.units = p.n_tiles;
  p.S = 1;
  p.epi.kind = EPI_SILU;
  p.epi.w_packed = 1;
  p.epi.act = act;
  p.epi.ldo = ff;
  p.wp = reinterpret_cast<const uint8_t*>(Wgu);
  p.dbg = (g_dbg && g_dbg_count++ == g_dbg_target) ? g_dbg : nullptr;
  FuseArgs f;  // host staging of the grid-constant argument (copied at launch; per call: thread-safe)
  memset(&f, 0, sizeof(f));
  GemmParams& q = f.p2;
  q = p;
  q.N = d;
  q.K = ff;
  q.kb = ff / 64;
  q.n_tiles = d / 256;
  q.units = q.n_tiles;
  q.epi = GemmEpi{};
  q.epi.kind = EPI_PARTIAL;
  q.epi.w_packed = 1;
  q.epi.part = part;
  q.epi.part_stride = part_stride;
  q.epi.ldo = d;
  q.wp = reinterpret_cast<const uint8_t*>(Wd);
  q.dbg = nullptr;
  const FuseSched fs = fuse_schedule(pairs, p.units, q.n_tiles, S2, p.kb, q.kb);
  if (!fs.ok) return 1;
  memcpy(f.n_items, fs.n_items, sizeof(f.n_items));
  memcpy(f.items, fs.items, sizeof(f.items));
  f.nA = p.units;
  f.S2 = S2;
  f.a_per_split = p.units / S2;
  f.done = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + fuse_ctr_offset(num_sms));
  f.exit_ctr = f.done + 32;
  const int stage_b = (p.m_blk >> 1) * 128;
  const int budget = 200 * 1024;
  const int xstages = stage_b <= 4096 ? 8 : (stage_b <= 8192 ? 6 : 4);
  int stages = (budget - xstages * stage_b) / kStageA;
  if (stages > 12) stages = 12;
  p.stages = q.stages = stages;
  p.xstages = q.xstages = xstages;
  p.acc_stages = q.acc_stages = 2;
  int tc = 32;
  while (tc < p.m_blk * 2) tc <<= 1;
  p.tmem_cols = q.tmem_cols = tc;
  CUtensorMap tmW, tmX;
  const uint64_t rowsA = (uint64_t)(p.N / 128) * p.kb * 128, rowsB = (uint64_t)(q.N / 128) * q.kb * 128;
  if (tma_encode_2d(&tmW, Wgu, rowsA, 64, 128, 128, 64, 2, false)) return -2;
  if (tma_encode_2d(&f.tmW2, Wd, rowsB, 64, 128, 128, 64, 2, false)) return -2;
  if (tma_encode_2d(&tmX, X, M, d, (uint64_t)d * 2, p.m_blk >> 1, 64, 2, true)) return -2;
  if (tma_encode_2d(&f.tmX2, act, M, ff, (uint64_t)ff * 2, p.m_blk >> 1, 64, 2, true)) return -2;
  const size_t rings = (size_t)stages * kStageA + (size_t)xstages * stage_b;
  const size_t smem = 1024 + rings + (2 * stages + 2 * xstages + 4) * 8 + 16 + 2 * kXchFloats * 4 + kRowTab * 4;
  if (once_per_device(kOnceGemmMlp))
    cudaFuncSetAttribute(gemm_pair_mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (tuning().verbose)
    fprintf(stderr, "gemm(mlp) M=%d ff=%d d=%d unitsA=%d itemsB=%d S2=%d stages=%d/%d smem=%zu\n", M, ff, d, p.units,
            S2 * q.n_tiles, S2, stages, xstages, smem);
  const int rc = launch_k(gemm_pair_mlp_kernel, dim3(2 * pairs), dim3(kGemmThreads), smem, stream, 2, tmW, tmX, p, f) ==
                         cudaSuccess
                     ? 0
                     : -3;
  if (rc) cudaGetLastError();
  return rc;
}

int gemm_partial_split(int M, int N, int K, int num_sms) {
  const int pair_sel = tuning().gemm_pair;
  const bool off = !tuning().partial_norm;
  const bool pair = pair_sel >= 0 ? pair_sel > 0 : M >= 128;
  if (off || M <= 0 || K % 64) return 1;
  if (!pair) {  // single-CTA kernel (H = 1 in partial mode) -- opt-in (srl_tuning.partial_small_m):
    // measured r01 neutral on the 32B slice (O / down -0.37 ms, the norms +0.25 ms per step)
    if (!tuning().partial_small_m) return 1;
    const int m_blk = pick_mblk(M);
    const int units = (N + 127) / 128 * ((M + m_blk - 1) / m_blk);
    return single_partial_split(units, K / 64, num_sms);
  }
  GemmEpi e{};
  e.kind = EPI_PARTIAL;
  e.w_packed = 1;
  int S = 1;
  if (gemm_pair_fused(nullptr, M, nullptr, N, K, e, num_sms, nullptr, &S) != 0) return 1;
  return S;
}

int gemm_bf16_fused(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, const GemmEpi& epi,
                    int num_sms, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return 0;
  if (K % 64 != 0) return -1;
  if (epi.kind == EPI_SILU && N % 128 != 0) return -1;  // N counts interleaved gate/up rows
  const int pair_sel = tuning().gemm_pair;
  const bool pair = pair_sel >= 0 ? pair_sel > 0 : M >= 128;
  if (pair) {
    const int r = gemm_pair_fused(X, M, W, N, K, epi, num_sms, stream);
    if (r <= 0) return r;
  }
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = N;
  p.K = K;
  p.m_blk = pick_mblk(M);
  p.m_blocks = (M + p.m_blk - 1) / p.m_blk;
  p.kb = K / 64;
  // split-K over a cluster only when the units alone cannot occupy the SMs; all
  // clusters must be co-resident (GPC packing can hold fewer than num_sms / S
  // clusters), else a second wave doubles the time
  auto pick_s = [&](int units) {
    int S = 1;
    if (units < num_sms) {
      S = num_sms / units;
      if (S > 8) S = 8;
      if (S > p.kb) S = p.kb;
      while (S > 1 && units > max_clusters(S)) --S;
    }
    return S;
  };
  // H (128-row halves per tile): 2 when it keeps more SMs streaming -- e.g. the
  // 32B shapes at M = 64: QKV 56 tiles x S 2 = 112 CTAs vs 28 x 5 = 140
  auto util = [&](int H) {
    const int units = (N + 128 * H - 1) / (128 * H) * p.m_blocks;
    if (units >= num_sms) return (double)units / ((double)((units + num_sms - 1) / num_sms) * num_sms);
    return (double)units * pick_s(units) / num_sms;
  };
  const int h_env = tuning().gemm_h;
  // packed weights pad rows to 128 only: H = 2 needs an even number of 128-row tiles
  const bool h2_ok = !(epi.w_packed && ((N + 127) / 128) % 2);
  const bool part = epi.kind == EPI_PARTIAL;
  p.H = h_env ? h_env : ((h2_ok && util(2) > util(1) + 0.02) ? 2 : 1);
  if (!h2_ok || part) p.H = 1;
  p.n_tiles = (N + 128 * p.H - 1) / (128 * p.H);
  p.units = p.n_tiles * p.m_blocks;
  p.epi = epi;
  p.dbg = (g_dbg && g_dbg_count++ == g_dbg_target) ? g_dbg : nullptr;
  // EPI_PARTIAL: the splits are independent CTAs (no cluster), <= 4 (what the RMSNorm sums)
  const int S = part ? single_partial_split(p.units, p.kb, num_sms) : pick_s(p.units);
  if (part && S < 2) return -1;  // caller must ask gemm_partial_split
  p.S = S;
  // smem: a short ring of activation k-slices and a deep ring of weight k-slices
  const int stage_a = p.H * kStageA;
  const int stage_b = p.m_blk * 128;
  const int budget = 200 * 1024;
  const int xs_env = tuning().gemm_xstages;
  const int ws_env = tuning().gemm_stages;
  int xstages = stage_b <= 8192 ? 4 : (stage_b <= 16384 ? 3 : 2);
  if (xs_env) xstages = xs_env;
  int stages = (budget - xstages * stage_b) / stage_a;
  if (stages > 12) stages = 12;
  if (ws_env && ws_env < stages) stages = ws_env;
  if (stages < 2 || xstages < 1) return -1;
  p.stages = stages;
  p.xstages = xstages;
  const size_t rings = (size_t)stages * stage_a + (size_t)xstages * stage_b;
  const size_t half_red = (size_t)p.m_blk * 512;  // one 128-row half's fp32 partial
  p.hp = (size_t)p.H * half_red <= rings ? p.H : 1;
  if (half_red > rings) return -1;
  p.acc_stages = (S == 1 && 2 * p.H * p.m_blk <= 512) ? 2 : 1;
  int tc = 32;
  while (tc < p.H * p.m_blk * p.acc_stages) tc <<= 1;
  p.tmem_cols = tc;
  CUtensorMap tmW, tmX;
  memset(&tmW, 0, sizeof(tmW));
  if (epi.w_packed) {
    p.wp = reinterpret_cast<const uint8_t*>(W);
  } else if (tma_encode_2d(&tmW, W, N, K, (uint64_t)K * 2, 128 * p.H, 64, 2, true)) {
    return -2;
  }
  if (tma_encode_2d(&tmX, X, M, K, (uint64_t)K * 2, p.m_blk, 64, 2, true)) return -2;
  const size_t smem = 1024 + rings + (2 * stages + 2 * xstages + 4) * 8 + 16 + 2 * kXchFloats * 4 + kRowTab * 4;
  if (once_per_device(kOnceGemmSingle)) {  // a per-device function attribute
    cudaFuncSetAttribute(gemm_bf16_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(gemm_bf16_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  if (S == 1) {
    const int grid = p.units < num_sms ? p.units : num_sms;
    launch_k(gemm_bf16_tc_kernel<0>, dim3(grid), dim3(kGemmThreads), smem, stream, 1, tmW, tmX, p);
  } else {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.units * S);
    cfg.blockDim = dim3(kGemmThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (tuning().verbose) {
      int ncl = -1;
      cudaOccupancyMaxActiveClusters(&ncl, gemm_bf16_tc_kernel<1>, &cfg);
      fprintf(stderr, "gemm M=%d N=%d K=%d H=%d units=%d S=%d hp=%d stages=%d smem=%zu max_active_clusters=%d\n", M,
              N, K, p.H, p.units, S, p.hp, stages, smem, ncl);
    }
    launch_k(gemm_bf16_tc_kernel<1>, dim3(p.units * S), dim3(kGemmThreads), smem, stream, part ? 1 : S, tmW, tmX, p);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// ---------------------------------------------------------------- weight packing
// one thread per 16-byte chunk of the packed image
__global__ void pack_weight_kernel(const __nv_bfloat16* __restrict__ src, int N, int K, uint4* __restrict__ dst,
                                   long long nchunks) {
  const int kb = K / 64;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < nchunks;
       g += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(g & 7);               // 16-byte chunk within the 128-byte row segment
    const int r = (int)((g >> 3) & 127);      // row within the 128-row block
    const long long blk = g >> 10;            // (t, k) block index
    const int t = (int)(blk / kb), k = (int)(blk % kb);
    const int row = t * 128 + r;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < N) v = __ldg(reinterpret_cast<const uint4*>(src + (size_t)row * K + (size_t)k * 64) + c);
    dst[blk * 1024 + r * 8 + (c ^ (r & 7))] = v;
  }
}

size_t packed_weight_bytes(int N, int K) { return (size_t)((N + 127) / 128) * 128 * (size_t)K * 2; }

// source row i -> packed row (i / rb) * bs + off + i % rb (the gate / up interleave)
__global__ void pack_weight_rows_kernel(const __nv_bfloat16* __restrict__ src, int n, int K, uint4* __restrict__ dst,
                                        int rb, int bs, int off, long long nchunks) {
  const int kb = K / 64;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < nchunks;
       g += (long long)gridDim.x * blockDim.x) {
    const long long cpr = (long long)K / 8;  // 16-byte chunks per source row
    const int i = (int)(g / cpr);
    const int cc = (int)(g % cpr);
    const int k = cc >> 3, c = cc & 7;
    const int row = (i / rb) * bs + off + i % rb;
    const int t = row >> 7, r = row & 127;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(src + (size_t)i * K) + cc);
    dst[((long long)t * kb + k) * 1024 + r * 8 + (c ^ (r & 7))] = v;
  }
}

int pack_weight_rows(const __nv_bfloat16* src, int n, int K, void* dst, int rb, int bs, int off, cudaStream_t stream) {
  if (n <= 0 || K <= 0 || K % 64 || rb <= 0) return -1;
  const long long nchunks = (long long)n * K / 8;
  long long blocks = (nchunks + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  pack_weight_rows_kernel<<<(int)blocks, 256, 0, stream>>>(src, n, K, reinterpret_cast<uint4*>(dst), rb, bs, off,
                                                           nchunks);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

int pack_weight(const __nv_bfloat16* src, int N, int K, void* dst, cudaStream_t stream) {
  if (N <= 0 || K <= 0 || K % 64) return -1;
  const long long nchunks = (long long)packed_weight_bytes(N, K) / 16;
  long long blocks = (nchunks + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  pack_weight_kernel<<<(int)blocks, 256, 0, stream>>>(src, N, K, reinterpret_cast<uint4*>(dst), nchunks);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace srl
