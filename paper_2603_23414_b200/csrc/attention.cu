// attention.cu — paged decode attention with GQA and split-KV (SURVEY §8(a)
// a6; "loading of model weights and KV caches"
// PagedAttention).  For each row r (a sequence at position pos_r, ctx =
// pos_r + 1) and query head h with kv head h / G:
//     o[r,h] = softmax_j(q[r,h] . K_j / sqrt(dh)) V_j ,  j < ctx
// Work item = (row, kv head, chunk of kChunkPages 64-token pages).
//
// bf16 KV (the production path): a persistent kernel; one producer warp
// streams (page, head) K/V blocks with 2-D TMA (128B swizzle) into a 4-stage
// mbarrier ring, four consumer warps each take 16 tokens of the page and use
// mma.sync m16n8k16 with the KV tokens on the M side and the G query heads
// of the kv head on N (S^T = K Q^T; O^T += V^T P^T, P^T transposed in
// registers with movmatrix), warp-shuffle online softmax in the log2 domain,
// and a cross-warp merge.  Per-chunk partials (o, m, l) are merged by
// attn_combine in chunk order.
// fp32 KV (test mode): a plain FFMA kernel with the same item/partial format.
#include <cstdlib>

#include "common.cuh"
#include "launch.hpp"
#include "layers.hpp"
#include "tma.hpp"

namespace srl {

constexpr float kLog2e = 1.4426950408889634f;

// ---------------------------------------------------------------- plan
// Split-KV only when the (row, kv head) pairs alone cannot fill the GPU (the
// drain phase of a rollout: few long sequences); otherwise one item per pair
// and the attention kernel writes the normalised output itself.
// Split-KV only when the (row, kv head) pairs alone leave SMs idle, into ~2 items
// per SM (measured r01, tools/bench_attn.py: every split item costs a partial
// write and a merge, so more, smaller items are slower; at 256-512 pairs the
// longest-first dynamic schedule balances whole rows better than any split)
constexpr int kMinItems = 148;
constexpr int kTargetItems = 2 * 148;
__global__ void attn_plan_kernel(AttnArgs a, int split, int min_items, int target_items) {
  __shared__ int wsum[32];
  __shared__ int base_s, active_s, pages_s;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) {
    base_s = 0;
    active_s = 0;
    pages_s = 0;
  }
  __syncthreads();
  int my_active = 0, my_pages = 0;
  for (int m = threadIdx.x; m < a.M; m += blockDim.x) {
    my_active += a.row_pos[m] >= 0;
    my_pages += (a.row_pos[m] + 1 + 63) / 64;
  }
  atomicAdd(&active_s, my_active);
  atomicAdd(&pages_s, my_pages);
  __syncthreads();
  if (active_s * a.Hkv >= min_items) split = 0;
  // split-KV chunk: about kTargetItems items over all (row, head) pairs, never
  // below kChunkPages pages (per-item overhead: q load, 4-warp merge, partials)
  const int cp = max(kChunkPages, min(256, (pages_s * a.Hkv + target_items - 1) / target_items));
  if (threadIdx.x == 0) *a.chunk_pages = cp;
  const int chunk_tok = 64 * cp;
  for (int b0 = 0; b0 < a.M; b0 += blockDim.x) {
    const int m = b0 + threadIdx.x;
    int nch = 0;
    if (m < a.M) {
      const int ctx = a.row_pos[m] + 1;
      nch = ctx <= 0 ? 0 : (split ? (ctx + chunk_tok - 1) / chunk_tok : 1);
    }
    const int cnt = nch * a.Hkv;
    // block exclusive scan of cnt
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = cnt;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int s = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const int excl = base_s + (w ? wsum[w - 1] : 0) + x - cnt;
    if (m < a.M) {
      a.row_item0[m] = excl;
      a.row_nchunk[m] = nch;
      for (int h = 0; h < a.Hkv; ++h)
        for (int c = 0; c < nch; ++c) {
          const int it = excl + h * nch + c;
          if (it < a.max_items) {
            a.items[it * 3 + 0] = m;
            a.items[it * 3 + 1] = h;
            a.items[it * 3 + 2] = c;
          }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) base_s += wsum[31];
    __syncthreads();
  }
  const int n = min(base_s, a.max_items);
  if (threadIdx.x == 0) *a.n_items = n;
  for (int i = threadIdx.x; i < a.n_ctr; i += blockDim.x) a.work_ctr[i] = 0;
  if (a.merge_ctr)
    for (int i = threadIdx.x; i < a.M * a.Hkv; i += blockDim.x) a.merge_ctr[i] = 0;
  // rows without context get no item: their (bf16) output is zeroed here, once per
  // forward, so the O projection never reads stale values for them (all threads
  // over the inactive rows' elements, 8 bf16 per store)
  {
    __shared__ int n_idle;
    __shared__ int idle[1024];
    if (threadIdx.x == 0) n_idle = 0;
    __syncthreads();
    for (int m = threadIdx.x; m < a.M; m += blockDim.x)
      if (a.row_pos[m] < 0) {
        const int k = atomicAdd(&n_idle, 1);
        if (k < 1024) idle[k] = m;
      }
    __syncthreads();
    const int per = a.Hq * a.dh / 8;  // uint4 per row (Hq * dh % 8 == 0)
    const int ni = min(n_idle, 1024);
    for (int i = threadIdx.x; i < ni * per; i += blockDim.x)
      reinterpret_cast<uint4*>(a.out + (size_t)idle[i / per] * a.Hq * a.dh)[i % per] = make_uint4(0u, 0u, 0u, 0u);
    for (int m = 0; n_idle > 1024 && m < a.M; ++m)  // (more than 1024 idle rows: rare, slow path)
      if (a.row_pos[m] < 0)
        for (int i = threadIdx.x; i < a.Hq * a.dh; i += blockDim.x) a.out[(size_t)m * a.Hq * a.dh + i] = __float2bfloat16(0.f);
  }
  // processing order: counting sort by descending page count (longest first:
  // the persistent CTAs then pull items LPT-style from a counter)
  __shared__ int hist[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  auto bucket = [&](int it) {
    const int m = a.items[it * 3], c = a.items[it * 3 + 2];
    const int npages = (a.row_pos[m] + 1 + 63) / 64;
    const int pg = a.row_nchunk[m] == 1 ? npages : min(npages - c * cp, cp);
    return 1023 - min(pg, 1023);
  };
  for (int it = threadIdx.x; it < n; it += blockDim.x) atomicAdd(&hist[bucket(it)], 1);
  __syncthreads();
  {  // exclusive scan of the 1024 buckets, one per thread
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int v = threadIdx.x < 1024 ? hist[threadIdx.x] : 0;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int s = wsum[lane];
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    if (threadIdx.x < 1024) hist[threadIdx.x] = (w ? wsum[w - 1] : 0) + x - v;
    __syncthreads();
  }
  for (int it = threadIdx.x; it < n; it += blockDim.x) a.order[atomicAdd(&hist[bucket(it)], 1)] = it;
}

int attn_max_items(int M, int Hkv, int max_ctx) {
  const int chunk_tok = 64 * kChunkPages;
  return M * Hkv * ((max_ctx + chunk_tok - 1) / chunk_tok);
}

// ---------------------------------------------------------------- combine
template <bool F32OUT>
__global__ void attn_combine_kernel(AttnArgs a, float* out_f32) {
  pdl_trigger();
  pdl_wait();
  const int G = a.Hq / a.Hkv;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= a.M * a.Hq) return;
  const int m = gw / a.Hq, h = gw % a.Hq;
  const int kvh = h / G, g = h % G;
  const int nch = a.row_nchunk[m];
  if (nch == 1) return;  // written by the attention kernel
  if (nch == 0) {
    for (int d = lane; d < a.dh; d += 32) {
      if (F32OUT) out_f32[((size_t)m * a.Hq + h) * a.dh + d] = 0.f;
      a.out[((size_t)m * a.Hq + h) * a.dh + d] = __float2bfloat16(0.f);
    }
    return;
  }
  const int it0 = a.row_item0[m] + kvh * nch;
  float mx = -INFINITY;
  for (int c = 0; c < nch; ++c) mx = fmaxf(mx, a.part_ml[((size_t)(it0 + c) * G + g) * 2 + 0]);
  float l = 0.f;
  for (int c = 0; c < nch; ++c) {
    const float* ml = a.part_ml + ((size_t)(it0 + c) * G + g) * 2;
    l += ml[1] * exp2f(ml[0] - mx);
  }
  const float inv = 1.f / l;
  for (int d = lane; d < a.dh; d += 32) {
    float acc = 0.f;
    for (int c = 0; c < nch; ++c) {
      const float mc = a.part_ml[((size_t)(it0 + c) * G + g) * 2 + 0];
      acc += a.part_o[((size_t)(it0 + c) * G + g) * a.dh + d] * exp2f(mc - mx);
    }
    const float o = acc * inv;
    if (F32OUT) out_f32[((size_t)m * a.Hq + h) * a.dh + d] = o;
    a.out[((size_t)m * a.Hq + h) * a.dh + d] = __float2bfloat16(o);
  }
}

// ---------------------------------------------------------------- fp32 KV (FFMA, test mode)
constexpr int kF32Threads = 128;
__global__ void __launch_bounds__(kF32Threads) attn_f32_kernel(AttnArgs a) {
  extern __shared__ float sm[];
  pdl_trigger();
  pdl_wait();
  const int G = a.Hq / a.Hkv;
  const int chunk_tok = 64 * kChunkPages;  // scores staged per block (smem); a chunk spans several
  const int item_tok = 64 * *a.chunk_pages;
  float* sq = sm;                       // [G][dh]
  float* ss = sq + G * a.dh;            // [G][chunk_tok]
  const int n_items = *a.n_items;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int m = a.items[it * 3], kvh = a.items[it * 3 + 1], c = a.items[it * 3 + 2];
    const int ctx = a.row_pos[m] + 1;
    const int nch = a.row_nchunk[m];
    const int t0 = nch == 1 ? 0 : c * item_tok;
    const int t1 = nch == 1 ? ctx : min(ctx, t0 + item_tok);
    const int slot = a.row_slot[m];
    const float* qrow = reinterpret_cast<const float*>(a.q) + ((size_t)m * a.Hq + kvh * G) * a.dh;
    const float* kp = reinterpret_cast<const float*>(a.k_pool);
    const float* vp = reinterpret_cast<const float*>(a.v_pool);
    __syncthreads();
    for (int i = threadIdx.x; i < G * a.dh; i += blockDim.x) sq[i] = qrow[i];
    float run_m[8], run_l[8];
    for (int g = 0; g < G; ++g) {
      run_m[g] = -INFINITY;
      run_l[g] = 0.f;
    }
    // o accumulators: thread owns (g, d) pairs i = threadIdx.x + k*blockDim
    float acc[8];
    for (int k = 0; k < 8; ++k) acc[k] = 0.f;
    for (int b0 = t0; b0 < t1; b0 += chunk_tok) {
      const int b1 = min(t1, b0 + chunk_tok);
      __syncthreads();
      const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int j = b0 + w; j < b1; j += kF32Threads / 32) {
        const int page = a.page_table[(size_t)slot * a.max_pages + j / 64];
        const float* krow = kp + (((size_t)page * a.Hkv + kvh) * 64 + j % 64) * a.dh;
        for (int g = 0; g < G; ++g) {
          float p = 0.f;
          for (int d = lane; d < a.dh; d += 32) p += sq[g * a.dh + d] * krow[d];
          for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
          if (lane == 0) ss[g * chunk_tok + (j - b0)] = p * a.scale * kLog2e;
        }
      }
      __syncthreads();
      for (int g = 0; g < G; ++g) {
        float bm = -INFINITY;
        for (int j = 0; j < b1 - b0; ++j) bm = fmaxf(bm, ss[g * chunk_tok + j]);
        const float nm = fmaxf(run_m[g], bm);
        const float alpha = run_m[g] == -INFINITY ? 0.f : exp2f(run_m[g] - nm);
        float lsum = 0.f;
        for (int j = 0; j < b1 - b0; ++j) lsum += exp2f(ss[g * chunk_tok + j] - nm);
        run_l[g] = run_l[g] * alpha + lsum;
        for (int k = 0; k < 8; ++k) {
          const int i = threadIdx.x + k * blockDim.x;
          if (i < G * a.dh && i / a.dh == g) acc[k] *= alpha;
        }
        run_m[g] = nm;
      }
      for (int k = 0; k < 8; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        if (i >= G * a.dh) break;
        const int g = i / a.dh, d = i % a.dh;
        float o = acc[k];
        for (int j = b0; j < b1; ++j) {
          const int page = a.page_table[(size_t)slot * a.max_pages + j / 64];
          const float v = vp[(((size_t)page * a.Hkv + kvh) * 64 + j % 64) * a.dh + d];
          o += exp2f(ss[g * chunk_tok + (j - b0)] - run_m[g]) * v;
        }
        acc[k] = o;
      }
    }
    if (nch == 1) {  // the whole context in one item: final normalised output
      for (int k = 0; k < 8; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        if (i >= G * a.dh) break;
        const int g = i / a.dh;
        const float o = acc[k] / run_l[g];
        const size_t oi = ((size_t)m * a.Hq + kvh * G) * a.dh + i;
        a.out[oi] = __float2bfloat16(o);
        if (a.out_f32) a.out_f32[oi] = o;
      }
    } else {
      for (int k = 0; k < 8; ++k) {
        const int i = threadIdx.x + k * blockDim.x;
        if (i >= G * a.dh) break;
        a.part_o[(size_t)it * G * a.dh + i] = acc[k];
      }
      if (threadIdx.x < G) {
        a.part_ml[((size_t)it * G + threadIdx.x) * 2 + 0] = run_m[threadIdx.x];
        a.part_ml[((size_t)it * G + threadIdx.x) * 2 + 1] = run_l[threadIdx.x];
      }
    }
  }
}

// ---------------------------------------------------------------- bf16 KV (TMA + mma.sync)
constexpr int kStagesDefault = 4;  // K/V ring depth (srl_tuning.attn_stages: 4 or 6)
constexpr int kConsumerWarps = 4;
constexpr int kFinishWarp = kConsumerWarps + 1;          // fused QKV finish (idle otherwise)
constexpr int kAttnThreads = (kConsumerWarps + 2) * 32;
constexpr int kFQ = 2;  // finished items handed from the finish warp to the producer

template <int DH>
struct AttnCfg {
  static constexpr int kBoxCols = DH < 64 ? DH : 64;       // elements per TMA box row
  static constexpr int kBoxes = DH / kBoxCols;             // boxes per 64-token block
  static constexpr int kBoxBytes = 64 * kBoxCols * 2;
  static constexpr int kBlockBytes = kBoxes * kBoxBytes;   // one page x one head, K or V
  static constexpr int kStageBytes = 2 * kBlockBytes;      // K + V
  static constexpr bool kSwz = kBoxCols == 64;             // 128B swizzle
};

template <int DH>
__device__ __forceinline__ uint32_t kv_addr(uint32_t block_base, int tok, int chunk16) {
  using C = AttnCfg<DH>;
  constexpr int kChunksPerBox = C::kBoxCols / 8;
  const int b = chunk16 / kChunksPerBox, c = chunk16 % kChunksPerBox;
  const int cc = C::kSwz ? (c ^ (tok & 7)) : c;
  return block_base + b * C::kBoxBytes + tok * (C::kBoxCols * 2) + (cc << 4);
}

struct ItemInfo {
  int m, kvh, p0, p1, ctx, slot;
};

__device__ __forceinline__ ItemInfo item_info(const AttnArgs& a, int it) {
  ItemInfo r;
  r.m = a.items[it * 3];
  r.kvh = a.items[it * 3 + 1];
  const int c = a.items[it * 3 + 2];
  r.ctx = a.row_pos[r.m] + 1;
  const int npages = (r.ctx + 63) / 64;
  if (a.row_nchunk[r.m] == 1) {
    r.p0 = 0;
    r.p1 = npages;
  } else {
    const int cp = *a.chunk_pages;
    r.p0 = c * cp;
    r.p1 = min(npages, r.p0 + cp);
  }
  r.slot = a.row_slot[r.m];
  return r;
}

// Fused QKV finish for one item (the whole producer warp): q of the item's G query
// heads and, for the item holding the row's last page, the new token's k / v --
// sum of the qkv_S partials in split order, + bias, RoPE on q / k (rotate-half pairs
// (i, i + dh/2), the EPI_QKV epilogue's arithmetic), stored as bf16.
template <int DH>
__device__ __forceinline__ void qkv_finish_item(const AttnArgs& a, const ItemInfo& ii, int G, bool last, int lane) {
  constexpr int HALF = DH / 2;
  const int pos = ii.ctx - 1;
  const float* cs = a.rope_cos + (size_t)pos * HALF;
  const float* sn = a.rope_sin + (size_t)pos * HALF;
  const size_t rowoff = (size_t)ii.m * a.Nqkv;
  // heads of this item: G query heads, then (last) the k and v head
  const int nh = G + (last ? 2 : 0);
  for (int t = lane; t < nh * (HALF / 4); t += 32) {
    const int hh = t / (HALF / 4), i = (t % (HALF / 4)) * 4;
    int col;  // first column of the head in the QKV output
    if (hh < G) col = (ii.kvh * G + hh) * DH;
    else if (hh == G) col = (a.Hq + ii.kvh) * DH;
    else col = (a.Hq + a.Hkv + ii.kvh) * DH;
    float x0[4] = {0.f, 0.f, 0.f, 0.f}, x1[4] = {0.f, 0.f, 0.f, 0.f};
    for (int sp = 0; sp < a.qkv_S; ++sp) {  // split (= k) order
      const float* pp = a.qkv_part + sp * a.qkv_part_stride + rowoff + col;
      const float4 u0 = __ldcg(reinterpret_cast<const float4*>(pp + i));
      const float4 u1 = __ldcg(reinterpret_cast<const float4*>(pp + i + HALF));
      x0[0] += u0.x; x0[1] += u0.y; x0[2] += u0.z; x0[3] += u0.w;
      x1[0] += u1.x; x1[1] += u1.y; x1[2] += u1.z; x1[3] += u1.w;
    }
    if (a.qkv_bias) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        x0[k] += __bfloat162float(a.qkv_bias[col + i + k]);
        x1[k] += __bfloat162float(a.qkv_bias[col + i + HALF + k]);
      }
    }
    float y0[4], y1[4];
    if (hh <= G) {  // q and k heads are rotated
      const float4 c = __ldg(reinterpret_cast<const float4*>(cs + i));
      const float4 s = __ldg(reinterpret_cast<const float4*>(sn + i));
      const float cc[4] = {c.x, c.y, c.z, c.w}, ss[4] = {s.x, s.y, s.z, s.w};
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
    __nv_bfloat16* dst;
    if (hh < G) {
      dst = const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(a.q)) +
            ((size_t)ii.m * a.Hq + ii.kvh * G + hh) * DH;
    } else {
      const int page = a.page_table[(size_t)ii.slot * a.max_pages + pos / 64];
      const size_t off = (((size_t)page * a.Hkv + ii.kvh) * 64 + pos % 64) * DH;
      dst = const_cast<__nv_bfloat16*>(reinterpret_cast<const __nv_bfloat16*>(hh == G ? a.k_pool : a.v_pool)) + off;
    }
    *reinterpret_cast<uint2*>(dst + i) = make_uint2(pack_bf16(y0[0], y0[1]), pack_bf16(y0[2], y0[3]));
    *reinterpret_cast<uint2*>(dst + i + HALF) = make_uint2(pack_bf16(y1[0], y1[1]), pack_bf16(y1[2], y1[3]));
  }
  // the new k / v are read back by this CTA's TMA (async proxy) and q by its
  // consumer warps: order the generic stores before both (the hand-off to the
  // producer is a release / acquire on an mbarrier)
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncwarp();
}

template <int DH, int kStages>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_bf16_kernel(AttnArgs a, const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV) {
  using C = AttnCfg<DH>;
  constexpr int MT = DH / 16;  // 16-dim tiles
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stages = smem;
  float* mrg = reinterpret_cast<float*>(stages + kStages * C::kStageBytes);  // [4 warps][G q][DH + 2]
  pdl_trigger();
  pdl_wait();
  const int G = a.Hq / a.Hkv;
  // merge-buffer rows per warp: the 8-wide MMA N side, or (the 2-CTA-per-SM ring) only
  // the G real query heads; it is also the split-KV merge's scratch (3 nch G floats,
  // capacity checked at launch)
  const int MR = kStages == 3 ? G : 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(mrg + kConsumerWarps * MR * (DH + 2));
  uint64_t* empty = full + kStages;
  volatile int* hdr = reinterpret_cast<volatile int*>(empty + kStages);  // [kStages] item of each staged page
  volatile int* merge_flag = hdr + kStages;

  __shared__ uint64_t fq_full[kFQ], fq_empty[kFQ];
  __shared__ int fq_item[kFQ];

  const int w = warp_id(), lane = lane_id();
  const int n_items = *a.n_items;
  const bool fin = a.qkv_part != nullptr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    for (int s = 0; s < kFQ; ++s) {
      mbar_init(&fq_full[s], 1);
      mbar_init(&fq_empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (w == kFinishWarp) {
    // ---------------- fused QKV finish warp: takes the items (longest first) and
    // finishes each one's q / k / v kFQ items ahead of the producer, so the partial
    // reads and stores stay off the TMA issue path
    if (!fin) return;
    for (int n = 0;; ++n) {
      const int s = n % kFQ;
      mbar_wait(&fq_empty[s], ((n / kFQ) & 1) ^ 1);
      int j = 0;
      if (lane == 0) j = atomicAdd(a.work_ctr, 1);
      j = __shfl_sync(0xffffffffu, j, 0);
      const int it = j < n_items ? a.order[j] : -1;
      if (it >= 0) {
        const ItemInfo ii = item_info(a, it);
        qkv_finish_item<DH>(a, ii, G, ii.p1 == (ii.ctx + 63) / 64, lane);
      }
      if (lane == 0) {
        fq_item[s] = it;
        mbar_arrive(&fq_full[s]);  // release: the item's q / k / v stores before the hand-off
      }
      if (it < 0) break;
    }
    return;
  }

  if (w == kConsumerWarps) {
    // ---------------- producer warp (lane 0 issues the TMA loads)
    {
      if (lane == 0) {
        tma_prefetch(&tmK);
        tma_prefetch(&tmV);
      }
      const uint64_t pol = policy_evict_first();
      int q = 0;
      for (int nf = 0; lane == 0; ++nf) {
        // longest remaining item first, pulled dynamically (balances the tail) -- from
        // the finish warp's hand-off queue when it runs
        int it;
        if (fin) {
          const int s = nf % kFQ;
          mbar_wait(&fq_full[s], (nf / kFQ) & 1);
          it = fq_item[s];
          mbar_arrive(&fq_empty[s]);
          asm volatile("fence.proxy.async.global;" ::: "memory");  // the finished k / v, read by TMA below
        } else {
          const int j = atomicAdd(a.work_ctr, 1);
          it = j < n_items ? a.order[j] : -1;
        }
        if (it < 0) break;
        const ItemInfo ii = item_info(a, it);
        const int* pt = a.page_table + (size_t)ii.slot * a.max_pages;
        int page_next = ii.p0 < ii.p1 ? pt[ii.p0] : 0;
        for (int p = ii.p0; p < ii.p1; ++p, ++q) {
          const int s = q % kStages;
          const uint32_t ph = (q / kStages) & 1;
          // the next page id is loaded one page ahead: its L2 round trip overlaps the
          // wait for a free stage instead of delaying the TMA issue
          const int page = page_next;
          if (p + 1 < ii.p1) page_next = pt[p + 1];
          mbar_wait(&empty[s], ph ^ 1);
          const int row = (page * a.Hkv + ii.kvh) * 64;
          uint8_t* kb = stages + s * C::kStageBytes;
          uint8_t* vb = kb + C::kBlockBytes;
          hdr[s] = it;  // published by the arrive below (release), read after the consumers' wait
          mbar_arrive_expect_tx(&full[s], C::kStageBytes);
          if (a.l2_prefetch > 0 && p + a.l2_prefetch < ii.p1) {  // more HBM requests in flight
            const int page2 = a.page_table[(size_t)ii.slot * a.max_pages + p + a.l2_prefetch];
            const int row2 = (page2 * a.Hkv + ii.kvh) * 64;
#pragma unroll
            for (int b = 0; b < C::kBoxes; ++b) {
              tma_prefetch_l2_2d(&tmK, b * C::kBoxCols, row2);
              tma_prefetch_l2_2d(&tmV, b * C::kBoxCols, row2);
            }
          }
#pragma unroll
          for (int b = 0; b < C::kBoxes; ++b) {
            tma_load_2d_hint(kb + b * C::kBoxBytes, &tmK, &full[s], b * C::kBoxCols, row, pol);
            tma_load_2d_hint(vb + b * C::kBoxBytes, &tmV, &full[s], b * C::kBoxCols, row, pol);
          }
        }
      }
      // end of work: a stage with no data and item -1
      if (lane == 0) {
        const int s = q % kStages;
        mbar_wait(&empty[s], ((q / kStages) & 1) ^ 1);
        hdr[s] = -1;
        mbar_arrive(&full[s]);
      }
    }
    return;
  }

  // ---------------- consumer warps
  const float scale2 = a.scale * kLog2e;
  int q = 0;
  for (;;) {
    {  // the next item is announced in the header of its first staged page
      const int s = q % kStages;
      mbar_wait(&full[s], (q / kStages) & 1);
    }
    const int it = hdr[q % kStages];
    if (it < 0) break;
    const ItemInfo ii = item_info(a, it);
    // Q^T fragments (B operand): n = query index lane/4 (< G), k = dims
    uint32_t bq[MT][2];
    {
      const int n = lane >> 2;
      const __nv_bfloat16* qrow =
          reinterpret_cast<const __nv_bfloat16*>(a.q) + ((size_t)ii.m * a.Hq + ii.kvh * G + n) * DH;
#pragma unroll
      for (int kk = 0; kk < MT; ++kk) {
        const int d0 = kk * 16 + 2 * (lane & 3);
        bq[kk][0] = n < G ? *reinterpret_cast<const uint32_t*>(qrow + d0) : 0u;
        bq[kk][1] = n < G ? *reinterpret_cast<const uint32_t*>(qrow + d0 + 8) : 0u;
      }
    }
    float o[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    for (int p = ii.p0; p < ii.p1; ++p, ++q) {
      const int s = q % kStages;
      const uint32_t ph = (q / kStages) & 1;
      mbar_wait(&full[s], ph);
      const uint32_t kb = smem_u32(stages + s * C::kStageBytes);
      const uint32_t vb = kb + C::kBlockBytes;
      const int tok0 = w * 16;
      const int tbase = p * 64 + tok0;  // absolute position of the warp's first token
      if (tbase < ii.ctx) {
        // two accumulators (even / odd 16-dim tiles): half the dependent MMA chain
        float sacc[4] = {0.f, 0.f, 0.f, 0.f}, sodd[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < MT; ++kk) {
          uint32_t a0, a1, a2, a3;
          ldmatrix_x4(kv_addr<DH>(kb, tok0 + (lane & 15), 2 * kk + (lane >> 4)), a0, a1, a2, a3);
          if (kk & 1) mma_bf16_16816(sodd, a0, a1, a2, a3, bq[kk][0], bq[kk][1]);
          else mma_bf16_16816(sacc, a0, a1, a2, a3, bq[kk][0], bq[kk][1]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) sacc[j] += sodd[j];
        // sacc: [0]=(tok r, q c0) [1]=(tok r, q c1) [2]=(tok r+8, q c0) [3]=(tok r+8, q c1)
        const int r = lane >> 2;
        const bool v0 = tbase + r < ii.ctx, v1 = tbase + r + 8 < ii.ctx;
        float x0 = v0 ? sacc[0] * scale2 : -INFINITY;
        float x1 = v0 ? sacc[1] * scale2 : -INFINITY;
        float x2 = v1 ? sacc[2] * scale2 : -INFINITY;
        float x3 = v1 ? sacc[3] * scale2 : -INFINITY;
        float bm0 = fmaxf(x0, x2), bm1 = fmaxf(x1, x3);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, off));
          bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, off));
        }
        const float nm0 = fmaxf(m0, bm0), nm1 = fmaxf(m1, bm1);
        const float al0 = m0 == -INFINITY ? 0.f : exp2f(m0 - nm0);
        const float al1 = m1 == -INFINITY ? 0.f : exp2f(m1 - nm1);
        const float p0 = exp2f(x0 - nm0), p1 = exp2f(x1 - nm1), p2 = exp2f(x2 - nm0), p3 = exp2f(x3 - nm1);
        // running sums stay per lane (the rescale factors are uniform over the 8 lanes
        // of a query column); reduced across the lanes once, at the end of the item
        l0 = l0 * al0 + (p0 + p2);
        l1 = l1 * al1 + (p1 + p3);
        m0 = nm0;
        m1 = nm1;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          o[mt][0] *= al0;
          o[mt][2] *= al0;
          o[mt][1] *= al1;
          o[mt][3] *= al1;
        }
        const uint32_t pb0 = movmatrix_trans(pack_bf16(p0, p1));
        const uint32_t pb1 = movmatrix_trans(pack_bf16(p2, p3));
        const int vtok = tok0 + (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t a0, a1, a2, a3;
          ldmatrix_x4_trans(kv_addr<DH>(vb, vtok, 2 * mt + ((lane >> 3) & 1)), a0, a1, a2, a3);
          mma_bf16_16816(o[mt], a0, a1, a2, a3, pb0, pb1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    // ---- merge the 4 warps' partial states (columns c0 = 2*(lane&3), c1 = c0+1)
    // (rows >= G of the 8-wide MMA N side are padding: never stored)
    float* my = mrg + w * MR * (DH + 2);
    const int c0 = 2 * (lane & 3);
    const bool r0 = c0 < G, r1 = c0 + 1 < G;
    if ((lane >> 2) == 0) {
      if (r0) {
        my[c0 * (DH + 2) + DH] = m0;
        my[c0 * (DH + 2) + DH + 1] = l0;
      }
      if (r1) {
        my[(c0 + 1) * (DH + 2) + DH] = m1;
        my[(c0 + 1) * (DH + 2) + DH + 1] = l1;
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int d = mt * 16 + (lane >> 2);
      if (r0) {
        my[c0 * (DH + 2) + d] = o[mt][0];
        my[c0 * (DH + 2) + d + 8] = o[mt][2];
      }
      if (r1) {
        my[(c0 + 1) * (DH + 2) + d] = o[mt][1];
        my[(c0 + 1) * (DH + 2) + d + 8] = o[mt][3];
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32));
    const bool single = a.row_nchunk[ii.m] == 1;
    for (int i = threadIdx.x; i < G * DH; i += kConsumerWarps * 32) {
      const int g = i / DH, d = i % DH;
      float mx = -INFINITY;
      for (int ww = 0; ww < kConsumerWarps; ++ww) mx = fmaxf(mx, mrg[(ww * MR + g) * (DH + 2) + DH]);
      float acc = 0.f, l = 0.f;
      for (int ww = 0; ww < kConsumerWarps; ++ww) {
        const float* e = mrg + (ww * MR + g) * (DH + 2);
        const float f = e[DH] == -INFINITY ? 0.f : exp2f(e[DH] - mx);
        acc += e[d] * f;
        l += e[DH + 1] * f;
      }
      if (single) {  // the whole context in one item: final normalised output
        const float o = acc / l;
        const size_t oi = ((size_t)ii.m * a.Hq + ii.kvh * G + g) * DH + d;
        a.out[oi] = __float2bfloat16(o);
        if (a.out_f32) a.out_f32[oi] = o;
      } else {
        a.part_o[((size_t)it * G + g) * DH + d] = acc;
        if (d == 0) {
          a.part_ml[((size_t)it * G + g) * 2 + 0] = mx;
          a.part_ml[((size_t)it * G + g) * 2 + 1] = l;
        }
      }
    }
    if (!single && a.merge_ctr) {
      // split-KV: the CTA completing the last chunk of (row, kv head) merges all
      // chunks in chunk order (deterministic whoever arrives last; no second kernel)
      // CTA barrier, then one fenced atomic by one thread (CUTLASS semaphore pattern)
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32));
      const int nch = a.row_nchunk[ii.m];
      int* ctr = a.merge_ctr + ii.m * a.Hkv + ii.kvh;
      if (threadIdx.x == 0) {
        __threadfence();  // release: the CTA's partials (ordered by the barrier) before the count
        const int last = atomicAdd(ctr, 1) == nch - 1;
        if (last) *ctr = 0;
        __threadfence();
        *merge_flag = last;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32));
      if (*merge_flag) {
        const int it0 = a.row_item0[ii.m] + ii.kvh * nch;
        constexpr int kT = kConsumerWarps * 32;
        // the chunks' (max, sum) go to shared memory once (the 4-warp merge buffer is
        // free here); per-(chunk, head) scale factors and 1/l are computed there, then
        // every output element sums its chunks' partials with the loads of four chunks
        // in flight -- the merge is L2-latency-bound otherwise (chunk order kept:
        // deterministic)
        float* sm_m = mrg;
        float* sm_l = sm_m + nch * G;
        float* sm_inv = sm_l + nch * G;
        for (int j = threadIdx.x; j < nch * G; j += kT) {
          const int cc = j / G, g = j % G;
          sm_m[j] = __ldcg(a.part_ml + ((size_t)(it0 + cc) * G + g) * 2);
          sm_l[j] = __ldcg(a.part_ml + ((size_t)(it0 + cc) * G + g) * 2 + 1);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kT));
        for (int g = threadIdx.x; g < G; g += kT) {
          float mx = -INFINITY;
          for (int cc = 0; cc < nch; ++cc) mx = fmaxf(mx, sm_m[cc * G + g]);
          float l = 0.f;
          for (int cc = 0; cc < nch; ++cc) {
            const float mc = sm_m[cc * G + g];
            const float f = mc == -INFINITY ? 0.f : exp2f(mc - mx);
            sm_m[cc * G + g] = f;  // from here on: the chunk's scale factor
            l += sm_l[cc * G + g] * f;
          }
          sm_inv[g] = 1.f / l;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kT));
        for (int i = threadIdx.x; i < G * DH; i += kT) {
          const int g = i / DH, d = i % DH;
          float acc = 0.f;
          for (int c0 = 0; c0 < nch; c0 += 4) {
            float p[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              p[j] = c0 + j < nch ? __ldcg(a.part_o + ((size_t)(it0 + c0 + j) * G + g) * DH + d) : 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (c0 + j < nch) acc += p[j] * sm_m[(c0 + j) * G + g];
          }
          const float o = acc * sm_inv[g];
          const size_t oi = ((size_t)ii.m * a.Hq + ii.kvh * G + g) * DH + d;
          a.out[oi] = __float2bfloat16(o);
          if (a.out_f32) a.out_f32[oi] = o;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32));
  }
}

template <int DH, int NS>
static void launch_bf16_ns(const AttnArgs& a, const void* tk, const void* tv, cudaStream_t st, int once_slot) {
  using C = AttnCfg<DH>;
  const int G = a.Hq / a.Hkv, MR = NS == 3 ? G : 8;
  const size_t smem = 1024 + NS * C::kStageBytes + (size_t)kConsumerWarps * MR * (DH + 2) * 4 + 2 * NS * 8 + 64;
  if (once_per_device(once_slot))  // per-device attribute
    cudaFuncSetAttribute(attn_bf16_kernel<DH, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = 148;
  const int occ = (int)((228 * 1024) / (smem + 1024));
  grid *= occ < 1 ? 1 : occ;
  launch_k(attn_bf16_kernel<DH, NS>, dim3(grid), dim3(kAttnThreads), smem, st, 1, a,
           *reinterpret_cast<const CUtensorMap*>(tk), *reinterpret_cast<const CUtensorMap*>(tv));
}

template <int DH>
static void launch_bf16(const AttnArgs& a, const void* tk, const void* tv, cudaStream_t st) {
  const int slot = DH == 128 ? kOnceAttn128 : (DH == 64 ? kOnceAttn64 : kOnceAttn32);
  if (tuning().attn_stages == 6 && DH == 128)
    launch_bf16_ns<DH, 6>(a, tk, tv, st, kOnceAttn128s6);
  else if (tuning().attn_stages == 3 && DH == 128 && a.Hq / a.Hkv <= 4 &&
           3 * (a.max_pages / kChunkPages + 1) <= kConsumerWarps * (DH + 2))
    // 3 x 32 KB stages and a G-row merge buffer: two CTAs per SM (the split-KV merge
    // scratch, 3 nch G floats, fits the 4 G (DH + 2) of the buffer)
    launch_bf16_ns<DH, 3>(a, tk, tv, st, kOnceAttn128s3);
  else
    launch_bf16_ns<DH, kStagesDefault>(a, tk, tv, st, slot);
}

void attn_plan(const AttnArgs& a, int split, cudaStream_t st) {
  // split-KV planning (srl_tuning; 0 = the built-in values)
  const int mi = tuning().attn_min_items ? tuning().attn_min_items : kMinItems;
  const int ti = tuning().attn_target_items ? tuning().attn_target_items : kTargetItems;
  launch_k(attn_plan_kernel, dim3(1), dim3(1024), 0, st, 1, a, split, mi, ti);
}

void attn_run(const AttnArgs& a_in, bool kv_fp32, const void* tmap_k, const void* tmap_v, cudaStream_t st) {
  if (a_in.M <= 0) return;
  // srl_tuning.attn_l2_prefetch = <pages>: L2 prefetch beyond the ring -- measured r01
  // slower at every distance tried (2/4/8 pages: -3..-10 %), so off
  const int pf = tuning().attn_l2_prefetch;
  AttnArgs a = a_in;
  a.l2_prefetch = pf;
  if (kv_fp32) {
    const int G = a.Hq / a.Hkv;
    const size_t smem = (size_t)G * a.dh * 4 + (size_t)G * 64 * kChunkPages * 4;
    launch_k(attn_f32_kernel, dim3(148 * 4), dim3(kF32Threads), smem, st, 1, a);
  } else {
    switch (a.dh) {
      case 128: launch_bf16<128>(a, tmap_k, tmap_v, st); break;
      case 64: launch_bf16<64>(a, tmap_k, tmap_v, st); break;
      case 32: launch_bf16<32>(a, tmap_k, tmap_v, st); break;
      default: return;
    }
  }
  if (kv_fp32 || !a.merge_ctr) {  // the bf16 kernel merges split-KV chunks itself
    const int warps = a.M * a.Hq;
    launch_k(attn_combine_kernel<false>, dim3((warps + 7) / 8), dim3(256), 0, st, 1, a, (float*)nullptr);
  }
}

void attn_combine_f32(const AttnArgs& a, float* out_f32, cudaStream_t st) {
  const int warps = a.M * a.Hq;
  launch_k(attn_combine_kernel<true>, dim3((warps + 7) / 8), dim3(256), 0, st, 1, a, out_f32);
}

}  // namespace srl
