// gemm_pair.cuh — the decode GEMM on CTA pairs (tcgen05 cta_group::2), included
// by gemm_tc.cu after the single-CTA kernel (shares GemmParams, the epilogues
// and the cluster helpers).
//
// Why pairs: at a wide decode batch (M_b = 256) one SM streaming a 128-row weight
// tile must also stage the whole 256-row activation slice and feed both to the
// tensor core; shared-memory traffic per k-block (TMA writes + UMMA operand
// reads, ~96 KB) then bounds the mainloop, not HBM.  With cta_group::2 two SMs
// of a TPC run one M = 256 MMA: each holds 128 weight rows (A) and HALF of the
// activation rows (B), and the pair shares B, so per-SM staging and operand
// traffic drop by a third and each SM's W stream runs at the tensor rate.
//
// Pair unit = 256 weight rows (CTA r2 of the pair owns rows 128*r2..+127) x one
// <= 256-row batch block.  The leader CTA (even cluster rank) issues the MMAs;
// both CTAs' TMA loads signal the leader's "full" barriers (.cta_group::2); the
// leader's commits multicast "empty" / "tfull" arrivals to both CTAs; both
// CTAs' epilogue warps arrive on the leader's "tempty".  Each CTA's TMEM holds
// its 128 rows x N accumulator and it runs the same fused epilogues.
//
// Decomposition (SPLIT; host selection and measurements in gemm_tc.cu):
//  0  persistent pairs, whole pair units round-robin (gate/up, LM head, prefill);
//  1  split-K over the S pairs of a (2S)-CTA cluster (decode QKV / O / down):
//     every CTA pushes each 16-column chunk of its fp32 partial straight into the
//     shared memory of the CTA (same row half) that owns the chunk
//     (st.shared::cluster, fire-and-forget), and the owner sums the S partials
//     in pair (= k) order from local memory -- deterministic;
//  3  fused MLP (gemm_pair_mlp_kernel): the gate/up GEMM (EPI_SILU, whole units,
//     phase A) and the down GEMM (EPI_PARTIAL, S2 k-splits per tile, phase B) as
//     ONE persistent work list per pair (FuseArgs, a host-built static schedule).
//     A down k-split s reads act columns produced by a fixed range of gate/up units;
//     each of their CTAs bumps done[s] after its act stores (release), and the X
//     producer of a phase-B item waits for done[s] (acquire) before its first TMA of
//     act.  Phase-A items precede phase-B items on every pair and phase-A items never
//     wait, so with all CTAs co-resident (grid = 2 x pairs) nothing can deadlock.
//     The weight producer streams phase-B weights ahead regardless (they are
//     constant), so the down GEMM fills the gate/up GEMM's last partial wave instead
//     of starting after it (r02: 112 gate/up units on 74 pairs = 1.51 waves).
//  2  stream-K (opt-in, srl_tuning.gemm_split = 2): the flattened (unit, k-block) space
//     is cut into #pairs equal ranges; a unit cut between pairs is finished by
//     its LAST arriving piece: every piece stores its fp32 partial to an
//     L2-resident workspace slot and bumps the unit's counter, and the CTA
//     completing the count sums all pieces in k order and runs the epilogue.
//     Nobody waits on another CTA, so co-residency is never assumed.

SRL_DEV uint32_t mapa_u32(uint32_t local_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
  return r;
}
SRL_DEV void st_dsmem_f4(uint32_t cluster_addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(cluster_addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
SRL_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
SRL_DEV void mbar_expect_tx_only(uint64_t* bar, uint32_t tx) { mbar_arrive_expect_tx(bar, tx); }
// 2-D TMA load into this CTA's shared memory whose completion is counted on the
// pair leader's mbarrier (cluster address)
SRL_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
SRL_DEV void tc_mma_bf16_pair(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate));
}
SRL_DEV void tc_commit_pair(uint64_t* bar, uint16_t cta_mask) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"(cta_mask)
               : "memory");
}
SRL_DEV void tmem_alloc_pair(uint32_t* holder, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(holder)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
SRL_DEV void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// stream-K: first flattened k-block of pair q's range
__device__ __forceinline__ long long sk_bound(const GemmParams& p, int q) {
  return (long long)q * p.sk_total / p.sk_pairs;
}
// piece i of pair `pid` (unit, k0, k1); *n = piece count when i < 0.  Stream-K
// pieces of the remainder units first, then (hybrid) the pair's whole units.
__device__ __forceinline__ Seg sk_piece(const GemmParams& p, int pid, int i, int* n = nullptr) {
  long long g = sk_bound(p, pid);
  const long long e = sk_bound(p, pid + 1);
  Seg sg{0, 0, 0};
  int j = 0;
  while (g < e) {
    const int r = (int)(g / p.kb);
    sg.u = p.sk_unit0 + r;
    sg.k0 = (int)(g - (long long)r * p.kb);
    sg.k1 = (int)min((long long)p.kb, sg.k0 + (e - g));
    if (j == i) return sg;
    g += sg.k1 - sg.k0;
    ++j;
  }
  for (int f = 0; f < p.sk_full; ++f, ++j)
    if (j == i) return Seg{pid + f * p.sk_pairs, 0, p.kb};
  if (n) *n = j;
  return sg;
}
// workspace slot of pair q's piece of unit u: 2q for its first piece, 2q + 1 for a later one
__device__ __forceinline__ int sk_slot(const GemmParams& p, int q, int u) {
  return 2 * q + (sk_bound(p, q) >= (long long)(u - p.sk_unit0) * p.kb ? 0 : 1);
}
// pairs whose ranges intersect unit u: [*q0, *q1]
__device__ __forceinline__ void sk_unit_pairs(const GemmParams& p, int u, int* q0, int* q1) {
  const long long a = (long long)(u - p.sk_unit0) * p.kb, b = a + p.kb - 1;
  int q = (int)(a * p.sk_pairs / p.sk_total);
  while (q > 0 && sk_bound(p, q) > a) --q;
  while (q + 1 < p.sk_pairs && sk_bound(p, q + 1) <= a) ++q;
  *q0 = q;
  while (q + 1 < p.sk_pairs && sk_bound(p, q + 1) <= b) ++q;
  *q1 = q;
}
__device__ __forceinline__ float4 ldcg_f4(const float4* a) { return __ldcg(a); }

// Fused MLP work list (SPLIT 3).  Item ids < nA: phase-A unit (ph 0); else
// j = id - nA: phase-B k-split j / p2.n_tiles of tile j % p2.n_tiles (ph 1,
// m_blocks == 1).
constexpr int kFuseMaxPairs = 80, kFuseMaxItems = 8;
struct FuseArgs {
  CUtensorMap tmW2, tmX2;  // phase B: down weights (packed), act [M][ff]
  GemmParams p2;
  int nA;                  // phase-A units
  int S2;                  // phase-B k-splits per tile
  int a_per_split;         // phase-A units whose act columns one k-split reads
  int* done;               // [S2] CTA completions of each split's phase-A units (self-resetting)
  int* exit_ctr;
  uint8_t n_items[kFuseMaxPairs];
  uint8_t items[kFuseMaxPairs][kFuseMaxItems];
};

SRL_DEV int ld_acquire_gpu(const int* a) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
SRL_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// pair unit u -> (pair tile, batch block); pair tile t covers weight rows 256t..256t+255
template <int SPLIT>
__device__ __forceinline__ void gemm_pair_body(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmParams& p,
                                               const FuseArgs* fz) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int stage_b = (p.m_blk >> 1) * 128;  // this CTA's half of the activation slice
  // H = 2 (whole units only): a pair unit is 512 weight rows, two M = 256 MMAs per
  // k-step sharing the activation slice -- per SM 32 KB of weights + 16 KB of
  // activations per k-block for twice the MACs (H = 1: 16 + 16); TMEM holds both
  // accumulators (512 columns, no double buffering).  Measured MMA-paced: 0.71 us per
  // k-block (1024 clk) vs 0.37-0.40 for H = 1; it pays where it halves the waves
  const int H = SPLIT == 0 ? p.H : 1;
  uint8_t* sA = smem;
  uint8_t* sB = smem + p.stages * kStageA * H;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + p.xstages * stage_b);
  uint64_t* empty = full + p.stages;
  uint64_t* xfull = empty + p.stages;
  uint64_t* xempty = xfull + p.xstages;
  uint64_t* tfull = xempty + p.xstages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tholder = reinterpret_cast<uint32_t*>(tempty + 2);
  float* xch = reinterpret_cast<float*>(tholder + 4);  // [2 groups][kXchFloats]
  int* rtab = reinterpret_cast<int*>(xch + 2 * kXchFloats);  // [kRowTab] (QKV row table)
  float* red = reinterpret_cast<float*>(smem);         // SPLIT: received partials, reuses the rings

  const int w = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const uint32_t r2 = rank & 1u, leader = rank & ~1u;
  const uint16_t pair_mask = (uint16_t)(3u << leader);
  const bool is_leader = r2 == 0;
  // units: SPLIT -> cluster id (one unit per cluster, pair index = k split);
  //        else  -> pair id, round-robin over pair units
  const int npairs = gridDim.x >> 1;
  const int pid = blockIdx.x >> 1;
  const int cl = SPLIT == 1 ? (int)(blockIdx.x / (2 * p.S)) : 0;
  // split index: the pair's rank in its (2S)-CTA cluster, or (EPI_PARTIAL, clusters of
  // one pair) its position among the unit's S consecutive pairs
  const int pi = SPLIT == 1 ? (p.split_pairs ? (int)((blockIdx.x >> 1) % p.S) : (int)(rank >> 1)) : 0;
  int nseg;
  if (SPLIT == 1) nseg = 1;
  else if (SPLIT == 2) sk_piece(p, pid, -1, &nseg);
  else if (SPLIT == 3) nseg = fz->n_items[pid];
  else nseg = pid < p.units ? (p.units - pid + npairs - 1) / npairs : 0;
  // piece i of this pair: (unit, k-block range[, phase])
  auto piece = [&](int i) -> Seg {
    if (SPLIT == 2) return sk_piece(p, pid, i);
    if (SPLIT == 1) return Seg{cl, pi * p.kb / p.S, (pi + 1) * p.kb / p.S};
    if (SPLIT == 3) {
      const int it = fz->items[pid][i];
      if (it < fz->nA) return Seg{it, 0, p.kb, 0};
      const int j = it - fz->nA, sp = j / fz->p2.n_tiles;
      return Seg{j % fz->p2.n_tiles, sp * fz->p2.kb / fz->S2, (sp + 1) * fz->p2.kb / fz->S2, 1};
    }
    return Seg{pid + i * npairs, 0, p.kb};
  };
  // the GEMM (and its tensor maps) a piece belongs to
  auto gp = [&](const Seg& sg) -> const GemmParams& { return (SPLIT == 3 && sg.ph) ? fz->p2 : p; };
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
      mbar_init(&tempty[a], 16);  // 8 epilogue warps x 2 CTAs (the leader's copy is used)
    }
    fence_barrier_init();
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
    if (SPLIT == 3) {
      tma_prefetch(&fz->tmW2);
      tma_prefetch(&fz->tmX2);
    }
  }
  if (w == 1) tmem_alloc_pair(tholder, p.tmem_cols);
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tbase = *tholder;
  if (threadIdx.x == 0) DBG(1);
  if (w != 0) pdl_wait();  // PDL: only the (constant) weight stream runs ahead of the predecessor

  if (w == 0) {
    if (lane == 0) {
      const uint64_t pol_w = p.w_shared ? policy_evict_normal() : policy_evict_first();
      const uint32_t full_l = mapa_u32(smem_u32(full), leader);
      int s = 0;
      uint32_t ph = 1;
      bool first = true;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = piece(i);
        const GemmParams& q = gp(sg);
        const CUtensorMap* tw = (SPLIT == 3 && sg.ph == 1) ? &fz->tmW2 : &tmW;
        const int u = sg.u;
        for (int k = sg.k0; k < sg.k1; ++k) {
          mbar_wait(&empty[s], ph);
          if (is_leader) mbar_arrive_expect_tx(&full[s], 2 * kStageA * H);  // both CTAs' halves
          for (int h = 0; h < H; ++h) {
            const int t128 = ((u % q.n_tiles) * H + h) * 2 + (int)r2;  // this CTA's 128-row tile of MMA h
            const int c1 = q.wp ? (t128 * q.kb + k) * 128 : t128 * 128;
            const int c0 = q.wp ? 0 : k * 64;
            tma_load_2d_pair(sA + (s * H + h) * kStageA, tw, full_l + 8u * s, c0, c1, pol_w);
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
      const uint64_t pol_x = policy_evict_last();
      const uint32_t xfull_l = mapa_u32(smem_u32(xfull), leader);
      bool xw = false;  // (profiling stamps of the first phase-B wait)
      int s = 0;
      uint32_t ph = 1;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = piece(i);
        const GemmParams& q = gp(sg);
        const CUtensorMap* tx = (SPLIT == 3 && sg.ph) ? &fz->tmX2 : &tmX;
        const uint32_t xbytes = 2u * (uint32_t)((q.m_blk >> 1) * 128);  // both CTAs' boxes (slots are stage_b apart)
        const int u = sg.u;
        const int ncol = unit_cols(q, u);
        const int mrow = (u / q.n_tiles) * q.m_blk + (int)r2 * (ncol >> 1);
        if (SPLIT == 3 && sg.ph == 1) {
          // phase B reads act columns [k0, k1) * 64: wait for the phase-A CTAs that
          // write them (acquire), then order the async-proxy (TMA) reads after it
          const int sp = sg.k0 * fz->S2 / q.kb;
          if (!xw) DBG(13);
          while (ld_acquire_gpu(fz->done + sp) < 2 * fz->a_per_split) __nanosleep(64);
          fence_proxy_async_global();
          if (!xw) DBG(15);
          xw = true;
        }
        for (int k = sg.k0; k < sg.k1; ++k) {
          mbar_wait(&xempty[s], ph);
          if (is_leader) mbar_arrive_expect_tx(&xfull[s], xbytes);
          tma_load_2d_pair(sB + s * stage_b, tx, xfull_l + 8u * s, k * 64, mrow, pol_x);
          if (++s == p.xstages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (w == 1) {
    if (lane == 0 && is_leader) {
      const uint64_t da0 = umma_desc_sw128(smem_u32(sA)), db0 = umma_desc_sw128(smem_u32(sB));
      const uint32_t sa16 = (uint32_t)(kStageA * H) >> 4, sb16 = (uint32_t)stage_b >> 4;
      int s = 0, sx = 0;
      uint32_t ph = 0, phx = 0;
      bool first = true;
      for (int i = 0; i < nseg; ++i) {
        const Seg sg = piece(i);
        const int u = sg.u;
        const uint32_t idesc = umma_idesc_bf16(256, unit_cols(gp(sg), u));
        const int a = i % p.acc_stages;
        mbar_wait(&tempty[a], ((i / p.acc_stages) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tacc = tbase + (uint32_t)(a * H * p.m_blk);
        uint32_t acc = 0;
        for (int k = sg.k0; k < sg.k1; ++k) {
          mbar_wait(&full[s], ph);
          mbar_wait(&xfull[sx], phx);
          tc_fence_after();
          const uint64_t db = db0 + (uint64_t)(sx * sb16);
          for (int h = 0; h < H; ++h) {
            const uint64_t da = da0 + (uint64_t)(s * sa16 + h * ((uint32_t)kStageA >> 4));
            const uint32_t th = tacc + (uint32_t)(h * p.m_blk);
            tc_mma_bf16_pair(th, da, db, idesc, acc);
            tc_mma_bf16_pair(th, da + 2, db + 2, idesc, 1u);
            tc_mma_bf16_pair(th, da + 4, db + 4, idesc, 1u);
            tc_mma_bf16_pair(th, da + 6, db + 6, idesc, 1u);
          }
          acc = 1;
          tc_commit_pair(&empty[s], pair_mask);  // frees both CTAs' slots once the MMAs retire
          tc_commit_pair(&xempty[sx], pair_mask);
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
        tc_commit_pair(&tfull[a], pair_mask);
      }
      DBG(5);
    }
    __syncwarp();
  } else if (SPLIT != 1) {
    // ------------------------------ epilogue warps (2..9): TMEM -> fused op
    const int qw = w & 3, n = qw * 32 + lane, eg = (w - 2) >> 2;
    float* xg = xch + eg * kXchFloats;
    const uint32_t tempty_l = mapa_u32(smem_u32(tempty), leader);
    volatile int& sh_last = *reinterpret_cast<volatile int*>(tholder + 2);  // (static smem would cap the dynamic 227 KB)
    const int cmax = p.m_blk >> 4;
    for (int i = 0; i < nseg; ++i) {
      const Seg sg = piece(i);
      const GemmParams& q = gp(sg);
      const int u = sg.u;
      const int unit_n0 = (u % q.n_tiles) * 256 + (int)r2 * 128, m_base = (u / q.n_tiles) * q.m_blk;
      const int ncol = unit_cols(q, u), nchunk = ncol >> 4;
      const int a = i % p.acc_stages;
      const bool whole = sg.k0 == 0 && sg.k1 == q.kb;
      fill_row_table(q, m_base, ncol, rtab, (int)threadIdx.x - 64);  // overlaps the MMAs
      mbar_wait(&tfull[a], (i / p.acc_stages) & 1);
      tc_fence_after();
      if (lane == 0 && qw == 0 && i < 3) DBG(6 + i);
      const uint32_t tl = tbase + ((uint32_t)(qw * 32) << 16) + (uint32_t)(a * p.m_blk);
      if (SPLIT == 3 && sg.ph) {
        // phase B: this k-split's fp32 partial of the down projection -> the next
        // RMSNorm (sums the S2 splits in order + residual), as EPI_PARTIAL
        const int sp = sg.k0 * fz->S2 / q.kb;
        if (unit_n0 < q.N) {
          float* dst = q.epi.part + (size_t)sp * q.epi.part_stride + unit_n0 + n;
          const bool rok = unit_n0 + n < q.N;
          for (int c = eg; c < nchunk; c += 2) {
            float v[16];
            tmem_ld16(tl + (uint32_t)(c * 16), v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int m = m_base + c * 16 + j;
              if (rok && m < q.M) dst[(size_t)m * q.epi.ldo] = v[j];  // a warp writes 128 contiguous bytes
            }
          }
        }
      } else if (whole) {
        for (int h = 0; h < H; ++h) {  // MMA h's 256 rows (H = 2: unit rows 512 t + 256 h)
          const int n0 = (u % q.n_tiles) * 256 * H + h * 256 + (int)r2 * 128;
          if (n0 >= p.N) break;
          const uint32_t tlh = tbase + ((uint32_t)(qw * 32) << 16) + (uint32_t)((a * H + h) * p.m_blk);
          for (int cc = eg * 16; cc < ncol; cc += 32) {
            float v[16];
            tmem_ld16(tlh + cc, v);
            apply_epilogue(p, n0, n, m_base + cc, v, xg, 1 + eg, rtab + cc);
          }
          if (lane == 0 && qw == 0 && eg == 0 && i == 0 && h == 0) DBG(15);  // (profiling) half 0 done
        }
      } else {
        // stream-K piece of a split unit: fp32 partial -> workspace slot (layout
        // [slot][row half][chunk][4 column quads][128 rows] float4, coalesced per warp)
        float4* dst = reinterpret_cast<float4*>(p.sk_ws) +
                      ((size_t)(sk_slot(p, pid, u) * 2 + (int)r2) * cmax) * 512 + n;
        int c = eg;
        for (; c + 2 < nchunk; c += 4) {  // two TMEM loads in flight per wait
          float va[16], vb[16];
          tmem_ld16x2(tl + (uint32_t)(c * 16), tl + (uint32_t)((c + 2) * 16), va, vb);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            __stcg(dst + (size_t)c * 512 + q4 * 128, make_float4(va[4 * q4], va[4 * q4 + 1], va[4 * q4 + 2], va[4 * q4 + 3]));
            __stcg(dst + (size_t)(c + 2) * 512 + q4 * 128,
                   make_float4(vb[4 * q4], vb[4 * q4 + 1], vb[4 * q4 + 2], vb[4 * q4 + 3]));
          }
        }
        for (; c < nchunk; c += 2) {
          float v[16];
          tmem_ld16(tl + (uint32_t)(c * 16), v);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            __stcg(dst + (size_t)c * 512 + q4 * 128, make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_l + 8u * a);  // TMEM buffer free: the next piece may accumulate
      if (lane == 0 && qw == 0 && i < 3) DBG(9 + i);
      if (SPLIT == 3 && !sg.ph) {
        // phase A: this CTA's act columns of unit u are stored -- count them into the
        // k-split of the down GEMM that reads them (release after a CTA barrier)
        fence_proxy_async_global();
        asm volatile("bar.sync 4, 256;" ::: "memory");
        if (w == 2 && lane == 0) {
          __threadfence();
          atomicAdd(fz->done + u / fz->a_per_split, 1);
        }
      }
      if (SPLIT == 2 && !whole) {
        // count the piece in; the CTA completing the count reduces the unit (this row half)
        int q0, q1;
        sk_unit_pairs(p, u, &q0, &q1);
        // CTA barrier, then one release by one thread (the CUTLASS semaphore pattern):
        // every epilogue thread's partial stores happen before the count
        asm volatile("bar.sync 4, 256;" ::: "memory");
        if (w == 2 && lane == 0) {
          __threadfence();
          const int old = atomicAdd(p.sk_cnt + 2 * u + (int)r2, 1);
          sh_last = old == q1 - q0;
          if (sh_last) {
            p.sk_cnt[2 * u + (int)r2] = 0;  // ready for the next launch
            __threadfence();
          }
        }
        asm volatile("bar.sync 4, 256;" ::: "memory");
        if (sh_last && unit_n0 < p.N) {
          for (int c = eg; c < nchunk; c += 2) {
            float v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = 0.f;
            // pair order = k order: deterministic.  Loads are issued in batches of
            // four pieces before the first add, so L2 latency is paid once per batch.
            for (int qb = q0; qb <= q1; qb += 4) {
              float4 x[4][4];
#pragma unroll
              for (int qq = 0; qq < 4; ++qq)
                if (qb + qq <= q1) {
                  const float4* src = reinterpret_cast<const float4*>(p.sk_ws) +
                                      ((size_t)(sk_slot(p, qb + qq, u) * 2 + (int)r2) * cmax + c) * 512 + n;
#pragma unroll
                  for (int q4 = 0; q4 < 4; ++q4) x[qq][q4] = ldcg_f4(src + q4 * 128);
                }
#pragma unroll
              for (int qq = 0; qq < 4; ++qq)
                if (qb + qq <= q1)
#pragma unroll
                  for (int q4 = 0; q4 < 4; ++q4) {
                    v[4 * q4] += x[qq][q4].x;
                    v[4 * q4 + 1] += x[qq][q4].y;
                    v[4 * q4 + 2] += x[qq][q4].z;
                    v[4 * q4 + 3] += x[qq][q4].w;
                  }
            }
            apply_epilogue(p, unit_n0, n, m_base + c * 16, v, xg, 1 + eg, rtab + c * 16);
          }
          if (w == 2 && lane == 0) DBG(15);
        }
      }
    }
    if (w == 2 && lane == 0) DBG(14);
  }

  if (SPLIT == 1) {
    // ------------------------------ split-K reduction: push partials to chunk owners
    const int u = cl;
    const int unit_n0 = (u % p.n_tiles) * 256 + (int)r2 * 128, m_base = (u / p.n_tiles) * p.m_blk;
    const int ncol = unit_cols(p, u), nchunk = ncol >> 4;
    const int cpr = ((p.m_blk >> 4) + p.S - 1) / p.S;  // receive slots per source pair
    const bool epi = w >= 2 && w <= 9;
    const int qw = w & 3, n = qw * 32 + lane, eg = (w - 2) >> 2;
    float* xg = xch + eg * kXchFloats;
    if (epi) {
      fill_row_table(p, m_base, ncol, rtab, (int)threadIdx.x - 64);
      mbar_wait(&tfull[0], 0);
      tc_fence_after();
      if (lane == 0 && qw == 0) DBG(6);
    }
    if (p.epi.kind == EPI_PARTIAL) {
      // hand the partial to the next RMSNorm (which sums the S splits in order and
      // adds the residual): no DSMEM exchange, no cluster barriers
      if (epi && unit_n0 < p.N) {
        const uint32_t tl = tbase + ((uint32_t)(qw * 32) << 16);
        float* dst = p.epi.part + (size_t)pi * p.epi.part_stride + unit_n0 + n;
        const bool rok = unit_n0 + n < p.N;
        for (int c = eg; c < nchunk; c += 2) {
          float v[16];
          tmem_ld16(tl + (uint32_t)(c * 16), v);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int m = m_base + c * 16 + j;
            if (rok && m < p.M) dst[(size_t)m * p.epi.ldo] = v[j];  // a warp writes 128 contiguous bytes
          }
        }
      }
    } else {
    cluster_sync_all();  // every CTA's mainloop is done: all rings may be overwritten
    if (threadIdx.x == 0) DBG(13);
    if (epi) {
      const uint32_t tl = tbase + ((uint32_t)(qw * 32) << 16);
      const uint32_t red_u32 = smem_u32(red);
      // chunk c is owned by pair j = the largest j with j * nchunk / S <= c
      auto push = [&](int c, const float (&v)[16]) {
        int j = (c * p.S) / nchunk;
        while (j + 1 < p.S && (j + 1) * nchunk / p.S <= c) ++j;
        while (j > 0 && j * nchunk / p.S > c) --j;
        const int cl0 = j * nchunk / p.S;
        const uint32_t dst = mapa_u32(red_u32, (uint32_t)(2 * j) + r2) +
                             (uint32_t)((((pi * cpr + (c - cl0)) * 4) * 128 + n) * 16);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          st_dsmem_f4(dst + (uint32_t)(q4 * 2048), make_float4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]));
      };
      int c = eg;
      for (; c + 2 < nchunk; c += 4) {  // two TMEM loads in flight per wait
        float va[16], vb[16];
        tmem_ld16x2(tl + (uint32_t)(c * 16), tl + (uint32_t)((c + 2) * 16), va, vb);
        push(c, va);
        push(c + 2, vb);
      }
      for (; c < nchunk; c += 2) {
        float v[16];
        tmem_ld16(tl + (uint32_t)(c * 16), v);
        push(c, v);
      }
    }
    cluster_sync_all();  // all partials delivered
    if (threadIdx.x == 0) DBG(14);
    if (epi && unit_n0 < p.N) {
      const int c0 = pi * nchunk / p.S, c1 = (pi + 1) * nchunk / p.S;
      RopePre pre_next;
      if (c0 + eg < c1) rope_prefetch(p, unit_n0, n, rtab + (c0 + eg) * 16, pre_next);
      for (int c = c0 + eg; c < c1; c += 2) {
        const RopePre pre = pre_next;
        if (c + 2 < c1) rope_prefetch(p, unit_n0, n, rtab + (c + 2) * 16, pre_next);  // one chunk ahead
        float v[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) v[jj] = 0.f;
        for (int src = 0; src < p.S; ++src) {  // pair order = k order: deterministic
          const float4* b = reinterpret_cast<const float4*>(red + (size_t)((src * cpr + (c - c0)) * 4) * 512) + n;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 x = b[q4 * 128];
            v[4 * q4] += x.x;
            v[4 * q4 + 1] += x.y;
            v[4 * q4 + 2] += x.z;
            v[4 * q4 + 3] += x.w;
          }
        }
        apply_epilogue(p, unit_n0, n, m_base + c * 16, v, xg, 1 + eg, rtab + c * 16, &pre);
      }
      if (w == 2 && lane == 0) DBG(15);
    }
    }  // EPI_PARTIAL else
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with the pair's TMEM before it is freed
  if (threadIdx.x == 0) DBG(12);
  if (w == 1) tmem_dealloc_pair(tbase, p.tmem_cols);
  if (SPLIT == 3 && threadIdx.x == 0) {
    // the last CTA out re-arms the split counters for the next launch (nobody waits
    // on them any more: every phase-B item of every CTA has been loaded)
    __threadfence();
    if (atomicAdd(fz->exit_ctr, 1) == (int)gridDim.x - 1) {
      for (int i = 0; i < fz->S2; ++i) fz->done[i] = 0;
      *fz->exit_ctr = 0;
      __threadfence();
    }
  }
}

template <int SPLIT>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p) {
  gemm_pair_body<SPLIT>(tmW, tmX, p, nullptr);
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_pair_mlp_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p,
                         const __grid_constant__ FuseArgs f) {
  gemm_pair_body<3>(tmW, tmX, p, &f);
}
