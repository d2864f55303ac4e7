// gemm_epi.cuh — fused GEMM epilogues (included by gemm_tc.cu after GemmParams).
//
// A 16-column chunk of the accumulator arrives one weight row per thread
// (thread n <-> TMEM lane n, 16 batch rows in registers).  The SiLU-mul pairs the
// gate and up rows of an output with one warp shuffle (kGuBlock interleave: lanes l
// and l + 16 of a warp) and needs no exchange.  Every other epilogue first
// transposes the chunk through shared memory so that thread t then owns batch
// row m0 + t/8 and a run of 16 consecutive weight rows: the global writes become
// 16- or 64-byte vectors along the contiguous output dimension instead of 2- or
// 4-byte scalars strided by the row pitch.
#pragma once

// named barrier of one epilogue group (4 warps covering the 128 TMEM lanes)
__device__ __forceinline__ void epi_bar(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kEpiThreads)); }

// SiLU(g) * u with the hardware exp2 / reciprocal: |rel err| ~ 2^-21, far below
// the bf16 rounding of the stored activation; g -> -inf gives 0 (fdividef by inf).
// (An FMA-only Newton reciprocal, one MUFU op fewer, measured 2.4x slower here: the
// epilogue's 8 warps are issue / latency bound.)
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.f + __expf(-g)) * u; }

constexpr int kXchPitch = 132;                   // floats per staged batch row (128 + 4: conflict-free)
constexpr int kXchFloats = 16 * kXchPitch;  // one staged 16-column chunk

__device__ __forceinline__ void store16_bf16(__nv_bfloat16* dst, const float (&y)[16]) {
  uint4 a, b;
  a.x = pack_bf16(y[0], y[1]);
  a.y = pack_bf16(y[2], y[3]);
  a.z = pack_bf16(y[4], y[5]);
  a.w = pack_bf16(y[6], y[7]);
  b.x = pack_bf16(y[8], y[9]);
  b.y = pack_bf16(y[10], y[11]);
  b.z = pack_bf16(y[12], y[13]);
  b.w = pack_bf16(y[14], y[15]);
  reinterpret_cast<uint4*>(dst)[0] = a;
  reinterpret_cast<uint4*>(dst)[1] = b;
}
__device__ __forceinline__ void store16_f32(float* dst, const float (&y)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) reinterpret_cast<float4*>(dst)[q] = make_float4(y[4 * q], y[4 * q + 1], y[4 * q + 2], y[4 * q + 3]);
}

// vector reduction into global memory (fire-and-forget; .ftz: denormals flush)
__device__ __forceinline__ void red_add_f4(float* dst, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// EPI_QKV: (position, KV page) of each batch row of a unit, looked up once per
// unit into shared memory by the 256 epilogue threads (named barrier 3) so the
// per-chunk epilogue does no dependent global loads.  tab[0..m_blk) positions
// (-1 past M), tab[256..256+m_blk) pages.
constexpr int kRowTab = 512;
__device__ __forceinline__ void fill_row_table(const GemmParams& p, int m_base, int ncol, int* tab, int t) {
  const GemmEpi& e = p.epi;
  if (e.kind != EPI_QKV) return;
  asm volatile("bar.sync 3, 256;" ::: "memory");  // previous unit's epilogue is done with the table
  for (int r = t; r < ncol; r += 256) {
    const int m = m_base + r;
    const int pos = m < p.M ? __ldg(e.row_pos + m) : -1;
    tab[r] = pos;
    tab[256 + r] = pos >= 0 ? __ldg(e.page_table + (size_t)__ldg(e.row_slot + m) * e.max_pages + pos / 64) : 0;
  }
  asm volatile("bar.sync 3, 256;" ::: "memory");
}

// EPI_QKV: the RoPE cos / sin run (16 values each) this thread will need for the
// chunk whose batch rows start at m0_local (rows of the unit's row table): loaded
// one chunk ahead by the split-K reduction loop, so the L2 latency overlaps the
// previous chunk's epilogue instead of stalling every chunk.
struct RopePre {
  float4 c[4], s[4];
  bool ok;
};
__device__ __forceinline__ void rope_prefetch(const GemmParams& p, int unit_n0, int n, const int* rtab_chunk, RopePre& r) {
  const GemmEpi& e = p.epi;
  r.ok = false;
  if (e.kind != EPI_QKV) return;
  const int ml = n >> 3, nb = (n & 7) * 16, ng0 = unit_n0 + nb;
  const int pos = rtab_chunk[ml];
  const int dh = e.dh, half = dh / 2, h = ng0 / dh, i0 = ng0 % dh;
  if (pos < 0 || ng0 >= p.N || h >= e.Hq + e.Hkv) return;
  const int d0 = i0 < half ? i0 : i0 - half;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    r.c[q] = __ldg(reinterpret_cast<const float4*>(e.rope_cos + (size_t)pos * half + d0) + q);
    r.s[q] = __ldg(reinterpret_cast<const float4*>(e.rope_sin + (size_t)pos * half + d0) + q);
  }
  r.ok = true;
}

// ---------------------------------------------------------------- fused epilogue
// v[j]: value of weight row unit_n0 + n for batch row m0 + j, j < 16.
// pre: optional prefetched RoPE run for this chunk (EPI_QKV).
// xch: this group's shared staging buffer (kXchFloats); bar: its named barrier;
// rtab: the unit's row table (fill_row_table) advanced to row m0.
__device__ __forceinline__ void apply_epilogue(const GemmParams& p, int unit_n0, int n, int m0, const float (&v)[16],
                                               float* xch, int bar, const int* rtab, const RopePre* pre = nullptr) {
  const GemmEpi& e = p.epi;
  if (e.kind == EPI_SILU) {
    // kGuBlock = 16 interleave: lane l < 16 holds gate row j = l of this warp's 16
    // outputs, lane l + 16 the up row of the same output.  Lane l computes batch rows
    // m0 .. m0+7 of output j, lane l + 16 rows m0+8 .. m0+15: each sends the partner
    // the 8 values it needs (one xor-16 shuffle each).
    static_assert(kGuBlock == 16, "the epilogue pairs lanes l and l + 16");
    const int l = n & 31;
    const bool up = l >= 16;
    const int o = (unit_n0 >> 1) + (n >> 5) * 16 + (l & 15);  // act column (output)
    const int mb = m0 + (up ? 8 : 0);
    __nv_bfloat16* dst = e.act + (size_t)mb * e.ldo + o;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float mine = up ? v[8 + k] : v[k];
      const float other = __shfl_xor_sync(0xffffffffu, up ? v[k] : v[8 + k], 16);
      const float a = up ? silu_mul(other, mine) : silu_mul(mine, other);
      if (mb + k < p.M) dst[(size_t)k * e.ldo] = __float2bfloat16_rn(a);
    }
    return;
  }
  const int* spos = rtab;
  const int* spage = rtab + 256;
#pragma unroll
  for (int j = 0; j < 16; ++j) xch[j * kXchPitch + n] = v[j];
  epi_bar(bar);
  const int ml = n >> 3;  // batch row within the chunk owned from here on
  const int m = m0 + ml;
  const float* row = xch + ml * kXchPitch;
  {
    const int nb = (n & 7) * 16;  // first of the thread's 16 weight rows
    const int ng0 = unit_n0 + nb;
    float r[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 t = *reinterpret_cast<const float4*>(row + nb + 4 * q);
      r[4 * q] = t.x;
      r[4 * q + 1] = t.y;
      r[4 * q + 2] = t.z;
      r[4 * q + 3] = t.w;
    }
    if (m < p.M && ng0 < p.N) {
      const bool full = ng0 + 16 <= p.N;
      switch (e.kind) {
        case EPI_SAMPLE:
          if (!e.out_f32) break;
          [[fallthrough]];
        case EPI_F32: {
          float* dst = e.out_f32 + (size_t)m * e.ldo + ng0;
          if (full) {
            store16_f32(dst, r);
          } else {
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (ng0 + k < p.N) dst[k] = r[k];
          }
          break;
        }
        case EPI_RESID: {
          // exactly one contribution per element per launch, so a fire-and-forget
          // vector reduction equals the read-modify-write without its read latency
          float* dst = e.x_res + (size_t)m * e.ldo + ng0;
          if (full) {
#pragma unroll
            for (int q = 0; q < 4; ++q) red_add_f4(dst + 4 * q, r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
          } else {
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (ng0 + k < p.N) dst[k] += r[k];
          }
          break;
        }
        case EPI_QKV: {
          // rows [q heads | k heads | v heads] x dh; a 16-row run stays inside one
          // half of one head (dh/2 is a multiple of 16)
          const int pos = spos[ml];
          if (pos < 0) break;
          const int dh = e.dh, half = dh / 2;
          const int h = ng0 / dh, i0 = ng0 % dh;
          float y[16];
          if (e.bias) {
#pragma unroll
            for (int k = 0; k < 16; ++k) r[k] += __bfloat162float(e.bias[ng0 + k]);
          }
          if (h < e.Hq + e.Hkv) {
            // RoPE pairs (i, i + half): the partner run is read from the staged chunk
            const bool lo = i0 < half;
            const int d0 = lo ? i0 : i0 - half;                  // frequency index of r[0]
            const int pn = lo ? nb + half : nb - half;           // partner rows in the tile
            float c[16], s[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const bool have = pre && pre->ok;
              const float4 cq = have ? pre->c[q] : __ldg(reinterpret_cast<const float4*>(e.rope_cos + (size_t)pos * half + d0) + q);
              const float4 sq = have ? pre->s[q] : __ldg(reinterpret_cast<const float4*>(e.rope_sin + (size_t)pos * half + d0) + q);
              c[4 * q] = cq.x; c[4 * q + 1] = cq.y; c[4 * q + 2] = cq.z; c[4 * q + 3] = cq.w;
              s[4 * q] = sq.x; s[4 * q + 1] = sq.y; s[4 * q + 2] = sq.z; s[4 * q + 3] = sq.w;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              float x1 = row[pn + k];
              if (e.bias) x1 += __bfloat162float(e.bias[unit_n0 + pn + k]);
              // lo half: y = x*c - x_hi*s ; hi half: y = x*c + x_lo*s
              y[k] = lo ? r[k] * c[k] - x1 * s[k] : r[k] * c[k] + x1 * s[k];
            }
          } else {
#pragma unroll
            for (int k = 0; k < 16; ++k) y[k] = r[k];
          }
          size_t off;
          void* base;
          if (h < e.Hq) {
            off = ((size_t)m * e.Hq + h) * dh + i0;
            base = e.q_out;
          } else {
            const int kvh = h < e.Hq + e.Hkv ? h - e.Hq : h - e.Hq - e.Hkv;
            off = (((size_t)spage[ml] * e.Hkv + kvh) * 64 + pos % 64) * dh + i0;
            base = h < e.Hq + e.Hkv ? e.k_pool : e.v_pool;
          }
          if (e.kv_f32)
            store16_f32(reinterpret_cast<float*>(base) + off, y);
          else
            store16_bf16(reinterpret_cast<__nv_bfloat16*>(base) + off, y);
          break;
        }
      }
    }
  }
  if (e.kind == EPI_SAMPLE) {
    // Gumbel-max over this thread's 16 vocab rows of batch row m, then over the 8
    // lanes holding the same row (128 vocab rows): the exact-RN score only where a
    // cheap bound says it could win (gumbel.cuh); ties -> lowest index; the online
    // LSE of z * invT for the behaviour logprob
    const int nb = (n & 7) * 16, ng0 = unit_n0 + nb;
    float bs = -INFINITY, bz = 0.f, mx = -INFINITY, sum = 0.f;
    int bj = 0x7fffffff;
    if (m < p.M && e.s_row_pos[m] >= 0) {
      const uint32_t nt = (uint32_t)e.s_row_n[m], tj = (uint32_t)e.s_row_traj[m], rs = (uint32_t)e.s_row_restarts[m];
      const uint2 key = make_uint2((uint32_t)(e.s_seed & 0xffffffffu), (uint32_t)(e.s_seed >> 32));
      const float invT = e.s_invT;
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const int j4 = ng0 + 4 * q4;
        if (j4 >= p.N) break;
        const uint4 w = philox4x32_10(make_uint4((uint32_t)(j4 >> 2), nt, tj, rs), key);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = j4 + q;
          if (j >= p.N) break;
          const float z = row[nb + 4 * q4 + q];
          const float zs = __fmul_rn(z, invT);
          if (__fadd_rn(zs, gumbel_fast(ws[q])) + kPrune + 1e-6f * fabsf(bs) >= bs) {
            const float sc = __fadd_rn(zs, gumbel_from_bits(ws[q]));
            if (better(sc, j, bs, bj)) {
              bs = sc;
              bj = j;
              bz = z;
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
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const float os = __shfl_xor_sync(0xffffffffu, bs, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      const float oz = __shfl_xor_sync(0xffffffffu, bz, o);
      if (better(os, oj, bs, bj)) {
        bs = os;
        bj = oj;
        bz = oz;
      }
      const float om = __shfl_xor_sync(0xffffffffu, mx, o);
      const float osum = __shfl_xor_sync(0xffffffffu, sum, o);
      const float nm = fmaxf(mx, om);
      sum = (mx == -INFINITY ? 0.f : sum * expf(mx - nm)) + (om == -INFINITY ? 0.f : osum * expf(om - nm));
      mx = nm;
    }
    if ((n & 7) == 0 && m < p.M && unit_n0 < p.N) {
      const size_t idx = (size_t)m * e.s_nblk + (unit_n0 >> 7);
      e.s_part[idx] = make_float4(bs, bz, mx, sum);
      e.s_part_j[idx] = bj;
    }
  }
  epi_bar(bar);  // the staging buffer is reused by the next chunk
}
