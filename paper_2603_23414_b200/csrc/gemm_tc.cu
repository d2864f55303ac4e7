// gemm_tc.cu — weight-streaming decode GEMM on tcgen05 tensor cores (sm_100a).
//
// Computes P[s][m][n] = sum_{k in split s} X[m][k] * W[n][k]   (fp32 partials)
// for the projection / MLP / LM-head contractions of the decode step
// (the paper's cost statement P:110
// "throughput is primarily constrained by limited HBM bandwidth, due to
// frequent loading of model weights").
//
// Swap-AB: the weight tile (128 rows of W) is the UMMA "A"/M side and the
// ragged decode batch X (M_b <= 256 rows, multiple of 16) is the UMMA "B"/N
// side, so a batch of 1..256 sequences always issues M=128 tcgen05.mma and
// the accumulator (128 lanes x M_b fp32 columns) lives in TMEM.
// One CTA = one (128-row weight tile, 256-row batch block, K split).
// Warp roles: w0 = TMA producer, w1 = TMEM allocator + single-thread MMA
// issuer, w2..w5 = epilogue (tcgen05.ld -> coalesced fp32 stores).
// K-split partials are reduced in a fixed order by the epilogue kernels
// (epilogue.cu), so results are bit-reproducible run to run.
#include "common.cuh"
#include "kernels.hpp"
#include "tma.hpp"

namespace srl {

struct GemmParams {
  int M, N, K;
  int m_blk;  // batch rows per CTA: multiple of 16, <= 256
  int n_tiles, m_blocks, splits, kb_total, stages, tmem_cols;
  float* out;  // [splits][M][N]
};

static constexpr int kStageA = 128 * 128;  // 128 weight rows x 64 bf16 (128 B)

__global__ void __launch_bounds__(192, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                        GemmParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int stage_b = p.m_blk * 128;
  uint8_t* sA = smem;
  uint8_t* sB = smem + p.stages * kStageA;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + p.stages * stage_b);
  uint64_t* empty = full + p.stages;
  uint64_t* tfull = empty + p.stages;
  uint32_t* tholder = reinterpret_cast<uint32_t*>(tfull + 1);

  const int bid = blockIdx.x;
  const int nt = bid % p.n_tiles;
  const int rest = bid / p.n_tiles;
  const int mb = rest % p.m_blocks;
  const int sp = rest / p.m_blocks;
  const int kb0 = (int)((long long)sp * p.kb_total / p.splits);
  const int kb1 = (int)((long long)(sp + 1) * p.kb_total / p.splits);
  const int nkb = kb1 - kb0;
  const int n0 = nt * 128, m0 = mb * p.m_blk;
  int nmma = p.M - m0;
  nmma = nmma > p.m_blk ? p.m_blk : nmma;
  nmma = (nmma + 15) & ~15;

  const int w = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
  }
  if (w == 1) tmem_alloc(tholder, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tholder;

  if (w == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
      const uint64_t pol_x = policy_evict_last();   // activations: re-read by every tile
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (i / p.stages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], kStageA + stage_b);
        tma_load_2d_hint(sA + s * kStageA, &tmW, &full[s], (kb0 + i) * 64, n0, pol_w);
        tma_load_2d_hint(sB + s * stage_b, &tmX, &full[s], (kb0 + i) * 64, m0, pol_x);
      }
    }
  } else if (w == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_bf16(128, nmma);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % p.stages;
        const uint32_t ph = (i / p.stages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a = smem_u32(sA + s * kStageA), b = smem_u32(sB + s * stage_b);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc_mma_bf16(tbase, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), idesc,
                      (i | k) != 0);
        tc_commit(&empty[s]);  // frees the smem stage when these MMAs retire
      }
      tc_commit(tfull);
    }
    __syncwarp();
  } else {
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int q = w & 3;  // TMEM lane quarter this warp may access
    const int n = n0 + q * 32 + lane;
    float* out = p.out + (size_t)sp * p.M * p.N;
    for (int c = 0; c < nmma; c += 16) {
      float v[16];
      tmem_ld16(tbase + ((uint32_t)(q * 32) << 16) + c, v);
      if (n < p.N) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int m = m0 + c + j;
          if (m < p.M) out[(size_t)m * p.N + n] = v[j];
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 1) tmem_dealloc(tbase, p.tmem_cols);
}

int gemm_choose_splits(int M, int N, int K, int num_sms) {
  const int n_tiles = (N + 127) / 128;
  const int m_blocks = (M + 255) / 256;
  const int units = n_tiles * m_blocks;
  const int kb = K / 64;
  int best = 1;
  double best_eff = 0;
  for (int s = 1; s <= 16 && s <= kb; ++s) {
    const long long ctas = (long long)units * s;
    const long long waves = (ctas + num_sms - 1) / num_sms;
    const double eff = (double)ctas / (double)(waves * num_sms);
    if (eff > best_eff + 0.03) {
      best_eff = eff;
      best = s;
    }
    if (units * s >= 4 * num_sms) break;
  }
  return best;
}

int gemm_bf16_partials(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, float* out,
                       int splits, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return 0;
  if (K % 64 != 0 || splits < 1 || splits > K / 64) return -1;
  static bool attr_set = false;
  GemmParams p;
  p.M = M;
  p.N = N;
  p.K = K;
  int mb = M < 256 ? M : 256;
  p.m_blk = (mb + 15) & ~15;
  p.n_tiles = (N + 127) / 128;
  p.m_blocks = (M + p.m_blk - 1) / p.m_blk;
  p.splits = splits;
  p.kb_total = K / 64;
  const int stage_bytes = kStageA + p.m_blk * 128;
  int stages = (200 * 1024) / stage_bytes;
  if (stages > 8) stages = 8;
  p.stages = stages;
  int tc = 32;
  while (tc < p.m_blk) tc <<= 1;
  p.tmem_cols = tc;
  p.out = out;
  CUtensorMap tmW, tmX;
  if (tma_encode_2d(&tmW, W, N, K, (uint64_t)K * 2, 128, 64, 2, true)) return -2;
  if (tma_encode_2d(&tmX, X, M, K, (uint64_t)K * 2, p.m_blk, 64, 2, true)) return -2;
  const size_t smem = 1024 + (size_t)stages * stage_bytes + (2 * stages + 1) * 8 + 16;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_bf16_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  const int grid = p.n_tiles * p.m_blocks * splits;
  gemm_bf16_tc_kernel<<<grid, 192, smem, stream>>>(tmW, tmX, p);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace srl
