// kernels.hpp — internal (C++) launcher declarations for the sm_100a GEMM.
// The public boundary is the C ABI in include/srl.h and include/srl_ops.h.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace srl {

enum EpiKind { EPI_F32 = 0, EPI_RESID = 1, EPI_SILU = 2, EPI_QKV = 3, EPI_SAMPLE = 4, EPI_PARTIAL = 5 };

struct GemmEpi {
  int kind;
  int w_packed;               // W in the packed layout of pack_weight() (else row-major [N, K])
  int ldo;                    // row stride of out_f32 / x_res / act
  float* out_f32;             // EPI_F32
  float* x_res;               // EPI_RESID
  __nv_bfloat16* act;         // EPI_SILU
  // EPI_QKV
  const __nv_bfloat16* bias;  // nullable
  const int* row_pos;
  const int* row_slot;
  const int* page_table;
  int max_pages;
  const float* rope_cos;
  const float* rope_sin;
  void* q_out;
  void* k_pool;
  void* v_pool;
  int Hq, Hkv, dh, kv_f32;
  // EPI_PARTIAL (split-K pair GEMM only, see gemm_partial_split): CTA pair j of the
  // split writes its fp32 partial to part + j * part_stride as [M][ldo] -- the
  // residual add and the sum over splits are left to the next RMSNorm
  float* part;
  size_t part_stride;
  // EPI_SAMPLE (LM head): logits as EPI_F32 (out_f32, may be null) plus, per batch
  // row and 128-row vocab block, the Gumbel-max partial of the seeded sampler
  // (best score, its logit, its index, online max / sum of exp) -- sampler.cu's
  // sample_reduce finishes the row
  const int *s_row_pos, *s_row_n, *s_row_traj, *s_row_restarts;
  float s_invT;
  unsigned long long s_seed;
  float4* s_part;  // [M][s_nblk] {best score, its logit, max, sum}
  int* s_part_j;   // [M][s_nblk]
  int s_nblk;
  // GEMM workspace (gemm_workspace_bytes, zero-filled before first use; every
  // launch leaves it zeroed): stream-K partial slots + arrival counters.  Null
  // disables stream-K (cluster split-K / whole units instead).
  void* ws;
};

// gate / up row interleave of the SiLU-mul GEMM (EPI_SILU): blocks of kGuBlock gate
// rows then the kGuBlock up rows of the same outputs, so in every 32-row warp slice
// of a 128-row tile lanes l and l + 16 hold the two operands of one output (the
// epilogue pairs them with one shuffle, no shared-memory exchange)
constexpr int kGuBlock = 16;
constexpr size_t kSkSlotBytes = 128 * 256 * 4;  // one CTA's fp32 partial: 128 rows x <= 256 batch columns
constexpr int kSkMaxUnits = 8192;               // stream-K counters: pair units per launch
size_t gemm_workspace_bytes(int num_sms);
// The split-K factor S the pair GEMM will use for this shape (> 1: EPI_PARTIAL is
// available and leaves S partials), else 1.
int gemm_partial_split(int M, int N, int K, int num_sms);

// ---- gemm_tc.cu
// Y = X[M,K] . W[N,K]^T with the fused epilogue `epi` (for EPI_SILU, W's
// N rows are the interleaved gate/up rows: kGuBlock gate rows, then the matching
// kGuBlock up rows, per 2 kGuBlock-row block).  One kernel launch, no workspace: split-K partials
// are reduced over distributed shared memory inside a thread-block cluster.
// Returns 0, -1 (bad shape) or -2/-3 (TMA encode / launch failure).
int gemm_bf16_fused(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, const GemmEpi& epi,
                    int num_sms, cudaStream_t stream);
void gemm_set_debug(unsigned long long* buf, int target);
// The decode MLP as one persistent tcgen05 kernel (gemm_pair.cuh SPLIT 3): act =
// silu(X Wg^T) * (X Wu^T) (EPI_SILU, interleaved packed gate/up weights Wgu [2ff, d])
// and the S2 k-split fp32 partials of act Wd^T (packed Wd [d, ff]) written to
// part + s * part_stride as [M][d] (the next RMSNorm sums them in split order).
// ws: the GEMM workspace (zero-filled once; left zeroed).  Returns 0, 1 (not
// applicable: the caller runs the two GEMMs) or < 0 (encode / launch failure).
int gemm_mlp_fused(const __nv_bfloat16* X, int M, const void* Wgu, int ff, int d, __nv_bfloat16* act, const void* Wd,
                   float* part, size_t part_stride, int S2, void* ws, int num_sms, cudaStream_t stream);

// Packed weight layout for the GEMM's weight stream: [ceil(N/128)][K/64] blocks of
// 16 KB, block (t, k) = rows 128t..128t+127 x cols 64k..64k+63 stored exactly as
// the SWIZZLE_128B shared-memory image (row r at r*128 B, its 16-byte chunk c at
// chunk c ^ (r % 8)); rows past N are zero.  One block = one contiguous bulk copy.
size_t packed_weight_bytes(int N, int K);
int pack_weight(const __nv_bfloat16* src, int N, int K, void* dst, cudaStream_t stream);
// pack n source rows into the packed image, source row i landing on row
// (i / rb) * bs + off + i % rb (rows of the other rb-blocks are left as they are)
int pack_weight_rows(const __nv_bfloat16* src, int n, int K, void* dst, int rb, int bs, int off, cudaStream_t stream);

}  // namespace srl
