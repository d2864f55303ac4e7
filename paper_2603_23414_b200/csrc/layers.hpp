// layers.hpp — launchers for layers.cu, attention.cu and sampler.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace srl {

void rope_table(float* cos_t, float* sin_t, int max_pos, int dh, double theta, cudaStream_t st);
constexpr int kNormMaxSplits = 8;  // split-K partials one RMSNorm can sum
// RMSNorm of the fp32 residual rows into the bf16 GEMM operand; with `embed`
// non-null the residual row is first set to the embedding of row_tok[m].
// part (optional): nsplit fp32 partials [M][d] (part_stride floats apart) of the
// previous split-K GEMM (EPI_PARTIAL), summed in order and added to x_res first.
void rmsnorm(float* x_res, const int* row_tok, const int* row_pos, int M, int d, const __nv_bfloat16* embed,
             const __nv_bfloat16* w, float eps, __nv_bfloat16* y, cudaStream_t st, const float* part = nullptr,
             int nsplit = 0, size_t part_stride = 0);
struct NormRowArgs;
void rmsnorm(const NormRowArgs& a, int M, cudaStream_t st);

// QKV projection finish from split-K partials (see layers.cu)
struct QkvFinishArgs {
  const float* part;
  size_t part_stride;
  int nsplit;
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
};
void qkv_finish(const QkvFinishArgs& a, int M, cudaStream_t st);

// ---- attention.cu
// Work item = (row, kv head, chunk of kChunkPages pages).  The plan kernel
// builds the item list from row_pos (ctx = pos + 1).
constexpr int kChunkPages = 4;  // smallest split-KV chunk (pages); the plan kernel picks >= this
struct AttnArgs {
  const void* q;         // [M][Hq][dh] bf16 or fp32
  const void* k_pool;    // [pages][Hkv][64][dh]
  const void* v_pool;
  const int* row_pos;    // [M]
  const int* row_slot;   // [M]
  const int* page_table; // [Q_g][max_pages]
  int max_pages, M, Hq, Hkv, dh;
  int* items;            // [max_items][3] (row, head, chunk)
  int* n_items;          // device counter
  int* row_item0;        // [M] first item of the row
  int* row_nchunk;       // [M]
  float* part_o;         // [max_items][G][dh]
  float* part_ml;        // [max_items][G][2]
  __nv_bfloat16* out;    // [M][Hq*dh]
  float* out_f32;        // optional fp32 copy of out (op-level tests)
  int max_items;
  float scale;
  // bf16 kernel scheduling: items are taken longest-first (order, built by the
  // plan kernel) from a dynamic counter -- LPT over the persistent CTAs
  int* order;            // [max_items] item ids by descending page count
  int* work_ctr;         // this launch's counter; the plan kernel zeroes work_ctr[0..n_ctr)
  int n_ctr;
  int* merge_ctr;        // [M * Hkv] split-KV chunk arrivals (zeroed by the plan kernel, reset by the merger)
  int* chunk_pages;      // device int: split-KV chunk size in pages, chosen by the plan kernel
  int l2_prefetch;       // bf16 kernel: pages of L2 prefetch beyond the smem ring (0 = none)
  // fused QKV finish (bf16 kernel, pure decode passes): when qkv_part is set, the QKV
  // projection left its qkv_S split-K fp32 partials [qkv_S][M][Nqkv] and the item's
  // producer warp sums them (split order) + bias, applies RoPE at the row's position,
  // writes q (bf16, a.q) and -- the item holding the row's last page -- the new
  // token's k / v into that page before the page is loaded
  const float* qkv_part;
  size_t qkv_part_stride;
  int qkv_S, Nqkv;
  const __nv_bfloat16* qkv_bias;  // nullable
  const float* rope_cos;
  const float* rope_sin;
};
void attn_plan(const AttnArgs& a, int split, cudaStream_t st);
void attn_run(const AttnArgs& a, bool kv_fp32, const void* tmap_k, const void* tmap_v, cudaStream_t st);
void attn_combine_f32(const AttnArgs& a, float* out_f32, cudaStream_t st);
int attn_max_items(int M, int Hkv, int max_ctx);

// ---- sampler.cu
struct SampleArgs {
  const float* logits;   // [M][V]
  int M, V;
  const int* row_pos;    // [M] (-1 inactive)
  const int* row_n;      // [M] generated-token index
  const int* row_traj;   // [M]
  const int* row_restarts;
  const int* row_slot;   // [M] output index of row m (null: m itself; < 0: inactive, nothing written)
  float invT;
  uint64_t seed;
  int* tok_out;          // [M]
  float* lp_out;         // [M]
  int top_k;             // > 0: draw from the k best (logit desc, index asc) only
  float top_p;           // < 1: then from the shortest ranked prefix of mass >= top_p
};
// top_k > 0 or top_p < 1 runs sample_trunc_kernel (truncation set by radix select).
void sample(const SampleArgs& a, cudaStream_t st);
// Finish the rows whose Gumbel-max partials the LM-head GEMM produced (EPI_SAMPLE):
// part / part_j [M][nblk] in vocab-block order -> token and behaviour logprob.
void sample_reduce(const SampleArgs& a, const float4* part, const int* part_j, int nblk, cudaStream_t st);

}  // namespace srl
