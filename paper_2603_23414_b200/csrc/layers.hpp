// layers.hpp — launchers for layers.cu, attention.cu and sampler.cu.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace srl {

void rope_table(float* cos_t, float* sin_t, int max_pos, int dh, double theta, cudaStream_t st);
void embed_norm(const int* row_tok, const int* row_pos, int M, int d, const __nv_bfloat16* embed,
                const __nv_bfloat16* w, float eps, float* x_res, __nv_bfloat16* xn, cudaStream_t st);
void resid_norm(const float* P, int S, int M, int d, const int* row_pos, float* x_res, const __nv_bfloat16* w,
                float eps, __nv_bfloat16* xn, cudaStream_t st);
void silu_mul(const float* P, int S, int M, int ff, __nv_bfloat16* act, cudaStream_t st);
void reduce_splits(const float* P, int S, long long n, float* out, cudaStream_t st);

struct QkvEpiArgs {
  const float* P;  // [S][M][(Hq+2Hkv)*dh]
  int S, M;
  const __nv_bfloat16* bias;  // nullable
  const int* row_pos;         // [M] (-1 inactive)
  const int* row_slot;        // [M] local slot -> page-table row
  const int* page_table;
  int max_pages;
  const float* rope_cos;
  const float* rope_sin;
  void* q_out;    // [M][Hq][dh] bf16 (bf16 KV) or fp32 (fp32 KV)
  void* k_pool;   // this layer's K pool [pages][Hkv][64][dh]
  void* v_pool;
  int Hq, Hkv, dh;
};
void qkv_epilogue(const QkvEpiArgs& a, bool kv_fp32, cudaStream_t st);

// ---- attention.cu
// Work item = (row, kv head, chunk of kChunkPages pages).  The plan kernel
// builds the item list from row_pos (ctx = pos + 1).
constexpr int kChunkPages = 4;  // 256 tokens per work item
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
  int max_items;
  float scale;
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
  float invT;
  uint64_t seed;
  int* tok_out;          // [M]
  float* lp_out;         // [M]
};
void sample(const SampleArgs& a, cudaStream_t st);

}  // namespace srl
