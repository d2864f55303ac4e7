// kernels.hpp — internal (C++) launcher declarations for the sm_100a GEMM.
// The public boundary is the C ABI in include/srl.h and include/srl_ops.h.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace srl {

enum EpiKind { EPI_F32 = 0, EPI_RESID = 1, EPI_SILU = 2, EPI_QKV = 3 };

struct GemmEpi {
  int kind;
  int w_blocked;              // W stored tile-blocked [N/128][K/64][128][64] (each TMA box contiguous)
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
};

// ---- gemm_tc.cu
// Y = X[M,K] . W[N,K]^T with the fused epilogue `epi` (for EPI_SILU, W holds
// 2N rows: gate rows [0,N) then up rows [N,2N)).  ws / counters: workspace of
// gemm_workspace_bytes(M, nt, num_sms) bytes and gemm_counter_count(M, N)
// zero-initialised ints (left zeroed on return).
int gemm_bf16_fused(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, const GemmEpi& epi,
                    float* ws, int* counters, int num_sms, cudaStream_t stream);
size_t gemm_workspace_bytes(int M, int nt, int num_sms);
size_t gemm_counter_count(int M, int N_units_rows);

}  // namespace srl
