// kernels.hpp — internal (C++) launcher declarations for the sm_100a kernels.
// The public boundary is the C ABI in include/srl.h and include/srl_ops.h.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace srl {

// ---- gemm_tc.cu
int gemm_choose_splits(int M, int N, int K, int num_sms);
int gemm_bf16_partials(const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K, float* out,
                       int splits, cudaStream_t stream);

}  // namespace srl
