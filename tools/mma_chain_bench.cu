// mma_chain_bench.cu — tcgen05.mma (M=128, K=16, cta_group::1) issue cost as a
// function of the accumulation dependency structure: C independent accumulators,
// interleaved per k-block (4 MMAs) or per MMA, with a commit (+ wait) every
// `cev` k-blocks.  Operands are static in shared memory (no TMA).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2603_23414_b200/csrc \
//        tools/mma_chain_bench.cu -o tools/mma_chain_bench.bin
#include <cstdio>

#include "common.cuh"

using namespace srl;

__global__ void chain_kernel(int N, int C, int per_mma, int cev, int kblocks, unsigned long long* out, int fresh, int balt) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = holder;
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N);
    const int cols = 512 / C;
    int ph = 0;
    for (int k = 0; k < kblocks; ++k) {
      const uint32_t a = smem_u32(sm + (k & (balt ? 1 : 3)) * 16384);
      const uint32_t b = smem_u32(sm + 65536 + (balt ? (k & 1) * N * 128 : 0));
      if (per_mma) {
        // MMA j of the k-block goes to accumulator j % C
        for (int kk = 0; kk < 4; ++kk)
          tc_mma_bf16(tbase + (kk % C) * cols, umma_desc_sw128(a + kk * 32), umma_desc_sw128(b + kk * 32), idesc,
                      (k > 0 || kk >= C) ? 1u : 0u);
      } else {
        const uint32_t acc = tbase + (k % C) * cols;
        for (int kk = 0; kk < 4; ++kk)
          tc_mma_bf16(acc, umma_desc_sw128(a + kk * 32), umma_desc_sw128(b + kk * 32), idesc,
                      ((k >= C && !fresh) || kk > 0) ? 1u : 0u);
      }
      if ((k % cev) == cev - 1) {
        tc_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, ph);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (threadIdx.x < 32) tmem_dealloc(tbase, 512);
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  const size_t smem = 1024 + 65536 + 65536;
  cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  printf("N C per_mma commit_every cycles_per_mma\n");
  const int kblocks = 2048;
  printf("(fresh balt) prefix\n");
  for (int fresh : {0, 1})
  for (int balt : {0, 1})
  for (int N : {16, 256})
    for (int C : {1, 2})
      for (int per_mma : {0})
        for (int cev : {8}) {
          if (C * N > 512) continue;
          chain_kernel<<<148, 64, smem>>>(N, C, per_mma, cev, 64, out, fresh, balt);
          chain_kernel<<<148, 64, smem>>>(N, C, per_mma, cev, kblocks, out, fresh, balt);
          cudaDeviceSynchronize();
          unsigned long long cyc[148];
          cudaMemcpy(cyc, out, sizeof(cyc), cudaMemcpyDeviceToHost);
          double avg = 0;
          for (int i = 0; i < 148; ++i) avg += cyc[i] / 148.0;
          printf("fresh=%d balt=%d  %d %d %d %d %.1f\n", fresh, balt, N, C, per_mma, cev, avg / (kblocks * 4.0));
        }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
