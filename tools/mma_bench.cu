// mma_bench.cu — achievable tcgen05.mma (kind::f16, cta_group::1, M=128) rate per
// SM on this GPU, alone and with concurrent TMA writes into shared memory
// (the decode GEMM's smem traffic), to locate the GEMM mainloop's limiter.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2603_23414_b200/csrc \
//        tools/mma_bench.cu -o tools/mma_bench.bin && tools/mma_bench.bin
#include <cstdio>

#include "common.cuh"

using namespace srl;

// mode bit 0: a producer thread streams `wbytes` per k-block into a separate
// ring with bulk copies (from an L2-resident source) while the MMAs run.
__global__ void mma_kernel(int N, int kblocks, int mode, int wbytes, const uint8_t* src, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // operands: A ring 2 x 16 KB, B ring 2 x N*128 B; copy ring 2 x 48 KB after that
  uint8_t* sA = sm;
  uint8_t* sB = sm + 2 * 16384;
  uint8_t* sC = sB + 2 * N * 128;
  __shared__ uint64_t bars[4];
  __shared__ uint32_t holder;
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  if (w == 0) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = holder;
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, N);
    for (int k = 0; k < kblocks; ++k) {
      const int s = k & 1;
      const uint32_t a = smem_u32(sA + s * 16384), b = smem_u32(sB + s * N * 128);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_bf16(tbase + (k & 1) * 256, umma_desc_sw128(a + kk * 32), umma_desc_sw128(b + kk * 32), idesc,
                    kk > 0 ? 1u : 0u);
      if (mode & 2) {  // serial: commit + wait every k-block (MMA round-trip latency)
        tc_commit(&bars[0]);
        mbar_wait(&bars[0], k & 1);
      } else if ((k & 7) == 7) {  // bound the number of outstanding MMAs
        tc_commit(&bars[0]);
        mbar_wait(&bars[0], ((k >> 3) & 1));
      }
    }
    tc_commit(&bars[1]);
    mbar_wait(&bars[1], 0);
  } else if (threadIdx.x == 32 && (mode & 1)) {
    // concurrent smem writer: wbytes per k-block, two buffers, as fast as the MMAs go
    const int per = wbytes;
    for (int k = 0; k < kblocks; k += 2) {
      for (int j = 0; j < 2; ++j) {
        mbar_arrive_expect_tx(&bars[2 + j], per);
        bulk_g2s(sC + j * 49152, src + ((blockIdx.x * 7 + k + j) & 63) * 49152, per, &bars[2 + j]);
      }
      for (int j = 0; j < 2; ++j) mbar_wait(&bars[2 + j], (k >> 1) & 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (w == 0) tmem_dealloc(tbase, 512);
}

int main() {
  uint8_t* src;
  cudaMalloc(&src, 64 * 49152);
  cudaMemset(src, 0, 64 * 49152);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("N mode wbytes kblocks us TFLOP/s cycles_per_mma(avg CTA)\n");
  const int kblocks = 4096;
  for (int N : {256, 128, 64, 16}) {
    for (int mode : {0, 1, 2}) {
      for (int wb : {16384, 32768, 49152}) {
        if (mode != 1 && wb != 16384) continue;
        const size_t smem = 1024 + 2 * 16384 + 2 * (size_t)N * 128 + 2 * 49152;
        mma_kernel<<<148, 64, smem>>>(N, 64, mode, wb, src, out);
        cudaEventRecord(e0);
        mma_kernel<<<148, 64, smem>>>(N, kblocks, mode, wb, src, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        unsigned long long cyc[148];
        cudaMemcpy(cyc, out, sizeof(cyc), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += cyc[i] / 148.0;
        const double flops = 2.0 * 128 * N * 64 * (double)kblocks * 148;
        printf("%d %d %d %d %.1f %.0f %.1f\n", N, mode, mode == 1 ? wb : 0, kblocks, ms * 1e3, flops / (ms * 1e-3) / 1e12,
               avg / (kblocks * 4.0));
      }
    }
  }
  printf("status %s (clock %d MHz)\n", cudaGetErrorString(cudaGetLastError()), clk_khz / 1000);
  return 0;
}
