// pipe_bench.cu — minimal weight-streaming pipeline: a producer thread streams
// 16 KB blocks from HBM into a ring with bulk copies, a consumer thread either
// releases each stage directly (mode 0), or issues tcgen05.mma on it and
// releases it with tcgen05.commit (mode 1), or releases it with a commit but
// no MMA (mode 2).  Isolates what the MMA/commit release path costs the stream.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2603_23414_b200/csrc \
//        tools/pipe_bench.cu -o tools/pipe_bench.bin
#include <cstdio>

#include "common.cuh"

using namespace srl;

__global__ void pipe_kernel(const uint8_t* src, long long per_cta, int stages, int mode, int nmma, int N,
                            unsigned long long* out, int l2src) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sB = sm + stages * 16384;  // fixed B operand (max(N, 128) x 64 bf16)
  __shared__ uint64_t full[16], empty[16];
  __shared__ uint32_t holder;
  const int w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  if (w == 1) tmem_alloc(&holder, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = holder;
  const long long nblk = per_cta / 16384;
  const uint8_t* base = src + blockIdx.x * per_cta;
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0 && mode < 6) {
    for (long long q = 0; q < nblk; ++q) {
      const int s = (int)(q % stages);
      mbar_wait(&empty[s], (uint32_t)(((q / stages) & 1) ^ 1));
      mbar_arrive_expect_tx(&full[s], 16384);
      // l2src: every CTA re-reads the same 2 MB (L2-resident) instead of streaming HBM
      const uint8_t* from = l2src ? src + (q & 127) * 16384 : base + q * 16384;
      bulk_g2s(sm + s * 16384, from, 16384, &full[s]);
    }
  } else if (threadIdx.x == 32 && mode >= 6) {
    // mode 6: MMAs on the ring slots with no barrier waits (pure MMA issue rate), commit every 8
    // mode 7: same, but a full-barrier wait on each stage's data (the producer idles: mode 7 has
    //         no producer, so the waits are for data loaded once below)
    const uint32_t idesc = umma_idesc_bf16(128, N);
    for (long long q = 0; q < nblk; ++q) {
      const int s = (int)(q % stages);
      const uint32_t a = smem_u32(sm + s * 16384), b = smem_u32(sB);
      for (int kk = 0; kk < nmma; ++kk)
        tc_mma_bf16(tbase, umma_desc_sw128(a + kk * 32), umma_desc_sw128(b + kk * 32), idesc, kk > 0 ? 1u : 0u);
      if ((q & 7) == 7) {
        tc_commit(&empty[0]);
        mbar_wait(&empty[0], (uint32_t)((q >> 3) & 1));
      }
    }
  } else if (threadIdx.x == 32) {
    const uint32_t idesc = umma_idesc_bf16(128, N);
    for (long long q = 0; q < nblk; ++q) {
      const int s = (int)(q % stages);
      mbar_wait(&full[s], (uint32_t)((q / stages) & 1));
      if (mode == 0) {
        mbar_arrive(&empty[s]);
        continue;
      }
      tc_fence_after();
      // mode 1: MMA on the stage, commit releases it
      // mode 3: MMA on a FIXED A buffer (not the stage just written), commit releases
      // mode 4: MMA on the stage, released at once by a plain arrive (timing only)
      const uint32_t a = smem_u32(mode == 3 ? sB : sm + s * 16384), b = smem_u32(sB);
      if (mode == 5) {  // MMAs only every 4th stage
        if ((q & 3) == 0)
          for (int kk = 0; kk < nmma; ++kk)
            tc_mma_bf16(tbase, umma_desc_sw128(a + kk * 32), umma_desc_sw128(b + kk * 32), idesc, kk > 0 ? 1u : 0u);
        tc_commit(&empty[s]);
        continue;
      }
      for (int kk = 0; kk < nmma; ++kk)
        tc_mma_bf16(tbase, umma_desc_sw128(a + kk * 32), umma_desc_sw128(b + kk * 32), idesc, kk > 0 ? 1u : 0u);
      if (mode == 4)
        mbar_arrive(&empty[s]);
      else
        tc_commit(&empty[s]);
    }
    // drain
    const int s = (int)((nblk - 1) % stages);
    (void)s;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  if (w == 1) tmem_dealloc(tbase, 256);
}

int main() {
  const long long total = 1ll << 30;
  uint8_t* src[2];
  for (auto& b : src) {
    cudaMalloc(&b, total);
    cudaMemset(b, 0, total);
  }
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("grid MB_per_cta stages mode nmma N us GB/s(total) GB/s(per CTA)\n");
  for (int l2src : {1})
  for (int grid : {148, 74}) {
    const long long per_cta = grid == 148 ? (1ll << 20) : (2ll << 20);  // 148 MB either way
    for (int stages : {12}) {
      for (int mode : {0, 1, 6}) {
        for (int nmma : {4}) {
          for (int N : {16}) {
            if (mode == 0 && N != 16) continue;
            const size_t smem = 1024 + (size_t)stages * 16384 + 16384;
            for (int i = 0; i < 2; ++i)
              pipe_kernel<<<grid, 64, smem>>>(src[i & 1], per_cta, stages, mode, nmma, N, out, l2src);
            const int it = 10;
            cudaEventRecord(e0);
            for (int i = 0; i < it; ++i) pipe_kernel<<<grid, 64, smem>>>(src[i & 1], per_cta, stages, mode, nmma, N, out, l2src);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / it;
            unsigned long long cyc[148];
            cudaMemcpy(cyc, out, sizeof(cyc), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; ++i) avg += (double)cyc[i] / grid;
            printf("l2src=%d %d %.1f %d %d %d %d %.2f %.0f %.1f  cyc/stage %.0f  eff_MHz %.0f\n", l2src, grid, per_cta / 1048576.0,
                   stages, mode, nmma, N, us, grid * per_cta / (us * 1e-6) / 1e9, per_cta / (us * 1e-6) / 1e9,
                   avg / (per_cta / 16384), avg / us);
          }
        }
      }
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
