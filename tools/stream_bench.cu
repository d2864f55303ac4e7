// stream_bench.cu — ground truth for weight streaming on this GPU: how fast can
// G CTAs pull B bytes from HBM into a shared-memory ring with bulk async
// copies (the GEMM's weight producer without the math)?
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2603_23414_b200/csrc \
//        tools/stream_bench.cu -o /tmp/stream_bench && /tmp/stream_bench
#include <cstdio>
#include <vector>

#include "common.cuh"
#include "tma.hpp"

using namespace srl;

__global__ void stream_kernel(const uint8_t* src, long long total, int chunk, int stages, int contiguous,
                              unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long nch = total / chunk;
  long long c0, cn, stride;
  if (contiguous) {
    c0 = nch * blockIdx.x / gridDim.x;
    cn = nch * (blockIdx.x + 1) / gridDim.x - c0;
    stride = 1;
  } else {
    c0 = blockIdx.x;
    cn = blockIdx.x < nch ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    stride = gridDim.x;
  }
  unsigned acc = 0;
  const long long pre = cn < stages ? cn : stages;
  for (long long i = 0; i < pre; ++i) {
    mbar_arrive_expect_tx(&full[i], chunk);
    bulk_g2s(sm + i * chunk, src + (c0 + i * stride) * chunk, chunk, &full[i]);
  }
  for (long long i = 0; i < cn; ++i) {
    const int s = (int)(i % stages);
    mbar_wait(&full[s], (uint32_t)((i / stages) & 1));
    acc += sm[s * chunk + (i & 1023)];
    const long long nx = i + stages;
    if (nx < cn) {
      mbar_arrive_expect_tx(&full[s], chunk);
      bulk_g2s(sm + s * chunk, src + (c0 + nx * stride) * chunk, chunk, &full[s]);
    }
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

// the GEMM's weight access: 2-D TMA boxes [128 rows x 64 cols] of a row-major [N, K] bf16
// matrix, CTA-persistent over 128-row tiles, k-blocks in order within a tile
__global__ void stream2d_kernel(const __grid_constant__ CUtensorMap tm, int n_tiles, int kb, int stages, int box_rows,
                                unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int chunk = box_rows * 128;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int nt = blockIdx.x < n_tiles ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const long long cn = (long long)nt * kb;
  unsigned acc = 0;
  auto issue = [&](long long i, int s) {
    const int t = blockIdx.x + (int)(i / kb) * gridDim.x, k = (int)(i % kb);
    mbar_arrive_expect_tx(&full[s], chunk);
    tma_load_2d(sm + s * chunk, &tm, &full[s], k * 64, t * box_rows);
  };
  for (long long i = 0; i < cn && i < stages; ++i) issue(i, (int)i);
  for (long long i = 0; i < cn; ++i) {
    const int s = (int)(i % stages);
    mbar_wait(&full[s], (uint32_t)((i / stages) & 1));
    acc += sm[s * chunk + (i & 1023)];
    if (i + stages < cn) issue(i + stages, s);
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
  const long long kBuf = 1ll << 30;  // rotate over 4 x 1 GiB: nothing stays in L2
  std::vector<uint8_t*> bufs(4);
  for (auto& b : bufs) {
    cudaMalloc(&b, kBuf);
    cudaMemset(b, 1, kBuf);
  }
  unsigned* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const long long totals[] = {33554432ll, 117440512ll, 234881024ll, 1050673152ll};
  const int grids[] = {148, 128, 112, 96, 74};
  const int rings[][2] = {{16384, 4}, {16384, 8}, {16384, 12}, {32768, 6}, {32768, 4}, {65536, 3}};
  printf("total_MB grid chunk_KB stages contiguous us GB/s\n");
  for (long long total : totals)
    for (int g : grids)
      for (auto& r : rings)
        for (int contig = 0; contig < 2; ++contig) {
          const size_t smem = 1024 + (size_t)r[0] * r[1] + 8 * r[1];
          const int it = total > 500000000ll ? 8 : 24;
          for (int i = 0; i < 3; ++i)
            stream_kernel<<<g, 32, smem>>>(bufs[i % 4], total, r[0], r[1], contig, sink);
          cudaEventRecord(e0);
          for (int i = 0; i < it; ++i)
            stream_kernel<<<g, 32, smem>>>(bufs[i % 4], total, r[0], r[1], contig, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double us = ms * 1e3 / it;
          printf("%.1f %d %d %d %d %.2f %.0f\n", total / 1048576.0, g, r[0] / 1024, r[1], contig, us,
                 total / (us * 1e-6) / 1e9);
        }
  cudaFuncSetAttribute(stream2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  printf("2d: N K grid box_rows stages us GB/s\n");
  const int shapes[][2] = {{4096, 4096}, {6144, 4096}, {28672, 4096}, {4096, 14336}, {128256, 4096}};
  for (auto& sh : shapes)
    for (int g : {148, 128, 112})
      for (int br : {128, 256})
        for (int st : {4, 8, 12}) {
          if (br * 128 * st > 200 * 1024) continue;
          std::vector<CUtensorMap> tms(4);
          for (int i = 0; i < 4; ++i) srl::tma_encode_2d(&tms[i], bufs[i], sh[0], sh[1], (uint64_t)sh[1] * 2, br, 64, 2, true);
          const size_t smem = 1024 + (size_t)br * 128 * st + 8 * st;
          const int n_tiles = sh[0] / br, kb = sh[1] / 64;
          const long long total = (long long)sh[0] * sh[1] * 2;
          const int it = 16;
          for (int i = 0; i < 3; ++i) stream2d_kernel<<<g, 32, smem>>>(tms[i % 4], n_tiles, kb, st, br, sink);
          cudaEventRecord(e0);
          for (int i = 0; i < it; ++i) stream2d_kernel<<<g, 32, smem>>>(tms[i % 4], n_tiles, kb, st, br, sink);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double us = ms * 1e3 / it;
          printf("2d %d %d %d %d %d %.2f %.0f\n", sh[0], sh[1], g, br, st, us, total / (us * 1e-6) / 1e9);
        }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
