// kv_stream_bench.cu — the read ceiling of the paged attention's access pattern, without
// the math: 148 persistent CTAs pull (page, kv head) blocks of a paged KV cache into a
// 4-stage shared-memory ring with bulk async copies, work items (row, kv head) taken
// from a counter, pages of a row scattered over the pool (random permutation).
//   mode 0: K and V from separate pools, 16 KB each per stage (the engine's layout)
//   mode 1: K and V of a (page, head) adjacent: one 32 KB copy per stage
//   mode 2: mode 0 with the pages of each row consecutive in the pool
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2603_23414_b200/csrc \
//        tools/kv_stream_bench.cu -o /tmp/kv_stream_bench && /tmp/kv_stream_bench
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "common.cuh"

using namespace srl;

constexpr int kBlk = 64 * 128 * 2;  // one page x one head, K or V
constexpr int kHkv = 8;

__global__ void kv_stream_kernel(const uint8_t* kpool, const uint8_t* vpool, const int* page_list, const int* row_p0,
                                 const int* row_np, int n_items, int* ctr, int stages, int mode, unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * 2 * kBlk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned acc = 0;
  long long q = 0;  // stages issued
  long long done = 0;
  auto consume = [&]() {
    const int s = (int)(done % stages);
    mbar_wait(&full[s], (uint32_t)((done / stages) & 1));
    acc += sm[(size_t)s * 2 * kBlk + (done & 1023)];
    ++done;
  };
  for (;;) {
    const int it = atomicAdd(ctr, 1);
    if (it >= n_items) break;
    const int row = it / kHkv, h = it % kHkv;
    for (int p = 0; p < row_np[row]; ++p) {
      if (q - done >= stages) consume();
      const int s = (int)(q % stages);
      const int page = page_list[row_p0[row] + p];
      uint8_t* dst = sm + (size_t)s * 2 * kBlk;
      mbar_arrive_expect_tx(&full[s], 2 * kBlk);
      if (mode == 1) {
        bulk_g2s(dst, kpool + ((size_t)page * kHkv + h) * 2 * kBlk, 2 * kBlk, &full[s]);
      } else {
        bulk_g2s(dst, kpool + ((size_t)page * kHkv + h) * kBlk, kBlk, &full[s]);
        bulk_g2s(dst + kBlk, vpool + ((size_t)page * kHkv + h) * kBlk, kBlk, &full[s]);
      }
      ++q;
    }
  }
  while (done < q) consume();
  if (acc == 0xdeadbeef) sink[0] = acc;
}

int main() {
  const int rows = 256;
  std::mt19937 rng(1);
  std::lognormal_distribution<double> ln(std::log(1700.0), 0.55);
  std::vector<int> np(rows), p0(rows);
  int tot = 0;
  for (int r = 0; r < rows; ++r) {
    const int ctx = std::min(8192, std::max(2, (int)ln(rng)));
    np[r] = (ctx + 63) / 64;
  }
  std::sort(np.begin(), np.end(), [](int x, int y) { return x > y; });  // items longest first (LPT)
  for (int r = 0; r < rows; ++r) {
    p0[r] = tot;
    tot += np[r];
  }
  const int n_pages = tot + 16;
  std::vector<int> perm(n_pages), seq(n_pages);
  for (int i = 0; i < n_pages; ++i) perm[i] = seq[i] = i;
  std::shuffle(perm.begin(), perm.end(), rng);
  uint8_t *kp, *vp;
  cudaMalloc(&kp, (size_t)n_pages * kHkv * 2 * kBlk);
  cudaMalloc(&vp, (size_t)n_pages * kHkv * kBlk);
  cudaMemset(kp, 1, (size_t)n_pages * kHkv * 2 * kBlk);
  cudaMemset(vp, 1, (size_t)n_pages * kHkv * kBlk);
  int *d_perm, *d_seq, *d_p0, *d_np, *ctr;
  unsigned* sink;
  cudaMalloc(&d_perm, n_pages * 4);
  cudaMalloc(&d_seq, n_pages * 4);
  cudaMalloc(&d_p0, rows * 4);
  cudaMalloc(&d_np, rows * 4);
  cudaMalloc(&ctr, 64 * 4);
  cudaMalloc(&sink, 4);
  cudaMemcpy(d_perm, perm.data(), n_pages * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_seq, seq.data(), n_pages * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_p0, p0.data(), rows * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_np, np.data(), rows * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(kv_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  const double bytes = (double)tot * kHkv * 2 * kBlk;
  printf("pages %d (mean ctx %.0f), bytes per pass %.3f GB\nmode stages us GB/s\n", tot, tot * 64.0 / rows, bytes / 1e9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int stages : {4, 6}) {
      const size_t smem = 1024 + (size_t)stages * 2 * kBlk + 8 * stages;
      const int* pl = mode == 2 ? d_seq : d_perm;
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(e0);
        kv_stream_kernel<<<148, 32, smem>>>(kp, vp, pl, d_p0, d_np, rows * kHkv, ctr, stages, mode, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
      }
      printf("%d %d %.1f %.0f\n", mode, stages, best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
