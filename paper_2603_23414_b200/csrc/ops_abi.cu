// ops_abi.cu — extern "C" op-level entry points (include/srl_ops.h).
#include <atomic>
#include <cstdio>
#include <string>

#include "kernels.hpp"
#include "srl_ops.h"
#include "tuning.hpp"

namespace srl {
thread_local std::string g_last_error = "ok";
void set_error(const char* fmt, const char* a = "", long b = 0) {
  char buf[512];
  snprintf(buf, sizeof(buf), fmt, a, b);
  g_last_error = buf;
}
}  // namespace srl

using namespace srl;

extern "C" const char* srl_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------------ tuning
namespace srl {
static const srl_tuning kDefaultTuning = {
    /*gemm_split*/ 1, /*gemm_pair*/ -1, /*gemm_h*/ 0, /*gemm_stages*/ 0, /*gemm_xstages*/ 0,
    /*partial_norm*/ 1, /*partial_small_m*/ 0, /*qkv_finish*/ 0, /*fused_sample*/ 0,
    /*attn_min_items*/ 0, /*attn_target_items*/ 0, /*attn_l2_prefetch*/ 0,
    /*pdl*/ 1, /*graphs*/ 1, /*mixed_prefill*/ 1, /*verbose*/ 0, /*fuse_mlp*/ 0, /*mlp_splits*/ 8,
    /*attn_stages*/ 4, /*qkv_attn*/ 1, /*pair_h2*/ 1};
srl_tuning g_tuning = kDefaultTuning;

bool once_per_device(int slot) {
  static std::atomic<unsigned long long> done[kOnceSlots];
  int dev = 0;
  cudaGetDevice(&dev);
  if (slot < 0 || slot >= kOnceSlots || dev < 0 || dev >= 64) return true;
  const unsigned long long bit = 1ull << dev;
  return (done[slot].fetch_or(bit) & bit) == 0;
}
}  // namespace srl

extern "C" void srl_default_tuning(srl_tuning* t) {
  if (!t) return;
  *t = srl::kDefaultTuning;
}

extern "C" int32_t srl_get_tuning(srl_tuning* t) {
  if (!t) {
    set_error("srl_get_tuning: %s", "null argument", 0);
    return -1;
  }
  *t = g_tuning;
  return 0;
}

extern "C" int32_t srl_set_tuning(const srl_tuning* t) {
  if (!t) {
    set_error("srl_set_tuning: %s", "null argument", 0);
    return -1;
  }
  if (t->gemm_split < 0 || t->gemm_split > 3 || t->gemm_pair < -1 || t->gemm_pair > 1 || t->gemm_h < 0 ||
      t->gemm_h > 2 || t->gemm_stages < 0 || t->gemm_xstages < 0 || t->attn_min_items < 0 ||
      t->attn_target_items < 0 || t->attn_l2_prefetch < 0 || t->attn_l2_prefetch > 16 || t->mlp_splits < 1 ||
      t->mlp_splits > 8 || (t->attn_stages != 3 && t->attn_stages != 4 && t->attn_stages != 6) || t->pair_h2 < 0 || t->pair_h2 > 1) {
    set_error("srl_set_tuning: %s", "field out of range", 0);
    return -1;
  }
  g_tuning = *t;
  return 0;
}

static int op_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

namespace srl {
void gemm_set_debug(unsigned long long* buf, int target);
}
// Profiling hook (not part of the public headers): per-CTA phase timestamps of
// the `target`-th GEMM launch after the call.
extern "C" void srl_debug_gemm_timestamps(unsigned long long* dev_buf, int32_t target) {
  srl::gemm_set_debug(dev_buf, target);
}

extern "C" int64_t srl_op_gemm_workspace(int32_t M, int32_t N, int32_t K, int32_t epi) {
  epi &= ~SRL_GEMM_W_PACKED;
  if (M <= 0 || N <= 0 || K <= 0 || epi < 0 || epi > 2) return -1;
  (void)K;
  return (int64_t)gemm_workspace_bytes(op_sms());
}

extern "C" int32_t srl_op_gemm_bf16(const void* X, int32_t M, const void* W, int32_t N, int32_t K, int32_t epi,
                                    void* out, void* workspace, void* stream) {
  const int packed = (epi & SRL_GEMM_W_PACKED) ? 1 : 0;
  epi &= ~SRL_GEMM_W_PACKED;
  if (M <= 0 || N <= 0 || K <= 0 || K % 64 || epi < 0 || epi > 2 || (epi == 2 && N % 64)) {
    set_error("srl_op_gemm_bf16: %s", "bad shape / epilogue", 0);
    return -1;
  }
  const int sms = op_sms();
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  GemmEpi e{};
  e.w_packed = packed;
  e.kind = epi == 0 ? EPI_F32 : (epi == 1 ? EPI_RESID : EPI_SILU);
  e.ldo = N;
  e.out_f32 = reinterpret_cast<float*>(out);
  e.x_res = reinterpret_cast<float*>(out);
  e.act = reinterpret_cast<__nv_bfloat16*>(out);
  e.ws = workspace;
  const int rows = epi == 2 ? 2 * N : N;  // SiLU-mul: interleaved gate/up rows
  int r = gemm_bf16_fused(reinterpret_cast<const __nv_bfloat16*>(X), M, reinterpret_cast<const __nv_bfloat16*>(W),
                          rows, K, e, sms, st);
  if (r) set_error("srl_op_gemm_bf16: %s (code %ld)", r == -1 ? "bad shape" : "launch/tma failure", r);
  return r;
}

extern "C" int32_t srl_op_mlp_bf16(const void* X, int32_t M, const void* Wgu_packed, const void* Wd_packed, int32_t d,
                                   int32_t ff, int32_t splits, void* act_out, float* part_out, void* workspace,
                                   void* stream) {
  if (!X || !Wgu_packed || !Wd_packed || !act_out || !part_out || !workspace || M <= 0 || d <= 0 || ff <= 0 ||
      splits < 1 || splits > 8) {
    set_error("srl_op_mlp_bf16: %s", "bad arguments", 0);
    return -1;
  }
  const int r = gemm_mlp_fused(reinterpret_cast<const __nv_bfloat16*>(X), M, Wgu_packed, ff, d,
                               reinterpret_cast<__nv_bfloat16*>(act_out), Wd_packed, part_out, (size_t)M * d, splits,
                               workspace, op_sms(), reinterpret_cast<cudaStream_t>(stream));
  if (r < 0) {
    set_error("srl_op_mlp_bf16: %s (code %ld)", "launch/tma failure", r);
    return -1;
  }
  return r;
}

extern "C" int64_t srl_op_packed_weight_bytes(int32_t N, int32_t K) {
  if (N <= 0 || K <= 0 || K % 64) return -1;
  return (int64_t)packed_weight_bytes(N, K);
}

extern "C" int32_t srl_op_pack_weight(const void* W, int32_t N, int32_t K, void* dst, void* stream) {
  if (!W || !dst || N <= 0 || K <= 0 || K % 64) {
    set_error("srl_op_pack_weight: %s", "bad shape / null pointer", 0);
    return -1;
  }
  const int r = pack_weight(reinterpret_cast<const __nv_bfloat16*>(W), N, K, dst, reinterpret_cast<cudaStream_t>(stream));
  if (r) set_error("srl_op_pack_weight: %s (code %ld)", "launch failure", r);
  return r;
}

// ---------------------------------------------------------------- attention op
#include "layers.hpp"
#include "tma.hpp"

static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

static size_t attn_ws_layout(int M, int Hq, int Hkv, int dh, int max_ctx, size_t* offs) {
  const int G = Hq / Hkv;
  const int items = attn_max_items(M, Hkv, max_ctx);
  size_t o = 0;
  offs[0] = o; o += al256(12ull * items);            // items
  offs[1] = o; o += al256(64);                        // n_items
  offs[2] = o; o += al256(4ull * M);                  // row_item0
  offs[3] = o; o += al256(4ull * M);                  // row_nchunk
  offs[4] = o; o += al256(4ull * items * G * dh);     // part_o
  offs[5] = o; o += al256(8ull * items * G);          // part_ml
  offs[6] = o; o += al256(2ull * M * Hq * dh);        // bf16 out
  offs[7] = o; o += al256(4ull * M);                  // row_slot identity
  offs[8] = o; o += al256(4ull * items);              // order
  offs[9] = o; o += al256(64);                        // work counter
  offs[10] = o; o += al256(4ull * M * Hkv);           // split-KV merge counters
  offs[11] = o; o += al256(64);                       // chunk size
  return o;
}

extern "C" int64_t srl_op_attention_workspace(int32_t M, int32_t Hq, int32_t Hkv, int32_t dh, int32_t max_ctx) {
  size_t offs[12];
  if (M <= 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || dh <= 0 || max_ctx <= 0) return -1;
  return (int64_t)attn_ws_layout(M, Hq, Hkv, dh, max_ctx, offs);
}

__global__ void iota_kernel(int* p, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i;
}

extern "C" int32_t srl_op_attention(const void* q, const void* k_pool, const void* v_pool, int32_t n_pages,
                                    const int32_t* page_table, int32_t max_pages, const int32_t* row_pos, int32_t M,
                                    int32_t Hq, int32_t Hkv, int32_t dh, int32_t kv_fp32, int32_t max_ctx,
                                    void* workspace, float* out_f32, void* stream) {
  if (M <= 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || Hq / Hkv > 8 || (dh != 32 && dh != 64 && dh != 128) ||
      n_pages <= 0 || max_ctx <= 0 || max_pages * 64 < max_ctx) {
    set_error("srl_op_attention: %s", "bad shape", 0);
    return -1;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  size_t offs[12];
  attn_ws_layout(M, Hq, Hkv, dh, max_ctx, offs);
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  AttnArgs a{};
  a.q = q;
  a.k_pool = k_pool;
  a.v_pool = v_pool;
  a.row_pos = row_pos;
  a.row_slot = reinterpret_cast<int*>(ws + offs[7]);
  a.page_table = page_table;
  a.max_pages = max_pages;
  a.M = M;
  a.Hq = Hq;
  a.Hkv = Hkv;
  a.dh = dh;
  a.items = reinterpret_cast<int*>(ws + offs[0]);
  a.n_items = reinterpret_cast<int*>(ws + offs[1]);
  a.row_item0 = reinterpret_cast<int*>(ws + offs[2]);
  a.row_nchunk = reinterpret_cast<int*>(ws + offs[3]);
  a.part_o = reinterpret_cast<float*>(ws + offs[4]);
  a.part_ml = reinterpret_cast<float*>(ws + offs[5]);
  a.out = reinterpret_cast<__nv_bfloat16*>(ws + offs[6]);
  a.out_f32 = out_f32;
  a.max_items = attn_max_items(M, Hkv, max_ctx);
  a.scale = 1.0f / sqrtf((float)dh);
  a.order = reinterpret_cast<int*>(ws + offs[8]);
  a.work_ctr = reinterpret_cast<int*>(ws + offs[9]);
  a.n_ctr = 1;
  a.merge_ctr = reinterpret_cast<int*>(ws + offs[10]);
  a.chunk_pages = reinterpret_cast<int*>(ws + offs[11]);
  iota_kernel<<<(M + 255) / 256, 256, 0, st>>>(const_cast<int*>(a.row_slot), M);
  CUtensorMap tk, tv;
  if (!kv_fp32) {
    const uint32_t bc = dh < 64 ? dh : 64;
    const uint64_t rows = (uint64_t)n_pages * Hkv * 64;
    if (tma_encode_2d(&tk, k_pool, rows, dh, (uint64_t)dh * 2, 64, bc, 2, bc == 64) ||
        tma_encode_2d(&tv, v_pool, rows, dh, (uint64_t)dh * 2, 64, bc, 2, bc == 64)) {
      set_error("srl_op_attention: %s", "TMA encode failed", 0);
      return -2;
    }
  }
  attn_plan(a, 1, st);
  attn_run(a, kv_fp32 != 0, &tk, &tv, st);
  attn_combine_f32(a, out_f32, st);
  if (cudaGetLastError() != cudaSuccess) {
    set_error("srl_op_attention: %s", "launch failure", 0);
    return -3;
  }
  return 0;
}

// ---------------------------------------------------------------- sampler op
extern "C" int32_t srl_op_sample(const float* logits, int32_t M, int32_t V, const int32_t* row_n,
                                 const int32_t* row_traj, const int32_t* row_restarts, float temperature,
                                 uint64_t seed, const int32_t* row_active, int32_t* tok_out, float* lp_out,
                                 void* stream) {
  if (M < 0 || V <= 0 || !(temperature > 0.f)) {
    set_error("srl_op_sample: %s", "bad arguments", 0);
    return -1;
  }
  SampleArgs a{};
  a.logits = logits;
  a.M = M;
  a.V = V;
  a.row_pos = row_active;
  a.row_n = row_n;
  a.row_traj = row_traj;
  a.row_restarts = row_restarts;
  a.invT = 1.0f / temperature;
  a.seed = seed;
  a.tok_out = tok_out;
  a.lp_out = lp_out;
  a.top_k = 0;
  a.top_p = 1.f;
  sample(a, reinterpret_cast<cudaStream_t>(stream));
  if (cudaGetLastError() != cudaSuccess) {
    set_error("srl_op_sample: %s", "launch failure", 0);
    return -3;
  }
  return 0;
}

extern "C" int32_t srl_op_sample_trunc(const float* logits, int32_t M, int32_t V, const int32_t* row_n,
                                       const int32_t* row_traj, const int32_t* row_restarts, float temperature,
                                       uint64_t seed, int32_t top_k, float top_p, const int32_t* row_active,
                                       int32_t* tok_out, float* lp_out, void* stream) {
  if (M < 0 || V <= 0 || !(temperature > 0.f) || top_k < 0 || !(top_p > 0.f && top_p <= 1.f)) {
    set_error("srl_op_sample_trunc: %s", "bad arguments", 0);
    return -1;
  }
  SampleArgs a{};
  a.logits = logits;
  a.M = M;
  a.V = V;
  a.row_pos = row_active;
  a.row_n = row_n;
  a.row_traj = row_traj;
  a.row_restarts = row_restarts;
  a.invT = 1.0f / temperature;
  a.seed = seed;
  a.tok_out = tok_out;
  a.lp_out = lp_out;
  a.top_k = top_k;
  a.top_p = top_p;
  sample(a, reinterpret_cast<cudaStream_t>(stream));
  if (cudaGetLastError() != cudaSuccess) {
    set_error("srl_op_sample_trunc: %s", "launch failure", 0);
    return -3;
  }
  return 0;
}
