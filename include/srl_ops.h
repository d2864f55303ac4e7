/* srl_ops.h — op-level C ABI of the SortedRL rollout hot path (sm_100a).
 *
 * These are the individual device steps that srl_decode_step (srl.h) chains;
 * they are exported so that tests can check each step against the CPU oracle
 * in isolation.  Conventions (same as srl.h):
 *   - every pointer argument is a DEVICE pointer unless its name ends in _host;
 *   - tensors are dense row-major, the last listed dimension contiguous;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *     asynchronous on that stream and never synchronise;
 *   - the return value is 0 on success, < 0 on a rejected argument or launch
 *     failure (see srl_last_error()); no output is written when < 0 is returned
 *     for an argument error.
 *   - memory is owned by the caller; nothing is retained after return.
 */
#ifndef SRL_OPS_H
#define SRL_OPS_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Decode projection GEMM with a fused epilogue (
 * PAPER.md P:110 §2.2 "frequent loading of model weights").  Y = X W^T with
 *   X [M, K] bf16, W [N, K] bf16 (a linear layer's weight), fp32 accumulation
 *   (tcgen05.mma kind::f16, accumulator in TMEM, operands staged by TMA,
 *   split-K only inside a thread-block cluster, reduced over DSMEM in a fixed
 *   order: bit-reproducible), and
 *   epi = 0: out fp32 [M, N]  = Y
 *   epi = 1: out fp32 [M, N] += Y                       (residual add)
 *   epi = 2: W has 2N rows, gate and up rows interleaved in 16-row blocks (rows
 *            [32b, 32b+16) = gate rows [16b, 16b+16), rows [32b+16, 32b+32) = the
 *            matching up rows: within a warp's 32 accumulator lanes the two operands
 *            of an output sit 16 lanes apart); out bf16 [M, N] = silu(Yg) * Yu
 * epi | SRL_GEMM_W_PACKED: W is in the packed layout written by srl_op_pack_weight
 *   (for epi 2: the packed image of the interleaved [2N, K] matrix) instead of
 *   row-major; the weight stream then moves contiguous 16 KB blocks.
 * workspace: device bytes >= srl_op_gemm_workspace(M, N, K, epi), ZERO-FILLED
 *   before its first use and not shared by concurrent launches; every launch
 *   leaves it zeroed.  It holds the stream-K fp32 partial slots and per-unit
 *   arrival counters (M >= 128, when whole units would leave SM pairs idle);
 *   NULL disables stream-K.
 * Requires K % 64 == 0 and, for epi 2, N % 64 == 0. */
#define SRL_GEMM_W_PACKED 0x100
int64_t srl_op_gemm_workspace(int32_t M, int32_t N, int32_t K, int32_t epi);
int32_t srl_op_gemm_bf16(const void* X, int32_t M, const void* W, int32_t N, int32_t K, int32_t epi, void* out,
                         void* workspace, void* stream);

/* The decode MLP (SURVEY §8(a) a8 + a9) as ONE persistent tcgen05 kernel, the
 * engine's path for 128 <= M <= 256 decode rows (srl_tuning.fuse_mlp):
 *   act  [M, ff] bf16 = silu(X Wg^T) * (X Wu^T)      (a8: the gate/up GEMM + SiLU-mul)
 *   part [splits][M, d] fp32, part[s] = act[:, ks] Wd[:, ks]^T over the s-th of
 *        `splits` equal k-ranges ks of ff               (a9: the down GEMM, k-split)
 * so that sum_s part[s] (in s order) = act Wd^T; the engine's next RMSNorm sums
 * them and adds the residual.  X [M, d] bf16 row-major; Wgu_packed = the packed
 * image (srl_op_pack_weight) of the interleaved [2ff, d] gate/up matrix (16 gate
 * rows then the matching 16 up rows per 32-row block, as epi 2 above); Wd_packed
 * = the packed image of Wd [d, ff].  workspace as srl_op_gemm_workspace (zeroed
 * before first use, left zeroed).  The down k-split s starts as soon as the
 * gate/up tiles producing its act columns are stored (device-scope counters).
 * Requires 128 <= M <= 256, d % 256 == 0, ff % (128 * splits) == 0, 1 <= splits
 * <= 8.  Returns 0, 1 (shape not supported by the fused kernel: nothing written)
 * or -1 (bad arguments / launch failure, srl_last_error()). */
int32_t srl_op_mlp_bf16(const void* X, int32_t M, const void* Wgu_packed, const void* Wd_packed, int32_t d, int32_t ff,
                        int32_t splits, void* act_out, float* part_out, void* workspace, void* stream);

/* Packed weight layout for srl_op_gemm_bf16 (and the engine's internal copy
 * of its projection weights; written by srl_load_policy_weights).  W [N, K] bf16
 * row-major -> dst of srl_op_packed_weight_bytes(N, K) bytes: blocks of 16 KB
 * ordered [ceil(N/128)][K/64]; block (t, k) holds rows 128t..128t+127 and columns
 * 64k..64k+63 exactly as the tcgen05 SWIZZLE_128B shared-memory image (row r at
 * byte r*128, its 16-byte chunk c at chunk position c ^ (r % 8)); rows >= N are
 * zero.  Requires K % 64 == 0.  srl_op_packed_weight_bytes returns -1 on bad
 * shapes. */
int64_t srl_op_packed_weight_bytes(int32_t N, int32_t K);
int32_t srl_op_pack_weight(const void* W, int32_t N, int32_t K, void* dst, void* stream);

/* Paged decode attention with GQA (PagedAttention).
 *   q          [M, Hq, dh]  bf16 (kv_fp32 = 0) or fp32 (kv_fp32 = 1)
 *   k_pool, v_pool [n_pages, Hkv, 64, dh] same dtype as q
 *   page_table [M, max_pages] int32: row r's token j lives in page page_table[r][j/64], row j%64
 *   row_pos    [M] int32: query position; ctx = row_pos+1 tokens are attended (row_pos < 0: output 0)
 *   out_f32    [M, Hq, dh] fp32: softmax_j(q . K_j / sqrt(dh)) V_j, query head h uses kv head h/(Hq/Hkv)
 *   workspace  device bytes >= srl_op_attention_workspace(M, Hq, Hkv, dh, max_ctx)
 * Requires dh in {32, 64, 128}, Hq/Hkv <= 8, max_ctx >= every ctx, max_pages*64 >= max_ctx. */
int64_t srl_op_attention_workspace(int32_t M, int32_t Hq, int32_t Hkv, int32_t dh, int32_t max_ctx);
int32_t srl_op_attention(const void* q, const void* k_pool, const void* v_pool, int32_t n_pages,
                         const int32_t* page_table, int32_t max_pages, const int32_t* row_pos, int32_t M,
                         int32_t Hq, int32_t Hkv, int32_t dh, int32_t kv_fp32, int32_t max_ctx, void* workspace,
                         float* out_f32, void* stream);

/* Seeded Gumbel-max sampling + log-probability.
 *   logits [M, V] fp32; per row r: n = row_n[r] (index of the generated token),
 *   traj = row_traj[r], restarts = row_restarts[r]; rows with row_active[r] < 0 are skipped
 *   (tok_out = -1).  tok_out[r] = argmax_j(z_j/T + Gumbel_j) with Gumbel_j from
 *   Philox4x32-10(key = seed, counter = (j>>2, n, traj, restarts))[j&3], ties -> lowest j;
 *   lp_out[r] = log softmax(z/T)[tok]. */
int32_t srl_op_sample(const float* logits, int32_t M, int32_t V, const int32_t* row_n, const int32_t* row_traj,
                      const int32_t* row_restarts, float temperature, uint64_t seed, const int32_t* row_active,
                      int32_t* tok_out, float* lp_out, void* stream);

/* The same with truncated sampling (srl_sched_cfg.top_k / top_p):
 * the argmax runs over the truncation set only -- the top_k best tokens by
 * (z/T desc, index asc) (0 = all), then the shortest ranked prefix whose mass
 * under their softmax reaches top_p (1 = all; the crossing token included) --
 * and lp_out is the log-probability under that truncated, renormalised
 * distribution.  The set is found by radix selection with integer fixed-point
 * masses (deterministic).  Errors: -1 for top_k < 0 or top_p outside (0, 1]. */
int32_t srl_op_sample_trunc(const float* logits, int32_t M, int32_t V, const int32_t* row_n, const int32_t* row_traj,
                            const int32_t* row_restarts, float temperature, uint64_t seed, int32_t top_k, float top_p,
                            const int32_t* row_active, int32_t* tok_out, float* lp_out, void* stream);

/* Thread-local description of the last error (never NULL). */
const char* srl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
