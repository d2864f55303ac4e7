/* srl.h — C ABI of the SortedRL rollout engine (B200 / sm_100a).
 *
 * The engine runs the rollout phase of SortedRL (arXiv 2603.23414): batched
 * autoregressive decode of a policy under online length-aware continuous
 * batching, with the paper's stateful controller and rollout buffer.
 * Citations "P:n" are PAPER.md line numbers; "Rn" are DESIGN.md readings.
 *
 *   srl_submit_prompts      feed the dataloader stream (P:147 step 1)
 *   srl_decode_step         one global decode step: refill free slots from the
 *                           pending queue (oversubscription), decode,
 *                           sample, stop-detect, compact finished sequences into
 *                           the rollout buffer, early-terminate when an update
 *                           group is ready
 *   srl_harvest_finished    the length-sorted update group (selective batching,
 *                           P:177) with tokens + behaviour logprobs
 *   srl_load_policy_weights refresh the policy after an update and apply the
 *                           off-policy cache bound K
 *
 * Conventions
 *   - Every call returns int32: SRL_OK (0), an informational status (> 0), or
 *     an error (< 0).  srl_last_error() describes the last error of the
 *     calling thread.  No C++ exception crosses this boundary.
 *   - One engine per GPU per process; an engine is NOT thread-safe (single
 *     owner).
 *   - Host arrays passed IN are copied before the call returns.  OUT arrays are
 *     caller-owned with an explicit capacity; counts are returned separately.
 *   - Device memory is allocated by the caller (the Python wrapper, via torch)
 *     and lent to the engine for its lifetime (srl_arena); the engine never
 *     frees it.  Sizes come from srl_arena_sizes().  `stream` is a
 *     cudaStream_t owned by the caller.
 *   - srl_decode_step, srl_harvest_finished and srl_load_policy_weights
 *     synchronise `stream` before returning (their results are host values).
 */
#ifndef SRL_H
#define SRL_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes */
#define SRL_OK 0
#define SRL_GROUP_READY 1 /* an update group is ready: harvest, then load weights */
#define SRL_DONE 2        /* stream exhausted and every trajectory emitted */
#define SRL_E_INVALID_ARG (-1)
#define SRL_E_STATE (-2)     /* call not allowed in the current state */
#define SRL_E_EMPTY (-3)     /* nothing submitted */
#define SRL_E_CAPACITY (-4)  /* buffer / KV pool too small */
#define SRL_E_DUPLICATE_ID (-5)
#define SRL_E_CUDA (-6)
#define SRL_E_NCCL (-7)

/* ---- enums */
/* SORTED: SortedRL.  SYNC: the synchronous baseline -- batches of
 * Q_tot admitted together, groups of U in completion order.  POSTHOC:
 * the paper's post-hoc sorting ablation -- a pool of pool_prompts*G
 * trajectories generated with refill, then, once ALL of it has finished, sorted
 * groups of U (the last group is |pool|/U - 1 versions stale). */
enum { SRL_MODE_SORTED = 0, SRL_MODE_SYNC = 1, SRL_MODE_POSTHOC = 2 };
enum { SRL_RESUME_KEEP_KV = 0, SRL_RESUME_REPREFILL = 1 };   /* reading R10 */
enum { SRL_BARRIER_TRAINED = 0, SRL_BARRIER_ADMITTED = 1 };  /* reading R8 */
enum { SRL_STOP_FORCED = 0, SRL_STOP_EOS = 1 };              /* reading R16 */
enum { SRL_KV_BF16 = 0, SRL_KV_FP32 = 1 };

/* Policy shape (LLaMA-3.1 / Qwen-2.5 family; reading R19). */
typedef struct srl_model_cfg {
  int32_t L, d, Hq, Hkv, dh, ff, V;
  float rope_theta, rms_eps;
  int32_t qkv_bias; /* Qwen-2.5 has q/k/v biases */
  /* 1: the weight region holds the projection matrices ONLY in the GEMM's packed
   * layout (no row-major staging copy: about half the bytes, what lets a
   * 65 GB Qwen-2.5-32B policy and its KV cache share one GPU).  Those tensors
   * are then installed with srl_load_policy_tensor and srl_weight_layout /
   * srl_weight_offset do not address them.  Needs Hq*dh, Hkv*dh % 128 == 0. */
  int32_t weights_compact;
} srl_model_cfg;

/* Scheduler.  Q_g slots per GPU, Q_tot = R * Q_g ("Q").
 * U   update-group size
 * K   cache bound in policy versions; -1 = infinity.  K = 0 is the paper's fully
 *     on-policy mode, K = -1 its partial mode; reading R9.
 * pool_prompts  n*b prompts loaded per epoch, G responses per prompt.
 * cap           max generation length; page_tokens must be 64.
 * kv_pages      KV pages per GPU; max_traj capacity of the trajectory table;
 * max_prompt    longest prompt accepted; prefill_chunk rows per prefill pass. */
typedef struct srl_sched_cfg {
  int32_t Q_g, U, K, pool_prompts, G, cap, page_tokens, kv_pages;
  int32_t mode, resume, barrier, stop, eos_id, kv_dtype;
  float temperature;
  uint64_t sample_seed;
  int32_t max_traj, max_prompt, prefill_chunk;
  /* N4 truncated sampling: top_k > 0 draws from the k best tokens (logit desc,
   * index asc); top_p < 1 then from the shortest ranked prefix of the top-k
   * softmax whose mass reaches top_p.  The cached behaviour logprob is that of
   * the truncated, renormalised distribution.  0 / 1 = off (R14). */
  int32_t top_k;
  float top_p;
  /* N4 prompt-prefix KV sharing (G > 1; P:235 several responses per prompt, P:387
   * RadixAttention): the full KV pages of prompt positions [0, prompt_len - 1) --
   * what every sample of a prompt prefills -- are held once per replica and
   * prompt, refcounted, and only shared with samples admitted under the policy
   * version they were computed with; a later sample prefills from the first
   * unshared position.  Page accounting = oracle/sched.py _prefix_pages.  0 / 1. */
  int32_t share_prefix;
  /* N1 chunked prefill (Sarathi; prompt ++ kept tokens on resume):
   * at most prefill_budget prefill positions per replica per step, served strictly
   * in admission order; a slot decodes from the step its prefill completes (reading
   * R30; oracle/sched.py _prefill).  0 = unlimited (every admission is prefilled in
   * its own step, R13).  Exclusive with share_prefix. */
  int32_t prefill_budget;
} srl_sched_cfg;

/* Data-parallel replicas (rows a14, a17).  R = world engines run
 * the SAME global step in lockstep: every rank holds the full (replicated)
 * controller state, decodes only its own slots g = s*R + rank, and after the
 * sampler an in-place all-gather of every replica's [Q_g] (token, logprob) rows
 * lets every rank run the identical controller END (stop, compaction, sorted
 * emission).  srl_load_policy_weights broadcasts rank 0's policy in place.
 * kind:
 *   SRL_COMM_NCCL   one process per GPU; nccl_unique_id from srl_nccl_unique_id
 *                   on rank 0, shared by the caller (e.g. torch.distributed);
 *                   world may be 1 (a one-rank communicator: same code path).
 *                   The communicator is created non-blocking and polled.
 *   SRL_COMM_LOCAL  `world` engines in one process, each driven by its own host
 *                   thread (any devices, several may share one GPU); local_group
 *                   from srl_local_group_create(world), destroyed after every
 *                   engine of the group.  Peer copies + CUDA events + a host
 *                   barrier.
 *   SRL_COMM_HOST   caller callbacks (`host`, an srl_host_transport that must
 *                   outlive the engine): rows staged through pinned host memory,
 *                   exchanged by the caller -- e.g. over a torch.distributed gloo
 *                   group, several processes sharing one GPU.  Slow; for tests
 *                   and GPU-less interconnects.
 * Failure handling: timeout_s (0 = 300 s) bounds communicator creation and every
 * wait on a step / update that contains a collective.  An asynchronous transport
 * error (ncclCommGetAsyncError) or a timeout aborts the communicator
 * (ncclCommAbort) and the call returns SRL_E_NCCL; every later call on that
 * engine returns SRL_E_NCCL too (destroy it).  A dead peer therefore fails the
 * surviving ranks instead of hanging them.
 * All ranks must make the same sequence of srl_submit_prompts /
 * srl_decode_step / srl_harvest_finished / srl_load_policy_weights calls. */
enum { SRL_COMM_NCCL = 0, SRL_COMM_LOCAL = 1, SRL_COMM_HOST = 2 };
/* SRL_COMM_HOST callbacks; return 0 on success, non-zero on failure.
 *   allgather(ctx, buf, seg): buf holds world segments of seg bytes; this rank's
 *     segment (offset rank*seg) is filled; on return every segment must hold its
 *     owner's bytes.
 *   broadcast(ctx, buf, bytes): rank 0's buf holds `bytes` bytes; on return every
 *     rank's buf must hold them. */
typedef struct srl_host_transport {
  int32_t (*allgather)(void* ctx, void* buf, uint64_t seg_bytes);
  int32_t (*broadcast)(void* ctx, void* buf, uint64_t bytes);
  void* ctx;
} srl_host_transport;
typedef struct srl_comm {
  int32_t rank, world;
  int32_t kind, timeout_s;
  void* local_group;
  const srl_host_transport* host;
  uint8_t nccl_unique_id[128];
} srl_comm;

/* Device memory lent by the caller, sized by srl_arena_sizes. */
typedef struct srl_arena {
  void* weights;  /* flat policy weights, layout from srl_weight_offset */
  void* kv;       /* KV cache pool */
  void* scratch;  /* activations, partials, controller state, buffers */
  uint64_t weights_bytes, kv_bytes, scratch_bytes;
} srl_arena;

typedef struct srl_step_info {
  int64_t k;          /* global step index of the step just run (-1 if none) */
  int32_t r_k;        /* running requests in that step (Eq. (bubble)) */
  int32_t n_finished; /* trajectories finished in that step */
  int32_t n_ready;    /* ready (finished, not emitted) trajectories */
  int32_t n_admitted; /* admissions in that step (all replicas) */
  int32_t n_prefill_tokens; /* prefill tokens processed on this GPU */
  int32_t v;          /* current policy version */
  float dt_ms;        /* device time of the step on this GPU (cudaEvent) */
  int64_t sum_ctx;    /* sum over this GPU's running rows of the attended context (KV tokens read per layer) */
  int32_t r_local;    /* running rows decoded on this GPU in that step (r_k counts all replicas) */
  int32_t pad_;
} srl_step_info;

/* Per-kernel-class device timing (CUDA events on the engine stream), enabled by
 * srl_set_profiling.  Classes: */
enum { SRL_K_GEMM_QKV = 0, SRL_K_GEMM_O = 1, SRL_K_GEMM_GU = 2, SRL_K_GEMM_DOWN = 3, SRL_K_LM_HEAD = 4,
       SRL_K_ATTN = 5, SRL_K_ELEMWISE = 6, SRL_K_SAMPLE = 7, SRL_K_CTL = 8, SRL_K_PREFILL = 9,
       SRL_K_COMM = 10 /* replica all-gather + weight broadcast */, SRL_K_NCLASS = 11 };

/* One harvested trajectory (SPEC BufferEntry / P:199). */
typedef struct srl_traj {
  int64_t prompt_id;   /* the caller's prompt id */
  int64_t tok_offset;  /* offset of its tokens in the caller's toks/logprobs/versions */
  int32_t traj_id, sample, len;
  int32_t v_first, v_last, finish_step, lifecycle, restarts;
  int32_t final_group; /* 1 when this is the epoch's final (possibly short) group */
  int32_t epoch;
} srl_traj;

/* Trace records: kind 0 = step (a = k, b = r_k); events (P:338 trace). */
enum { SRL_EV_STEP = 0, SRL_EV_LOAD = 1, SRL_EV_ADMIT = 2, SRL_EV_PREEMPT = 3, SRL_EV_FINISH = 4,
       SRL_EV_EMIT = 5, SRL_EV_DISCARD = 6, SRL_EV_SCAVENGE = 7, SRL_EV_EMIT_MEMBER = 8 };
typedef struct srl_trace_rec {
  int32_t kind, a, b, c, d, e;
} srl_trace_rec;
/* Field meaning per kind:
 *   STEP        a=k, b=r_k
 *   LOAD        a=k, b=epoch, c=first traj_id, d=count
 *   ADMIT       a=k, b=global slot, c=traj_id, d=kept tokens
 *   PREEMPT     a=k, b=global slot, c=traj_id, d=tokens kept (0/1)
 *   FINISH      a=k, b=global slot, c=traj_id, d=length
 *   EMIT        a=group index, b=version, c=count, d=final flag   (followed by c EMIT_MEMBER)
 *   EMIT_MEMBER a=group index, b=position in group, c=traj_id
 *   DISCARD     a=version, b=traj_id, c=where (1 pending, 2 running, 3 ready)
 *   SCAVENGE    a=version, b=traj_id, c=global slot */

typedef struct srl_engine srl_engine;

/* Byte sizes of the three arena regions for a configuration (weights = the
 * staging image of srl_weight_layout followed by the packed GEMM copies, see
 * srl_load_policy_weights).  Returns < 0 for
 * an invalid configuration (Q_g <= 0, U > pool*G in SORTED mode, ...). */
int32_t srl_arena_sizes(const srl_model_cfg* m, const srl_sched_cfg* s, int32_t world, uint64_t* weights_bytes,
                        uint64_t* kv_bytes, uint64_t* scratch_bytes);

/* Byte offset (of row 0) and element count of a named weight tensor inside the
 * flat weight region ("embed", "lm_head", "final_norm", "L<i>.wq", "L<i>.wk",
 * "L<i>.wv", "L<i>.bq", "L<i>.bk", "L<i>.bv", "L<i>.wo", "L<i>.attn_norm",
 * "L<i>.mlp_norm", "L<i>.wg", "L<i>.wu", "L<i>.wd"), bf16, in the shape of a
 * linear layer's weight [out, in].  Returns -1 if unknown.  All tensors are
 * dense row-major EXCEPT wg / wu, whose rows are interleaved in 16-row blocks
 * (see srl_weight_layout). */
int64_t srl_weight_offset(const srl_model_cfg* m, const char* name, int64_t* numel);

/* Full placement of a named tensor: row i (of `rows`, each `cols` bf16 elements)
 * starts at byte offset + ((i / row_block) * block_stride + i % row_block) * cols * 2.
 * Dense tensors have row_block = block_stride = rows.  L<i>.wg / L<i>.wu have
 * row_block = 16, block_stride = 32: each 32-row block of the gate/up region
 * holds 16 gate rows followed by the 16 up rows of the same outputs, so one
 * 128-row tensor-core tile carries both operands of the fused SiLU-mul and each
 * warp's 32 accumulator lanes hold both operands of 16 outputs. */
int32_t srl_weight_layout(const srl_model_cfg* m, const char* name, int64_t* offset, int64_t* rows, int64_t* cols,
                          int64_t* row_block, int64_t* block_stride);

int32_t srl_create(const srl_model_cfg* m, const srl_sched_cfg* s, int32_t device, void* stream,
                   const srl_arena* mem, const srl_comm* comm /* NULL => R = 1 */, srl_engine** out);
int32_t srl_destroy(srl_engine* e);

/* Append n prompts to the stream.  Prompt i has tokens toks[tok_off[i] .. tok_off[i+1])
 * (host arrays); trajectory ids are prompt_index*G + sample in submission order.
 * forced_len[n*G] (host; required in FORCED stop mode, each in [1, cap]).
 * All ranks must submit identical lists.  Errors: SRL_E_DUPLICATE_ID,
 * SRL_E_INVALID_ARG, SRL_E_CAPACITY (max_traj / prompt storage exceeded). */
int32_t srl_submit_prompts(srl_engine* e, int32_t n, const uint64_t* prompt_ids, const int32_t* tok_off,
                           const int32_t* toks, const int32_t* forced_len);

/* One global decode step.  Returns SRL_OK, SRL_GROUP_READY, SRL_DONE, or
 * SRL_E_STATE (a group awaits harvest/load, or no weights loaded),
 * SRL_E_EMPTY, SRL_E_CAPACITY.  `info` (optional) receives the step summary. */
int32_t srl_decode_step(srl_engine* e, srl_step_info* info);

/* Copy out the ready update group: records in group order (ascending
 * (len, traj_id) in SORTED mode; completion order in SYNC mode), and the
 * concatenated tokens / behaviour logprobs / generating policy versions.
 * Returns SRL_E_STATE when no group is ready and SRL_E_CAPACITY (nothing
 * consumed) when cap_recs or cap_toks is too small. */
int32_t srl_harvest_finished(srl_engine* e, int32_t cap_recs, srl_traj* recs, int32_t* n_out, int32_t* toks,
                             float* logprobs, int32_t* versions, int64_t cap_toks);

/* Device views of the group the last srl_harvest_finished copied out (the same
 * data: tokens / behaviour logprobs / generating versions concatenated in group
 * order, and the records with prompt_id = the engine's prompt index), for a
 * trainer on the same GPU (srl_learner.h) without a host round trip.  Valid
 * until the next srl_harvest_finished (also across srl_load_policy_weights);
 * *n_tok = total tokens.  SRL_E_STATE if nothing has been harvested yet. */
int32_t srl_harvest_device(srl_engine* e, const int32_t** toks, const float** logprobs, const int32_t** versions,
                           const srl_traj** recs, int32_t* n_recs, int64_t* n_tok);

/* Collective over the replicas.  Install policy version `version` (> current;
 * the first call may use any version >= 0).  flat_w: device pointer to a flat
 * weight image (srl_weight_offset layout) on rank 0 (ignored elsewhere), or
 * NULL when the caller already wrote the staging part of the engine's weight
 * region (the first srl_weight_layout bytes) -- on rank 0; other ranks receive
 * rank 0's installed tensors by an in-place broadcast (row a17) and
 * never read their own staging copy.  The projection matrices (wq/wk/wv,
 * wo, wg/wu, wd, lm_head) are repacked from the source into the GEMM's packed
 * layout (srl_op_pack_weight) in the rest of the weight region -- which is why
 * srl_arena_sizes reports about twice the model size -- so the staging copy of
 * those matrices is not read by decoding; the other tensors (embed, norms,
 * biases) are copied from flat_w when it is given and read in place.  Then applies
 * the cache bound: trajectories with version - v_first > K are discarded and
 * re-queued (tokens dropped); under REPREFILL running ones are scavenged.
 * SRL_E_STATE if a group is ready but not harvested or version <= current. */
int32_t srl_load_policy_weights(srl_engine* e, const void* flat_w, int64_t version);

/* Install ONE tensor of the next policy from a caller device buffer holding it
 * row-major [rows, cols] bf16 (the srl_weight_layout shape; wg / wu plain, not
 * interleaved): projection matrices are packed straight into the GEMM's weight
 * stream (for wq / wk / wv into their tile range of the fused QKV matrix, for
 * wg / wu into their 16-row interleave), the others are copied.  The source is
 * read on the engine stream; the caller keeps it alive until the next
 * synchronising call.  Then srl_load_policy_weights(e, NULL, version) makes the
 * installed tensors the new policy (and broadcasts them from rank 0).  Works
 * with and without weights_compact (without it the staging copy is updated
 * too).  Errors: SRL_E_INVALID_ARG (unknown name), SRL_E_STATE (a group awaits
 * harvest), SRL_E_CUDA. */
int32_t srl_load_policy_tensor(srl_engine* e, const char* name, const void* src);

/* Trace / event log since record index `from` (see srl_trace_rec).  *n_out
 * receives the number copied; *n_total the total recorded. */
int32_t srl_get_trace(srl_engine* e, int64_t from, int32_t cap, srl_trace_rec* out, int32_t* n_out,
                      int64_t* n_total);

/* Counters: raw generated tokens, discarded tokens, emitted trajectories,
 * groups, device-side kernel launches issued by the engine. */
int32_t srl_get_counters(srl_engine* e, int64_t* raw_tokens, int64_t* discarded_tokens, int64_t* emitted,
                         int64_t* groups, int64_t* kernel_launches);

/* Change K between updates (SRL_E_STATE while a group is pending). */
int32_t srl_set_cache_bound(srl_engine* e, int32_t K);

/* Enable (1) / disable (0) per-class timing; enabling resets the accumulators.
 * Only the classes in the profile mask (bit SRL_K_*; default all) are bracketed
 * by CUDA events.  Event records sit between kernels, so they also cut the
 * programmatic (PDL) edges of the decode graph: with profiling off the graph
 * holds no events at all.  Decode graphs are cached per (row bucket, bracketed
 * class set), so switching the mask between steps -- e.g. every class on a
 * sample of steps -- replays an already captured graph of each kind. */
int32_t srl_set_profiling(srl_engine* e, int32_t on);
int32_t srl_set_profile_mask(srl_engine* e, uint32_t class_mask);
/* ms[SRL_K_NCLASS]: accumulated device milliseconds per class over decode steps
 * (prefill passes are accumulated whole under SRL_K_PREFILL); launches[]: launch counts. */
int32_t srl_get_profile(srl_engine* e, double* ms, int64_t* launches);

/* Test accessor: copy the fp32 logits [Q_g, V] of the last decode step (local
 * slots; rows of empty slots are unspecified) to host memory. */
int32_t srl_debug_copy_logits(srl_engine* e, float* out_host, int64_t cap_floats);

/* Replica plumbing (see srl_comm).  srl_nccl_unique_id: 128 bytes for
 * srl_comm.nccl_unique_id (SRL_E_NCCL if libnccl cannot be loaded).
 * srl_local_group_create: an in-process group of `world` ranks (1..64). */
int32_t srl_nccl_unique_id(uint8_t* out128);
int32_t srl_local_group_create(int32_t world, void** out);
int32_t srl_local_group_destroy(void* group);

/* Kernel-selection settings, process-wide (all engines and op calls of the
 * process).  The defaults (srl_default_tuning) are the production choices; the
 * alternatives are kept selectable for measurement and for their parity tests
 * (DESIGN.md §7 gives each one's measured cost).  Nothing in the library reads
 * the environment.  Settings are read when a launch is planned:
 * an engine's captured decode graphs keep the settings they were captured
 * with, and `graphs` / `mixed_prefill` are read by srl_create -- so set them
 * before creating engines.  srl_set_tuning returns -1 (srl_last_error) for an
 * out-of-range field and changes nothing then. */
typedef struct srl_tuning {
  int32_t gemm_split;      /* decomposition when whole pair units leave SM pairs idle: 1 cluster split-K
                              (default), 0 batch split, 2 stream-K with L2 fix-up, 3 hybrid stream-K */
  int32_t gemm_pair;       /* -1 auto (CTA-pair tcgen05 kernel for M >= 128), 0 never, 1 always */
  int32_t gemm_h;          /* single-CTA kernel 128-row halves per tile: 0 auto, 1, 2 */
  int32_t gemm_stages;     /* weight ring depth cap (0 = auto) */
  int32_t gemm_xstages;    /* activation ring depth (0 = auto) */
  int32_t partial_norm;    /* 1: O / down split-K partials summed (in split order) by the next RMSNorm */
  int32_t partial_small_m; /* 1: the same for the single-CTA kernel (M < 128) */
  int32_t qkv_finish;      /* 1: QKV split-K partials + a bias/RoPE/KV-append kernel */
  int32_t fused_sample;    /* 1: Gumbel-max sampling fused into the LM head epilogue */
  int32_t attn_min_items, attn_target_items; /* split-KV planning (0 = built-in) */
  int32_t attn_l2_prefetch; /* pages of L2 prefetch beyond the attention TMA ring (0..16) */
  int32_t pdl;             /* 1: programmatic dependent launch across the decode chain */
  int32_t graphs;          /* 1: replay the decode tail from CUDA graphs */
  int32_t mixed_prefill;   /* 1: admitted prompts ride in the decode pass when they fit one chunk */
  int32_t verbose;         /* 1: print GEMM plans to stderr */
  int32_t fuse_mlp;        /* 1: gate/up and down GEMMs as one persistent kernel (128 <= M <= 256);
                              measured r02 equal to the two PDL-chained GEMMs, off */
  int32_t mlp_splits;      /* k-splits of the fused down GEMM (its partials go to the next RMSNorm), 1..8 */
  int32_t attn_stages;     /* attention K/V ring depth: 4 (default) or 6 (dh = 128); 3 (dh = 128): two
                              CTAs per SM when G = Hq / Hkv <= 4 fits both in shared memory */
  int32_t qkv_attn;        /* 1 (default): pure decode passes leave QKV split-K partials to the attention
                              kernel, whose finish warp completes q / k / v per item (bias, RoPE, KV
                              append) ahead of its TMA producer */
  int32_t pair_h2;         /* 1 (default): whole-unit pair GEMMs take 512-row units (two MMAs per
                              k-step share the activation slice) when that at least halves the
                              waves of 256-row units (decode gate/up); 0: 256-row units */
} srl_tuning;
void srl_default_tuning(srl_tuning* t);
int32_t srl_get_tuning(srl_tuning* t);
int32_t srl_set_tuning(const srl_tuning* t);

const char* srl_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
