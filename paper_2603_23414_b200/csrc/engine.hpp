// engine.hpp — device-side data layout of the SortedRL rollout engine.
//
// All controller state lives in HBM and is mutated only by the single-CTA
// controller kernels in ctl.cu (the host reads a small status block after
// each step).  Global slot g = s*R + r (local slot s on replica r), reading
// R24.  Every rank holds the full (replicated) integer state; each rank owns
// the KV pages / page-table rows of its own slots only.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "srl.h"

namespace srl {

constexpr int kPage = 64;       // tokens per KV page
constexpr int kMaxR = 64;       // max data-parallel replicas
constexpr int kCtlThreads = 1024;
constexpr int kMaxSortReady = 16384;  // bitonic-sort capacity of the ready list (128 KB of shared memory)
constexpr int kMaxGroup = 2048;      // largest update group that can be harvested

enum TrajState { TS_STREAM = 0, TS_PENDING = 1, TS_RUNNING = 2, TS_READY = 3, TS_EMITTED = 4 };
enum StepStatus { ST_CONTINUE = 100 };  // internal: BEGIN succeeded, run the forward

struct DevTraj {
  int prompt_idx, prompt_len, forced_len, epoch;
  int n_tok, v_first, lifecycle, restarts;
  int admit_step, finish_step, state, slot;
  int fresh, pages, sample;
  int shared;  // N4: prompt-prefix pages held through the replica's shared entry (page-table
               // entries [0, shared)); the private pages are entries [shared, shared + pages)
  int pre_next, pre_end;  // N1: next prefill position (-1: not started since admission) and the
                          //     end of the prefill range (prompt ++ kept tokens minus the last)
};

// Host-visible status block (mirrored to pinned memory after each phase).
struct CtlStatus {
  int status;
  int r_k;
  int n_fin;
  int n_ready;
  int n_admit;        // admissions this step (all replicas)
  int n_admit_local;  // admissions on this rank that need a prefill
  int m_pre;          // prefill rows on this rank
  int k;              // step index of the step (BEGIN) / next step (END)
  int v;
  int group_n, group_final, group_state;
  long long n_events, raw_tokens, discarded_tokens, emitted, n_groups;
  long long sum_ctx;  // sum of (pos + 1) over this rank's running rows (BEGIN)
  int r_local;        // running rows on this rank (BEGIN)
  int pad[3];
};

struct CtlState {
  int k, v, v_valid;
  int epoch, epoch_of_latest;
  int loaded, emitted, next_stream, n_stream, n_prompts;
  int fresh_head, n_resumed, n_ready;
  int group_state, group_n, group_final, n_groups;
  int K;
  int page_blocked;
  int own_top;
  long long n_events, raw_tokens, discarded_tokens, prompt_tok_used;
  int free_pages[kMaxR];
  CtlStatus st;
};

// Pointers + configuration passed by value to every controller kernel.
struct Ctl {
  // config
  int Q_g, R, rank, Q_tot, U, pool_traj, G, cap, kv_pages, max_pages;
  int mode, resume, barrier, stop, eos_id, max_traj, max_prompt, prefill_rows_max;
  int share_prefix, max_prompts, pfx_max;  // N4: sharing on, prompt-table size, shared pages per entry
  int prefill_budget;                      // N1: prefill positions per replica per step (0 = unlimited)
  long long ev_cap;
  // state
  CtlState* s;
  DevTraj* traj;
  int* slot_traj;      // [Q_tot]
  int* page_table;     // [Q_g][max_pages] (own slots)
  int* page_stack;     // [kv_pages] (own replica)
  int* resumed;        // [max_traj] tids sorted by (-lifecycle, tid)
  int* ready;          // [max_traj]
  int* group;          // [max_traj]
  int* tokens;         // [max_traj][cap]
  float* lps;          // [max_traj][cap]
  int* vers;           // [max_traj][cap]
  int* prompt_off;     // [max_prompts+1]
  int* prompt_tok;     // prompt token storage
  int* events;         // [ev_cap][6]
  // N4 prompt-prefix sharing (oracle/sched.py _prefix_pages), one entry per (replica, prompt)
  int* pfx_ref;        // [R][max_prompts] holders of the entry (replicated accounting)
  int* pfx_tag;        // [R][max_prompts] policy version the entry's KV was computed under
  int* pfx_pages;      // [max_prompts][pfx_max] page ids of this rank's entries
  int* pfx_valid;      // [R][max_prompts] the entry's shared positions have been prefilled (in an
                       //   earlier step or earlier in this step's rows) -- later holders skip them
  int* pre_list;       // [Q_g][3] this step's own prefill allocations (local slot, first position, count)
  // per-step rows (this rank)
  int* row_tok;        // [Q_g]
  int* row_pos;        // [Q_g]  (-1 = inactive)
  int* row_n;          // [Q_g]  generated index of the token being sampled
  int* row_traj;       // [Q_g]
  int* row_restarts;   // [Q_g]
  int* row_slot;       // [Q_g]  local slot of decode row i (-1: inactive row); rows are the running
                       //        local slots compacted in ascending slot order (BEGIN)
  int* pre_tok;        // [prefill_rows_max]
  int* pre_pos;
  int* pre_slot;       // local slot of the prefill row
  int* admit_local;    // [Q_g] local slot ids admitted this step (for prefill)
  int* samp;           // [R][2][Q_g]: per replica its sampled tokens, then their fp32 logprobs
                       // (bit pattern); rank r writes block r, the replica all-gather fills the rest
  // harvest staging
  int* h_tok;
  float* h_lp;
  int* h_ver;
  srl_traj* h_rec;
  long long h_cap_tok;
};

// ---- ctl.cu launchers
void ctl_begin(const Ctl& c, cudaStream_t st);
void ctl_end(const Ctl& c, cudaStream_t st);
void ctl_bump(const Ctl& c, int version, cudaStream_t st);
void ctl_harvest(const Ctl& c, cudaStream_t st);
void ctl_init(const Ctl& c, int K, cudaStream_t st);
void ctl_submit(const Ctl& c, int n_new_traj, int n_new_prompts, cudaStream_t st);

}  // namespace srl
