// ctl.cu — the SortedRL controller + stateful rollout buffer as single-CTA
// device kernels.
//
// Mirrors the state machine of PAPER.md §3.1–3.3 and P:353 with
// the DESIGN.md readings; per decode step the host launches
//   ctl_begin: emission pre-check, epoch load (cache-aware loading),
//              refill of free slots from the pending queue (oversubscription,
//              P:167), KV page growth / preemption, row + prefill lists;
//   ctl_end:   append the sampled token + logprob + version per running slot
//              (P:180), stop detection, ballot/prefix-sum compaction of the
//              finished slots into the ready list (ascending global slot),
//              trace record (Eq. (bubble)), early-termination check
//              |ready| >= U with the length-sorted update group
//              chosen by an in-shared-memory bitonic sort on (len, traj_id);
//   ctl_bump:  after load_policy_weights, the cache bound K (discard + requeue)
//              and REPREFILL scavenging.
// Per-slot work is spread over the 1024 threads with warp ballots; only the
// admission / page-growth loops (a handful of items per step) run on one
// thread, in ascending slot order, exactly as the oracle specifies.
#include "common.cuh"
#include "launch.hpp"
#include "engine.hpp"

namespace srl {

// ------------------------------------------------------------------ block utils
// Exclusive prefix sum of `v` over the 1024-thread block; *total = sum.
__device__ int block_scan(int v, int* total) {
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;
  }
  __syncthreads();
  const int base = w ? wsum[w - 1] : 0;
  const int tot = wsum[31];
  __syncthreads();
  if (total) *total = tot;
  return base + x - v;
}

__device__ int block_sum(int v) {
  int t;
  block_scan(v, &t);
  return t;
}

__device__ __forceinline__ long long sort_key_ready(const Ctl& c, int tid) {
  return ((long long)c.traj[tid].n_tok << 32) | (unsigned)tid;
}

// Bitonic sort of keys[0..n) ascending (n <= kMaxSortReady), all threads.
__device__ void bitonic_sort(long long* keys, int n) {
  int N = 1;
  while (N < n) N <<= 1;
  for (int i = n + threadIdx.x; i < N; i += blockDim.x) keys[i] = 0x7fffffffffffffffLL;
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const long long a = keys[i], b = keys[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ void log_event(const Ctl& c, long long idx, int kind, int a, int b, int cc, int d, int e) {
  int* ev = c.events + (idx % c.ev_cap) * 6;
  ev[0] = kind;
  ev[1] = a;
  ev[2] = b;
  ev[3] = cc;
  ev[4] = d;
  ev[5] = e;
}
// thread-0-only helper
__device__ void push_event(const Ctl& c, int kind, int a, int b, int cc, int d, int e = 0) {
  log_event(c, c.s->n_events, kind, a, b, cc, d, e);
  c.s->n_events++;
}

// ------------------------------------------------------------------ pending queue (thread 0)
__device__ bool pending_empty(const Ctl& c) {
  return c.s->n_resumed == 0 && c.s->fresh_head >= c.s->next_stream;
}
__device__ int pending_peek(const Ctl& c) {
  return c.s->n_resumed > 0 ? c.resumed[0] : c.s->fresh_head;
}
__device__ void pending_pop(const Ctl& c) {
  CtlState* s = c.s;
  if (s->n_resumed > 0) {
    for (int i = 1; i < s->n_resumed; ++i) c.resumed[i - 1] = c.resumed[i];
    s->n_resumed--;
  } else {
    s->fresh_head++;
  }
}
// insert a non-fresh trajectory keeping the (-lifecycle, tid) order
__device__ void resumed_insert(const Ctl& c, int tid) {
  CtlState* s = c.s;
  const long long key = ((long long)(1000000 - c.traj[tid].lifecycle) << 32) | (unsigned)tid;
  int i = s->n_resumed;
  while (i > 0) {
    const int o = c.resumed[i - 1];
    const long long ko = ((long long)(1000000 - c.traj[o].lifecycle) << 32) | (unsigned)o;
    if (ko < key) break;
    c.resumed[i] = o;
    --i;
  }
  c.resumed[i] = tid;
  s->n_resumed++;
}
__device__ void push_pending(const Ctl& c, int tid) {
  DevTraj& t = c.traj[tid];
  t.state = TS_PENDING;
  t.slot = -1;
  resumed_insert(c, tid);  // only non-fresh trajectories are ever re-pushed
}

// release slot g (thread 0): pages back to the replica pool
__device__ void free_slot(const Ctl& c, int g) {
  CtlState* s = c.s;
  const int tid = c.slot_traj[g];
  DevTraj& t = c.traj[tid];
  const int r = g % c.R;
  if (r == c.rank) {
    const int* row = c.page_table + (size_t)(g / c.R) * c.max_pages + t.shared;
    for (int i = t.pages - 1; i >= 0; --i) c.page_stack[s->own_top++] = row[i];
  }
  s->free_pages[r] += t.pages;
  if (t.shared) {  // N4: release the prompt-prefix entry; its last holder frees its pages
    const int key = r * c.max_prompts + t.prompt_idx;
    if (--c.pfx_ref[key] == 0) {
      s->free_pages[r] += t.shared;
      c.pfx_valid[key] = 0;
      if (r == c.rank) {
        const int* pp = c.pfx_pages + (size_t)t.prompt_idx * c.pfx_max;
        for (int i = t.shared - 1; i >= 0; --i) c.page_stack[s->own_top++] = pp[i];
      }
    }
    t.shared = 0;
  }
  t.pages = 0;
  t.slot = -1;
  c.slot_traj[g] = -1;
}

__device__ void drop_tokens(const Ctl& c, DevTraj& t) {
  c.s->discarded_tokens += t.n_tok;
  t.n_tok = 0;
  t.v_first = -1;
  t.restarts++;
}

// ------------------------------------------------------------------ load / emission
__device__ bool load_possible(const Ctl& c) {
  const CtlState* s = c.s;
  if (s->next_stream >= s->n_stream) return false;
  if (s->loaded == 0) return true;
  if (c.mode == SRL_MODE_SYNC || c.mode == SRL_MODE_POSTHOC || c.barrier == SRL_BARRIER_TRAINED)
    return s->emitted == s->loaded;
  if (s->fresh_head < s->next_stream) return false;  // the tail of the fresh range is the latest epoch
  for (int i = 0; i < s->n_resumed; ++i)
    if (c.traj[c.resumed[i]].epoch == s->epoch_of_latest) return false;
  return true;
}

__device__ void maybe_load(const Ctl& c) {  // thread 0
  CtlState* s = c.s;
  if (!load_possible(c)) return;
  const int want = c.mode == SRL_MODE_SYNC ? c.Q_tot : c.pool_traj;
  const int n = min(want, s->n_stream - s->next_stream);
  for (int i = 0; i < n; ++i) {
    DevTraj& t = c.traj[s->next_stream + i];
    t.epoch = s->epoch;
    t.state = TS_PENDING;
  }
  push_event(c, SRL_EV_LOAD, s->k, s->epoch, s->next_stream, n);
  s->next_stream += n;
  s->epoch_of_latest = s->epoch;
  s->epoch++;
  s->loaded += n;
}

// Early termination / selective batching (all threads).  Returns 1 if a group was
// emitted, 0 if not, -1 if the ready list outgrew the sort buffer (SRL_E_CAPACITY;
// validate() rules this out for every accepted configuration).
__device__ int emission_check(const Ctl& c, long long* keys) {
  CtlState* s = c.s;
  __shared__ int sh_flag, sh_final, sh_n;
  int occ = 0;
  for (int g = threadIdx.x; g < c.Q_tot; g += blockDim.x) occ += c.slot_traj[g] >= 0;
  occ = block_sum(occ);
  if (threadIdx.x == 0) {
    sh_flag = 0;
    const bool pe = pending_empty(c);
    if (c.mode == SRL_MODE_SYNC) {
      if (s->n_ready > 0 && occ == 0 && pe) {
        sh_flag = 1;
        sh_n = min(c.U, s->n_ready);
        sh_final = s->n_ready == sh_n;
      }
    } else if (c.mode != SRL_MODE_POSTHOC || (pe && occ == 0)) {
      // (POSTHOC: the sorted groups only once the whole loaded batch has finished)
      const bool drain = pe && occ == 0 && !load_possible(c);
      if (s->n_ready >= c.U) {
        sh_flag = 2;
        sh_n = c.U;
        sh_final = 0;
      } else if (drain && s->n_ready > 0) {
        sh_flag = 2;
        sh_n = s->n_ready;
        sh_final = 1;
      }
    }
  }
  __syncthreads();
  const int flag = sh_flag, n = sh_n;
  if (!flag) return 0;
  const int nr = s->n_ready;
  if (flag == 2 && nr > kMaxSortReady) return -1;  // uniform: every thread reads the same n_ready
  if (flag == 1) {  // SYNC: completion order, no sorting
    for (int i = threadIdx.x; i < n; i += blockDim.x) c.group[i] = c.ready[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = n; i < nr; ++i) c.ready[i - n] = c.ready[i];
    }
  } else {
    for (int i = threadIdx.x; i < nr; i += blockDim.x) keys[i] = sort_key_ready(c, c.ready[i]);
    __syncthreads();
    bitonic_sort(keys, nr);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int tid = (int)(keys[i] & 0xffffffffLL);
      c.group[i] = tid;
      c.traj[tid].state = TS_EMITTED;  // mark before compaction below
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // stable removal of the emitted ones (ready keeps compaction order)
      int w = 0;
      for (int i = 0; i < nr; ++i) {
        const int tid = c.ready[i];
        if (c.traj[tid].state != TS_EMITTED) c.ready[w++] = tid;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) c.traj[c.group[i]].state = TS_EMITTED;
    s->n_ready = nr - n;
    s->emitted += n;
    s->group_state = 1;
    s->group_n = n;
    s->group_final = sh_final;
    push_event(c, SRL_EV_EMIT, s->n_groups, s->v, n, sh_final);
    for (int i = 0; i < n; ++i) push_event(c, SRL_EV_EMIT_MEMBER, s->n_groups, i, c.group[i], 0);
    s->n_groups++;
  }
  __syncthreads();
  return 1;
}

__device__ void fill_status(const Ctl& c, int status) {
  CtlState* s = c.s;
  CtlStatus& st = s->st;
  st.status = status;
  st.k = s->k;
  st.v = s->v;
  st.n_ready = s->n_ready;
  st.group_n = s->group_n;
  st.group_final = s->group_final;
  st.group_state = s->group_state;
  st.n_events = s->n_events;
  st.raw_tokens = s->raw_tokens;
  st.discarded_tokens = s->discarded_tokens;
  st.emitted = s->emitted;
  st.n_groups = s->n_groups;
}

// ------------------------------------------------------------------ BEGIN
__global__ void __launch_bounds__(kCtlThreads, 1) ctl_begin_kernel(Ctl c) {
  extern __shared__ long long keys[];
  __shared__ int sh_free[1024];
  __shared__ int sh_nfree, sh_ngrow, sh_stop, sh_cap;
  CtlState* s = c.s;
  if (threadIdx.x == 0) {
    sh_stop = 0;
    sh_cap = 0;
    s->st.n_admit = s->st.n_admit_local = s->st.m_pre = s->st.r_k = s->st.n_fin = 0;
    if (s->group_state != 0 || !s->v_valid) {
      fill_status(c, SRL_E_STATE);
      sh_stop = 1;
    }
  }
  __syncthreads();
  if (sh_stop) return;
  // 0 pre: emission check (leftover ready >= U after an update / SYNC next group)
  if (const int em = emission_check(c, keys)) {
    if (threadIdx.x == 0) fill_status(c, em > 0 ? SRL_GROUP_READY : SRL_E_CAPACITY);
    return;
  }
  // 1 load
  if (threadIdx.x == 0) maybe_load(c);
  __syncthreads();
  // 2 refill: free slots in ascending global order (ballot compaction), admissions on thread 0
  for (int base = 0; base < c.Q_tot; base += blockDim.x) {
    const int g = base + threadIdx.x;
    const int f = (g < c.Q_tot && c.slot_traj[g] < 0) ? 1 : 0;
    int tot;
    const int pos = block_scan(f, &tot);
    if (f) sh_free[pos] = g;
    if (threadIdx.x == 0) sh_nfree = tot;
    __syncthreads();
    // only thread 0 may read sh_stop here (it writes it below): a volatile read is not
    // speculated past the thread test (compute-sanitizer racecheck)
    if (threadIdx.x == 0 && !*reinterpret_cast<volatile int*>(&sh_stop)) {
      s->page_blocked = 0;
      for (int i = 0; i < sh_nfree; ++i) {
        const int gg = sh_free[i];
        if (pending_empty(c)) {
          sh_stop = 1;
          break;
        }
        const int tid = pending_peek(c);
        DevTraj& t = c.traj[tid];
        const int need = (t.prompt_len + t.n_tok + kPage - 1) / kPage;
        const int r = gg % c.R;
        // N4 (oracle/sched.py _prefix_pages): the full pages of prompt positions
        // [0, prompt_len - 1) are shareable; a new holder shares an existing entry
        // only if it was computed under the current version
        const int S = c.share_prefix ? (t.prompt_len - 1) / kPage : 0;
        const int key = r * c.max_prompts + t.prompt_idx;
        const int ref = S > 0 ? c.pfx_ref[key] : 0;
        const bool share = S > 0 && (ref == 0 || c.pfx_tag[key] == s->v);
        const int cost = (share && ref > 0) ? need - S : need;
        if (s->free_pages[r] < cost || need > c.max_pages) {
          s->page_blocked = 1;
          sh_stop = 1;
          break;
        }
        pending_pop(c);
        s->free_pages[r] -= cost;
        t.pages = share ? need - S : need;
        t.shared = share ? S : 0;
        if (share) {
          if (ref == 0) {
            c.pfx_tag[key] = s->v;
            c.pfx_valid[key] = 0;  // computed by the first holder whose prefill reaches it
          }
          c.pfx_ref[key] = ref + 1;
        }
        t.pre_next = -1;
        t.pre_end = t.prompt_len + t.n_tok - 1;
        t.slot = gg;
        t.state = TS_RUNNING;
        t.fresh = 0;
        if (t.v_first < 0) t.v_first = s->v;
        t.admit_step = s->k;
        c.slot_traj[gg] = tid;
        push_event(c, SRL_EV_ADMIT, s->k, gg, tid, t.n_tok);
        s->st.n_admit++;
        if (r == c.rank) {
          int* row = c.page_table + (size_t)(gg / c.R) * c.max_pages;
          if (share) {
            int* pp = c.pfx_pages + (size_t)t.prompt_idx * c.pfx_max;
            if (ref == 0)  // a new entry: its pages are computed by the first surviving holder's prefill
              for (int p = 0; p < S; ++p) pp[p] = c.page_stack[--s->own_top];
            for (int p = 0; p < S; ++p) row[p] = pp[p];
          }
          for (int p = t.shared; p < need; ++p) row[p] = c.page_stack[--s->own_top];
          c.admit_local[s->st.n_admit_local++] = gg / c.R;
        }
      }
    }
    __syncthreads();
    if (sh_stop) break;
  }
  __syncthreads();
  // 3 page growth / preemption: slots needing a page, ascending g
  for (int base = 0; base < c.Q_tot; base += blockDim.x) {
    const int g = base + threadIdx.x;
    int f = 0;
    if (g < c.Q_tot) {
      const int tid = c.slot_traj[g];
      if (tid >= 0) {
        const DevTraj& t = c.traj[tid];
        f = (t.shared + t.pages) * kPage < t.prompt_len + t.n_tok;
      }
    }
    int tot;
    const int pos = block_scan(f, &tot);
    if (f) sh_free[pos] = g;
    if (threadIdx.x == 0) sh_ngrow = tot;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < sh_ngrow && !sh_cap; ++i) {
        const int gg = sh_free[i];
        const int tid = c.slot_traj[gg];
        if (tid < 0) continue;  // preempted earlier in this loop
        DevTraj& t = c.traj[tid];
        const int need = (t.prompt_len + t.n_tok + kPage - 1) / kPage - t.shared;  // private pages
        const int r = gg % c.R;
        while (t.pages < need && c.slot_traj[gg] == tid) {
          if (s->free_pages[r] > 0 && t.shared + t.pages < c.max_pages) {
            s->free_pages[r]--;
            if (r == c.rank)
              c.page_table[(size_t)(gg / c.R) * c.max_pages + t.shared + t.pages] = c.page_stack[--s->own_top];
            t.pages++;
            continue;
          }
          // victim: occupied slot of replica r with max (admit_step, slot)
          int victim = -1, vstep = -1, n_occ = 0;
          for (int h = r; h < c.Q_tot; h += c.R) {
            const int vt = c.slot_traj[h];
            if (vt < 0) continue;
            ++n_occ;
            const int as = c.traj[vt].admit_step;
            if (as > vstep || (as == vstep && h > victim)) {
              vstep = as;
              victim = h;
            }
          }
          if (n_occ == 1) {  // alone and still short of pages: it can never fit (reading R25)
            sh_cap = 1;
            break;
          }
          const int vt = c.slot_traj[victim];
          DevTraj& v = c.traj[vt];
          const bool keep = c.mode == SRL_MODE_SYNC || s->K != 0;
          free_slot(c, victim);
          v.lifecycle++;
          if (!keep) drop_tokens(c, v);
          else if (v.n_tok == 0) v.v_first = -1;
          push_event(c, SRL_EV_PREEMPT, s->k, victim, vt, keep ? 1 : 0);
          push_pending(c, vt);
        }
      }
    }
    __syncthreads();
  }
  if (sh_cap) {
    if (threadIdx.x == 0) fill_status(c, SRL_E_CAPACITY);
    return;
  }
  // running set
  int occ = 0;
  for (int g = threadIdx.x; g < c.Q_tot; g += blockDim.x) occ += c.slot_traj[g] >= 0;
  occ = block_sum(occ);
  if (occ == 0) {
    if (threadIdx.x == 0) {
      int st;
      if (!pending_empty(c)) st = SRL_E_CAPACITY;
      else if (s->n_stream == 0) st = SRL_E_EMPTY;
      else st = SRL_DONE;
      fill_status(c, st);
    }
    return;
  }
  // N1 prefill allocation (reading R30, oracle/sched.py _prefill), replicated over
  // every replica's slots: each replica serves its prefilling slots strictly in
  // admission order (admit_step, global slot) with at most prefill_budget positions
  // per step (0 = unlimited); a slot short of its prefill stops its replica's walk.
  // N4: a slot starts after its shared prompt pages when the entry is already valid.
  __shared__ int sh_npf, sh_nalloc, sh_used[kMaxR], sh_blk[kMaxR];
  if (threadIdx.x == 0) sh_npf = 0;
  __syncthreads();
  for (int base = 0; base < c.Q_tot; base += blockDim.x) {
    const int g = base + threadIdx.x;
    int f = 0;
    if (g < c.Q_tot) {
      const int tid = c.slot_traj[g];
      f = tid >= 0 && c.traj[tid].pre_next < c.traj[tid].pre_end;
    }
    int tot;
    const int pos = block_scan(f, &tot);
    if (f) keys[sh_npf + pos] = ((long long)c.traj[c.slot_traj[g]].admit_step << 32) | (unsigned)g;
    __syncthreads();
    if (threadIdx.x == 0) sh_npf += tot;
    __syncthreads();
  }
  const int npf = sh_npf;
  if (npf > 0) bitonic_sort(keys, npf);
  if (threadIdx.x == 0) {
    for (int r = 0; r < c.R; ++r) sh_used[r] = sh_blk[r] = 0;
    int na = 0, off = 0;
    for (int i = 0; i < npf; ++i) {
      const int g = (int)(keys[i] & 0xffffffffLL), r = g % c.R;
      if (sh_blk[r]) continue;
      DevTraj& t = c.traj[c.slot_traj[g]];
      const int key = r * c.max_prompts + t.prompt_idx;
      if (t.pre_next < 0) t.pre_next = (t.shared > 0 && c.pfx_valid[key]) ? t.shared * kPage : 0;
      int n = t.pre_end - t.pre_next;
      if (c.prefill_budget > 0 && n > c.prefill_budget - sh_used[r]) n = c.prefill_budget - sh_used[r];
      if (n > 0) {
        if (r == c.rank) {
          c.pre_list[3 * na] = g / c.R;
          c.pre_list[3 * na + 1] = t.pre_next;
          c.pre_list[3 * na + 2] = off;
          ++na;
          off += n;
        }
        t.pre_next += n;
        sh_used[r] += n;
      }
      if (t.shared > 0 && t.pre_next >= t.shared * kPage) c.pfx_valid[key] = 1;
      if (t.pre_next < t.pre_end) sh_blk[r] = 1;
    }
    sh_nalloc = na;
    c.pre_list[3 * na + 2] = off;  // sentinel: total rows (pre_list has room for Q_g + 1 entries)
  }
  __syncthreads();
  // decode rows: this rank's running slots whose prefill is complete, compacted in
  // ascending slot order (row i -> slot row_slot[i]), so the decode forward runs over
  // the first r_local rows only (the host picks a graph whose M covers them); rows
  // past them are inactive
  long long my_ctx = 0;
  int my_rows = 0, dec = 0;
  for (int g = threadIdx.x; g < c.Q_tot; g += blockDim.x) {
    const int tid = c.slot_traj[g];
    dec += tid >= 0 && c.traj[tid].pre_next >= c.traj[tid].pre_end;
  }
  dec = block_sum(dec);
  __shared__ int sh_rbase;
  if (threadIdx.x == 0) sh_rbase = 0;
  __syncthreads();
  for (int base = 0; base < c.Q_g; base += blockDim.x) {
    const int sl = base + threadIdx.x;
    int tid = sl < c.Q_g ? c.slot_traj[sl * c.R + c.rank] : -1;
    if (tid >= 0 && c.traj[tid].pre_next < c.traj[tid].pre_end) tid = -1;  // still prefilling
    int tot;
    const int rank_in = block_scan(tid >= 0 ? 1 : 0, &tot);
    if (tid >= 0) {
      const int i = sh_rbase + rank_in;
      const DevTraj& t = c.traj[tid];
      const int n = t.n_tok;
      c.row_tok[i] = n > 0 ? c.tokens[(size_t)tid * c.cap + n - 1]
                           : c.prompt_tok[c.prompt_off[t.prompt_idx] + t.prompt_len - 1];
      c.row_pos[i] = t.prompt_len + n - 1;
      my_ctx += t.prompt_len + n;
      my_rows++;
      c.row_n[i] = n;
      c.row_traj[i] = tid;
      c.row_restarts[i] = t.restarts;
      c.row_slot[i] = sl;
    }
    __syncthreads();
    if (threadIdx.x == 0) sh_rbase += tot;
    __syncthreads();
  }
  for (int i = sh_rbase + threadIdx.x; i < c.Q_g; i += blockDim.x) {
    c.row_tok[i] = 0;
    c.row_pos[i] = -1;
    c.row_n[i] = 0;
    c.row_traj[i] = -1;
    c.row_restarts[i] = 0;
    c.row_slot[i] = -1;
  }
  // prefill rows of this rank's allocations, in allocation order (prompt ++ kept[:-1])
  __shared__ unsigned long long sh_ctx;
  if (threadIdx.x == 0) sh_ctx = 0;
  __syncthreads();
  atomicAdd(&sh_ctx, (unsigned long long)my_ctx);
  my_rows = block_sum(my_rows);
  if (threadIdx.x == 0) {
    s->st.sum_ctx = (long long)sh_ctx;
    s->st.r_local = my_rows;
  }
  const int na = sh_nalloc;
  const int m_pre = c.pre_list[3 * na + 2];
  if (m_pre <= c.prefill_rows_max) {
    for (int a = 0; a < na; ++a) {
      const int sl = c.pre_list[3 * a], p0 = c.pre_list[3 * a + 1], off = c.pre_list[3 * a + 2];
      const int cnt = c.pre_list[3 * a + 5] - off;
      const DevTraj& t = c.traj[c.slot_traj[sl * c.R + c.rank]];
      const int* pt = c.prompt_tok + c.prompt_off[t.prompt_idx];
      const int* kt = c.tokens + (size_t)c.slot_traj[sl * c.R + c.rank] * c.cap;
      for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int q = p0 + i;
        c.pre_tok[off + i] = q < t.prompt_len ? pt[q] : kt[q - t.prompt_len];
        c.pre_pos[off + i] = q;
        c.pre_slot[off + i] = sl;
      }
    }
  }
  if (threadIdx.x == 0) {
    s->st.r_k = dec;
    s->st.m_pre = m_pre;
    fill_status(c, m_pre > c.prefill_rows_max ? SRL_E_CAPACITY : ST_CONTINUE);
  }
}

// ------------------------------------------------------------------ END
__global__ void __launch_bounds__(kCtlThreads, 1) ctl_end_kernel(Ctl c) {
  extern __shared__ long long keys[];
  __shared__ int sh_fin[1024];
  __shared__ int sh_nfin_total;
  pdl_trigger();
  pdl_wait();
  CtlState* s = c.s;
  const int v = s->v;
  if (threadIdx.x == 0) sh_nfin_total = 0;
  int occ = 0;
  for (int base = 0; base < c.Q_tot; base += blockDim.x) {
    const int g = base + threadIdx.x;
    int fin = 0;
    if (g < c.Q_tot) {
      const int tid = c.slot_traj[g];
      if (tid >= 0 && c.traj[tid].pre_next >= c.traj[tid].pre_end) {  // decoded this step (N1: prefill complete)
        occ++;
        DevTraj& t = c.traj[tid];
        const int n = t.n_tok;
        const int src = (g % c.R) * 2 * c.Q_g + g / c.R;
        const int tok = c.samp[src];
        c.tokens[(size_t)tid * c.cap + n] = tok;
        c.lps[(size_t)tid * c.cap + n] = __int_as_float(c.samp[src + c.Q_g]);
        c.vers[(size_t)tid * c.cap + n] = v;
        t.n_tok = n + 1;
        fin = (c.stop == SRL_STOP_FORCED && n + 1 == t.forced_len) ||
              (c.stop == SRL_STOP_EOS && tok == c.eos_id) || n + 1 == c.cap;
      }
    }
    int tot;
    const int pos = block_scan(fin, &tot);
    if (fin) sh_fin[pos] = g;
    __syncthreads();
    // compaction into the ready list, ascending global slot (parallel writes)
    const int nr0 = s->n_ready;
    const long long ev0 = s->n_events;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) {
      const int gg = sh_fin[i];
      const int tid = c.slot_traj[gg];
      DevTraj& t = c.traj[tid];
      t.finish_step = s->k;
      t.state = TS_READY;
      c.ready[nr0 + i] = tid;
      log_event(c, ev0 + i, SRL_EV_FINISH, s->k, gg, tid, t.n_tok, 0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < tot; ++i) free_slot(c, sh_fin[i]);
      s->n_ready = nr0 + tot;
      s->n_events = ev0 + tot;
      sh_nfin_total += tot;
    }
    __syncthreads();
  }
  occ = block_sum(occ);
  if (threadIdx.x == 0) {
    s->raw_tokens += occ;
    s->st.n_fin = sh_nfin_total;
    s->st.r_k = occ;
    push_event(c, SRL_EV_STEP, s->k, occ, 0, 0);
    s->k++;
  }
  __syncthreads();
  const int em = emission_check(c, keys);
  if (threadIdx.x == 0) fill_status(c, em > 0 ? SRL_GROUP_READY : (em < 0 ? SRL_E_CAPACITY : SRL_OK));
}

// ------------------------------------------------------------------ BUMP (load_policy_weights)
__device__ __forceinline__ long long resumed_key(const Ctl& c, int tid) {
  return ((long long)(1000000 - c.traj[tid].lifecycle) << 32) | (unsigned)tid;
}

__global__ void __launch_bounds__(kCtlThreads, 1) ctl_bump_kernel(Ctl c, int version) {
  extern __shared__ long long keys[];
  CtlState* s = c.s;
  __shared__ int sh_first, sh_rebuild;
  if (threadIdx.x == 0) {
    sh_first = !s->v_valid;
    s->v = version;
    s->v_valid = 1;
    s->group_state = 0;
    s->group_n = 0;
    sh_rebuild = 0;
  }
  __syncthreads();
  if (sh_first || c.mode == SRL_MODE_SYNC) {
    if (threadIdx.x == 0) fill_status(c, SRL_OK);
    return;
  }
  const int K = s->K;
  const int nlive = s->next_stream;
  // Enforcement in ascending traj_id (the oracle's event order), thread 0.
  if (threadIdx.x == 0) {
    bool ch_ready = false;
    for (int tid = 0; tid < nlive; ++tid) {
      DevTraj& t = c.traj[tid];
      if (t.state != TS_PENDING && t.state != TS_RUNNING && t.state != TS_READY) continue;
      if (K >= 0 && t.v_first >= 0 && version - t.v_first > K) {
        const int where = t.state == TS_PENDING ? 1 : (t.state == TS_RUNNING ? 2 : 3);
        push_event(c, SRL_EV_DISCARD, version, tid, where, 0);
        if (t.state == TS_RUNNING) free_slot(c, t.slot);
        if (t.state == TS_READY) ch_ready = true;
        drop_tokens(c, t);
        t.lifecycle++;
        t.state = TS_PENDING;
        t.fresh = 0;
        sh_rebuild = 1;
      } else if (c.resume == SRL_RESUME_REPREFILL && t.state == TS_RUNNING) {
        push_event(c, SRL_EV_SCAVENGE, version, tid, t.slot, 0);
        free_slot(c, t.slot);
        t.lifecycle++;
        t.state = TS_PENDING;
        sh_rebuild = 1;
      }
    }
    if (ch_ready) {  // stable removal of discarded ready entries
      int w = 0;
      for (int i = 0; i < s->n_ready; ++i) {
        const int tid = c.ready[i];
        if (c.traj[tid].state == TS_READY) c.ready[w++] = tid;
      }
      s->n_ready = w;
    }
  }
  __syncthreads();
  if (sh_rebuild) {
    // resumed list = every non-fresh pending trajectory, sorted by (-lifecycle, traj_id)
    int n = 0;
    for (int base = 0; base < nlive; base += blockDim.x) {
      const int tid = base + threadIdx.x;
      const int f = (tid < nlive && c.traj[tid].state == TS_PENDING && !c.traj[tid].fresh) ? 1 : 0;
      int tot;
      const int pos = block_scan(f, &tot);
      if (f && n + pos < kMaxSortReady) keys[n + pos] = resumed_key(c, tid);
      n += tot;
      __syncthreads();
    }
    if (n > kMaxSortReady) {
      if (threadIdx.x == 0) fill_status(c, SRL_E_CAPACITY);
      return;
    }
    bitonic_sort(keys, n);
    for (int i = threadIdx.x; i < n; i += blockDim.x) c.resumed[i] = (int)(keys[i] & 0xffffffffLL);
    if (threadIdx.x == 0) s->n_resumed = n;
  }
  __syncthreads();
  if (threadIdx.x == 0) fill_status(c, SRL_OK);
}

// ------------------------------------------------------------------ HARVEST gather
__global__ void __launch_bounds__(kCtlThreads, 1) ctl_harvest_kernel(Ctl c) {
  CtlState* s = c.s;
  __shared__ long long sh_off[kMaxGroup + 1];
  const int n = min(s->group_n, kMaxGroup);
  if (threadIdx.x == 0) {
    long long off = 0;
    for (int i = 0; i < n; ++i) {
      sh_off[i] = off;
      off += c.traj[c.group[i]].n_tok;
    }
    sh_off[n] = off;
  }
  __syncthreads();
  const long long total = sh_off[n];
  if (total > c.h_cap_tok || n > kMaxGroup) {
    if (threadIdx.x == 0) fill_status(c, SRL_E_CAPACITY);
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int tid = c.group[i];
    const DevTraj& t = c.traj[tid];
    srl_traj r;
    r.traj_id = tid;
    r.prompt_id = t.prompt_idx;
    r.sample = t.sample;
    r.len = t.n_tok;
    r.v_first = t.v_first;
    r.v_last = t.n_tok > 0 ? c.vers[(size_t)tid * c.cap + t.n_tok - 1] : -1;
    r.finish_step = t.finish_step;
    r.lifecycle = t.lifecycle;
    r.restarts = t.restarts;
    r.tok_offset = sh_off[i];
    r.final_group = s->group_final;
    r.epoch = t.epoch;
    c.h_rec[i] = r;
  }
  for (int i = 0; i < n; ++i) {
    const int tid = c.group[i];
    const int len = c.traj[tid].n_tok;
    const long long o = sh_off[i];
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      c.h_tok[o + j] = c.tokens[(size_t)tid * c.cap + j];
      c.h_lp[o + j] = c.lps[(size_t)tid * c.cap + j];
      c.h_ver[o + j] = c.vers[(size_t)tid * c.cap + j];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fill_status(c, SRL_OK);
    s->st.m_pre = (int)total;  // tokens staged (host marks the group harvested after copy-out)
  }
}

// ------------------------------------------------------------------ init / submit
__global__ void ctl_init_kernel(Ctl c, int K) {
  CtlState* s = c.s;
  for (int g = threadIdx.x; g < c.Q_tot; g += blockDim.x) c.slot_traj[g] = -1;
  for (int p = threadIdx.x; p < c.kv_pages; p += blockDim.x) c.page_stack[p] = c.kv_pages - 1 - p;
  for (int i = threadIdx.x; i < c.R * c.max_prompts; i += blockDim.x) c.pfx_ref[i] = c.pfx_tag[i] = 0;
  for (int i = threadIdx.x; i < c.R * c.max_prompts; i += blockDim.x) c.pfx_valid[i] = 0;
  if (threadIdx.x == 0) {
    memset(s, 0, sizeof(CtlState));
    s->K = K;
    s->own_top = c.kv_pages;
    for (int r = 0; r < c.R; ++r) s->free_pages[r] = c.kv_pages;
    s->epoch_of_latest = -1;
  }
}

__global__ void ctl_submit_kernel(Ctl c, int n_traj, int n_prompts) {
  if (threadIdx.x == 0) {
    c.s->n_stream += n_traj;
    c.s->n_prompts += n_prompts;
  }
}

static size_t sort_smem() {
  if (once_per_device(kOnceCtl)) {  // > 48 KB of dynamic shared memory: a per-device attribute
    cudaFuncSetAttribute(ctl_begin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSortReady * 8);
    cudaFuncSetAttribute(ctl_end_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSortReady * 8);
    cudaFuncSetAttribute(ctl_bump_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSortReady * 8);
  }
  return (size_t)kMaxSortReady * sizeof(long long);
}

void ctl_begin(const Ctl& c, cudaStream_t st) { ctl_begin_kernel<<<1, kCtlThreads, sort_smem(), st>>>(c); }
void ctl_end(const Ctl& c, cudaStream_t st) { launch_k(ctl_end_kernel, dim3(1), dim3(kCtlThreads), sort_smem(), st, 1, c); }
void ctl_bump(const Ctl& c, int version, cudaStream_t st) {
  ctl_bump_kernel<<<1, kCtlThreads, sort_smem(), st>>>(c, version);
}
void ctl_harvest(const Ctl& c, cudaStream_t st) { ctl_harvest_kernel<<<1, kCtlThreads, 0, st>>>(c); }
void ctl_init(const Ctl& c, int K, cudaStream_t st) { ctl_init_kernel<<<1, kCtlThreads, 0, st>>>(c, K); }
void ctl_submit(const Ctl& c, int n_traj, int n_prompts, cudaStream_t st) {
  ctl_submit_kernel<<<1, 32, 0, st>>>(c, n_traj, n_prompts);
}

}  // namespace srl
