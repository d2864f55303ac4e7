// engine.cu — host orchestration of one rollout decode step and the C ABI
// of include/srl.h.  All arithmetic of the step runs in the device kernels
// (gemm_tc.cu, layers.cu, attention.cu, sampler.cu, ctl.cu); this file plans
// memory, chains the launches on the caller's stream and mirrors a handful
// of host-side counters.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "comm.hpp"
#include "engine.hpp"
#include "kernels.hpp"
#include "layers.hpp"
#include "tma.hpp"
#include "tuning.hpp"

namespace srl {
extern thread_local std::string g_last_error;
void set_error(const char* fmt, const char* a, long b);
}  // namespace srl

using namespace srl;

namespace {

constexpr size_t kAlign = 1024;
constexpr int kMaxSmsPlan = 160;  // GEMM workspace sized for up to this many SMs
inline size_t al(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct LayerW {
  __nv_bfloat16 *attn_norm, *wqkv, *bqkv, *wo, *mlp_norm, *wgu, *wd;  // staging (srl_weight_layout)
  uint8_t *pqkv, *po, *pgu, *pd;                                     // packed GEMM copies (pack_weight)
};

bool is_packed_tensor(const std::string& n);
constexpr size_t kNoOff = ~size_t(0);  // compact weights: tensor held only in packed form

// ------------------------------------------------------------------ weight layout
struct WeightLayout {
  // row i of a tensor lives at byte off + ((i / row_block) * block_stride + i % row_block) * cols * 2
  struct Ent {
    std::string name;
    size_t off, numel;
    size_t rows, cols, row_block, block_stride;
  };
  std::vector<Ent> ents;
  size_t total = 0;
  bool compact = false;  // projection matrices get no staging storage
  void add(const std::string& n, size_t rows, size_t cols) {
    if (compact && is_packed_tensor(n)) {
      ents.push_back({n, kNoOff, rows * cols, rows, cols, rows, rows});
      return;
    }
    ents.push_back({n, total, rows * cols, rows, cols, rows, rows});
    total += al(rows * cols * 2);
  }
  // q/k/v (and their biases) must be contiguous: add them unaligned in one run
  void add_run(const std::vector<std::pair<std::string, size_t>>& run, size_t cols) {
    if (compact && is_packed_tensor(run[0].first)) {
      for (auto& e : run) ents.push_back({e.first, kNoOff, e.second * cols, e.second, cols, e.second, e.second});
      return;
    }
    size_t off = total;
    for (auto& e : run) {
      ents.push_back({e.first, off, e.second * cols, e.second, cols, e.second, e.second});
      off += e.second * cols * 2;
    }
    total = al(off);
  }
  // gate / up rows interleaved in kGuBlock-row blocks: one 128-row GEMM tile holds the
  // gate and up rows of the same 64 outputs, each warp's 32 rows those of 16 outputs
  // (fused SiLU-mul epilogue, gemm_epi.cuh)
  void add_gate_up(const std::string& g, const std::string& u, size_t ff, size_t cols) {
    const size_t o = compact ? kNoOff : total;
    ents.push_back({g, o, ff * cols, ff, cols, (size_t)kGuBlock, 2 * (size_t)kGuBlock});
    ents.push_back({u, compact ? kNoOff : total + kGuBlock * cols * 2, ff * cols, ff, cols, (size_t)kGuBlock,
                    2 * (size_t)kGuBlock});
    if (!compact) total += al(2 * ff * cols * 2);
  }
  const Ent* find(const std::string& n) const {
    for (auto& e : ents)
      if (e.name == n) return &e;
    return nullptr;
  }
};

WeightLayout make_layout(const srl_model_cfg& m) {
  WeightLayout w;
  w.compact = m.weights_compact != 0;
  const size_t d = m.d, qd = (size_t)m.Hq * m.dh, kd = (size_t)m.Hkv * m.dh, ff = m.ff;
  w.add("embed", m.V, d);
  for (int l = 0; l < m.L; ++l) {
    const std::string p = "L" + std::to_string(l) + ".";
    w.add(p + "attn_norm", d, 1);
    w.add_run({{p + "wq", qd}, {p + "wk", kd}, {p + "wv", kd}}, d);
    if (m.qkv_bias) w.add_run({{p + "bq", qd}, {p + "bk", kd}, {p + "bv", kd}}, 1);
    w.add(p + "wo", d, qd);
    w.add(p + "mlp_norm", d, 1);
    w.add_gate_up(p + "wg", p + "wu", ff, d);
    w.add(p + "wd", d, ff);
  }
  w.add("final_norm", d, 1);
  w.add("lm_head", m.V, d);
  return w;
}

// Packed copies of the projection matrices (the GEMM weight stream), placed after
// the staging region: per layer qkv, o, gate/up (interleaved rows), down; then lm_head.
struct PackedLayout {
  size_t base = 0, per_layer = 0, qkv = 0, o = 0, gu = 0, dn = 0, lm = 0, total = 0;
};
PackedLayout make_packed(const srl_model_cfg& m, size_t staging_total) {
  PackedLayout p;
  const int d = m.d, qd = m.Hq * m.dh, nqkv = (m.Hq + 2 * m.Hkv) * m.dh;
  p.base = al(staging_total);
  p.qkv = 0;
  p.o = p.qkv + al(packed_weight_bytes(nqkv, d));
  p.gu = p.o + al(packed_weight_bytes(d, qd));
  p.dn = p.gu + al(packed_weight_bytes(2 * m.ff, d));
  p.per_layer = p.dn + al(packed_weight_bytes(d, m.ff));
  p.lm = (size_t)m.L * p.per_layer;
  p.total = p.base + p.lm + al(packed_weight_bytes(m.V, d));
  return p;
}
// compact weights pack q / k / v separately: each must cover whole 128-row tiles
bool compact_ok(const srl_model_cfg& m) { return (m.Hq * m.dh) % 128 == 0 && (m.Hkv * m.dh) % 128 == 0; }

bool is_packed_tensor(const std::string& n) {
  static const char* kSuffix[] = {".wq", ".wk", ".wv", ".wo", ".wg", ".wu", ".wd"};
  if (n == "lm_head") return true;
  for (const char* x : kSuffix) {
    const size_t k = strlen(x);
    if (n.size() > k && n.compare(n.size() - k, k, x) == 0) return true;
  }
  return false;
}

// ------------------------------------------------------------------ scratch layout
struct ScratchPlan {
  size_t total = 0;
  size_t take(size_t bytes) {
    size_t o = total;
    total += al(bytes);
    return o;
  }
};

struct Sizes {
  int Q_g, R, Q_tot, max_pages, max_ctx, max_prompts, mmax, prefill_rows_max, max_items, G;
  int pfx_max;  // N4: shared prompt-prefix pages per (replica, prompt) entry
  long long ev_cap, h_cap_tok;
  size_t qkv_n;
};

int validate(const srl_model_cfg* m, const srl_sched_cfg* s, int world, std::string& why) {
  if (!m || !s) return why = "null config", -1;
  if (m->L <= 0 || m->d <= 0 || m->Hq <= 0 || m->Hkv <= 0 || m->dh <= 0 || m->ff <= 0 || m->V <= 0)
    return why = "model dims must be positive", -1;
  if (m->Hq % m->Hkv) return why = "Hq must be a multiple of Hkv", -1;
  if (m->Hq / m->Hkv > 8) return why = "GQA group > 8 not supported", -1;
  if (m->dh != 32 && m->dh != 64 && m->dh != 128) return why = "dh must be 32, 64 or 128", -1;
  if (m->d % 128 || (m->Hq * m->dh) % 64 || m->ff % 128) return why = "d, ff must be multiples of 128 and Hq*dh of 64", -1;
  if (m->d > 8192) return why = "d must be <= 8192", -1;
  if (m->weights_compact && !compact_ok(*m)) return why = "compact weights need Hq*dh and Hkv*dh multiples of 128", -1;
  if (s->Q_g <= 0 || s->U <= 0 || s->G <= 0 || s->cap <= 0 || s->pool_prompts <= 0 || s->kv_pages <= 0)
    return why = "Q_g, U, G, cap, pool_prompts, kv_pages must be positive", -1;
  if (s->page_tokens != kPage) return why = "page_tokens must be 64", -1;
  if (world < 1 || world > kMaxR) return why = "world out of range", -1;
  if ((long long)s->Q_g * world > 4096) return why = "Q_tot must be <= 4096", -1;
  if (s->mode < SRL_MODE_SORTED || s->mode > SRL_MODE_POSTHOC) return why = "mode", -1;
  if (s->mode != SRL_MODE_SYNC && s->U > s->pool_prompts * s->G) return why = "U larger than the prompt pool (S:252)", -1;
  if (s->U > kMaxGroup) return why = "U too large", -1;
  // the emission sort holds the whole ready list in shared memory: before a step it
  // has < U entries (>= U emits first), a step adds <= Q_tot finishes; POSTHOC keeps
  // the whole pool until it has finished
  if (s->mode == SRL_MODE_SORTED && (long long)s->U - 1 + (long long)s->Q_g * world > kMaxSortReady)
    return why = "U - 1 + Q_tot exceeds the emission sort capacity (16384)", -1;
  if (s->mode == SRL_MODE_POSTHOC && (long long)s->pool_prompts * s->G + s->U - 1 > kMaxSortReady)
    return why = "POSTHOC pool_prompts * G exceeds the emission sort capacity (16384)", -1;
  if (s->stop == SRL_STOP_EOS && s->eos_id < 0) return why = "EOS stop needs eos_id", -1;
  if (s->temperature <= 0.f) return why = "temperature must be > 0", -1;
  if (s->max_traj <= 0 || s->max_prompt <= 0 || s->prefill_chunk <= 0) return why = "max_traj, max_prompt, prefill_chunk must be positive", -1;
  if (s->kv_dtype != SRL_KV_BF16 && s->kv_dtype != SRL_KV_FP32) return why = "kv_dtype", -1;
  if (s->top_k < 0 || !(s->top_p > 0.f && s->top_p <= 1.f)) return why = "top_k must be >= 0 and top_p in (0, 1]", -1;
  if (s->share_prefix != 0 && s->share_prefix != 1) return why = "share_prefix must be 0 or 1", -1;
  if (s->prefill_budget < 0) return why = "prefill_budget must be >= 0 (0 = unlimited)", -1;
  if (s->prefill_budget > 0 && s->share_prefix && s->G > 1)
    return why = "prefill_budget and share_prefix are exclusive (reading R30)", -1;
  return 0;
}

Sizes compute_sizes(const srl_model_cfg* m, const srl_sched_cfg* s, int world) {
  Sizes z;
  z.Q_g = s->Q_g;
  z.R = world;
  z.Q_tot = s->Q_g * world;
  z.max_ctx = s->max_prompt + s->cap;
  z.max_pages = (z.max_ctx + kPage - 1) / kPage;
  z.max_prompts = (s->max_traj + s->G - 1) / s->G + 1;
  z.pfx_max = s->max_prompt > 1 ? (s->max_prompt - 1) / kPage : 0;
  if (z.pfx_max < 1) z.pfx_max = 1;
  z.prefill_rows_max = s->Q_g * (z.max_ctx);
  z.mmax = s->Q_g + s->prefill_chunk;  // a mixed pass: Q_g decode rows + up to prefill_chunk prompt rows
  z.G = m->Hq / m->Hkv;
  const int a1 = attn_max_items(s->Q_g, m->Hkv, z.max_ctx);
  const int a2 = (s->Q_g + s->prefill_chunk) * m->Hkv;  // mixed / prefill passes never split the KV
  z.max_items = a1 > a2 ? a1 : a2;
  z.ev_cap = 1LL << 20;
  const int gmax = s->max_traj < kMaxGroup ? s->max_traj : kMaxGroup;
  z.h_cap_tok = (long long)gmax * s->cap;
  z.qkv_n = (size_t)(m->Hq + 2 * m->Hkv) * m->dh;

  return z;
}

}  // namespace

// ------------------------------------------------------------------ the engine
struct srl_engine {
  srl_model_cfg m;
  srl_sched_cfg s;
  Sizes z;
  int rank = 0, world = 1, device = 0, num_sms = 148;
  cudaStream_t st = nullptr;
  Comm* comm = nullptr;  // replica exchange (NCCL or in-process); null for a lone engine
  bool kv_f32 = false;
  // arena
  uint8_t *W = nullptr, *KV = nullptr, *S = nullptr;
  WeightLayout wl;
  std::vector<LayerW> lw;
  __nv_bfloat16 *embed = nullptr, *final_norm = nullptr, *lm_head = nullptr;
  uint8_t* plm_head = nullptr;  // packed copy
  PackedLayout pk;
  std::vector<void*> kpool, vpool;
  std::vector<CUtensorMap> tmK, tmV;
  // scratch
  float* x_res = nullptr;
  __nv_bfloat16 *xn = nullptr, *attn_out = nullptr, *act = nullptr;
  void* qbuf = nullptr;
  float* logits = nullptr;
  float *rope_cos = nullptr, *rope_sin = nullptr;
  void* gemm_ws = nullptr;     // GEMM stream-K workspace (zeroed at create, left zeroed by every launch)
  float* qkv_part = nullptr;     // split-K partials of the QKV projection for qkv_finish
  size_t qkv_part_floats = 0;
  float* norm_part = nullptr;    // split-K partials of the O / down projections for the next RMSNorm
  size_t norm_part_floats = 0;
  float4* samp_part = nullptr;  // [Q_g][ceil(V/128)] Gumbel-max partials of the fused LM head
  int* samp_part_j = nullptr;
  size_t gemm_ws_bytes = 0;
  AttnArgs attn{};
  Ctl ctl{};
  CtlStatus* hst = nullptr;  // pinned
  // host mirrors
  std::unordered_set<uint64_t> ids;
  std::vector<uint64_t> prompt_ids;
  long long n_traj = 0, n_prompts = 0, prompt_tok_used = 0, prompt_tok_cap = 0;
  int group_state = 0;  // 0 none, 1 ready, 2 harvested
  bool v_valid = false;
  long long v = -1;
  long long launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // profiling: event pairs bracketing kernel classes.  `direct` is refilled every
  // step; `gset` belongs to the captured decode graph and is re-recorded by
  // every replay.
  struct EvSet {
    std::vector<cudaEvent_t> ev;
    size_t used = 0;
    std::vector<int> cls, nl;
  };
  bool prof = false;
  uint32_t prof_mask = 0xffffffffu;  // classes bracketed while profiling
  bool capturing = false;
  EvSet direct;
  EvSet* gset = nullptr;  // event set of the graph being captured / replayed
  double prof_ms[SRL_K_NCLASS] = {0};
  long long prof_launch[SRL_K_NCLASS] = {0};
  // CUDA graph of the static decode tail (forward + sampler + ctl_end)
  bool use_graph = true;
  // one graph per decode-row bucket M (rows = the running slots, compacted):
  // at low occupancy (epoch drains) the GEMMs stream the weights for M rows, not Q_g
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    long long launches = 0;
    int direct = 0;  // direct runs of this bucket (the first step of a bucket runs uncaptured)
    EvSet gset;
  };
  // keyed by (decode rows M, profiled-class mask): switching the mask between steps
  // (e.g. every class on sampled steps, one class otherwise) replays a graph of
  // each kind instead of recapturing
  std::map<std::pair<int, uint32_t>, Graph> graphs;
  int last_m = 0;  // decode rows of the last step
  bool mixed_ok = true;
  long long comm_timeout_ms = 300000;
  bool comm_dead = false;
  long long last_harvest_tok = 0;  // tokens / records of the last harvested group (srl_harvest_device)
  int last_harvest_n = 0;
  bool harvest_valid = false;        // the replica transport failed or timed out: every call fails
  cudaEvent_t ev_sync = nullptr;
  int launch_rc = 0;             // first failed launch of the current step (note_launch)
  const char* launch_what = "";
};

namespace {

// Brackets a group of launches of one kernel class with CUDA events on the
// engine stream (only when profiling is on).
struct Prof {
  srl_engine* e;
  srl_engine::EvSet* S = nullptr;
  int cls;
  int nl;
  Prof(srl_engine* e_, int cls_, int nlaunch = 1) : e(e_), cls(cls_), nl(nlaunch) {
    if (cls < 0) return;
    // Only profiled classes get event records: an event node between two kernels
    // of the captured graph replaces their programmatic (PDL) edge by a full one.
    if (!e->prof || !((e->prof_mask >> cls) & 1u)) return;
    S = e->capturing ? e->gset : &e->direct;
    if (S->used + 2 > S->ev.size()) {
      for (int i = 0; i < 256; ++i) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        S->ev.push_back(ev);
      }
    }
    record(S->ev[S->used]);
  }
  // inside a stream capture the record must be an external event-record node
  void record(cudaEvent_t ev) {
    if (e->capturing)
      cudaEventRecordWithFlags(ev, e->st, cudaEventRecordExternal);
    else
      cudaEventRecord(ev, e->st);
  }
  ~Prof() {
    if (!S) return;
    record(S->ev[S->used + 1]);
    S->cls.push_back(cls);
    S->nl.push_back(nl);
    S->used += 2;
  }
};

void prof_collect(srl_engine* e, srl_engine::EvSet& S, bool keep) {  // after a stream sync
  if (e->prof) {
    for (size_t i = 0; i < S.cls.size(); ++i) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, S.ev[2 * i], S.ev[2 * i + 1]) != cudaSuccess) {
        cudaGetLastError();  // timing unavailable: never poison the engine's error state
        ms = 0.f;
      }
      e->prof_ms[S.cls[i]] += ms;
      e->prof_launch[S.cls[i]] += S.nl[i];
    }
  }
  if (!keep) {
    S.cls.clear();
    S.nl.clear();
    S.used = 0;
  }
}

int cuda_fail(const char* what, cudaError_t e = cudaSuccess) {
  if (e == cudaSuccess) e = cudaGetLastError();
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
  g_last_error = buf;
  return SRL_E_CUDA;
}

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

void plan_scratch(srl_engine* e, ScratchPlan& p, bool assign) {
  const Sizes& z = e->z;
  const srl_model_cfg& m = e->m;
  const srl_sched_cfg& s = e->s;
  uint8_t* B = e->S;
  auto P = [&](size_t bytes) -> void* { size_t o = p.take(bytes); return assign ? (void*)(B + o) : nullptr; };
  Ctl& c = e->ctl;
  c.s = (CtlState*)P(sizeof(CtlState));
  c.traj = (DevTraj*)P(sizeof(DevTraj) * s.max_traj);
  c.slot_traj = (int*)P(4 * z.Q_tot);
  c.page_table = (int*)P(4ull * z.Q_g * z.max_pages);
  c.page_stack = (int*)P(4ull * s.kv_pages);
  c.resumed = (int*)P(4ull * s.max_traj);
  c.ready = (int*)P(4ull * s.max_traj);
  c.group = (int*)P(4ull * s.max_traj);
  c.tokens = (int*)P(4ull * s.max_traj * s.cap);
  c.lps = (float*)P(4ull * s.max_traj * s.cap);
  c.vers = (int*)P(4ull * s.max_traj * s.cap);
  c.prompt_off = (int*)P(4ull * (z.max_prompts + 1));
  c.prompt_tok = (int*)P(4ull * z.max_prompts * s.max_prompt);
  c.events = (int*)P(24ull * z.ev_cap);
  c.pfx_ref = (int*)P(4ull * z.R * z.max_prompts);
  c.pfx_tag = (int*)P(4ull * z.R * z.max_prompts);
  c.pfx_pages = (int*)P(4ull * z.max_prompts * z.pfx_max);
  c.pfx_valid = (int*)P(4ull * z.R * z.max_prompts);
  c.pre_list = (int*)P(12ull * (z.Q_g + 1));
  // decode rows [0, Q_g) and prefill rows [Q_g, ...) are one array each, so one
  // forward can run both (the mixed pass of a step with admissions)
  c.row_tok = (int*)P(4ull * (z.Q_g + z.prefill_rows_max));
  c.row_pos = (int*)P(4ull * (z.Q_g + z.prefill_rows_max));
  c.row_n = (int*)P(4 * z.Q_g);
  c.row_traj = (int*)P(4 * z.Q_g);
  c.row_restarts = (int*)P(4 * z.Q_g);
  c.row_slot = (int*)P(4ull * (z.Q_g + z.prefill_rows_max));
  c.pre_tok = c.row_tok + z.Q_g;
  c.pre_pos = c.row_pos + z.Q_g;
  c.pre_slot = c.row_slot + z.Q_g;
  c.admit_local = (int*)P(4 * z.Q_g);
  c.samp = (int*)P(8 * z.Q_tot);
  c.h_tok = (int*)P(4ull * z.h_cap_tok);
  c.h_lp = (float*)P(4ull * z.h_cap_tok);
  c.h_ver = (int*)P(4ull * z.h_cap_tok);
  c.h_rec = (srl_traj*)P(sizeof(srl_traj) * kMaxGroup);
  // S <= 4 splits of <= 512 rows (gemm_partial_split), <= kNormMaxSplits of <= 256 rows (fused MLP)
  e->norm_part_floats = std::max(4ull * (z.Q_g > 512 ? z.Q_g : 512), (unsigned long long)kNormMaxSplits * 256) * m.d;
  e->norm_part = (float*)P(4ull * e->norm_part_floats);
  e->qkv_part_floats = 4ull * (z.Q_g > 512 ? z.Q_g : 512) * z.qkv_n;
  e->qkv_part = (float*)P(4ull * e->qkv_part_floats);
  e->samp_part = (float4*)P(16ull * z.Q_g * ((m.V + 127) / 128));
  e->samp_part_j = (int*)P(4ull * z.Q_g * ((m.V + 127) / 128));
  e->gemm_ws_bytes = gemm_workspace_bytes(kMaxSmsPlan);
  e->gemm_ws = P(e->gemm_ws_bytes);
  e->x_res = (float*)P(4ull * z.mmax * m.d);
  e->xn = (__nv_bfloat16*)P(2ull * z.mmax * m.d);
  e->attn_out = (__nv_bfloat16*)P(2ull * z.mmax * m.Hq * m.dh);
  e->act = (__nv_bfloat16*)P(2ull * z.mmax * m.ff);
  e->qbuf = P((e->kv_f32 ? 4ull : 2ull) * z.mmax * m.Hq * m.dh);
  e->logits = (float*)P(4ull * z.Q_g * m.V);
  e->rope_cos = (float*)P(4ull * z.max_ctx * (m.dh / 2));
  e->rope_sin = (float*)P(4ull * z.max_ctx * (m.dh / 2));
  AttnArgs& a = e->attn;
  a.items = (int*)P(12ull * z.max_items);
  a.order = (int*)P(4ull * z.max_items);
  a.work_ctr = (int*)P(4ull * m.L);
  a.n_ctr = m.L;
  a.merge_ctr = (int*)P(4ull * z.mmax * m.Hkv);
  a.chunk_pages = (int*)P(64);
  a.n_items = (int*)P(64);
  a.row_item0 = (int*)P(4ull * z.mmax);
  a.row_nchunk = (int*)P(4ull * z.mmax);
  a.part_o = (float*)P(4ull * z.max_items * z.G * m.dh);
  a.part_ml = (float*)P(8ull * z.max_items * z.G);
}

size_t kv_bytes_for(const srl_model_cfg& m, const srl_sched_cfg& s) {
  const size_t el = s.kv_dtype == SRL_KV_FP32 ? 4 : 2;
  return al((size_t)s.kv_pages * m.Hkv * kPage * m.dh * el) * 2 * m.L;
}

// LM head + sampler fusion (EPI_SAMPLE + sample_reduce), opt-in (srl_tuning.fused_sample).
// Measured r01 (cfg2): the Gumbel-max work in the LM head's 8 epilogue warps per SM
// outlasts the MMAs it should hide behind (LM head 0.21 -> 0.77 ms per step) while
// the stand-alone sampler, 256 CTAs x 16 warps, costs 0.22 ms -- so it stays off.
bool fused_sample() { return tuning().fused_sample != 0; }

// Records the first failed launch of a step (reported by srl_decode_step as
// SRL_E_CUDA; the launchers clear the non-sticky error they saw).
void note_launch(srl_engine* e, const char* what, int rc) {
  if (rc == 0 || e->launch_rc) return;
  e->launch_rc = rc;
  e->launch_what = what;
}

// ---- fused GEMM helper
// one fused GEMM launch, profiled under `cls`
void run_gemm(srl_engine* e, int cls, const __nv_bfloat16* X, int M, const __nv_bfloat16* W, int N, int K,
              const GemmEpi& epi) {
  Prof p(e, cls);
  if (cudaError_t pre = cudaGetLastError()) note_launch(e, "launch before a GEMM", (int)pre);
  note_launch(e, "GEMM launch", gemm_bf16_fused(X, M, W, N, K, epi, e->num_sms, e->st));
  e->launches++;
}

// One forward pass over M rows (decode: rows = local slots; prefill: rows = prompt tokens).
// m_lm: rows that get logits (the decode rows, first in the batch); -1 = M.
// split: allow split-KV attention (decode passes; never with prompt rows).
void forward(srl_engine* e, int M, const int* row_tok, const int* row_pos, const int* row_slot, bool decode,
             int m_lm = -1, int split = -1) {
  const srl_model_cfg& m = e->m;
  cudaStream_t st = e->st;
  const int d = m.d, qd = m.Hq * m.dh;
  const int Nqkv = (int)e->z.qkv_n;
  AttnArgs a = e->attn;
  a.q = e->qbuf;
  a.row_pos = row_pos;
  a.row_slot = row_slot;
  a.page_table = e->ctl.page_table;
  a.max_pages = e->z.max_pages;
  a.M = M;
  a.Hq = m.Hq;
  a.Hkv = m.Hkv;
  a.dh = m.dh;
  a.out = e->attn_out;
  a.max_items = e->z.max_items;
  a.scale = 1.0f / sqrtf((float)m.dh);
  const int D = decode ? 0 : -1000;  // profiling class offset (prefill is timed as a whole)
  {
    Prof p1(e, D + SRL_K_ATTN);
    attn_plan(a, split >= 0 ? split : (decode ? 1 : 0), st);
  }
  {
    Prof p2(e, D + SRL_K_ELEMWISE);
    rmsnorm(e->x_res, row_tok, row_pos, M, d, e->embed, e->lw[0].attn_norm, m.rms_eps, e->xn, st);
  }
  e->launches += 2;
  GemmEpi qe{};
  qe.kind = EPI_QKV;
  qe.row_pos = row_pos;
  qe.row_slot = row_slot;
  qe.page_table = e->ctl.page_table;
  qe.max_pages = e->z.max_pages;
  qe.rope_cos = e->rope_cos;
  qe.rope_sin = e->rope_sin;
  qe.q_out = e->qbuf;
  qe.Hq = m.Hq;
  qe.Hkv = m.Hkv;
  qe.dh = m.dh;
  qe.kv_f32 = e->kv_f32 ? 1 : 0;
  qe.w_packed = 1;
  qe.ws = e->gemm_ws;
  GemmEpi re{};
  re.w_packed = 1;
  re.ws = e->gemm_ws;
  re.kind = EPI_RESID;
  re.x_res = e->x_res;
  re.ldo = d;
  // split-K O / down projections hand their partials to the next RMSNorm (which
  // sums them in split order and adds the residual: the same fp32 operations the
  // GEMM's own DSMEM reduction + residual add would do) when the pair GEMM splits
  int S_o = gemm_partial_split(M, d, qd, e->num_sms), S_d = gemm_partial_split(M, d, m.ff, e->num_sms);
  if ((size_t)S_o * M * d > e->norm_part_floats || S_o > 4) S_o = 1;  // rmsnorm sums <= 4 splits
  if ((size_t)S_d * M * d > e->norm_part_floats || S_d > 4) S_d = 1;
  // fused MLP (decode rows 128..256 on the pair kernel): down k-splits for the RMSNorm
  int mlp_S = tuning().fuse_mlp ? tuning().mlp_splits : 0;
  if (mlp_S > kNormMaxSplits || (size_t)mlp_S * M * d > e->norm_part_floats) mlp_S = 0;
  // the QKV projection can likewise leave its partials to qkv_finish (bias, RoPE, KV
  // append) -- opt-in (srl_tuning.qkv_finish): measured r01 even with the in-GEMM
  // reduction (QKV class -0.02 ms, attention +0.1 ms per step)
  int S_q = tuning().qkv_finish ? gemm_partial_split(M, Nqkv, d, e->num_sms) : 1;
  if ((size_t)S_q * M * Nqkv > e->qkv_part_floats) S_q = 1;
  // ... or to the attention kernel, whose producer warps finish q / k / v per item
  // (pure decode passes: every row's KV append precedes only its own attention)
  const bool pure_decode = decode && (m_lm < 0 || m_lm >= M);
  int S_qa = (pure_decode && !e->kv_f32 && tuning().qkv_attn) ? gemm_partial_split(M, Nqkv, d, e->num_sms) : 1;
  if ((size_t)S_qa * M * Nqkv > e->qkv_part_floats) S_qa = 1;
  if (S_qa > 1) S_q = 1;
  a.qkv_part = nullptr;
  a.qkv_part_stride = (size_t)M * Nqkv;
  a.qkv_S = S_qa;
  a.Nqkv = Nqkv;
  a.rope_cos = e->rope_cos;
  a.rope_sin = e->rope_sin;
  GemmEpi pq{};
  pq.kind = EPI_PARTIAL;
  pq.w_packed = 1;
  pq.ws = e->gemm_ws;
  pq.part = e->qkv_part;
  pq.part_stride = (size_t)M * Nqkv;
  pq.ldo = Nqkv;
  GemmEpi pe = re;
  pe.kind = EPI_PARTIAL;
  pe.part = e->norm_part;
  pe.part_stride = (size_t)M * d;
  pe.ldo = d;
  GemmEpi se{};
  se.w_packed = 1;
  se.ws = e->gemm_ws;
  se.kind = EPI_SILU;
  se.act = e->act;
  se.ldo = m.ff;
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = e->lw[l];
    qe.bias = m.qkv_bias ? w.bqkv : nullptr;
    qe.k_pool = e->kpool[l];
    qe.v_pool = e->vpool[l];
    a.qkv_part = nullptr;
    if (S_qa > 1) {  // split-K partials, finished inside the attention kernel
      run_gemm(e, D + SRL_K_GEMM_QKV, e->xn, M, (const __nv_bfloat16*)w.pqkv, Nqkv, d, pq);
      a.qkv_part = e->qkv_part;
      a.qkv_bias = qe.bias;
    } else if (S_q > 1) {  // split-K partials, then bias + RoPE + KV append in one elementwise pass
      run_gemm(e, D + SRL_K_GEMM_QKV, e->xn, M, (const __nv_bfloat16*)w.pqkv, Nqkv, d, pq);
      {
        Prof p(e, D + SRL_K_GEMM_QKV);
        QkvFinishArgs fa{};
        fa.part = e->qkv_part;
        fa.part_stride = (size_t)M * Nqkv;
        fa.nsplit = S_q;
        fa.bias = qe.bias;
        fa.row_pos = row_pos;
        fa.row_slot = row_slot;
        fa.page_table = e->ctl.page_table;
        fa.max_pages = e->z.max_pages;
        fa.rope_cos = e->rope_cos;
        fa.rope_sin = e->rope_sin;
        fa.q_out = e->qbuf;
        fa.k_pool = e->kpool[l];
        fa.v_pool = e->vpool[l];
        fa.Hq = m.Hq;
        fa.Hkv = m.Hkv;
        fa.dh = m.dh;
        fa.kv_f32 = e->kv_f32 ? 1 : 0;
        qkv_finish(fa, M, st);
        e->launches++;
      }
    } else {
      run_gemm(e, D + SRL_K_GEMM_QKV, e->xn, M, (const __nv_bfloat16*)w.pqkv, Nqkv, d, qe);
    }
    a.k_pool = e->kpool[l];
    a.v_pool = e->vpool[l];
    a.work_ctr = e->attn.work_ctr + l;  // one counter per layer, all zeroed by attn_plan
    {
      Prof p(e, D + SRL_K_ATTN, 2);
      attn_run(a, e->kv_f32, &e->tmK[l], &e->tmV[l], st);
    }
    run_gemm(e, D + SRL_K_GEMM_O, e->attn_out, M, (const __nv_bfloat16*)w.po, d, qd, S_o > 1 ? pe : re);
    {
      Prof p(e, D + SRL_K_ELEMWISE);
      rmsnorm(e->x_res, row_tok, row_pos, M, d, nullptr, w.mlp_norm, m.rms_eps, e->xn, st,
              S_o > 1 ? e->norm_part : nullptr, S_o, (size_t)M * d);
    }
    // gate/up (SiLU-mul) and down: one persistent kernel whose down k-splits fill the
    // gate/up tail (gemm_pair.cuh SPLIT 3), else two GEMMs
    int S_dn = S_d, fused = 1;
    if (mlp_S > 1) {
      Prof p(e, D + SRL_K_GEMM_GU);
      fused = gemm_mlp_fused(e->xn, M, w.pgu, m.ff, d, e->act, w.pd, e->norm_part, (size_t)M * d, mlp_S, e->gemm_ws,
                             e->num_sms, st);
      if (fused < 0) note_launch(e, "fused MLP launch", fused);
      if (fused == 0) S_dn = mlp_S;
      e->launches += fused == 0;
    }
    if (fused != 0) {
      run_gemm(e, D + SRL_K_GEMM_GU, e->xn, M, (const __nv_bfloat16*)w.pgu, 2 * m.ff, d, se);  // interleaved gate/up
      run_gemm(e, D + SRL_K_GEMM_DOWN, e->act, M, (const __nv_bfloat16*)w.pd, d, m.ff, S_d > 1 ? pe : re);
    }
    {
      Prof p(e, D + SRL_K_ELEMWISE);
      const __nv_bfloat16* next = l + 1 < m.L ? e->lw[l + 1].attn_norm : e->final_norm;
      rmsnorm(e->x_res, row_tok, row_pos, M, d, nullptr, next, m.rms_eps, e->xn, st,
              S_dn > 1 ? e->norm_part : nullptr, S_dn, (size_t)M * d);
    }
    e->launches += 4;  // attention (2 launches) + the two RMSNorms
  }
  if (decode) {
    GemmEpi fe{};
    fe.kind = EPI_F32;
    fe.out_f32 = e->logits;
    fe.ldo = m.V;
    fe.w_packed = 1;
    fe.ws = e->gemm_ws;
    if (fused_sample() && e->s.top_k == 0 && e->s.top_p >= 1.f) {  // Gumbel-max in the LM head's epilogue
      const Ctl& c = e->ctl;
      fe.kind = EPI_SAMPLE;
      fe.s_row_pos = row_pos;
      fe.s_row_n = c.row_n;
      fe.s_row_traj = c.row_traj;
      fe.s_row_restarts = c.row_restarts;
      fe.s_invT = 1.0f / e->s.temperature;
      fe.s_seed = e->s.sample_seed;
      fe.s_part = e->samp_part;
      fe.s_part_j = e->samp_part_j;
      fe.s_nblk = (m.V + 127) / 128;
    }
    run_gemm(e, SRL_K_LM_HEAD, e->xn, m_lm >= 0 ? m_lm : M, (const __nv_bfloat16*)e->plm_head, m.V, d, fe);
  }
}

// Decode-row bucket for r running local rows: the GEMM batch M.  Fine steps where
// the weight stream dominates (few rows), coarser ones near full occupancy;
// always a multiple of 16 (the UMMA N granularity) up to Q_g.
int decode_rows(const srl_engine* e, int r) {
  const int Q = e->s.Q_g;
  int m;
  if (r <= 64) m = (r + 15) / 16 * 16;
  else if (r <= 256) m = (r + 31) / 32 * 32;
  else m = (r + 63) / 64 * 64;
  if (m < 16) m = 16;
  return m < Q ? m : Q;
}

// decode forward over the local slots, sampler and (alone) controller END --
// static shapes.  With a replica exchange the END runs after the all-gather.
// M_pre > 0: the mixed pass of a step with admissions -- the decode rows [0, M) are
// followed (from row Q_g) by the admitted prompts' rows, all in one forward, so
// the prompts ride on the step's weight stream instead of a pass of their own
// (chunked prefill); logits and sampling cover the decode rows only.
void decode_tail(srl_engine* e, bool with_end, int M, int M_pre = 0) {
  const Ctl& c = e->ctl;
  cudaStream_t st = e->st;
  if (M_pre > 0)
    forward(e, e->s.Q_g + M_pre, c.row_tok, c.row_pos, c.row_slot, true, M, 0);
  else
    forward(e, M, c.row_tok, c.row_pos, c.row_slot, true);
  SampleArgs sa{};
  sa.logits = e->logits;
  sa.M = M;
  sa.row_slot = c.row_slot;
  sa.V = e->m.V;
  sa.row_pos = c.row_pos;
  sa.row_n = c.row_n;
  sa.row_traj = c.row_traj;
  sa.row_restarts = c.row_restarts;
  sa.invT = 1.0f / e->s.temperature;
  sa.seed = e->s.sample_seed;
  sa.top_k = e->s.top_k;
  sa.top_p = e->s.top_p;
  sa.tok_out = c.samp + (size_t)e->rank * 2 * e->s.Q_g;
  sa.lp_out = (float*)(c.samp + (size_t)e->rank * 2 * e->s.Q_g + e->s.Q_g);
  {
    Prof p(e, SRL_K_SAMPLE);
    if (fused_sample() && sa.top_k == 0 && sa.top_p >= 1.f)
      sample_reduce(sa, e->samp_part, e->samp_part_j, (e->m.V + 127) / 128, st);
    else
      sample(sa, st);
  }
  e->launches++;
  if (!with_end) return;
  {
    Prof p(e, SRL_K_CTL);
    ctl_end(c, st);
  }
  e->launches++;
}

// Rows a14 + a12/a13: every replica's (token, logprob) rows reach every rank, then
// the replicated controller END runs identically everywhere (reading R24).
int exchange_and_end(srl_engine* e) {
  std::string err;
  {
    Prof p(e, SRL_K_COMM);
    if (e->comm->allgather_inplace(e->ctl.samp, 8ull * e->s.Q_g, e->st, err)) {
      e->comm->abort();
      e->comm_dead = true;
      return fail(SRL_E_NCCL, "srl_decode_step: replica all-gather: " + err);
    }
  }
  {
    Prof p(e, SRL_K_CTL);
    ctl_end(e->ctl, e->st);
  }
  e->launches++;
  return SRL_OK;
}

// Waits for the engine stream.  Alone: a plain synchronise.  With replicas the
// stream may hold a collective whose peer died, so the wait is a poll with a
// deadline that also watches the transport's asynchronous error; on either the
// communicator is aborted and the engine is dead (SRL_E_NCCL from then on).
int stream_wait(srl_engine* e, const char* what) {
  if (!e->comm) {
    const cudaError_t ce = cudaStreamSynchronize(e->st);
    return ce == cudaSuccess ? 0 : cuda_fail(what, ce);
  }
  if (cudaEventRecord(e->ev_sync, e->st) != cudaSuccess) return cuda_fail(what);
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaEventQuery(e->ev_sync);
    if (q == cudaSuccess) return 0;
    if (q != cudaErrorNotReady) return cuda_fail(what, q);
    std::string err;
    const bool late = std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(e->comm_timeout_ms);
    if (e->comm->poll_error(err) || late) {
      e->comm->abort();
      e->comm_dead = true;
      return fail(SRL_E_NCCL, std::string(what) + ": replica transport " + (late ? "timed out" : "failed: " + err) +
                                  " -- communicator aborted");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

int read_status(srl_engine* e, const char* what = "status read-back") {
  cudaMemcpyAsync(e->hst, &e->ctl.s->st, sizeof(CtlStatus), cudaMemcpyDeviceToHost, e->st);
  return stream_wait(e, what);
}

}  // namespace

// ================================================================== C ABI

// end of a decode step: status read-back, profiling, step info
static int32_t finish_step(srl_engine* e, const CtlStatus& b, srl_step_info* info, srl_engine::EvSet* gset) {
  cudaStream_t st = e->st;
  if (e->launch_rc) {  // a launch of this step failed: its outputs are stale, say so
    const int rc = e->launch_rc;
    e->launch_rc = 0;
    cudaGetLastError();
    char buf[160];
    snprintf(buf, sizeof(buf), "srl_decode_step: %s failed (code %d)", e->launch_what, rc);
    return fail(SRL_E_CUDA, buf);
  }
  cudaEventRecord(e->ev1, st);
  if (int rc = read_status(e, "srl_decode_step")) return rc;
  if (cudaError_t ce = cudaGetLastError()) return cuda_fail("decode step", ce);
  prof_collect(e, e->direct, false);
  if (gset) prof_collect(e, *gset, true);
  const CtlStatus& en = *e->hst;
  if (info) {
    info->k = en.k - 1;
    info->r_k = en.r_k;
    info->n_finished = en.n_fin;
    info->n_ready = en.n_ready;
    info->n_admitted = b.n_admit;
    info->n_prefill_tokens = b.m_pre;
    info->sum_ctx = b.sum_ctx;
    info->r_local = b.r_local;
    info->v = en.v;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e->ev0, e->ev1);
    info->dt_ms = ms;
  }
  if (en.status == SRL_GROUP_READY) e->group_state = 1;
  return en.status;
}

extern "C" {

int32_t srl_arena_sizes(const srl_model_cfg* m, const srl_sched_cfg* s, int32_t world, uint64_t* wb, uint64_t* kb,
                        uint64_t* sb) {
  std::string why;
  if (validate(m, s, world, why)) return fail(SRL_E_INVALID_ARG, "srl_arena_sizes: " + why);
  srl_engine tmp;
  tmp.m = *m;
  tmp.s = *s;
  tmp.z = compute_sizes(m, s, world);
  tmp.kv_f32 = s->kv_dtype == SRL_KV_FP32;
  ScratchPlan p;
  plan_scratch(&tmp, p, false);
  if (wb) *wb = make_packed(*m, make_layout(*m).total).total;
  if (kb) *kb = kv_bytes_for(*m, *s);
  if (sb) *sb = p.total;
  return SRL_OK;
}

int64_t srl_weight_offset(const srl_model_cfg* m, const char* name, int64_t* numel) {
  if (!m || !name) return -1;
  WeightLayout w = make_layout(*m);
  const WeightLayout::Ent* e = w.find(name);
  if (!e || e->off == kNoOff) return -1;
  if (numel) *numel = (int64_t)e->numel;
  return (int64_t)e->off;
}

int32_t srl_weight_layout(const srl_model_cfg* m, const char* name, int64_t* offset, int64_t* rows, int64_t* cols,
                          int64_t* row_block, int64_t* block_stride) {
  if (!m || !name) return fail(SRL_E_INVALID_ARG, "srl_weight_layout: null argument");
  WeightLayout w = make_layout(*m);
  const WeightLayout::Ent* e = w.find(name);
  if (!e) return fail(SRL_E_INVALID_ARG, std::string("srl_weight_layout: unknown tensor ") + name);
  if (e->off == kNoOff)
    return fail(SRL_E_INVALID_ARG, std::string("srl_weight_layout: ") + name +
                                       " is held only in packed form (compact weights): use srl_load_policy_tensor");
  if (offset) *offset = (int64_t)e->off;
  if (rows) *rows = (int64_t)e->rows;
  if (cols) *cols = (int64_t)e->cols;
  if (row_block) *row_block = (int64_t)e->row_block;
  if (block_stride) *block_stride = (int64_t)e->block_stride;
  return SRL_OK;
}

int32_t srl_create(const srl_model_cfg* m, const srl_sched_cfg* s, int32_t device, void* stream, const srl_arena* mem,
                   const srl_comm* comm, srl_engine** out) {
  if (!out || !mem) return fail(SRL_E_INVALID_ARG, "srl_create: null argument");
  const int world = comm ? comm->world : 1;
  std::string why;
  if (validate(m, s, world, why)) return fail(SRL_E_INVALID_ARG, "srl_create: " + why);
  if (comm && (comm->rank < 0 || comm->rank >= world || comm->kind < SRL_COMM_NCCL || comm->kind > SRL_COMM_HOST ||
               comm->timeout_s < 0))
    return fail(SRL_E_INVALID_ARG, "srl_create: bad srl_comm (rank / kind / timeout)");
  uint64_t wb, kb, sb;
  srl_arena_sizes(m, s, world, &wb, &kb, &sb);
  if (mem->weights_bytes < wb || mem->kv_bytes < kb || mem->scratch_bytes < sb || !mem->weights || !mem->kv || !mem->scratch)
    return fail(SRL_E_CAPACITY, "srl_create: arena smaller than srl_arena_sizes");
  if (cudaSetDevice(device) != cudaSuccess) return cuda_fail("cudaSetDevice");
  srl_engine* e = new srl_engine();
  e->m = *m;
  e->s = *s;
  e->world = world;
  e->rank = comm ? comm->rank : 0;
  e->device = device;
  e->st = (cudaStream_t)stream;
  e->kv_f32 = s->kv_dtype == SRL_KV_FP32;
  e->z = compute_sizes(m, s, world);
  e->use_graph = tuning().graphs != 0 && stream != nullptr;  // the legacy stream cannot be captured
  e->mixed_ok = tuning().mixed_prefill != 0;
  if (comm) {
    e->comm_timeout_ms = (comm->timeout_s > 0 ? comm->timeout_s : 300) * 1000LL;
    if (comm->kind == SRL_COMM_NCCL)
      e->comm = comm_create_nccl(comm->nccl_unique_id, comm->rank, world, (int)e->comm_timeout_ms, why);
    else if (comm->kind == SRL_COMM_LOCAL)
      e->comm = comm_create_local(comm->local_group, comm->rank, world, (int)e->comm_timeout_ms, why);
    else
      e->comm = comm_create_host(comm->host, comm->rank, world, why);
    if (!e->comm) {
      delete e;
      return fail(SRL_E_NCCL, "srl_create: replica communicator: " + why);
    }
  }
  cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, device);
  e->W = (uint8_t*)mem->weights;
  e->KV = (uint8_t*)mem->kv;
  e->S = (uint8_t*)mem->scratch;
  // weights
  e->wl = make_layout(*m);
  auto wp = [&](const std::string& n) -> __nv_bfloat16* {
    const WeightLayout::Ent* en = e->wl.find(n);
    return en && en->off != kNoOff ? (__nv_bfloat16*)(e->W + en->off) : nullptr;
  };
  e->embed = wp("embed");
  e->final_norm = wp("final_norm");
  e->lm_head = wp("lm_head");
  e->pk = make_packed(*m, e->wl.total);
  e->plm_head = e->W + e->pk.base + e->pk.lm;
  for (int l = 0; l < m->L; ++l) {
    const std::string p = "L" + std::to_string(l) + ".";
    LayerW w;
    uint8_t* lp = e->W + e->pk.base + (size_t)l * e->pk.per_layer;
    w.pqkv = lp + e->pk.qkv;
    w.po = lp + e->pk.o;
    w.pgu = lp + e->pk.gu;
    w.pd = lp + e->pk.dn;
    w.attn_norm = wp(p + "attn_norm");
    w.wqkv = wp(p + "wq");
    w.bqkv = m->qkv_bias ? wp(p + "bq") : nullptr;
    w.wo = wp(p + "wo");
    w.mlp_norm = wp(p + "mlp_norm");
    w.wgu = wp(p + "wg");
    w.wd = wp(p + "wd");
    e->lw.push_back(w);
  }
  // KV pools + TMA maps
  const size_t el = e->kv_f32 ? 4 : 2;
  const size_t pool = al((size_t)s->kv_pages * m->Hkv * kPage * m->dh * el);
  e->tmK.resize(m->L);
  e->tmV.resize(m->L);
  for (int l = 0; l < m->L; ++l) {
    e->kpool.push_back(e->KV + (2 * (size_t)l) * pool);
    e->vpool.push_back(e->KV + (2 * (size_t)l + 1) * pool);
    if (!e->kv_f32) {
      const uint32_t bc = m->dh < 64 ? m->dh : 64;
      const uint64_t rows = (uint64_t)s->kv_pages * m->Hkv * kPage;
      if (tma_encode_2d(&e->tmK[l], e->kpool[l], rows, m->dh, (uint64_t)m->dh * 2, 64, bc, 2, bc == 64) ||
          tma_encode_2d(&e->tmV[l], e->vpool[l], rows, m->dh, (uint64_t)m->dh * 2, 64, bc, 2, bc == 64)) {
        delete e;
        return fail(SRL_E_CUDA, "srl_create: TMA descriptor encode failed");
      }
    }
  }
  ScratchPlan p;
  plan_scratch(e, p, true);
  Ctl& c = e->ctl;
  c.Q_g = s->Q_g;
  c.R = world;
  c.rank = e->rank;
  c.Q_tot = e->z.Q_tot;
  c.U = s->U;
  c.pool_traj = s->pool_prompts * s->G;
  c.G = s->G;
  c.cap = s->cap;
  c.kv_pages = s->kv_pages;
  c.max_pages = e->z.max_pages;
  c.mode = s->mode;
  c.resume = s->resume;
  c.barrier = s->barrier;
  c.stop = s->stop;
  c.eos_id = s->eos_id;
  c.max_traj = s->max_traj;
  c.max_prompt = s->max_prompt;
  c.prefill_rows_max = e->z.prefill_rows_max;
  c.share_prefix = s->share_prefix && s->G > 1;
  c.prefill_budget = s->prefill_budget;
  c.max_prompts = e->z.max_prompts;
  c.pfx_max = e->z.pfx_max;
  c.ev_cap = e->z.ev_cap;
  c.h_cap_tok = e->z.h_cap_tok;
  e->prompt_tok_cap = (long long)e->z.max_prompts * s->max_prompt;
  // init device state
  cudaMemsetAsync(e->KV, 0, mem->kv_bytes, e->st);  // finite values in never-written KV rows
  cudaMemsetAsync(e->gemm_ws, 0, e->gemm_ws_bytes, e->st);
  int zero = 0;
  cudaMemcpyAsync(c.prompt_off, &zero, 4, cudaMemcpyHostToDevice, e->st);
  ctl_init(c, s->K, e->st);
  rope_table(e->rope_cos, e->rope_sin, e->z.max_ctx, m->dh, (double)m->rope_theta, e->st);
  if (cudaHostAlloc((void**)&e->hst, sizeof(CtlStatus), cudaHostAllocDefault) != cudaSuccess) {
    delete e;
    return cuda_fail("cudaHostAlloc");
  }
  cudaEventCreate(&e->ev0);
  cudaEventCreate(&e->ev1);
  cudaEventCreateWithFlags(&e->ev_sync, cudaEventDisableTiming);
  if (cudaStreamSynchronize(e->st) != cudaSuccess) {
    delete e;
    return cuda_fail("srl_create init");
  }
  *out = e;
  return SRL_OK;
}

int32_t srl_destroy(srl_engine* e) {
  if (!e) return SRL_OK;
  if (e->hst) cudaFreeHost(e->hst);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  if (e->ev_sync) cudaEventDestroy(e->ev_sync);
  for (cudaEvent_t ev : e->direct.ev) cudaEventDestroy(ev);
  for (auto& kv : e->graphs) {
    for (cudaEvent_t ev : kv.second.gset.ev) cudaEventDestroy(ev);
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  }
  delete e->comm;
  delete e;
  return SRL_OK;
}

int32_t srl_submit_prompts(srl_engine* e, int32_t n, const uint64_t* prompt_ids, const int32_t* tok_off,
                           const int32_t* toks, const int32_t* forced_len) {
  if (!e || n < 0 || (n > 0 && (!prompt_ids || !tok_off || !toks))) return fail(SRL_E_INVALID_ARG, "srl_submit_prompts: bad arguments");
  if (n == 0) return SRL_OK;
  const srl_sched_cfg& s = e->s;
  std::unordered_set<uint64_t> seen;
  for (int i = 0; i < n; ++i) {
    if (e->ids.count(prompt_ids[i]) || !seen.insert(prompt_ids[i]).second)
      return fail(SRL_E_DUPLICATE_ID, "srl_submit_prompts: duplicate prompt id (S:114)");
    const int len = tok_off[i + 1] - tok_off[i];
    if (len < 1 || len > s.max_prompt) return fail(SRL_E_INVALID_ARG, "srl_submit_prompts: prompt length outside [1, max_prompt]");
  }
  if (s.stop == SRL_STOP_FORCED && !forced_len) return fail(SRL_E_INVALID_ARG, "srl_submit_prompts: FORCED stop needs forced_len");
  if (forced_len)
    for (long long i = 0; i < (long long)n * s.G; ++i)
      if (forced_len[i] < 1 || forced_len[i] > s.cap) return fail(SRL_E_INVALID_ARG, "srl_submit_prompts: forced_len outside [1, cap]");
  const long long ntok = tok_off[n] - tok_off[0];
  if (e->n_traj + (long long)n * s.G > s.max_traj || e->prompt_tok_used + ntok > e->prompt_tok_cap ||
      e->n_prompts + n > e->z.max_prompts - 1)
    return fail(SRL_E_CAPACITY, "srl_submit_prompts: max_traj / prompt storage exceeded");
  std::vector<int> offs(n);
  for (int i = 0; i < n; ++i) offs[i] = (int)(e->prompt_tok_used + (tok_off[i + 1] - tok_off[0]));
  std::vector<DevTraj> tr((size_t)n * s.G);
  for (int i = 0; i < n; ++i)
    for (int g = 0; g < s.G; ++g) {
      DevTraj& t = tr[(size_t)i * s.G + g];
      memset(&t, 0, sizeof(t));
      t.prompt_idx = (int)(e->n_prompts + i);
      t.prompt_len = tok_off[i + 1] - tok_off[i];
      t.forced_len = forced_len ? forced_len[(size_t)i * s.G + g] : s.cap;
      t.epoch = -1;
      t.v_first = -1;
      t.admit_step = -1;
      t.finish_step = -1;
      t.state = TS_STREAM;
      t.slot = -1;
      t.fresh = 1;
      t.sample = g;
    }
  Ctl& c = e->ctl;
  cudaMemcpyAsync(c.prompt_tok + e->prompt_tok_used, toks + tok_off[0], 4 * ntok, cudaMemcpyHostToDevice, e->st);
  cudaMemcpyAsync(c.prompt_off + e->n_prompts + 1, offs.data(), 4 * n, cudaMemcpyHostToDevice, e->st);
  cudaMemcpyAsync(c.traj + e->n_traj, tr.data(), sizeof(DevTraj) * tr.size(), cudaMemcpyHostToDevice, e->st);
  ctl_submit(c, n * s.G, n, e->st);
  e->launches++;
  if (cudaStreamSynchronize(e->st) != cudaSuccess) return cuda_fail("srl_submit_prompts");
  for (int i = 0; i < n; ++i) {
    e->ids.insert(prompt_ids[i]);
    e->prompt_ids.push_back(prompt_ids[i]);
  }
  e->n_traj += (long long)n * s.G;
  e->n_prompts += n;
  e->prompt_tok_used += ntok;
  return SRL_OK;
}

int32_t srl_decode_step(srl_engine* e, srl_step_info* info) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_decode_step: null engine");
  if (e->comm_dead) return fail(SRL_E_NCCL, "srl_decode_step: the replica transport failed earlier (destroy the engine)");
  if (info) {
    memset(info, 0, sizeof(*info));
    info->k = -1;
  }
  if (e->group_state != 0) return fail(SRL_E_STATE, "srl_decode_step: a group awaits harvest/load_policy_weights (P:30)");
  if (!e->v_valid) return fail(SRL_E_STATE, "srl_decode_step: no policy weights loaded");
  cudaStream_t st = e->st;
  cudaEventRecord(e->ev0, st);
  {
    Prof p(e, SRL_K_CTL);
    ctl_begin(e->ctl, st);
  }
  e->launches++;
  if (int rc = read_status(e, "srl_decode_step")) return rc;
  if (cudaError_t ce = cudaGetLastError()) return cuda_fail("ctl_begin", ce);
  CtlStatus b = *e->hst;
  if (info) {
    info->v = b.v;
    info->n_ready = b.n_ready;
  }
  if (b.status != ST_CONTINUE) {
    prof_collect(e, e->direct, false);
    if (b.status == SRL_GROUP_READY) e->group_state = 1;
    if (b.status < 0) return fail(b.status, b.status == SRL_E_CAPACITY ? "srl_decode_step: KV pool / prefill capacity"
                                                                     : (b.status == SRL_E_EMPTY ? "srl_decode_step: nothing submitted"
                                                                                                 : "srl_decode_step: state"));
    return b.status;
  }
  const Ctl& c = e->ctl;
  if (b.r_local == 0) {
    // N1 (prefill budget): every running slot of this GPU is still prefilling -- the
    // step is its prefill rows only, then the (replicated) controller END
    for (int r0 = 0; r0 < b.m_pre; r0 += e->s.prefill_chunk) {
      const int mc = b.m_pre - r0 < e->s.prefill_chunk ? b.m_pre - r0 : e->s.prefill_chunk;
      Prof p(e, SRL_K_PREFILL, 2 + 8 * e->m.L);
      forward(e, mc, c.pre_tok + r0, c.pre_pos + r0, c.pre_slot + r0, false);
    }
    e->last_m = 0;
    if (e->comm) {
      if (int rc = exchange_and_end(e)) return rc;
    } else {
      Prof p(e, SRL_K_CTL);
      ctl_end(c, st);
      e->launches++;
    }
    return finish_step(e, b, info, nullptr);
  }
  if (e->mixed_ok && b.m_pre > 0 && b.m_pre <= e->s.prefill_chunk) {
    // steady state: the few admitted prompts join the decode pass (direct launches:
    // the row count varies)
    e->last_m = e->s.Q_g;
    decode_tail(e, e->comm == nullptr, e->s.Q_g, b.m_pre);
    if (e->comm)
      if (int rc = exchange_and_end(e)) return rc;
    return finish_step(e, b, info, nullptr);
  }
  // prefill of newly admitted sequences (prompt ++ kept tokens), in chunks
  for (int r0 = 0; r0 < b.m_pre; r0 += e->s.prefill_chunk) {
    const int mc = b.m_pre - r0 < e->s.prefill_chunk ? b.m_pre - r0 : e->s.prefill_chunk;
    Prof p(e, SRL_K_PREFILL, 2 + 8 * e->m.L);
    forward(e, mc, c.pre_tok + r0, c.pre_pos + r0, c.pre_slot + r0, false);
  }
  // decode of the running local slots (compacted rows) + sampling + stop /
  // compaction / emission: a static launch sequence per row bucket, replayed from
  // a CUDA graph from the bucket's second step on
  const int M = decode_rows(e, b.r_local);
  e->last_m = M;
  srl_engine::Graph& G = e->graphs[std::make_pair(M, e->prof ? e->prof_mask : 0u)];
  e->gset = &G.gset;
  if (e->use_graph && G.direct >= 1 && !G.exec) {
    const long long l0 = e->launches;
    cudaGraph_t g = nullptr;
    e->capturing = true;
    bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      decode_tail(e, e->comm == nullptr, M);
      ok = cudaStreamEndCapture(st, &g) == cudaSuccess && g;
    }
    e->capturing = false;
    if (ok) ok = cudaGraphInstantiate(&G.exec, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    G.launches = e->launches - l0;
    e->launches = l0;
    if (!ok) {  // fall back to direct launches for good
      G.exec = nullptr;
      e->use_graph = false;
      G.gset.cls.clear();
      G.gset.nl.clear();
      G.gset.used = 0;
    }
  }
  if (G.exec) {
    if (cudaError_t ge = cudaGraphLaunch(G.exec, st)) note_launch(e, "decode graph launch", (int)ge);
    e->launches += G.launches;
  } else {
    decode_tail(e, e->comm == nullptr, M);
    G.direct++;
  }
  if (e->comm)
    if (int rc = exchange_and_end(e)) return rc;
  return finish_step(e, b, info, G.exec ? &G.gset : nullptr);
}

int32_t srl_harvest_finished(srl_engine* e, int32_t cap_recs, srl_traj* recs, int32_t* n_out, int32_t* toks,
                             float* logprobs, int32_t* versions, int64_t cap_toks) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_harvest_finished: null engine");
  if (e->comm_dead) return fail(SRL_E_NCCL, "srl_harvest_finished: the replica transport failed earlier");
  if (e->group_state != 1) return fail(SRL_E_STATE, "srl_harvest_finished: no group is ready");
  e->harvest_valid = false;  // the staging buffers are rewritten now
  ctl_harvest(e->ctl, e->st);
  e->launches++;
  if (int rc = read_status(e, "srl_harvest_finished")) return rc;
  const CtlStatus& h = *e->hst;
  if (h.status == SRL_E_CAPACITY) return fail(SRL_E_CAPACITY, "srl_harvest_finished: engine staging too small");
  const int n = h.group_n;
  const long long total = h.m_pre;
  e->last_harvest_tok = total;
  e->last_harvest_n = n;
  if (n_out) *n_out = n;
  if (n > cap_recs || total > cap_toks || !recs) return fail(SRL_E_CAPACITY, "srl_harvest_finished: caller buffers too small");
  cudaMemcpyAsync(recs, e->ctl.h_rec, sizeof(srl_traj) * n, cudaMemcpyDeviceToHost, e->st);
  if (toks) cudaMemcpyAsync(toks, e->ctl.h_tok, 4 * total, cudaMemcpyDeviceToHost, e->st);
  if (logprobs) cudaMemcpyAsync(logprobs, e->ctl.h_lp, 4 * total, cudaMemcpyDeviceToHost, e->st);
  if (versions) cudaMemcpyAsync(versions, e->ctl.h_ver, 4 * total, cudaMemcpyDeviceToHost, e->st);
  const int two = 2;
  cudaMemcpyAsync(&e->ctl.s->group_state, &two, 4, cudaMemcpyHostToDevice, e->st);
  if (int rc = stream_wait(e, "srl_harvest_finished")) return rc;
  for (int i = 0; i < n; ++i) {
    const long long pi = recs[i].prompt_id;
    recs[i].prompt_id = (pi >= 0 && pi < (long long)e->prompt_ids.size()) ? (int64_t)e->prompt_ids[pi] : -1;
  }
  e->group_state = 2;
  e->harvest_valid = true;
  return SRL_OK;
}

int32_t srl_harvest_device(srl_engine* e, const int32_t** toks, const float** logprobs, const int32_t** versions,
                           const srl_traj** recs, int32_t* n_recs, int64_t* n_tok) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_harvest_device: null engine");
  if (!e->harvest_valid) return fail(SRL_E_STATE, "srl_harvest_device: no harvested group");
  if (toks) *toks = e->ctl.h_tok;
  if (logprobs) *logprobs = e->ctl.h_lp;
  if (versions) *versions = e->ctl.h_ver;
  if (recs) *recs = e->ctl.h_rec;
  if (n_recs) *n_recs = e->last_harvest_n;
  if (n_tok) *n_tok = e->last_harvest_tok;
  return SRL_OK;
}

int32_t srl_load_policy_weights(srl_engine* e, const void* flat_w, int64_t version) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_load_policy_weights: null engine");
  if (e->comm_dead) return fail(SRL_E_NCCL, "srl_load_policy_weights: the replica transport failed earlier");
  if (e->group_state == 1) return fail(SRL_E_STATE, "srl_load_policy_weights: harvest the ready group first");
  if (version < 0 || (e->v_valid && version <= e->v))
    return fail(SRL_E_STATE, "srl_load_policy_weights: policy version must increase");
  // Pack the projection matrices from the staging-layout source straight into the
  // GEMM weight stream's layout; the remaining tensors (embedding, norms, biases)
  // are read in place, so copy those when the source is the caller's buffer.
  if (e->m.weights_compact && flat_w)
    return fail(SRL_E_INVALID_ARG, "srl_load_policy_weights: compact weights are loaded with srl_load_policy_tensor");
  const uint8_t* src = flat_w ? (const uint8_t*)flat_w : e->W;
  // with replicas only rank 0 reads a source (the rest receive); compact weights
  // were already installed tensor by tensor
  const bool root = e->rank == 0 && !e->m.weights_compact;
  if (root && src != e->W) {
    for (const auto& en : e->wl.ents)
      if (!is_packed_tensor(en.name))
        cudaMemcpyAsync(e->W + en.off, src + en.off, en.numel * 2, cudaMemcpyDeviceToDevice, e->st);
  }
  if (root) {
    const srl_model_cfg& m = e->m;
    const int d = m.d, qd = m.Hq * m.dh, nqkv = (m.Hq + 2 * m.Hkv) * m.dh;
    auto sp = [&](const std::string& n) {
      return (const __nv_bfloat16*)(src + e->wl.find(n)->off);
    };
    int rc = 0;
    for (int l = 0; l < m.L; ++l) {
      const std::string p = "L" + std::to_string(l) + ".";
      const LayerW& w = e->lw[l];
      rc |= pack_weight(sp(p + "wq"), nqkv, d, w.pqkv, e->st);
      rc |= pack_weight(sp(p + "wo"), d, qd, w.po, e->st);
      rc |= pack_weight(sp(p + "wg"), 2 * m.ff, d, w.pgu, e->st);
      rc |= pack_weight(sp(p + "wd"), d, m.ff, w.pd, e->st);
      e->launches += 4;
    }
    rc |= pack_weight(sp("lm_head"), m.V, d, e->plm_head, e->st);
    e->launches++;
    if (rc) return cuda_fail("srl_load_policy_weights: pack_weight", cudaGetLastError());
  }
  if (e->comm) {
    // Row a17: rank 0's installed policy -> every replica, in place: the packed GEMM
    // stream (one contiguous region) plus the tensors read in place (embedding,
    // norms, biases).  Packed staging matrices are not decoded from, so not sent.
    std::vector<Range> rr;
    for (const auto& en : e->wl.ents)
      if (!is_packed_tensor(en.name) && en.off != kNoOff) rr.push_back({e->W + en.off, en.numel * 2});
    rr.push_back({e->W + e->pk.base, e->pk.total - e->pk.base});
    std::string err;
    Prof p(e, SRL_K_COMM);
    if (e->comm->broadcast_inplace(rr, e->st, err)) {
      e->comm->abort();
      e->comm_dead = true;
      return fail(SRL_E_NCCL, "srl_load_policy_weights: broadcast: " + err);
    }
  }
  ctl_bump(e->ctl, (int)version, e->st);
  e->launches++;
  if (int rc = read_status(e, "srl_load_policy_weights")) return rc;
  if (cudaError_t ce = cudaGetLastError()) return cuda_fail("srl_load_policy_weights", ce);
  if (e->hst->status < 0) return fail(e->hst->status, "srl_load_policy_weights: capacity (resumed list)");
  e->v = version;
  e->v_valid = true;
  e->group_state = 0;
  return SRL_OK;
}

int32_t srl_get_trace(srl_engine* e, int64_t from, int32_t cap, srl_trace_rec* out, int32_t* n_out, int64_t* n_total) {
  if (!e || from < 0 || cap < 0) return fail(SRL_E_INVALID_ARG, "srl_get_trace: bad arguments");
  long long total = 0;
  cudaMemcpyAsync(&total, &e->ctl.s->n_events, 8, cudaMemcpyDeviceToHost, e->st);
  cudaStreamSynchronize(e->st);
  if (n_total) *n_total = total;
  long long lo = total - e->z.ev_cap;
  if (lo < 0) lo = 0;
  if (from < lo) from = lo;
  long long cnt = total - from;
  if (cnt > cap) cnt = cap;
  if (cnt < 0) cnt = 0;
  long long done = 0;
  while (done < cnt) {
    const long long idx = (from + done) % e->z.ev_cap;
    long long run = e->z.ev_cap - idx;
    if (run > cnt - done) run = cnt - done;
    cudaMemcpyAsync(out + done, e->ctl.events + idx * 6, 24 * run, cudaMemcpyDeviceToHost, e->st);
    done += run;
  }
  if (cudaStreamSynchronize(e->st) != cudaSuccess) return cuda_fail("srl_get_trace");
  if (n_out) *n_out = (int32_t)cnt;
  return SRL_OK;
}

int32_t srl_get_counters(srl_engine* e, int64_t* raw, int64_t* disc, int64_t* emitted, int64_t* groups, int64_t* launches) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_get_counters: null engine");
  CtlState st;
  cudaMemcpyAsync(&st, e->ctl.s, sizeof(CtlState), cudaMemcpyDeviceToHost, e->st);
  if (cudaStreamSynchronize(e->st) != cudaSuccess) return cuda_fail("srl_get_counters");
  if (raw) *raw = st.raw_tokens;
  if (disc) *disc = st.discarded_tokens;
  if (emitted) *emitted = st.emitted;
  if (groups) *groups = st.n_groups;
  if (launches) *launches = e->launches;
  return SRL_OK;
}

int32_t srl_set_profile_mask(srl_engine* e, uint32_t class_mask) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_set_profile_mask: null engine");
  e->prof_mask = class_mask;  // graphs are cached per (rows, mask): nothing to recapture
  return SRL_OK;
}

int32_t srl_set_profiling(srl_engine* e, int32_t on) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_set_profiling: null engine");
  e->prof = on != 0;
  for (int i = 0; i < SRL_K_NCLASS; ++i) {
    e->prof_ms[i] = 0;
    e->prof_launch[i] = 0;
  }
  e->direct.cls.clear();
  e->direct.nl.clear();
  e->direct.used = 0;
  return SRL_OK;
}

int32_t srl_get_profile(srl_engine* e, double* ms, int64_t* launches) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_get_profile: null engine");
  for (int i = 0; i < SRL_K_NCLASS; ++i) {
    if (ms) ms[i] = e->prof_ms[i];
    if (launches) launches[i] = e->prof_launch[i];
  }
  return SRL_OK;
}

int32_t srl_set_cache_bound(srl_engine* e, int32_t K) {
  if (!e) return fail(SRL_E_INVALID_ARG, "srl_set_cache_bound: null engine");
  if (e->group_state == 1) return fail(SRL_E_STATE, "srl_set_cache_bound: a group is pending");
  if (K < -1) return fail(SRL_E_INVALID_ARG, "srl_set_cache_bound: K must be >= -1");
  e->s.K = K;
  cudaMemcpyAsync(&e->ctl.s->K, &K, 4, cudaMemcpyHostToDevice, e->st);
  if (cudaStreamSynchronize(e->st) != cudaSuccess) return cuda_fail("srl_set_cache_bound");
  return SRL_OK;
}

}  // extern "C"

extern "C" int32_t srl_debug_copy_logits(srl_engine* e, float* out_host, int64_t cap_floats) {
  if (!e || !out_host) return fail(SRL_E_INVALID_ARG, "srl_debug_copy_logits: bad arguments");
  const long long n = (long long)e->s.Q_g * e->m.V;
  if (cap_floats < n) return fail(SRL_E_CAPACITY, "srl_debug_copy_logits: buffer too small");
  // decode rows are compacted running slots: put row i back at its slot
  std::vector<int> rs(e->s.Q_g);
  cudaMemcpyAsync(rs.data(), e->ctl.row_slot, 4 * e->s.Q_g, cudaMemcpyDeviceToHost, e->st);
  if (cudaStreamSynchronize(e->st) != cudaSuccess) return cuda_fail("srl_debug_copy_logits");
  for (int i = 0; i < e->last_m && i < e->s.Q_g; ++i)
    if (rs[i] >= 0)
      cudaMemcpyAsync(out_host + (size_t)rs[i] * e->m.V, e->logits + (size_t)i * e->m.V, 4ull * e->m.V,
                      cudaMemcpyDeviceToHost, e->st);
  if (cudaStreamSynchronize(e->st) != cudaSuccess) return cuda_fail("srl_debug_copy_logits");
  return SRL_OK;
}

// ------------------------------------------------------------------ replica plumbing
extern "C" int32_t srl_nccl_unique_id(uint8_t* out128) {
  if (!out128) return fail(SRL_E_INVALID_ARG, "srl_nccl_unique_id: null argument");
  std::string err;
  if (nccl_unique_id(out128, err)) return fail(SRL_E_NCCL, "srl_nccl_unique_id: " + err);
  return SRL_OK;
}

extern "C" int32_t srl_local_group_create(int32_t world, void** out) {
  if (!out || world < 1 || world > kMaxR) return fail(SRL_E_INVALID_ARG, "srl_local_group_create: bad arguments");
  *out = local_group_create(world);
  return SRL_OK;
}

extern "C" int32_t srl_local_group_destroy(void* group) {
  local_group_destroy(group);
  return SRL_OK;
}

// ------------------------------------------------------------------ compact weights: one tensor at a time
extern "C" int32_t srl_load_policy_tensor(srl_engine* e, const char* name, const void* src) {
  if (!e || !name || !src) return fail(SRL_E_INVALID_ARG, "srl_load_policy_tensor: null argument");
  if (e->group_state == 1) return fail(SRL_E_STATE, "srl_load_policy_tensor: harvest the ready group first");
  const std::string n(name);
  const WeightLayout::Ent* en = e->wl.find(n);
  if (!en) return fail(SRL_E_INVALID_ARG, "srl_load_policy_tensor: unknown tensor " + n);
  const __nv_bfloat16* s = (const __nv_bfloat16*)src;
  const srl_model_cfg& m = e->m;
  int rc = 0;
  if (!is_packed_tensor(n)) {
    if (cudaMemcpyAsync(e->W + en->off, src, en->numel * 2, cudaMemcpyDeviceToDevice, e->st) != cudaSuccess) rc = -3;
  } else if (n == "lm_head") {
    rc = pack_weight(s, m.V, m.d, e->plm_head, e->st);
  } else {
    const int l = atoi(n.c_str() + 1);
    const std::string t = n.substr(n.find('.') + 1);
    const LayerW& w = e->lw[l];
    const size_t kbq = (size_t)m.d / 64, tile = 128ull * 128;  // one packed 128-row x 64-col block, bytes
    const int qd = m.Hq * m.dh, kd = m.Hkv * m.dh;
    if (t == "wq") rc = pack_weight(s, qd, m.d, w.pqkv, e->st);
    else if (t == "wk") rc = pack_weight(s, kd, m.d, w.pqkv + (size_t)(qd / 128) * kbq * tile, e->st);
    else if (t == "wv") rc = pack_weight(s, kd, m.d, w.pqkv + (size_t)((qd + kd) / 128) * kbq * tile, e->st);
    else if (t == "wo") rc = pack_weight(s, m.d, qd, w.po, e->st);
    else if (t == "wd") rc = pack_weight(s, m.d, m.ff, w.pd, e->st);
    else if (t == "wg") rc = pack_weight_rows(s, m.ff, m.d, w.pgu, kGuBlock, 2 * kGuBlock, 0, e->st);
    else if (t == "wu") rc = pack_weight_rows(s, m.ff, m.d, w.pgu, kGuBlock, 2 * kGuBlock, kGuBlock, e->st);
    else return fail(SRL_E_INVALID_ARG, "srl_load_policy_tensor: not loadable: " + n);
  }
  if (is_packed_tensor(n) && !e->m.weights_compact && en->off != kNoOff) {
    // keep the staging image consistent too (srl_load_policy_weights(NULL) re-packs
    // from it); wg / wu: the source is plain row-major, the staging image
    // interleaves row_block-row blocks at block_stride rows -- scatter block-wise
    const size_t rowb = en->cols * 2;
    if (en->row_block == en->rows) {
      if (cudaMemcpyAsync(e->W + en->off, src, en->numel * 2, cudaMemcpyDeviceToDevice, e->st) != cudaSuccess) rc = -3;
    } else if (en->rows % en->row_block == 0) {
      if (cudaMemcpy2DAsync(e->W + en->off, en->block_stride * rowb, src, en->row_block * rowb, en->row_block * rowb,
                            en->rows / en->row_block, cudaMemcpyDeviceToDevice, e->st) != cudaSuccess)
        rc = -3;
    } else {
      rc = -1;
    }
  }
  e->launches++;
  if (rc || cudaGetLastError() != cudaSuccess) return cuda_fail("srl_load_policy_tensor");
  return SRL_OK;
}
