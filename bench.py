#!/usr/bin/env python
"""SortedRL rollout benchmark (BASELINE.json metric: rollout tokens/s + bubble
ratio @1/2/4/8 B200; decode %HBM roofline).

A "step" is one early-update round of the rollout -- SortedRL's unit of work
(P:169-177): srl_decode_step repeatedly (refill/admission + prefill of
admitted prompts, the policy's decode forward over the ragged batch -- tcgen05
GEMMs, paged attention -- Philox sampling, stop detection, compaction into the
rollout buffer) until the length-sorted update group is ready, then its
harvest and the policy refresh (load_policy_weights with the cache bound).
Every SURVEY §8(a) row runs in every step.

Workload (configs[1], "cfg2"): LLaMA-3.1-8B-shaped random-init policy on one
B200, rollout batch Q=256, max 8k tokens, update group U=64, K=inf (partial
mode), pool 4*Q prompts per epoch, 256-token prompts, lognormal(1600, 0.55) +
3% cap FORCED response lengths (DESIGN.md input recipe).  At least W untimed
rounds, placed so that the K timed rounds straddle the first epoch boundary;
the prompts live in pinned host memory and are submitted epoch by epoch
through the public API (PromptStream), inside the rounds that need them.
One timed region: CUDA events on the engine stream give `value` (tokens per
second of device time, barrier + max over ranks); the wall clock of the same
rounds -- prompt uploads and group copy-backs included -- gives `e2e`.

  python bench.py [--gpus N] [--steps K] [--warmup W]    (N > 1: self-launches N ranks)
  python bench.py --impl reference ...   # the CPU oracle on a bounded sample
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workload.configs import (BARRIER_ADMITTED, BARRIER_TRAINED, K_INF, KV_BF16, LLAMA8B, MODE_POSTHOC,  # noqa: E402
                              MODE_SORTED, MODE_SYNC, QWEN32B, RESUME_KEEP_KV, RESUME_REPREFILL,
                              STOP_FORCED, SchedConfig)
from workload.lengths import LengthModel, sample_lengths  # noqa: E402
from workload.prompts import make_prompts  # noqa: E402

METRIC = "rollout tokens/s + bubble ratio @1/2/4/8 B200; decode %HBM roofline"
WORKLOAD = ("cfg2: LLaMA-3.1-8B-shaped random-init bf16 policy, rollout batch Q_g=256 per GPU, "
            "max 8192 new tokens, update group U=64, K=inf (partial), pool 1024 prompts per GPU per epoch, "
            "256-token prompts, FORCED lognormal(1600,0.55)+3%-at-cap lengths, TRAINED barrier, KEEP_KV; "
            "N>1: lockstep replicas (global slots g=s*N+r, per-step all-gather of sampled rows, "
            "weight broadcast after every update group)")
N_PROMPTS_PER_EPOCH = 1024
PROMPT_LEN = 256
WORKLOAD_32B = ("cfg4 per GPU: Qwen-2.5-32B-shaped random-init bf16 policy (qkv bias, compact packed-only weights "
                "65.5 GB), rollout batch Q_g=64 per GPU, max 16384 new tokens, update group U=64, K=inf (partial), "
                "pool 256 prompts per GPU per epoch, 256-token prompts, FORCED lognormal(1600,0.55)+3%-at-cap lengths, "
                "TRAINED barrier, KEEP_KV; policy refresh = version bump (no trainer copy fits beside the engine)")
# model -> (shape, Q_g, cap, kv_pages, prompts per GPU per epoch, compact weights, trainer copy, workload text)
MODELS = {"llama8b": (LLAMA8B, 256, 8192, 11000, 1024, False, True, None),
          "qwen32b": (QWEN32B, 64, 16384, 5000, 256, True, False, WORKLOAD_32B)}
EPOCHS = 4          # prompt stream long enough for the untimed + timed rounds
U_MAX = 2048        # harvest buffer capacity (records)


def cfg2_sched(world=1, Q_g=256, cap=8192, pool=N_PROMPTS_PER_EPOCH, kv_pages=11000):
    return SchedConfig(Q_g=Q_g, R=world, U=64, K=K_INF, pool_prompts=pool * world, G=1, cap=cap,
                       page_tokens=64,
                       kv_pages=kv_pages, mode=MODE_SORTED, resume=RESUME_KEEP_KV, barrier=BARRIER_TRAINED,
                       stop=STOP_FORCED, kv_dtype=KV_BF16, temperature=1.0, sample_seed=3)


def workload_inputs(world=1, epochs=2, pool=N_PROMPTS_PER_EPOCH, V=LLAMA8B.V, cap=8192, G=1):
    """The prompt stream every replica submits (identical on all ranks; the replicated
    pending queue shards it over the global slots).  `pool` counts trajectories per
    GPU per epoch: pool / G prompts of G responses each (G = 8: LogicRL's 128 x 8,
    P:235)."""
    n = pool * world * epochs // G
    off, toks = make_prompts(1, n, V, PROMPT_LEN)
    L = sample_lengths(LengthModel(median=1600, sigma=0.55, tail=0.03, floor=1, cap=cap), 0, n * G)
    return off, toks, L


def aggregate_over_ranks(dist, raw, useful, ms, device="cuda"):
    """Whole-job rates: tokens of all ranks / the slowest rank's device time."""
    import torch
    t = torch.tensor([raw, useful, ms], dtype=torch.float64, device=device)
    tot = t.clone()
    dist.all_reduce(tot)
    mx = t.clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    return tot[0].item() / (mx[2].item() * 1e-3), tot[1].item() / (mx[2].item() * 1e-3), mx[2].item()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ model byte / flop model
def step_bytes_flops(m, r, sum_ctx):
    wl = m.L * ((m.Hq + 2 * m.Hkv) * m.dh * m.d + m.d * m.Hq * m.dh + 3 * m.d * m.ff) * 2
    w_step = wl + m.V * m.d * 2
    kvb = 2 * m.L * m.Hkv * m.dh * 2                       # KV bytes per token (all layers)
    B = w_step + kvb * sum_ctx + kvb * r                    # weights + KV read + KV append
    p_mm = w_step / 2
    a = 4 * m.L * m.Hq * m.dh                               # attention flops per context position
    F = 2 * p_mm * r + a * sum_ctx
    return B, F, w_step, kvb


# ------------------------------------------------------------------ the GPU arm
class PromptStream:
    """The dataloader: the prompt stream in PINNED host memory, submitted to the
    engine one epoch (pool_prompts * world prompts) at a time through the public
    API.  TRAINED barrier: the next epoch is submitted just in time -- when
    every loaded trajectory has been emitted, the only moment the controller can
    load it -- so prompts are copied host -> device inside the round that consumes
    them.  ADMITTED barrier: one epoch is kept queued ahead of the controller."""

    def __init__(self, eng, off, toks, L, ids, per_epoch, trained, torch, G=1):
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        self.eng, self.off, self.G = eng, off, G
        self.toks, self.L, self.ids = pin(toks), pin(L), pin(ids)
        self.per_epoch, self.trained = per_epoch, trained
        self.next = 0            # prompts submitted
        self.loaded = 0          # trajectories the controller has loaded (LOAD events)
        self.ev_from = 0         # trace records read so far
        self.h2d = 0             # bytes copied host -> device by submissions
        self.admits = []         # (k, traj_id) of every ADMIT event seen
        self.submits = []        # (first traj_id, count) per submission

    def poll(self):
        """Read the new trace records: LOAD counts and ADMIT events."""
        tr, tot = self.eng.trace(self.ev_from)
        for kind, a, b, c, d, e in tr:
            if kind == 1:        # LOAD: a=k, b=epoch, c=first traj, d=count
                self.loaded += d
            elif kind == 2:      # ADMIT: a=k, b=slot, c=traj
                self.admits.append((a, c))
        self.ev_from = tot

    def submit_epoch(self):
        lo, hi = self.next, min(len(self.ids), self.next + self.per_epoch)
        if hi <= lo:
            return 0
        o = self.off[lo:hi + 1]
        self.eng.submit_prompts(self.ids[lo:hi], (o - o[0]).astype(np.int32), self.toks[o[0]:o[-1]],
                               self.L[lo * self.G:hi * self.G])
        self.h2d += int((o[-1] - o[0]) * 4 + (hi - lo) * (8 + 4 + 4 * self.G) + 4)
        self.submits.append((lo, hi - lo))
        self.next = hi
        return hi - lo

    def feed(self, emitted):
        """Called between rounds (after the harvest and the policy refresh)."""
        self.poll()
        if self.trained:
            if emitted == self.loaded and self.next == self.loaded:
                self.submit_epoch()
        elif self.next - self.loaded < self.per_epoch:
            self.submit_epoch()


def run_gpu(args, rank, world, dist):
    import torch
    if args.tuning:
        from paper_2603_23414_b200 import _lib
        _lib.set_tuning(**{k: int(v) for k, v in (kv.split("=") for kv in args.tuning.split(","))})
    from paper_2603_23414_b200.engine import DONE, GROUP_READY, RolloutEngine
    from workload.weights import fill_engine_weights
    torch.cuda.set_device(rank % max(1, torch.cuda.device_count()))
    dev = torch.cuda.current_device()
    from paper_2603_23414_b200.engine import share_nccl_unique_id
    model, Q_g, cap, kv_pages, pool, compact, keep_trainer, _ = MODELS[args.model]
    sched = cfg2_sched(world, Q_g=Q_g, cap=cap, pool=pool, kv_pages=kv_pages)
    # scheduler variants (the paper's comparisons; defaults = SortedRL partial mode)
    sched = dataclasses.replace(sched, mode={"sorted": MODE_SORTED, "sync": MODE_SYNC, "posthoc": MODE_POSTHOC}[args.mode],
                                K=args.K, U=args.U,
                                barrier={"trained": BARRIER_TRAINED, "admitted": BARRIER_ADMITTED}[args.barrier],
                                resume={"keep_kv": RESUME_KEEP_KV, "reprefill": RESUME_REPREFILL}[args.resume],
                                G=args.G, pool_prompts=pool * world // args.G, share_prefix=int(args.share_prefix),
                                prefill_budget=args.prefill_budget)
    off, toks, L = workload_inputs(world, epochs=EPOCHS, pool=pool, V=model.V, cap=cap, G=args.G)
    ids = np.arange(len(off) - 1, dtype=np.uint64) + 1
    max_traj = EPOCHS * pool * world
    rep = {}
    if world > 1:
        rep = dict(rank=rank, world=world, nccl_id=share_nccl_unique_id(dist, rank))
    eng = RolloutEngine(model, sched, max_traj=max_traj, max_prompt=PROMPT_LEN, prefill_chunk=4096, device=dev,
                        compact_weights=compact, **rep)
    fill_engine_weights(eng, model, 0)
    # the trainer's copy of the refreshed policy on rank 0 (K13: the same bytes are
    # re-emitted); the other replicas receive it through the engine's broadcast
    trainer = eng.W.clone() if rank == 0 and keep_trainer else None
    eng.load_policy_weights(0)
    torch.cuda.synchronize()
    stream = eng.stream              # the stream every engine kernel is launched on
    per_epoch = pool * world // sched.G      # prompts per epoch
    trained = sched.barrier == BARRIER_TRAINED or sched.mode != MODE_SORTED
    loader = PromptStream(eng, off, toks, L, ids, per_epoch, trained, torch, G=sched.G)
    st = {"v": 0, "useful": 0, "d2h": 0, "done": False, "emitted": 0, "steps": 0}
    trace = []                       # every decode step: (r_k, sum_ctx, dt_ms, prefill_tokens, n_fin, r_local)
    ATT = ["attention"]
    prof_all_every = max(1, args.prof_every)
    att_every = max(1, args.attn_every)
    att_ctx = []                     # sum_ctx of the decode steps whose attention launches were timed

    def step(sample_all=False):
        # profiled window: every class on 1 step in prof_every, attention alone on 1 in
        # attn_every, nothing on the rest (a bracketed class loses its PDL edges)
        timed_att = False
        if sample_all is not None:
            i = st["steps"]
            if sample_all:
                eng.set_profile_mask(None)
                timed_att = True
            elif i % att_every == 0:
                eng.set_profile_mask(ATT)
                timed_att = True
            else:
                eng.set_profile_mask([])
        s_, info = eng.decode_step()
        if s_ == DONE:
            st["done"] = True
            return None
        if info.k >= 0:
            trace.append((info.r_k, info.sum_ctx, info.dt_ms, info.n_prefill_tokens, info.n_finished,
                          info.r_local))
            st["steps"] += 1
            if timed_att:
                att_ctx.append(info.sum_ctx)
        if s_ == GROUP_READY:        # rows a15-a17: sorted group out, refreshed policy in
            h = eng.harvest_finished(cap_recs=U_MAX, cap_toks=U_MAX * sched.cap)
            st["useful"] += sum(r["len"] for r in h.records)
            st["emitted"] += len(h.records)
            st["d2h"] += sum(r["len"] for r in h.records) * 12 + len(h.records) * 64
            st["v"] += 1
            eng.load_policy_weights(st["v"], trainer)
            return True
        return False

    def one_round(profiled=False):
        """One early-update round: decode steps until the length-sorted update group
        is ready, its harvest and the policy refresh (the bench's "step"), then the
        dataloader's turn."""
        got = False
        while not st["done"]:
            r = step((st["steps"] % prof_all_every == 0) if profiled else None)
            if r:
                got = True
                break
        loader.feed(st["emitted"])
        return got

    loader.submit_epoch()            # epoch 1 (before anything is timed)
    if args.full:
        # the whole job: every epoch from the first admission to the last emitted
        # group, device-timed end to end (epoch-start prefill bursts, drains)
        loader.submit_epoch()        # the 2-epoch job, both resident
        loader.per_epoch = 0         # nothing else is streamed
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0 = eng.counters()
        with ClockSampler(dev) as clk:
            e0.record(stream)
            rounds = 0
            while one_round():
                rounds += 1
            e1.record(stream)
            torch.cuda.synchronize()
        c1 = eng.counters()
        ms = e0.elapsed_time(e1)
        eng.close()
        return dict(ms=ms, ran=rounds, raw=(c1["raw_tokens"] - c0["raw_tokens"]) / world, useful=st["useful"] / world,
                    stats=trace, prof={"attention": (0.0, 0)}, launches=c1["kernel_launches"] - c0["kernel_launches"],
                    clocks=clk.summary(), e2e=None, trace=trace, breakdown={}, n_break=0, warmup_rounds=0,
                    window=None)
    # ---------------- untimed rounds: at least W warm-up rounds, and enough of them that
    # the timed window is centred on the first epoch boundary (the job's cost includes the
    # epoch drain and the next epoch's prefill burst, and the streamed epoch is admitted
    # inside the window)
    groups_per_epoch = max(1, per_epoch * sched.G // sched.U)
    n_pre = max(args.warmup, groups_per_epoch - args.steps // 2)
    warm = 0
    while warm < n_pre and one_round():
        warm += 1
    # ---------------- the timed window: K rounds through the public API.  `value` = raw
    # tokens / device time (CUDA events on the engine stream); `e2e` = the same tokens /
    # wall time of the same rounds, which include the dataloader's pinned host -> device
    # prompt copies and the device -> host copies of every harvested group
    eng.set_profiling(True, classes=ATT)
    t0 = len(trace)
    u0, c0, h2d0, d2h0, ev0 = st["useful"], eng.counters(), loader.h2d, st["d2h"], len(loader.admits)
    sub0 = len(loader.submits)
    s0 = st["steps"]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ran = 0
    with ClockSampler(dev) as clk:
        w0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            ran += one_round(profiled=True)
        e1.record(stream)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
    if dist:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    prof = eng.profile()
    eng.set_profiling(False)
    c1 = eng.counters()
    raw, useful = c1["raw_tokens"] - c0["raw_tokens"], st["useful"] - u0
    launches = c1["kernel_launches"] - c0["kernel_launches"]
    stats = trace[t0:]
    n_dec = len(stats)
    n_sampled = sum(1 for i in range(s0, st["steps"]) if i % prof_all_every == 0)
    # streamed prompts admitted inside the window
    streamed = loader.submits[sub0:]
    first_streamed = min((lo for lo, n in streamed), default=None)
    adm = loader.admits[ev0:]
    n_stream_adm = 0 if first_streamed is None else sum(1 for _, t in adm if t >= first_streamed * sched.G)
    steps_e2e = max(1, ran)
    n_status = (st["steps"] - s0) * 2 + ran * 2                 # status read-backs per step + per round
    e2e = {"value": raw / (w1 - w0), "unit": "tokens/s", "tokens": int(raw),
           "h2d_bytes_per_step": int((loader.h2d - h2d0) / steps_e2e),
           "d2h_bytes_per_step": int((st["d2h"] - d2h0 + n_status * 96) / steps_e2e),
           "wall_ms_per_step": (w1 - w0) * 1e3 / steps_e2e, "steps": ran,
           "window": "the same rounds as value (one timed region: device events and wall clock)",
           "streamed_prompts": int(sum(n for _, n in streamed)),
           "streamed_admitted_in_window": int(n_stream_adm)}
    eng.close()
    del eng
    return dict(ms=ms, ran=ran, raw=raw / world, useful=useful / world, stats=stats, prof=prof, launches=launches,
                clocks=clk.summary(), e2e=e2e, trace=trace, breakdown=prof, n_break=n_sampled, n_dec=n_dec,
                warmup_rounds=warm, window=(warm, warm + ran), att_ctx=att_ctx)


# ------------------------------------------------------------------ CPU oracle (the reference arm)
ORACLE_ROWS, ORACLE_CTX = 8, 1024


class OracleSlice:
    """A bounded sample of the cfg2 workload on the CPU oracle (fp64, oracle/model.py):
    ORACLE_ROWS sequences at context ORACLE_CTX decoding one token each through ONE of
    the 32 LLaMA-8B-shaped layers plus 1/32 of the LM head (the full 32 layers would
    need 64 GB of fp64 weights).  `step()` runs it once and returns its wall time;
    tokens/s of the full model = rows / (32 t_layer + 32 t_lm_slice)."""

    def __init__(self):
        from oracle.model import Model
        from workload.weights import bf16_bits_to_f32, gen_weight_np
        m1 = LLAMA8B.with_layers(1)
        W = {}
        for name in ["L0.attn_norm", "L0.wq", "L0.wk", "L0.wv", "L0.wo", "L0.mlp_norm", "L0.wg", "L0.wu", "L0.wd"]:
            W[name] = bf16_bits_to_f32(gen_weight_np(m1, name)).astype(np.float64)
        W["lm_head"] = bf16_bits_to_f32(gen_weight_np(m1, "lm_head", rows=np.arange(LLAMA8B.V // 32))).astype(np.float64)
        W["final_norm"] = bf16_bits_to_f32(gen_weight_np(m1, "final_norm")).astype(np.float64)
        self.W, self.mdl = W, Model(m1, W)
        rng = np.random.default_rng(0)
        self.hist = [(list(rng.normal(size=(ORACLE_CTX - 1, LLAMA8B.Hkv, LLAMA8B.dh))),
                      list(rng.normal(size=(ORACLE_CTX - 1, LLAMA8B.Hkv, LLAMA8B.dh))),
                      rng.normal(size=LLAMA8B.d)) for _ in range(ORACLE_ROWS)]

    def step(self):
        t_layer = t_lm = 0.0
        for k_hist, v_hist, x0 in self.hist:
            K_, V_ = list(k_hist), list(v_hist)
            t0 = time.perf_counter()
            x = self.mdl.layer(0, x0, ORACLE_CTX - 1, K_, V_)
            t1 = time.perf_counter()
            _ = self.W["lm_head"] @ self.mdl.hidden(x)
            t2 = time.perf_counter()
            t_layer += t1 - t0
            t_lm += t2 - t1
        return t_layer + t_lm, ORACLE_ROWS / (LLAMA8B.L * t_layer + 32 * t_lm)

    SAMPLE = (f"oracle fp64 decode (oracle/model.py) of {ORACLE_ROWS} rows at context {ORACLE_CTX} through one "
              f"LLaMA-8B-shaped layer + 1/32 of the LM head per step; tokens/s of the full 32-layer model = rows / "
              f"(32 t_layer + 32 t_lm_slice)")


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return 1


def oracle_tiny_end_to_end():
    """BASELINE configs[0] (cfg1) end to end on the oracle: the SortedRL controller with
    the tiny fp64 model (16 prompts, Q = 16, U = 4): generated tokens / wall second."""
    from oracle.model import ModelRunner, load_weights
    from oracle.sched import Controller
    from workload.configs import TINY
    off, toks = make_prompts(1, 16, TINY.V, 4, 16)
    L = sample_lengths(LengthModel(median=12, sigma=0.6, tail=0.1, floor=1, cap=64), 0, 16)
    W = load_weights(TINY)
    cfg = SchedConfig(Q_g=16, U=4, K=K_INF, pool_prompts=16, cap=64, kv_pages=256)
    runner = ModelRunner(TINY, lambda v: W, lambda t: toks[off[t.prompt_id]:off[t.prompt_id + 1]], seed=3)
    c = Controller(cfg, runner)
    c.submit_prompts(range(16), np.diff(off), L)
    t0 = time.perf_counter()
    c.run()
    dt = time.perf_counter() - t0
    return {"value": c.raw_tokens / dt, "unit": "tokens/s", "tokens": c.raw_tokens, "decode_steps": len(c.trace),
            "wall_s": dt, "workload": "cfg1 (BASELINE configs[0]): tiny fp64 model + SortedRL controller, 16 prompts"}


def oracle_sample(seconds_budget=20.0):
    """cpu_baseline of the GPU arm: the oracle slice on all host cores for about
    `seconds_budget` seconds (median over steps), plus the same slice on one thread."""
    sl = OracleSlice()
    vals, t0 = [], time.perf_counter()
    while time.perf_counter() - t0 < seconds_budget or len(vals) < 3:
        vals.append(sl.step()[1])
    one = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1):
            one = float(np.median([sl.step()[1] for _ in range(2)]))
    except Exception:
        pass
    return {"value": float(np.median(vals)), "unit": "tokens/s", "cores": blas_threads(), "kind": "oracle",
            "host_cpus": os.cpu_count(), "single_thread_value": one,
            "sample": OracleSlice.SAMPLE + f"; median of {len(vals)} steps"}


def run_reference(args):
    """--impl reference: the tier's reference arm is the CPU oracle as it stands.  Each
    step is one OracleSlice step (a bounded sample of the cfg2 workload, timed for real);
    warm-up steps are run and discarded; one thread and the cfg1 end-to-end run are
    reported beside it.  With N > 1 ranks only rank 0 works (the others count themselves
    in over a CPU process group and exit)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    ranks = 1
    if world > 1:
        import torch
        import torch.distributed as td
        td.init_process_group("gloo")
        t = torch.ones(1)
        td.all_reduce(t)
        ranks = int(t.item())
        td.destroy_process_group()
    if rank != 0:
        return
    sl = OracleSlice()
    for _ in range(args.warmup):
        sl.step()
    wall, vals = [], []
    for _ in range(max(1, args.steps)):
        w, v = sl.step()
        wall.append(w)
        vals.append(v)
    value = float(np.median(vals))
    one = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1):
            one = sl.step()[1]
    except Exception:
        pass
    tiny = oracle_tiny_end_to_end()
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": max(1, args.steps),
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(wall)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "ranks": ranks,
            "config": {"workload": MODELS[args.model][7] or WORKLOAD, "sample": OracleSlice.SAMPLE,
                       "step": "one OracleSlice step (wall time = ms_per_step)"},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": blas_threads(), "kind": "oracle",
                             "host_cpus": os.cpu_count(), "single_thread_value": one,
                             "sample": OracleSlice.SAMPLE + f"; median of {len(vals)} steps"},
            "tiny_end_to_end": tiny,
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(n):
    """`bench.py --gpus N` run without a launcher: start N ranks of this script (one
    process per GPU, torch.distributed rendezvous on 127.0.0.1) and wait for them;
    a rank that fails takes the others down."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rc = 0
    while procs:
        for p in list(procs):
            code = p.poll()
            if code is None:
                continue
            procs.remove(p)
            if code != 0:
                rc = code
                for q in procs:        # a failed rank would leave its peers blocked in a collective
                    q.terminate()
        time.sleep(0.2)
    return rc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3, help="timed early-update rounds")
    ap.add_argument("--warmup", type=int, default=3, help="untimed rounds before them (at least)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="llama8b", choices=sorted(MODELS),
                    help="llama8b = BASELINE configs[1] (default); qwen32b = the per-GPU slice of configs[3]")
    ap.add_argument("--mode", default="sorted", choices=["sorted", "sync", "posthoc"],
                    help="scheduler: SortedRL (default), the synchronous baseline, post-hoc sorting (P:349)")
    ap.add_argument("--K", type=int, default=K_INF, help="cache bound in policy versions (-1 = inf, 0 = on-policy)")
    ap.add_argument("--U", type=int, default=64, help="update group size")
    ap.add_argument("--barrier", default="trained", choices=["trained", "admitted"], help="cache-aware loading barrier")
    ap.add_argument("--attn-every", type=int, default=4,
                    help="time the attention launches on 1 decode step in N (the roofline's measured kernel)")
    ap.add_argument("--tuning", default="", help="srl_tuning overrides for measurement, e.g. fuse_mlp=0,mlp_splits=4")
    ap.add_argument("--G", type=int, default=1, help="responses per prompt (trajectories per epoch unchanged)")
    ap.add_argument("--share-prefix", action="store_true", help="N4: G samples share their prompt-prefix KV pages")
    ap.add_argument("--prefill-budget", type=int, default=0, help="N1: prefill tokens per GPU per step (0 = unlimited)")
    ap.add_argument("--resume", default="keep_kv", choices=["keep_kv", "reprefill"],
                    help="how kept partial trajectories resume (reading R10): keep their KV (default) or re-prefill "
                         "prompt + generated tokens (P:180 literal)")
    ap.add_argument("--prof-every", type=int, default=8,
                    help="every class is bracketed by events on one decode step in this many (the breakdown); "
                         "the rest bracket attention only (the roofline)")
    ap.add_argument("--trace-out", default=None, help="write every decode step's (r_k, sum_ctx, dt_ms, prefill "
                    "tokens, finished, r_local) as .npy")
    ap.add_argument("--full", action="store_true",
                    help="time the whole 2-epoch rollout (every round, incl. epoch starts and drains) instead")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:          # no launcher: start the N ranks ourselves
        sys.exit(self_launch(args.gpus))
    world = max(1, world)
    if world != args.gpus:
        raise SystemExit(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.impl == "reference":
        return run_reference(args)
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import datetime

        import torch
        import torch.distributed as td
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        td.init_process_group("nccl", timeout=datetime.timedelta(seconds=600))
        dist = td
    r = run_gpu(args, rank, world, dist)
    if args.trace_out and rank == 0:
        np.save(args.trace_out, np.array(r["trace"], dtype=np.float64))
    m = MODELS[args.model][0]
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    # per-rank aggregates over the timed rounds
    stats = r["stats"]
    sum_ctx = sum(x[1] for x in stats)
    steps = r["ran"]
    n_dec = len(stats)
    attn_ms, attn_n = r["prof"]["attention"]
    # dominant kernel: paged attention, bracketed by CUDA events on the engine stream in
    # the sampled decode steps of the timed window (a class's events sit outside its
    # launches, inside the graph); units = those steps' context tokens per layer
    per_unit = 2 * m.Hkv * m.dh * 2                             # K+V bytes per context token per layer
    att_ctx = r.get("att_ctx") or [x[1] for x in stats]
    units = sum(att_ctx)                                         # context tokens read per layer, timed launches
    achieved = per_unit * units * m.L / (attn_ms * 1e-3) / 1e9 if attn_ms > 0 else None
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if os.path.exists(tp):                                       # committed ncu --set full capture (one launch)
        with open(tp) as fh:
            traffic_src = json.load(fh)
        traffic = traffic_src["dram_bytes_per_launch"]
    roof = {"bound": "hbm", "kernel": "attn_bf16_kernel (paged GQA decode attention)", "achieved": achieved,
            "peak": hbm, "unit": "GB/s", "frac": achieved / hbm if achieved else None, "traffic": traffic,
            "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum of the one attention launch captured with "
                            "ncu --set full (traffic_capture: its own algorithmic bytes beside it)",
            "traffic_capture": traffic_src,
            "per_unit_bytes": per_unit, "unit_def": "one context token of one layer (K+V, bf16)",
            "units_per_launch": units / max(1, len(att_ctx)), "launches": attn_n,
            "peak_source": peak_src + " (MEASURED_PEAKS.json copy bandwidth; a read-only stream may exceed it)"}
    # decode roofline fraction of the whole step
    t_roof = 0.0
    for (rk, sc, dt, npre, nfin, rl) in stats:
        B, F, _, _ = step_bytes_flops(m, rl, sc)                 # this GPU's rows and context
        t_roof += max(B / (hbm * 1e9), F / (tf_sust * 1e12))
    dec_frac = t_roof / (r["ms"] * 1e-3) if r["ms"] > 0 else None
    tok_s = r["raw"] / (r["ms"] * 1e-3)
    Q = MODELS[args.model][1] * world                           # Q_tot (reading R1)

    def bubble(tr):
        if not tr:
            return None, None
        ab = sum(Q - x[0] for x in tr) / (Q * len(tr))
        tw = sum((Q - x[0]) * x[2] for x in tr) / (Q * max(1e-9, sum(x[2] for x in tr)))
        return ab, tw
    b_win, b_win_t = bubble(stats)
    b_all, b_all_t = bubble(r["trace"])
    e2e = r["e2e"]
    if dist:
        tok_s, useful_s, ms = aggregate_over_ranks(dist, r["raw"], r["useful"], r["ms"])
        if e2e:   # whole-job e2e: all replicas' tokens (the replicated counters) / the slowest rank's wall
            import torch
            t = torch.tensor([e2e["wall_ms_per_step"]], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e = dict(e2e, value=e2e["tokens"] / (t.item() * max(1, e2e["steps"]) * 1e-3), wall_ms_per_step=t.item())
    else:
        useful_s = r["useful"] / (r["ms"] * 1e-3)
        ms = r["ms"]
    if rank != 0:
        dist.barrier() if dist else None
        return
    nb = max(1, r["n_break"])
    bd = {k: v[0] / nb for k, v in r["breakdown"].items()}
    if att_ctx:
        bd["attention"] = attn_ms / len(att_ctx)                 # per timed step (1 in attn_every + the sampled ones)
    win = r.get("window")
    line = {
        "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world, "steps": steps,
        "warmup": r.get("warmup_rounds", args.warmup), "ms_per_step": ms / max(1, steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": MODELS[args.model][7] or WORKLOAD,
                   "scheduler": {"mode": args.mode, "K": args.K, "U": args.U, "barrier": args.barrier,
                                 "resume": args.resume, "G": args.G, "share_prefix": bool(args.share_prefix),
                                 "prefill_budget": args.prefill_budget},
                   "step": "one early-update round: decode steps (refill, prefill, decode GEMMs, paged attention, "
                           "Philox sampling, stop detection, compaction) until the length-sorted update group of "
                           f"U={args.U} is ready, its harvest, and the policy refresh (load_policy_weights, K bound)",
                   "window": (f"the whole 2-epoch rollout: {steps} rounds, {n_dec} decode steps" if args.full else
                              f"rounds {win[0] + 1}..{win[1]} of the job (the first epoch boundary mid-window: "
                              f"epoch drain + next epoch's prefill burst inside), {n_dec} decode steps; "
                              f"{r.get('warmup_rounds')} untimed rounds before"),
                   "l2": "no flush needed: every decode step streams 15 GB of weights + the KV cache (>> 126 MB L2)",
                   "parallelism": f"dp{world} lockstep replicas (NCCL)" if world > 1 else "dp1",
                   **({"tuning": args.tuning} if args.tuning else {})},
        "decode_steps": n_dec,
        "ms_per_decode_step": ms / max(1, n_dec),
        "useful_tokens_per_s": useful_s,
        "bubble_ratio": {"window_abstract": b_win, "window_time_weighted": b_win_t,
                         "since_start_abstract": b_all, "since_start_time_weighted": b_all_t,
                         "since_start_steps": len(r["trace"]),
                         "definition": "Eq.(bubble) P:339-342, Q = Q_tot; abstract (dt=1) and measured dt"},
        "decode_roofline_frac": {"value": dec_frac, "definition": "sum_k max(B_k/BW, F_k/TC) / sum_k dt_k (SURVEY 8(d))",
                                 "BW_GBs": hbm, "TC_TFs": tf_sust},
        "roofline": roof,
        "kernel_ms_per_decode_step": bd,
        "kernel_breakdown_note": (f"inside the timed window: every class bracketed by CUDA events on 1 decode step in "
                                  f"{args.prof_every} ({r['n_break']} steps; those steps lose their PDL edges), "
                                  f"attention alone on 1 in {args.attn_every} more ({len(r.get('att_ctx') or [])} "
                                  f"attention-timed steps in all); prefill passes counted under 'prefill'"),
        "paper_context": {"note": "context, not the target: P:336-339, H100/MI300X mix (P:239), GPU type/count, engine "
                                  "capacity and length trace unstated",
                          "bubble": {"sync_baseline": 0.74, "sortedrl_on_policy": 0.0581, "sortedrl_partial": 0.0337},
                          "tokens_per_s": {"sync_baseline": 3987, "sortedrl_on_policy": 4289, "sortedrl_partial": 5559}},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "e2e": e2e,
        "mean_ctx": sum_ctx / max(1, sum(x[5] for x in stats)),
    }
    if not args.no_cpu and world == 1 and args.model == "llama8b":
        line["cpu_baseline"] = oracle_sample()
    elif not args.no_cpu:
        line["cpu_baseline"] = None
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()


if __name__ == "__main__":
    main()
