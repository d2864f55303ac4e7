"""BASELINE configs[4] ("cfg5"): the off-policy cache sweep -- cache bound
K in {0, 1, 2, 4, inf} x update group U in {32, 64, 128}, plus the synchronous
baseline -- on the per-GPU cfg2 engine (LLaMA-3.1-8B shape, Q_g = 256, cap 8k,
pools of 1024 prompts, TRAINED barrier, KEEP_KV), each point a fixed window of
the first N decode steps of the job ("GPU runs use a fixed
10k-step window"; full-length numbers come from the oracle).

For every point the GPU's (k, r_k) trace and event log over the window must be
BIT-IDENTICAL to the CPU oracle's (oracle/sched.py, computed in parallel on the
host while the GPU runs), and so must the per-token staleness histogram of the
emitted groups.  Reported per point: useful tokens/s (tokens of emitted
trajectories / device time), raw tokens/s, Eq. (bubble) over the window
(abstract dt = 1 and measured dt), staleness (per token v_emit - version), groups.
Test tooling (imports oracle/).

  python tools/cfg5_sweep.py [--steps N] [--out profiles/r02_cfg5_sweep.json]
"""
import argparse
import dataclasses
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from workload.configs import K_INF, MODE_SORTED, MODE_SYNC  # noqa: E402

POINTS = ([("sync", dict(mode=MODE_SYNC, U=64))] +
          [(f"K={'inf' if K < 0 else K} U={U}", dict(K=K, U=U)) for K in (0, 1, 2, 4, K_INF) for U in (32, 64, 128)])


def _digest(events):
    return hashlib.sha256(repr(events).encode()).hexdigest()


def oracle_point(args):
    """The oracle's first `n` decode steps of the job (same loop as the GPU's)."""
    name, over, n = args
    from oracle.sched import GROUP_READY, Controller
    cfg = dataclasses.replace(bench.cfg2_sched(1), **over)
    off, toks, L = bench.workload_inputs(1, epochs=2)
    c = Controller(cfg)
    c.submit_prompts(np.arange(len(L)) + 1, np.diff(off), L)
    c.load_policy_weights(0)
    stale = {}
    v = 0
    t0 = time.time()
    while len(c.trace) < n:
        st = c.decode_step()
        if st == 2:
            break
        if st == GROUP_READY:
            for r in c.harvest():
                for ver in r["vers"]:
                    stale[v - ver] = stale.get(v - ver, 0) + 1
            v += 1
            c.load_policy_weights(v)
    return name, dict(trace=c.trace, events=_digest(c.events), n_events=len(c.events), stale=stale,
                      raw=c.raw_tokens, wall=time.time() - t0)


def gpu_point(name, over, n):
    import torch
    from paper_2603_23414_b200.engine import DONE, GROUP_READY, RolloutEngine, events_to_oracle_form
    from workload.weights import fill_engine_weights
    cfg = dataclasses.replace(bench.cfg2_sched(1), **over)
    off, toks, L = bench.workload_inputs(1, epochs=2)
    eng = RolloutEngine(bench.LLAMA8B, cfg, max_traj=len(L), max_prompt=bench.PROMPT_LEN, prefill_chunk=4096)
    fill_engine_weights(eng, bench.LLAMA8B, 0)
    trainer = eng.W.clone()
    eng.load_policy_weights(0)
    eng.submit_prompts(np.arange(len(L), dtype=np.uint64) + 1, np.asarray(off, np.int32), toks, L)
    torch.cuda.synchronize()
    stream = eng.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps, useful, stale, dts, rks, v = 0, 0, {}, [], [], 0
    e0.record(stream)
    while steps < n:
        st, info = eng.decode_step()
        if st == DONE:
            break
        if info.k >= 0:
            steps += 1
            dts.append(info.dt_ms)
            rks.append(info.r_k)
        if st == GROUP_READY:
            h = eng.harvest_finished(cap_recs=4096, cap_toks=4096 * cfg.cap)
            useful += int(sum(r["len"] for r in h.records))
            for ver, cnt in zip(*np.unique(v - h.versions, return_counts=True)):
                stale[int(ver)] = stale.get(int(ver), 0) + int(cnt)
            v += 1
            eng.load_policy_weights(v, trainer)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    cnt = eng.counters()
    tr, _ = eng.trace()
    ev, trace = events_to_oracle_form(tr)
    eng.close()
    del trainer
    torch.cuda.empty_cache()
    Q = cfg.Q_tot
    dts = np.array(dts)
    rk = np.array(rks)
    return dict(trace=trace, events=_digest(ev), n_events=len(ev), stale=stale, ms=ms, steps=steps,
                useful_tok_s=useful / (ms * 1e-3), raw_tok_s=cnt["raw_tokens"] / (ms * 1e-3), groups=v,
                discarded=cnt["discarded_tokens"],
                bubble_abstract=float((Q - rk).sum() / (Q * len(rk))),
                bubble_time=float(((Q - rk) * dts).sum() / (Q * dts.sum())))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="comma-separated point names")
    args = ap.parse_args()
    pts = [p for p in POINTS if not args.only or p[0] in args.only.split(",")]
    with ProcessPoolExecutor(max_workers=min(len(pts), max(1, (os.cpu_count() or 2) - 2))) as ex:
        fut = ex.map(oracle_point, [(name, over, args.steps) for name, over in pts])
        gpu = {}
        for name, over in pts:
            t = time.time()
            gpu[name] = gpu_point(name, over, args.steps)
            g = gpu[name]
            print(f"{name:14s} gpu {g['steps']} steps {g['ms'] / 1e3:6.1f} s  useful {g['useful_tok_s']:8.0f} tok/s  raw "
                  f"{g['raw_tok_s']:8.0f}  bubble {g['bubble_abstract']:.3f}/{g['bubble_time']:.3f}  groups {g['groups']}"
                  f"  ({time.time() - t:.0f} s wall)", flush=True)
        orc = dict(fut)
    rows = []
    for name, over in pts:
        g, o = gpu[name], orc[name]
        same = g["trace"] == o["trace"] and g["events"] == o["events"] and g["stale"] == o["stale"]
        toks = sum(o["stale"].values())
        rows.append(dict(point=name, scheduler=over, steps=g["steps"], device_s=g["ms"] / 1e3,
                         useful_tokens_per_s=g["useful_tok_s"], raw_tokens_per_s=g["raw_tok_s"],
                         bubble_abstract=g["bubble_abstract"], bubble_time_weighted=g["bubble_time"],
                         groups=g["groups"], discarded_tokens=g["discarded"],
                         staleness_mean=(sum(k * v for k, v in o["stale"].items()) / toks) if toks else None,
                         staleness_max=max(o["stale"]) if o["stale"] else None,
                         oracle_bit_identical=bool(same), oracle_events=o["n_events"]))
        print(f"{name:14s} oracle-identical {same}  staleness mean {rows[-1]['staleness_mean']} max "
              f"{rows[-1]['staleness_max']}", flush=True)
    out = dict(workload="cfg5 on the per-GPU cfg2 engine (LLaMA-3.1-8B shape, Q_g=256, cap 8192, pools of 1024 "
                        "prompts, 2 epochs, TRAINED barrier, KEEP_KV), first %d decode steps of the job" % args.steps,
               points=rows)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)
    assert all(r["oracle_bit_identical"] for r in rows), [r["point"] for r in rows if not r["oracle_bit_identical"]]


if __name__ == "__main__":
    main()
