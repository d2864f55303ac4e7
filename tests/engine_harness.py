"""Test-side helpers: build a RolloutEngine on seeded synthetic inputs and run
the rollout loop of SURVEY §3 item 2 (submit -> decode_step* -> harvest ->
load_policy_weights)."""
from __future__ import annotations

import numpy as np

from workload.configs import SchedConfig
from workload.lengths import LengthModel, sample_lengths
from workload.prompts import make_prompts
from workload.weights import fill_engine_weights


def fill_weights(eng, model, version, seed=2, flat=None):
    """Write version-`version` weights (workload recipe) into the engine's weight
    region, or into `flat` (a uint8 tensor with the same layout) if given."""
    fill_engine_weights(eng, model, version, seed=seed, flat=flat)


def tiny_workload(n_prompts=16, G=1, seed_len=0, seed_prompt=1, V=512, cap=64, lm=None, plen=(4, 16)):
    lm = lm or LengthModel(median=12, sigma=0.6, tail=0.1, floor=1, cap=cap)
    off, toks = make_prompts(seed_prompt, n_prompts, V, plen[0], plen[1])
    L = sample_lengths(lm, seed_len, n_prompts * G)
    return off, toks, L


def make_engine(model, cfg: SchedConfig, max_traj, max_prompt, prefill_chunk=256, **replica):
    """`replica`: rank / world / local_group / nccl_id for a lockstep replica engine."""
    from paper_2603_23414_b200.engine import RolloutEngine
    eng = RolloutEngine(model, cfg, max_traj=max_traj, max_prompt=max_prompt, prefill_chunk=prefill_chunk,
                        **replica)
    fill_weights(eng, model, 0)
    eng.load_policy_weights(0)
    return eng


def run_engine(eng, model, off, toks, L, *, refresh_weights=True, record_logits=False, max_steps=100000):
    """Returns dict(groups=[(harvest, version_at_emit)], events, steps, logits=[per step], infos)."""
    import torch
    from paper_2603_23414_b200.engine import DONE, GROUP_READY, events_to_oracle_form
    n = len(off) - 1
    eng.submit_prompts(np.arange(n, dtype=np.uint64) + 1000, off, toks, L)
    flat = torch.empty_like(eng.W) if refresh_weights else None
    groups, logits, infos = [], [], []
    v = 0
    for _ in range(max_steps):
        st, info = eng.decode_step()
        if st == DONE:
            break
        if info.k >= 0:                       # a decode step ran (GROUP_READY may follow it)
            infos.append(info)
            if record_logits:
                logits.append(eng.debug_logits())
        if st == GROUP_READY:
            h = eng.harvest_finished(cap_recs=4096)
            groups.append((h, v))
            v += 1
            if refresh_weights:
                fill_weights(eng, model, v, flat=flat)
                eng.load_policy_weights(v, flat)
            else:
                eng.load_policy_weights(v)
    tr, _ = eng.trace()
    ev, steps = events_to_oracle_form(tr)
    return dict(groups=groups, events=ev, steps=steps, logits=logits, infos=infos)
