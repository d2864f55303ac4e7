"""Pins for oracle/sched.py + oracle/metrics.py: the SortedRL controller in
abstract time (dt = 1 per decode step).  CPU only.

Each pin comes from somewhere other than the oracle itself: SPEC.md worked
examples, closed forms derived from the schedule definition (SURVEY §8(c)
P2/P3), a hand-derived example (tests/golden/sched_worked_example.json),
numeric integration of the length distribution, and invariants.
"""
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle.metrics import bubble_ratio
from oracle.sched import DONE, GROUP_READY, Controller, SchedError
from workload.configs import (BARRIER_ADMITTED, BARRIER_TRAINED, K_INF, MODE_POSTHOC, MODE_SORTED, MODE_SYNC,
                              RESUME_KEEP_KV, RESUME_REPREFILL, SchedConfig)
from workload.lengths import LengthModel, sample_lengths

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def run(lengths, prompt_len=4, **kw):
    cfg = SchedConfig(**kw)
    c = Controller(cfg)
    n = len(lengths) // cfg.G
    c.submit_prompts(range(n), [prompt_len] * n, lengths)
    groups = c.run()
    return c, groups


# ---------------------------------------------------------------- Eq. (bubble)
def test_bubble_ratio_spec_examples():
    """all full -> 0; Q=2, [(4 units, r=2), (6 units, r=1)] -> 0.3."""
    assert bubble_ratio([(0, 4), (1, 4)], 4) == 0
    assert abs(bubble_ratio([(0, 2), (1, 1)], 2, dts=[4.0, 6.0]) - 0.3) < 1e-15
    with pytest.raises(ValueError):
        bubble_ratio([], 2)


def test_engine_trace_spec_example():
    """Q=2, lengths 4 and 10 -> r = [2,2,2,2,1,1,1,1,1,1]."""
    c, groups = run([4, 10], Q_g=2, U=2, pool_prompts=2, cap=16)
    assert [r for _, r in c.trace] == [2, 2, 2, 2, 1, 1, 1, 1, 1, 1]
    assert [[r["len"] for r in g] for g in groups] == [[4, 10]]


def test_harvest_trace_spec_example():
    """8 requests of lengths 1..8, Q=4, target 4 -> first 4 harvested after 4 steps."""
    c, groups = run(list(range(1, 9)), Q_g=4, U=4, pool_prompts=8, cap=16)
    assert [r["len"] for r in groups[0]] == [1, 2, 3, 4]
    first_emit = [e for e in c.events if e[0] == "EMIT"][0]
    finishes = [e for e in c.events if e[0] == "FINISH" and e[3] in first_emit[3]]
    assert max(e[1] for e in finishes) == 3          # steps 0..3 -> 4 steps


def test_select_train_batches_spec_example():
    """lengths [5,1,3,2], batch size 2 -> [[1,2],[3,5]] (all start together)."""
    c, groups = run([5, 1, 3, 2], Q_g=4, U=2, pool_prompts=4, cap=8)
    assert [[r["len"] for r in g] for g in groups] == [[1, 2], [3, 5]]


# ---------------------------------------------------------------- worked example
def test_worked_example_golden():
    with open(os.path.join(GOLD, "sched_worked_example.json")) as fh:
        gold = json.load(fh)
    L = gold["lengths"]
    for key, K in (("K_inf", K_INF), ("K_0", 0)):
        c, groups = run(L, Q_g=gold["Q"], U=gold["U"], pool_prompts=len(L), cap=16, K=K)
        g = gold[key]
        assert [[r["traj_id"] for r in grp] for grp in groups] == g["groups"]
        assert len(c.trace) == g["T"]
        assert bubble_ratio(c.trace, gold["Q"]) == Fraction(*g["bubble"])
        assert c.raw_tokens == g["raw"]
        assert sum(r["len"] for grp in groups for r in grp) == g["useful"]


# ---------------------------------------------------------------- closed forms
def _p2_closed_form(L, Q, U):
    """K=inf, Q >= N, one epoch: groups = consecutive U-slices of sort(len, id);
    T = max L; B = 1 - sum L / (Q max L); group j (0-based) staleness = j."""
    order = sorted(range(len(L)), key=lambda i: (L[i], i))
    groups = [order[i:i + U] for i in range(0, len(order), U)]
    T = max(L)
    return groups, T, 1 - Fraction(sum(L), Q * T)


def _p3_closed_form(L, Q, U):
    """K=0, Q >= N: rounds; round length = U-th smallest remaining (len, id) (max if
    fewer than U remain); busy_j = sum over remaining of min(len, lambda_j)."""
    rem = sorted(range(len(L)), key=lambda i: (L[i], i))
    T, busy, groups = 0, 0, []
    while rem:
        take = rem[:U]
        lam = L[take[-1]]
        busy += sum(min(L[i], lam) for i in rem)
        T += lam
        groups.append(take)
        rem = rem[U:]
    return groups, T, 1 - Fraction(busy, Q * T), busy


@pytest.mark.parametrize("seed", range(40))
def test_closed_form_partial_mode_p2(seed):
    rng = random.Random(seed)
    N = rng.randint(1, 24)
    U = rng.randint(1, max(1, N))
    Q = rng.randint(N, N + 5)
    L = [rng.randint(1, 20) for _ in range(N)]
    c, groups = run(L, Q_g=Q, U=U, pool_prompts=N, cap=20, K=K_INF)
    want_groups, T, B = _p2_closed_form(L, Q, U)
    assert [[r["traj_id"] for r in g] for g in groups] == want_groups
    assert len(c.trace) == T
    assert bubble_ratio(c.trace, Q) == B
    for j, g in enumerate(groups):
        for r in g:
            assert r["v_first"] == 0 and r["vers"][-1] <= j


@pytest.mark.parametrize("seed", range(40))
def test_closed_form_on_policy_mode_p3(seed):
    rng = random.Random(1000 + seed)
    N = rng.randint(1, 24)
    U = rng.randint(1, max(1, N))
    Q = rng.randint(N, N + 5)
    L = [rng.randint(1, 20) for _ in range(N)]
    c, groups = run(L, Q_g=Q, U=U, pool_prompts=N, cap=20, K=0)
    want_groups, T, B, busy = _p3_closed_form(L, Q, U)
    assert [[r["traj_id"] for r in g] for g in groups] == want_groups
    assert len(c.trace) == T
    assert bubble_ratio(c.trace, Q) == B
    assert c.raw_tokens == busy
    for j, g in enumerate(groups):          # fully on-policy: every token from the emitting version
        for r in g:
            assert set(r["vers"]) == {j} and r["v_first"] == j


@pytest.mark.parametrize("seed", range(30))
def test_posthoc_sorting_definition(seed):
    """P:349 post-hoc sorting: each loaded pool is generated to completion (with
    refill when Q < pool) before anything is emitted; then its trajectories go out
    as the U-slices of sort(len, traj_id), one per policy version -- group j of a
    pool is j versions stale, and every token of the pool is from the version it
    started under.  With Q >= pool each pool takes exactly max(len) steps."""
    rng = random.Random(3000 + seed)
    P = rng.randint(1, 12)
    n_pools = rng.randint(1, 3)
    N = P * n_pools
    U = rng.randint(1, P)
    Q = rng.randint(max(1, P // 2), P + 3)
    L = [rng.randint(1, 15) for _ in range(N)]
    c, groups = run(L, Q_g=Q, U=U, pool_prompts=P, cap=15, K=K_INF, mode=MODE_POSTHOC)
    want, v = [], 0
    for e in range(n_pools):
        ids = sorted(range(e * P, (e + 1) * P), key=lambda t: (L[t], t))
        want += [ids[i:i + U] for i in range(0, P, U)]
    assert [[r["traj_id"] for r in g] for g in groups] == want
    ev = c.events
    for e in range(n_pools):                     # no emission of a pool before its last finish
        pool = set(range(e * P, (e + 1) * P))
        last_fin = max(i for i, x in enumerate(ev) if x[0] == "FINISH" and x[3] in pool)
        first_emit = min(i for i, x in enumerate(ev) if x[0] == "EMIT" and set(x[3]) <= pool)
        assert first_emit > last_fin
    v = 0
    for e in range(n_pools):
        ng = (P + U - 1) // U
        for j in range(ng):
            for r in groups[v + j]:
                assert set(r["vers"]) == {v} and r["v_first"] == v      # generated before any update
        v += ng
    if Q >= P:
        assert len(c.trace) == sum(max(L[e * P:(e + 1) * P]) for e in range(n_pools))


@pytest.mark.parametrize("seed", range(20))
def test_sync_closed_form(seed):
    """SYNC: B = 1 - sum L / (Q * sum_batches max L) with batches of Q in traj order."""
    rng = random.Random(2000 + seed)
    Q = rng.randint(1, 8)
    nb = rng.randint(1, 4)
    N = Q * nb - rng.randint(0, Q - 1)
    L = [rng.randint(1, 15) for _ in range(N)]
    U = rng.randint(1, Q)
    c, groups = run(L, Q_g=Q, U=U, pool_prompts=Q, cap=15, mode=MODE_SYNC)
    batches = [L[i:i + Q] for i in range(0, N, Q)]
    T = sum(max(b) for b in batches)
    assert len(c.trace) == T
    assert bubble_ratio(c.trace, Q) == 1 - Fraction(sum(L), Q * T)
    # groups: completion order (finish_step, slot) within each batch, ceil(b/U) per batch
    assert len(groups) == sum((len(b) + U - 1) // U for b in batches)
    for g in groups:
        fs = [(r["finish_step"], r["traj_id"]) for r in g]
        assert fs == sorted(fs)


def test_equal_lengths_bubble():
    """All lengths equal, N = mQ -> B = 0; N = mQ + j -> B = 1 - N/((m+1)Q)."""
    c, _ = run([7] * 12, Q_g=4, U=4, pool_prompts=12, cap=8)
    assert bubble_ratio(c.trace, 4) == 0
    c, _ = run([7] * 10, Q_g=4, U=2, pool_prompts=10, cap=8)
    assert bubble_ratio(c.trace, 4) == 1 - Fraction(10, 3 * 4)


def test_expected_sync_bubble_matches_numeric_integration():
    """E[B_sync] = 1 - E[L] / E[max of Q lengths], from the length CDF by numeric
    integration (independent of the simulator), at the tiny config (cap 64, Q=16)."""
    lm = LengthModel(median=12, sigma=0.6, tail=0.1, floor=1, cap=64)
    from scipy.stats import norm
    xs = np.arange(1, 65)
    # P(L <= x) for the recipe: body clamp(rint(exp(mu + s z))) plus tail at cap
    edges = np.log(xs + 0.5)
    Fb = norm.cdf((edges - np.log(lm.median)) / lm.sigma)
    Fb[-1] = 1.0
    F = (1 - lm.tail) * Fb
    F[-1] = 1.0
    p = np.diff(np.concatenate([[0.0], F]))
    EL = (xs * p).sum()
    Q = 16
    Emax = (xs * np.diff(np.concatenate([[0.0], F ** Q]))).sum()
    expected = 1 - EL / Emax
    N = Q * 400
    L = sample_lengths(lm, 0, N).tolist()
    c, _ = run(L, Q_g=Q, U=4, pool_prompts=Q, cap=64, mode=MODE_SYNC)
    got = float(bubble_ratio(c.trace, Q))
    assert abs(expected - 0.672) < 0.01          # SURVEY Appendix B value
    assert abs(got - expected) < 0.02


def test_throughput_identity_flat_cost():
    """with dt = 1, raw tokens = Q (1 - B) #steps exactly."""
    for seed in range(30):
        rng = random.Random(3000 + seed)
        Q = rng.randint(1, 6)
        L = [rng.randint(1, 12) for _ in range(rng.randint(1, 30))]
        c, _ = run(L, Q_g=Q, U=rng.randint(1, 4), pool_prompts=rng.randint(4, 12), cap=12,
                   K=rng.choice([K_INF, 0, 1]))
        B = bubble_ratio(c.trace, Q)
        assert c.raw_tokens == Q * (1 - B) * len(c.trace)


# ---------------------------------------------------------------- invariants
def _random_cfg(rng):
    R = rng.choice([1, 1, 2, 4])
    return dict(Q_g=rng.randint(1, 5), R=R, U=rng.randint(1, 6), K=rng.choice([K_INF, 0, 1, 2]),
                pool_prompts=rng.randint(2, 10), G=rng.choice([1, 1, 2]), cap=rng.randint(4, 30),
                page_tokens=rng.choice([2, 4, 64]), kv_pages=rng.choice([4, 8, 16, 1 << 20]),
                resume=rng.choice([RESUME_KEEP_KV, RESUME_REPREFILL]),
                barrier=rng.choice([BARRIER_TRAINED, BARRIER_ADMITTED]),
                mode=rng.choice([MODE_SORTED, MODE_SORTED, MODE_SYNC, MODE_POSTHOC]),
                share_prefix=rng.choice([0, 1]), prefill_budget=rng.choice([0, 0, 1, 3, 8]))


@pytest.mark.parametrize("seed", range(500))
def test_invariants_random_runs(seed):
    rng = random.Random(seed)
    kw = _random_cfg(rng)
    if kw["share_prefix"] and kw["G"] > 1 and kw["prefill_budget"]:
        with pytest.raises(SchedError):
            Controller(SchedConfig(**kw))
        kw["prefill_budget"] = 0
    cfg = SchedConfig(**kw)
    n_prompts = rng.randint(1, 16)
    N = n_prompts * cfg.G
    L = [rng.randint(1, cfg.cap) for _ in range(N)]
    plen = [rng.randint(1, 6) if rng.random() < 0.5 else rng.randint(1, 20) for _ in range(n_prompts)]
    if cfg.mode in (MODE_SORTED, MODE_POSTHOC) and cfg.U > cfg.pool_prompts * cfg.G:
        with pytest.raises(SchedError):
            Controller(cfg)
        return
    c = Controller(cfg)
    c.submit_prompts(range(n_prompts), plen, L)
    # a trajectory must fit the pool on its own, else admission can deadlock (CAPACITY)
    need_max = max((plen[i // cfg.G] + cfg.cap - 1 + cfg.page_tokens - 1) // cfg.page_tokens for i in range(N))
    groups_v = []
    try:
        c.load_policy_weights(0)
        while True:
            st = c.decode_step()
            assert all(r <= cfg.Q_tot for _, r in c.trace)
            if st == DONE:
                break
            if st == GROUP_READY:
                groups_v.append((c.harvest(), c.v, c.group_final))
                c.load_policy_weights(c.v + 1)
    except SchedError as e:
        assert e.code == "CAPACITY" and need_max * 1 > cfg.kv_pages // 2, e
        return
    if cfg.kv_pages >= (1 << 20):                                  # no preemption possible
        assert all(c.work_conserving)
    emitted = [r["traj_id"] for recs, _, _ in groups_v for r in recs]
    assert sorted(emitted) == list(range(N))                      # each exactly once
    for recs, v_emit, final in groups_v:
        if cfg.mode in (MODE_SORTED, MODE_POSTHOC):
            keys = [(r["len"], r["traj_id"]) for r in recs]
            assert keys == sorted(keys)                           # sorted within group
            assert len(recs) == cfg.U or final                    # batch exactness
            if cfg.K >= 0:
                for r in recs:
                    assert v_emit - r["v_first"] <= cfg.K         # cache bound
        for r in recs:
            assert r["len"] == len(r["tokens"]) == len(r["lps"]) == len(r["vers"])
            assert r["len"] == L[r["traj_id"]]                   # FORCED stop exact
            assert r["vers"] == sorted(r["vers"])                  # segment versions nondecreasing
            # v_first is stamped at admission (R30): with a prefill budget the first token
            # may come after a version bump
            assert r["vers"][0] == r["v_first"] if not cfg.prefill_budget else r["vers"][0] >= r["v_first"]
    # N1: the per-replica budget holds every step; with no interruption and no
    # sharing every admission prefills exactly prompt_len - 1 positions
    assert len(c.prefill_trace) == len(c.trace)
    if cfg.prefill_budget:
        assert all(x <= cfg.prefill_budget for _, pre in c.prefill_trace for x in pre)
    if not any(e[0] in ("PREEMPT", "DISCARD", "SCAVENGE") for e in c.events) and not (cfg.share_prefix and cfg.G > 1):
        assert sum(sum(pre) for _, pre in c.prefill_trace) == sum(plen[i // cfg.G] - 1 for i in range(N))
    # page conservation (incl. shared prompt prefixes, N4): every page back at DONE
    assert c.free_pages == [cfg.kv_pages] * cfg.R and all(v == 0 for v in c.pfx_ref.values())
    # token conservation: raw = emitted + discarded (nothing in flight at DONE)
    assert c.raw_tokens == sum(L) + c.discarded_tokens
    # lifecycle counts interruptions: events PREEMPT + DISCARD + SCAVENGE per traj
    inter = {}
    for e in c.events:
        if e[0] in ("PREEMPT",):
            inter[e[3]] = inter.get(e[3], 0) + 1
        elif e[0] in ("DISCARD", "SCAVENGE"):
            inter[e[2]] = inter.get(e[2], 0) + 1
    for recs, _, _ in groups_v:
        for r in recs:
            assert r["lifecycle"] == inter.get(r["traj_id"], 0)
    # TRAINED barrier: no admission of epoch e+1 before epoch e fully emitted
    if cfg.barrier == BARRIER_TRAINED or cfg.mode in (MODE_SYNC, MODE_POSTHOC):
        loads = [e for e in c.events if e[0] == "LOAD"]
        emit_idx = {}
        for i, e in enumerate(c.events):
            if e[0] == "EMIT":
                for t in e[3]:
                    emit_idx[t] = i
        for i, e in enumerate(c.events):
            if e[0] == "LOAD" and e[2] > 0:
                prev = [x for x in loads if x[2] == e[2] - 1][0]
                for t in range(prev[3], prev[3] + prev[4]):
                    assert emit_idx[t] < i


def test_r_invariance_event_logs():
    """(R, Q_g) and (1, R*Q_g) give identical event logs with ample pages (slot g = s*R + r)."""
    for seed in range(20):
        rng = random.Random(4000 + seed)
        L = [rng.randint(1, 25) for _ in range(40)]
        base = dict(U=rng.randint(1, 6), K=rng.choice([K_INF, 0, 1]), pool_prompts=rng.randint(6, 40), cap=25,
                    resume=rng.choice([RESUME_KEEP_KV, RESUME_REPREFILL]))
        R = rng.choice([2, 4, 8])
        Qg = rng.randint(1, 3)
        c1, g1 = run(L, Q_g=R * Qg, R=1, **base)
        c2, g2 = run(L, Q_g=Qg, R=R, **base)
        assert c1.events == c2.events
        assert c1.trace == c2.trace


def test_micro_curriculum_statistical():
    """P:175/P:507 'short-short-short-long': with the default workload and n=4, the
    last group of an epoch is >= 1.5x longer than the first."""
    lm = LengthModel(median=400, sigma=0.55, tail=0.03, cap=2048)
    Q, b = 32, 32
    L = sample_lengths(lm, 5, 4 * b * 3).tolist()
    c, groups = run(L, Q_g=Q, U=32, pool_prompts=4 * b, cap=2048, K=K_INF)
    per_epoch = {}
    for g in groups:
        e = c.stream[g[0]["traj_id"]].epoch
        per_epoch.setdefault(e, []).append(np.mean([r["len"] for r in g]))
    ratios = [v[-1] / v[0] for v in per_epoch.values()]
    assert min(ratios) >= 1.5, ratios


def test_state_errors():
    cfg = SchedConfig(Q_g=2, U=1, pool_prompts=2, cap=4)
    c = Controller(cfg)
    with pytest.raises(SchedError):
        c.decode_step()                      # no weights
    c.load_policy_weights(0)
    with pytest.raises(SchedError):
        c.submit_prompts([1, 1], [2, 2], [1, 1])   # duplicate id
    with pytest.raises(SchedError):
        c.submit_prompts([1], [2], [9])             # forced_len > cap
    c.submit_prompts([1, 2], [2, 2], [1, 2])
    assert c.decode_step() == GROUP_READY
    with pytest.raises(SchedError):
        c.decode_step()                      # group pending
    with pytest.raises(SchedError):
        c.load_policy_weights(1)             # not harvested
    c.harvest()
    with pytest.raises(SchedError):
        c.harvest()
    with pytest.raises(SchedError):
        c.load_policy_weights(0)             # version must increase
    c.load_policy_weights(1)
    with pytest.raises(SchedError):
        Controller(SchedConfig(Q_g=0))


# ---------------------------------------------------------------- metrics pins
def test_staleness_spec_segment_example():
    """S:366 (P:180 partial mode): segments (v3: 5 tokens)(v4: 7)(v5: 2) emitted at
    version 5 -> per-token staleness 2 x5, 1 x7, 0 x2; the trajectory's v_emit - v_first = 2."""
    from oracle.metrics import staleness
    rec = {"v_first": 3, "vers": [3] * 5 + [4] * 7 + [5] * 2}
    tok, traj = staleness([([rec], 5)])
    assert tok == {2: 5, 1: 7, 0: 2} and traj == {2: 1}


def test_staleness_sync_baseline_four_off_policy_updates():
    """P:263 (section 4.3): rollout batch 512, update batch 128 -> '4 off-policy updates in
    each iteration': the k-th group of a SYNC batch (0-based) is emitted k versions after
    the batch was generated, so the last one has staleness 3 on every token.  Scaled to a
    rollout batch of 8 and update groups of 2 (the same 4:1 ratio)."""
    from oracle.metrics import staleness
    L = [3, 1, 4, 1, 5, 9, 2, 6]
    c, groups = run(L, Q_g=8, U=2, pool_prompts=8, cap=16, mode=MODE_SYNC)
    assert len(groups) == 4
    for k, g in enumerate(groups):
        tok, traj = staleness([(g, k)])
        assert set(tok) == {k} and set(traj) == {k}
    tok, _ = staleness([(g, k) for k, g in enumerate(groups)])
    assert tok[3] == sum(r["len"] for r in groups[-1])


def test_curriculum_profile_worked_example():
    """golden/sched_worked_example.json (K = inf, Q >= N, one epoch): groups are the
    consecutive U-slices of the sorted lengths [1,1 | 2,3 | 4,5 | 6,9], so the profile
    of group means is [1, 2.5, 4.5, 7.5] -- the short-to-long micro-curriculum."""
    from oracle.metrics import curriculum_profile
    c, groups = run([3, 1, 4, 1, 5, 9, 2, 6], Q_g=8, U=2, pool_prompts=8, cap=16, K=K_INF)
    prof = curriculum_profile([(g, c.stream[g[0]["traj_id"]].epoch) for g in groups])
    assert prof == {0: [1.0, 2.5, 4.5, 7.5]}
    # two epochs of the same lengths: the profile restarts short in each epoch
    c, groups = run([3, 1, 4, 1, 5, 9, 2, 6] * 2, Q_g=8, U=2, pool_prompts=8, cap=16, K=K_INF)
    prof = curriculum_profile([(g, c.stream[g[0]["traj_id"]].epoch) for g in groups])
    assert prof == {0: [1.0, 2.5, 4.5, 7.5], 1: [1.0, 2.5, 4.5, 7.5]}


def test_throughput_function_identity():
    """metrics.throughput over the abstract trace (dt = 1) equals Q (1 - B)."""
    from oracle.metrics import throughput
    c, _ = run([3, 1, 4, 1, 5, 9, 2, 6], Q_g=4, U=2, pool_prompts=8, cap=16, K=K_INF)
    B = bubble_ratio(c.trace, 4)
    assert throughput(c.raw_tokens, Fraction(len(c.trace))) == 4 * (1 - B)
    with pytest.raises(ValueError):
        throughput(5, 0)


# ---------------------------------------------------------------- N4: shared prompt prefixes
def _pfx_run(kv_pages, share, L=(5, 5, 5, 5), plen=200, **kw):
    cfg = SchedConfig(Q_g=4, U=2, pool_prompts=1, G=4, cap=16, kv_pages=kv_pages, share_prefix=share, **kw)
    c = Controller(cfg)
    c.submit_prompts([7], [plen], list(L))
    c.load_policy_weights(0)
    return c


def test_prefix_sharing_page_accounting_hand_example():
    """One prompt of 200 tokens, G = 4 samples, 64-token pages: positions [0, 199) are
    prefilled by every sample, so floor(199 / 64) = 3 full pages are shareable; each
    sample needs ceil((200 + 1) / 64) = 4 pages after its first token.  Shared: 3 + 4 x 1
    = 7 pages; unshared: 16."""
    for share, used in ((1, 7), (0, 16)):
        c = _pfx_run(100, share)
        c.decode_step()
        assert c.free_pages == [100 - used]
        assert [t.shared for t in c.stream] == ([3] * 4 if share else [0] * 4)


def test_prefix_sharing_admits_more_when_page_limited():
    """kv_pages = 10: unshared, two 4-page samples fit (8) and the third blocks; shared,
    all four fit (7 pages).  Hand-derived r_0 = 2 vs 4."""
    c0 = _pfx_run(10, 0)
    c0.decode_step()
    c1 = _pfx_run(10, 1)
    c1.decode_step()
    assert c0.trace[0] == (0, 2) and c1.trace[0] == (0, 4)


def test_prefix_sharing_only_within_a_policy_version():
    """After a version bump a newly admitted sample does not share the prefix computed
    under the old weights: it holds a private copy of its whole prompt, and the
    old entry is freed when its last holder finishes."""
    cfg = SchedConfig(Q_g=2, U=1, pool_prompts=1, G=3, cap=16, kv_pages=100, share_prefix=1)
    c = Controller(cfg)
    c.submit_prompts([7], [200], [2, 6, 6])
    c.load_policy_weights(0)
    st = c.decode_step()                      # samples 0, 1 admitted, sharing 3 pages
    assert st == 0 and [t.shared for t in c.stream[:2]] == [3, 3] and c.free_pages == [100 - 3 - 2]
    assert c.decode_step() == GROUP_READY     # sample 0 (length 2) finishes and is emitted
    c.harvest()
    c.load_policy_weights(1)
    c.decode_step()                           # sample 2 admitted under version 1
    t2 = c.stream[2]
    assert t2.shared == 0 and t2.pages == 4   # its own copy of the prompt (4 pages)
    assert c.free_pages == [100 - (3 + 1) - 4]


def test_prefix_sharing_same_schedule_with_ample_pages():
    """With pages to spare sharing changes no scheduling decision: identical event logs."""
    rng = random.Random(9)
    for _ in range(40):
        G = rng.choice([2, 4, 8])
        n = rng.randint(1, 6)
        L = [rng.randint(1, 30) for _ in range(n * G)]
        plen = [rng.randint(1, 300) for _ in range(n)]
        kw = dict(Q_g=rng.randint(2, 8), U=rng.randint(1, 4), pool_prompts=rng.randint(1, 4), G=G, cap=30,
                  K=rng.choice([K_INF, 0, 1]), resume=rng.choice([RESUME_KEEP_KV, RESUME_REPREFILL]))
        ev = []
        for share in (0, 1):
            c = Controller(SchedConfig(share_prefix=share, **kw))
            c.submit_prompts(range(n), plen, L)
            c.run()
            ev.append(c.events)
        assert ev[0] == ev[1]


# ---------------------------------------------------------------- N1: per-step prefill budget
def test_prefill_budget_worked_example():
    """Hand-derived (reading R30).  Prompts of 100, 50, 30, 10 tokens need 99, 49, 29, 9
    prefill positions; budget 64 per step, served strictly in admission order:
      k=0: slot 0 gets 64 (35 left)                          -> prefill 64, no decode row
      k=1: slot 0 35 (done), slot 1 29 (20 left)              -> prefill 64, decode {0}
      k=2: slot 1 20, slot 2 29, slot 3 9 (all done)          -> prefill 58, decode {0,1,2,3}
      k=3: slot 0 emits its 3rd token and finishes            -> decode 4
      k=4: slots 1, 2, 3 finish                               -> decode 3, group of 4."""
    cfg = SchedConfig(Q_g=4, U=4, pool_prompts=4, cap=8, prefill_budget=64)
    c = Controller(cfg)
    c.submit_prompts([1, 2, 3, 4], [100, 50, 30, 10], [3, 3, 3, 3])
    c.load_policy_weights(0)
    st = [c.decode_step() for _ in range(5)]
    assert st == [0, 0, 0, 0, GROUP_READY]
    assert c.trace == [(0, 0), (1, 1), (2, 4), (3, 4), (4, 3)]
    assert c.prefill_trace == [(0, (64,)), (1, (64,)), (2, (58,)), (3, (0,)), (4, (0,))]
    fin = [(e[1], e[2]) for e in c.events if e[0] == "FINISH"]
    assert fin == [(3, 0), (4, 1), (4, 2), (4, 3)]
    # unlimited: every prompt prefilled in step 0, all four finish at step 2 (R13)
    c0 = Controller(SchedConfig(Q_g=4, U=4, pool_prompts=4, cap=8))
    c0.submit_prompts([1, 2, 3, 4], [100, 50, 30, 10], [3, 3, 3, 3])
    c0.load_policy_weights(0)
    while c0.decode_step() != GROUP_READY:
        pass
    assert c0.trace == [(0, 4), (1, 4), (2, 4)] and c0.prefill_trace[0] == (0, (99 + 49 + 29 + 9,))


def test_prefill_budget_large_equals_unlimited():
    """A budget no step can exhaust reproduces the unlimited schedule exactly (R13 is the
    budget's limit), on random instances incl. preemption, discards and REPREFILL."""
    for seed in range(60):
        rng = random.Random(7000 + seed)
        kw = _random_cfg(rng)
        kw["share_prefix"] = 0
        kw["mode"] = rng.choice([MODE_SORTED, MODE_SYNC])
        kw["U"] = min(kw["U"], kw["pool_prompts"] * kw["G"])
        n = rng.randint(1, 12)
        L = [rng.randint(1, kw["cap"]) for _ in range(n * kw["G"])]
        plen = [rng.randint(1, 20) for _ in range(n)]
        runs = []
        for C in (0, 10 ** 6):
            c = Controller(SchedConfig(**dict(kw, prefill_budget=C)))
            c.submit_prompts(range(n), plen, L)
            try:
                c.run()
            except SchedError as e:
                assert e.code == "CAPACITY"
                c = None
            runs.append(c)
        if runs[0] is None:
            assert runs[1] is None
            continue
        assert runs[0].events == runs[1].events and runs[0].trace == runs[1].trace
        assert runs[0].prefill_trace == runs[1].prefill_trace


def test_prefill_budget_fifo_and_first_token():
    """Without interruptions: prefills complete in admission order per replica, and a
    trajectory admitted at step a whose prefill needs P positions emits its first token
    no earlier than step a + ceil(P / C) - 1 (the budget is the only limit)."""
    for seed in range(40):
        rng = random.Random(9100 + seed)
        C = rng.choice([1, 5, 16, 40])
        R = rng.choice([1, 2])
        cfg = SchedConfig(Q_g=rng.randint(1, 6), R=R, U=2, pool_prompts=8, cap=20, prefill_budget=C)
        n = 8
        plen = [rng.randint(1, 60) for _ in range(n)]
        L = [rng.randint(1, 20) for _ in range(n)]
        c = Controller(cfg)
        c.submit_prompts(range(n), plen, L)
        c.run()
        admit = {e[3]: (e[1], e[2]) for e in c.events if e[0] == "ADMIT"}
        fin = {e[3]: e[1] for e in c.events if e[0] == "FINISH"}
        first = {t: fin[t] - L[t] + 1 for t in fin}          # FORCED: one token per step once decoding
        for t, (a, g) in admit.items():
            P = plen[t] - 1
            assert first[t] >= a + max(0, -(-P // C) - 1), (t, a, P, C, first[t])
        for r in range(R):
            order = sorted((a, g, t) for t, (a, g) in admit.items() if g % R == r)
            starts = [first[t] for _, _, t in order]
            assert starts == sorted(starts)


def test_prefill_budget_rejected_with_sharing():
    with pytest.raises(SchedError):
        Controller(SchedConfig(G=2, share_prefix=1, prefill_budget=64))
    with pytest.raises(SchedError):
        Controller(SchedConfig(prefill_budget=-1))
