"""Rollout metrics.  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

Bubble ratio, PAPER.md Eq. (bubble), §4.4.1:
    B = sum_k (Q - r_k) * dt_k / (T * Q),   T = sum_k dt_k
with Q the running-queue size, r_k the running requests and dt_k the duration
of step k.  Throughput = output tokens / T.
"""
from __future__ import annotations

from fractions import Fraction


def bubble_ratio(trace, Q: int, dts=None):
    """trace: [(k, r_k)]; dts: durations (default 1 each -> exact Fraction)."""
    if Q <= 0 or not trace:
        raise ValueError("bubble ratio needs Q > 0 and a non-empty trace (S:455)")
    if dts is None:
        T = len(trace)
        idle = sum(Q - r for _, r in trace)
        return Fraction(idle, T * Q)
    T = float(sum(dts))
    return sum((Q - r) * dt for (_, r), dt in zip(trace, dts)) / (T * Q)


def throughput(total_tokens: int, T: float) -> float:
    if T <= 0:
        raise ValueError("zero-duration trace")
    return total_tokens / T


def staleness(groups):
    """Per-token (v_emit - version) and per-trajectory (v_emit - v_first) histograms,
    where v_emit is the policy version current when the group was emitted."""
    tok, traj = {}, {}
    for recs, v_emit in groups:
        for r in recs:
            d = v_emit - r["v_first"]
            traj[d] = traj.get(d, 0) + 1
            for v in r["vers"]:
                tok[v_emit - v] = tok.get(v_emit - v, 0) + 1
    return tok, traj


def curriculum_profile(groups_with_epoch):
    """Mean response length of each emitted group, grouped by epoch."""
    prof = {}
    for recs, epoch in groups_with_epoch:
        prof.setdefault(epoch, []).append(sum(r["len"] for r in recs) / len(recs))
    return prof
