"""The learner-side consumer of a harvested update group --
plain fp64 definitions.  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

PAPER.md §2 defines what a SortedRL update group feeds:
  Eq. (1) P:59-69  the clipped surrogate objective
        J = E[ min( rho_t A_t, clip(rho_t, 1 - eps, 1 + eps) A_t ) ],
        rho_t = pi_theta(o_t | q, o_<t) / pi_theta_old(o_t | q, o_<t)
      with pi_theta_old the behaviour log-probabilities the rollout cached per
      token ("every token can use the exact log probability value that
      was used to generate each token during importance sampling") and the
      DAPO clip-higher variant ("training tricks from DAPO ... including
      clip-higher"): lower bound 1 - eps_low, upper bound 1 + eps_high
      (SPEC S:393-402);
  Eq. (2) P:74-80  PPO's GAE advantage
        A_t = sum_{l=0}^{T-t-1} (gamma lambda)^l delta_{t+l},
        delta_t = r_t + gamma V(s_{t+1}) - V(s_t),
      evaluated by the backward recursion A_t = delta_t + gamma lambda A_{t+1}
      (values carry the bootstrap V(s_T));
  Eq. (3) P:81-85  Reinforce++'s batch-normalised advantage
        A_i = (R_i - mu_batch) / sigma_batch
      with the population standard deviation; sigma = 0 gives all zeros
      (SPEC S:373-381 degenerate-batch rule); a batch of one is an error.
Staleness: per token, version at the update minus the version
that generated it.
"""
from __future__ import annotations

import math

import numpy as np


class LearnerError(ValueError):
    pass


def reinforcepp_advantages(rewards) -> np.ndarray:
    """Eq. (3): one advantage per trajectory of the batch."""
    R = [float(r) for r in rewards]
    n = len(R)
    if n < 2:
        raise LearnerError("Reinforce++ batch normalisation needs >= 2 trajectories (S:377)")
    mu = sum(R) / n
    var = sum((r - mu) ** 2 for r in R) / n          # population variance
    sigma = math.sqrt(var)
    if sigma == 0.0:
        return np.zeros(n)
    return np.array([(r - mu) / sigma for r in R])


def gae_advantages(rewards, values, gamma: float, lam: float) -> np.ndarray:
    """Eq. (2) for one trajectory: rewards r_0..r_{T-1}, values V(s_0)..V(s_T)."""
    T = len(rewards)
    if len(values) != T + 1:
        raise LearnerError("GAE needs len(values) == len(rewards) + 1 (bootstrap value, S:381)")
    A = np.zeros(T)
    acc = 0.0
    for t in range(T - 1, -1, -1):
        delta = float(rewards[t]) + gamma * float(values[t + 1]) - float(values[t])
        acc = delta + gamma * lam * acc
        A[t] = acc
    return A


def ppo_terms(new_lp, old_lp, adv, eps_low: float, eps_high: float):
    """Eq. (1) per token: (ratio, term, d term / d new_lp) and the objective = mean term.
    The derivative follows the branch min() takes: rho A when the unclipped branch is
    the minimum (ties included), 0 when the clipped constant is."""
    new_lp, old_lp, adv = (np.asarray(x, dtype=np.float64) for x in (new_lp, old_lp, adv))
    if not (len(new_lp) == len(old_lp) == len(adv)):
        raise LearnerError("equal lengths required (S:391)")
    if not (np.isfinite(new_lp).all() and np.isfinite(old_lp).all() and np.isfinite(adv).all()):
        raise LearnerError("non-finite inputs (S:393)")
    ratio = np.empty(len(adv))
    term = np.empty(len(adv))
    grad = np.empty(len(adv))
    for t in range(len(adv)):
        rho = math.exp(new_lp[t] - old_lp[t])
        unclipped = rho * adv[t]
        clipped = min(max(rho, 1.0 - eps_low), 1.0 + eps_high) * adv[t]
        ratio[t] = rho
        if unclipped <= clipped:
            term[t], grad[t] = unclipped, rho * adv[t]
        else:
            term[t], grad[t] = clipped, 0.0
    return ratio, term, grad, (float(term.sum() / len(term)) if len(term) else 0.0)


def token_staleness(versions, v_update: int) -> dict:
    """Histogram over tokens of v_update - generating version."""
    h = {}
    for v in versions:
        d = int(v_update) - int(v)
        h[d] = h.get(d, 0) + 1
    return h
