"""Seeded Gumbel-max sampler + chosen-token log-probability (fp32 decision).

TEST INFRASTRUCTURE ONLY (oracle/__init__.py).  Follows SURVEY §8(c) O-S:

    u_j  = Philox word (seed; j>>2, n, traj_id, restarts)[j&3] -> (0,1)
    g_j  = -LOG(-LOG(u_j))                    (oracle/logf.py, fp32)
    s_j  = z_j * invT + g_j                   (fp32: one multiply, one add)
    tok  = argmax_j s_j                       (ties -> lowest j)
    lp   = z_tok*invT - (m + log sum_j exp(z_j*invT - m)),  m = max_j z_j*invT

Gumbel-max: argmax_j(z_j/T + Gumbel_j) is a draw from softmax(z/T) (the
Gumbel-max trick), so `tok` is a sample from the policy at temperature T and
`lp` is log pi(tok) — the behaviour log-probability PAPER.md P:180 caches
("the exact log probability value that was used to generate each token").
The token decision is taken in fp32 (the kernel's precision, task rule ③);
`lp` is computed here in fp64 and compared with a tolerance.
"""
from __future__ import annotations

import numpy as np

from .logf import logf
from .philox import bits_to_uniform, sampler_bits


def inv_temperature(T: float) -> np.float32:
    return np.float32(1.0) / np.float32(T)


def gumbel(seed: int, V: int, n: int, traj_id: int, restarts: int) -> np.ndarray:
    u = bits_to_uniform(sampler_bits(seed, np.arange(V), n, traj_id, restarts))
    return -logf(-logf(u))


def truncation_set(zs: np.ndarray, top_k: int = 0, top_p: float = 1.0):
    """The tokens a top-k / top-p (nucleus) sampler may draw from (
    the paper's runs use neither, reading R14).  Candidates are ranked by
    (scaled logit desc, index asc); top-k keeps the first k (k <= 0: all); top-p
    then keeps, of those, the shortest prefix of the ranking whose probability
    under softmax restricted to the top-k set reaches top_p (the token that
    crosses it is included; top_p >= 1: all).  Probabilities in fp64.
    Returns (bool mask [V], cumulative mass just before the last kept token,
    cumulative mass including it) -- the last two say how close the top-p cut was."""
    V = zs.shape[0]
    order = np.lexsort((np.arange(V), -zs.astype(np.float64)))      # zs desc, then index asc
    keep = order if top_k <= 0 else order[:top_k]
    lo = hi = 1.0
    if top_p < 1.0:
        z64 = zs.astype(np.float64)[keep]
        w = np.exp(z64 - z64.max())
        P = w / w.sum()
        c = 0.0
        for i in range(len(keep)):
            lo, c = c, c + P[i]
            if c >= top_p:
                keep = keep[:i + 1]
                break
        hi = c
    mask = np.zeros(V, dtype=bool)
    mask[keep] = True
    return mask, lo, hi


def sample_row(z: np.ndarray, invT: np.float32, seed: int, n: int, traj_id: int, restarts: int,
               top_k: int = 0, top_p: float = 1.0):
    """Return (token, logprob fp64, perturbed scores fp32) for one logits row z (fp32).
    With top_k / top_p the argmax runs over truncation_set only and the logprob is
    that of the truncated, renormalised distribution the token was drawn from
    (the exact probability used to generate it); excluded tokens get score -inf."""
    z = np.asarray(z, dtype=np.float32)
    g = gumbel(seed, z.shape[0], n, traj_id, restarts)
    zs = z * np.float32(invT)
    s = zs + g
    zs64 = zs.astype(np.float64)
    if top_k > 0 or top_p < 1.0:
        mask = truncation_set(zs, top_k, top_p)[0]
        s = np.where(mask, s, np.float32(-np.inf)).astype(np.float32)
        zs64 = np.where(mask, zs64, -np.inf)
    tok = int(np.argmax(s))
    m = zs64.max()
    lse = m + np.log(np.exp(zs64 - m).sum())
    return tok, float(zs64[tok] - lse), s
