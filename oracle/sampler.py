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


def sample_row(z: np.ndarray, invT: np.float32, seed: int, n: int, traj_id: int, restarts: int):
    """Return (token, logprob fp64, perturbed scores fp32) for one logits row z (fp32)."""
    z = np.asarray(z, dtype=np.float32)
    g = gumbel(seed, z.shape[0], n, traj_id, restarts)
    zs = z * np.float32(invT)
    s = zs + g
    tok = int(np.argmax(s))
    zs64 = zs.astype(np.float64)
    m = zs64.max()
    lse = m + np.log(np.exp(zs64 - m).sum())
    return tok, float(zs64[tok] - lse), s
