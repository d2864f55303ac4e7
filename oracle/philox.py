"""Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
as 1, 2, 3", SC'11) — the counter-based generator SURVEY §8(c) O-S fixes for
the rollout sampler.  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Round function (one of 10), with multipliers M0, M1 and Weyl key increments W0, W1:
    (hi0, lo0) = M0 * c0 ;  (hi1, lo1) = M1 * c2          (32x32 -> 64 bit)
    c' = (hi1 ^ c1 ^ k0,  lo1,  hi0 ^ c3 ^ k1,  lo0)
    k' = (k0 + W0, k1 + W1)                                (between rounds)

Counter/key assignment for the sampler (O-S):
    key = (seed_lo, seed_hi), counter = (j >> 2, n, traj_id, restarts), word j & 3,
    where j is the vocabulary index and n the 0-based index of the generated token.
Uniform: u = float(2*(x >> 9) + 1) * 2^-24, exact in fp32 and inside (0, 1).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
_M32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Vectorised Philox4x32-10.  c* are uint32-valued arrays (broadcastable)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & _M32 for c in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    ka, kb = int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            ka = (ka + W0) & 0xFFFFFFFF
            kb = (kb + W1) & 0xFFFFFFFF
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _M32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _M32
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(ka), lo1, hi0 ^ c3 ^ np.uint64(kb), lo0
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def sampler_bits(seed: int, j: np.ndarray, n: int, traj_id: int, restarts: int) -> np.ndarray:
    """32-bit Philox word for vocabulary indices j of generated token n of a trajectory."""
    j = np.asarray(j, dtype=np.uint64)
    words = philox4x32_10(j >> np.uint64(2), n, traj_id, restarts, seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    w = np.stack(words, axis=0)  # [4, ...]
    sel = (j & np.uint64(3)).astype(np.int64)
    return np.take_along_axis(w, sel[None, ...], axis=0)[0]


def bits_to_uniform(x: np.ndarray) -> np.ndarray:
    """u = float(2*(x>>9)+1) * 2^-24 (exact in fp32, strictly inside (0,1))."""
    x = np.asarray(x, dtype=np.uint32)
    return ((x >> np.uint32(9)).astype(np.float32) * np.float32(2.0) + np.float32(1.0)) * np.float32(2.0 ** -24)
