"""Long-tailed response-length targets (FORCED stop lengths).

Calibrated to PAPER.md P:114 §2.3 ("while 80% of samples are generated within
3K tokens, the remaining 5% can extend up to the token limit") and used for
P:336's "sampling parameters ... let generation lengths be exactly the same
as baseline".  Recipe (reading R18):

    with probability `tail`:  L = cap
    otherwise:                L = clamp(rint(exp(ln(median) + sigma * Phi^-1(u))), floor, cap)

Inverse-CDF sampling from an explicit counter-based uniform stream, so that
raising `cap` never lowers a sample drawn from the same uniforms.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import ndtri

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def uniform01(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based uniforms in (0, 1) with 53-bit resolution."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = splitmix64(np.array([seed * 1000003 + stream], dtype=np.uint64))[0]
        h = splitmix64(idx ^ key)
    return ((h >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


@dataclass(frozen=True)
class LengthModel:
    median: float = 1600.0
    sigma: float = 0.55
    tail: float = 0.03
    floor: int = 1
    cap: int = 8192

    def __post_init__(self):
        if self.sigma < 0 or self.floor < 1 or self.floor > self.cap or not (0.0 <= self.tail <= 1.0):
            raise ValueError(f"invalid LengthModel {self}")


def sample_lengths(model: LengthModel, seed: int, n: int, offset: int = 0) -> np.ndarray:
    """n int32 lengths in [floor, cap] for trajectory indices offset..offset+n-1."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    u_tail = uniform01(seed, 0, idx)
    u_body = uniform01(seed, 1, idx)
    body = np.exp(np.log(model.median) + model.sigma * ndtri(u_body))
    body = np.clip(np.rint(body), model.floor, model.cap)
    out = np.where(u_tail < model.tail, model.cap, body)
    return out.astype(np.int32)
