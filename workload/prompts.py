"""Synthetic prompts: seeded uniform token ids in [1, V).

Prompt lengths follow SURVEY §8(c) reading Q17 (App. A prompts are ~150–300
tokens): a fixed length (256 for the 8B/32B configs) or a
uniform range (U[4,16] for the tiny config).
"""
from __future__ import annotations

import numpy as np

from .lengths import uniform01


def make_prompts(seed: int, n: int, vocab: int, len_lo: int, len_hi: int | None = None):
    """Return (tok_off[n+1] int32, toks[int32]) for n prompts.

    len_hi None -> every prompt has len_lo tokens; else lengths ~ U[len_lo, len_hi].
    """
    idx = np.arange(n, dtype=np.uint64)
    if len_hi is None or len_hi == len_lo:
        lens = np.full(n, len_lo, dtype=np.int64)
    else:
        u = uniform01(seed, 7, idx)
        lens = len_lo + np.floor(u * (len_hi - len_lo + 1)).astype(np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    tot = int(off[-1])
    u = uniform01(seed, 8, np.arange(tot, dtype=np.uint64))
    toks = 1 + np.floor(u * (vocab - 1)).astype(np.int64)
    return off.astype(np.int32), toks.astype(np.int32)
