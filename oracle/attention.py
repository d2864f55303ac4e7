"""Brute-force paged decode attention (fp64).  TEST INFRASTRUCTURE ONLY.

Definition: for each query row r (a sequence at
position pos_r) and query head h, with kv head h // (Hq/Hkv):
    o[r, h] = softmax_j( q[r,h] . K[j] / sqrt(dh) ) V[j],  j = 0 .. ctx_r - 1
where token j of the sequence lives at page pt[r][j // page], row j % page
of the paged pool pool[page, Hkv, page_tokens, dh] (PagedAttention).
"""
from __future__ import annotations

import numpy as np

from .model import attention


def gather_paged(pool: np.ndarray, page_row: np.ndarray, ctx: int) -> np.ndarray:
    """pool [P, Hkv, T, dh], page_row [n_pages] -> dense [ctx, Hkv, dh]."""
    T = pool.shape[2]
    out = np.empty((ctx, pool.shape[1], pool.shape[3]), dtype=np.float64)
    for j in range(ctx):
        out[j] = pool[page_row[j // T], :, j % T, :]
    return out


def paged_attention(q: np.ndarray, k_pool: np.ndarray, v_pool: np.ndarray, page_table: np.ndarray,
                    ctx: np.ndarray) -> np.ndarray:
    """q [R, Hq, dh]; page_table [R, max_pages]; ctx [R] -> o [R, Hq, dh] (fp64)."""
    R = q.shape[0]
    o = np.zeros(q.shape, dtype=np.float64)
    for r in range(R):
        if ctx[r] <= 0:
            continue
        K = gather_paged(k_pool, page_table[r], int(ctx[r]))
        V = gather_paged(v_pool, page_table[r], int(ctx[r]))
        o[r] = attention(q[r].astype(np.float64), K, V)
    return o
