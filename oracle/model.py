"""Naive fp64 decoder-only transformer (LLaMA-3.1 / Qwen-2.5 family) with a
per-trajectory KV list.  TEST INFRASTRUCTURE ONLY (oracle/__init__.py).

PAPER.md names the policy families but prints no architecture;
the definition below is the public pre-norm LLaMA/Qwen block (DESIGN.md
readings R19):

    h   = x + Wo . Attn(RoPE(Wq n1(x) + bq), RoPE(Wk n1(x) + bk), Wv n1(x) + bv)
    x'  = h + Wd . (silu(Wg n2(h)) * (Wu n2(h)))
    n(x) = x / sqrt(mean(x^2) + eps) * w
    logits = W_lm . n_f(x_L)

RoPE rotates the pairs (i, i + dh/2) of every head by pos * theta^(-2i/dh)
("rotate_half" convention).  Attention: query head h reads kv head
h // (Hq/Hkv), causal over all cached positions, scale 1/sqrt(dh), softmax.
All arithmetic in float64 on the bf16 weight values (exactly upcast).
"""
from __future__ import annotations

import numpy as np

from workload.configs import ModelShape
from workload.weights import bf16_bits_to_f32, gen_weight_np, weight_names


def load_weights(m: ModelShape, seed: int = 2, version: int = 0, skip=()):
    """Dict name -> float64 array of the version-`version` policy."""
    W = {}
    for name in weight_names(m):
        if name in skip:
            continue
        W[name] = bf16_bits_to_f32(gen_weight_np(m, name, seed, version)).astype(np.float64)
    return W


def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * w


def rope(x: np.ndarray, pos: int, theta: float) -> np.ndarray:
    """x [H, dh] -> rotated copy (rotate_half pairs (i, i+dh/2))."""
    H, dh = x.shape
    half = dh // 2
    i = np.arange(half, dtype=np.float64)
    ang = pos * theta ** (-2.0 * i / dh)
    c, s = np.cos(ang), np.sin(ang)
    a, b = x[:, :half], x[:, half:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=1)


def attention(q: np.ndarray, K: np.ndarray, V: np.ndarray) -> np.ndarray:
    """q [Hq, dh]; K, V [ctx, Hkv, dh] -> o [Hq, dh] (softmax(q K^T / sqrt(dh)) V)."""
    Hq, dh = q.shape
    Hkv = K.shape[1]
    grp = Hq // Hkv
    o = np.empty_like(q)
    for h in range(Hq):
        kv = h // grp
        s = K[:, kv, :] @ q[h] / np.sqrt(dh)
        p = np.exp(s - s.max())
        p /= p.sum()
        o[h] = p @ V[:, kv, :]
    return o


def silu(x):
    return x / (1.0 + np.exp(-x))


def bf16_round(x) -> np.ndarray:
    """x rounded to the nearest bfloat16 value (ties to even), returned as float64.
    bfloat16 is the top 16 bits of an IEEE binary32; x is first rounded to binary32
    (as a GPU kernel holds it), then the low 16 bits are rounded off RNE."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


# Where a bf16 decode path stores values in bf16 (reading R29): the
# normalised activations that feed the projection GEMMs, the RoPE'd query, the
# KV cache (K after RoPE, V), the softmax numerators before the P.V product, the
# attention output (O-projection operand), silu(g)*u (down-projection operand)
# and the final-norm output (LM-head operand).  Everything else stays exact.
STORAGE_POINTS = ("xn", "q", "kv", "p", "o", "act", "xf")


class Model:
    def __init__(self, m: ModelShape, W: dict):
        self.m = m
        self.W = W

    def embed(self, tok: int) -> np.ndarray:
        return self.W["embed"][tok].copy()

    def layer(self, l: int, x: np.ndarray, pos: int, cache_k: list, cache_v: list) -> np.ndarray:
        m, W = self.m, self.W
        p = f"L{l}."
        h = rmsnorm(x, W[p + "attn_norm"], m.rms_eps)
        q = W[p + "wq"] @ h
        k = W[p + "wk"] @ h
        v = W[p + "wv"] @ h
        if m.qkv_bias:
            q = q + W[p + "bq"]
            k = k + W[p + "bk"]
            v = v + W[p + "bv"]
        q = rope(q.reshape(m.Hq, m.dh), pos, m.rope_theta)
        k = rope(k.reshape(m.Hkv, m.dh), pos, m.rope_theta)
        cache_k.append(k)
        cache_v.append(v.reshape(m.Hkv, m.dh))
        o = attention(q, np.stack(cache_k), np.stack(cache_v))
        x = x + W[p + "wo"] @ o.reshape(-1)
        h2 = rmsnorm(x, W[p + "mlp_norm"], m.rms_eps)
        x = x + W[p + "wd"] @ (silu(W[p + "wg"] @ h2) * (W[p + "wu"] @ h2))
        return x

    def hidden(self, x: np.ndarray) -> np.ndarray:
        return rmsnorm(x, self.W["final_norm"], self.m.rms_eps)

    def logits(self, x: np.ndarray) -> np.ndarray:
        return self.W["lm_head"] @ self.hidden(x)

    def decode_token(self, tok: int, pos: int, kv) -> np.ndarray:
        """Process one token at position `pos`, appending to kv[l] = (Klist, Vlist); return final x."""
        x = self.embed(tok)
        for l in range(self.m.L):
            x = self.layer(l, x, pos, kv[l][0], kv[l][1])
        return x

    def new_kv(self):
        return [([], []) for _ in range(self.m.L)]

    def full_forward(self, toks, positions=None, storage_bf16=()) -> np.ndarray:
        """Non-incremental causal forward over a whole sequence; returns logits [T, V]
        (or only the rows `positions`).  Pins the incremental decode (prefill ==
        step-by-step decode).

        storage_bf16: names from STORAGE_POINTS (or True for all of them) at which
        the value is rounded to bf16 (bf16_round) before it is used, exactly where a
        bf16 decode path stores it (reading R29); the softmax denominator sums the
        unrounded numerators.  Default: none -- the plain fp64 definition."""
        m, W = self.m, self.W
        pts = set(STORAGE_POINTS) if storage_bf16 is True else set(storage_bf16)
        assert pts <= set(STORAGE_POINTS), pts

        def r(a, key):
            return bf16_round(a) if key in pts else a
        T = len(toks)
        X = np.stack([self.embed(t) for t in toks])
        for l in range(m.L):
            p = f"L{l}."
            H = r(rmsnorm(X, W[p + "attn_norm"], m.rms_eps), "xn")
            Qm, Km, Vm = H @ W[p + "wq"].T, H @ W[p + "wk"].T, H @ W[p + "wv"].T
            if m.qkv_bias:
                Qm, Km, Vm = Qm + W[p + "bq"], Km + W[p + "bk"], Vm + W[p + "bv"]
            Qr = r(np.stack([rope(Qm[t].reshape(m.Hq, m.dh), t, m.rope_theta) for t in range(T)]), "q")
            Kr = r(np.stack([rope(Km[t].reshape(m.Hkv, m.dh), t, m.rope_theta) for t in range(T)]), "kv")
            Vr = r(Vm.reshape(T, m.Hkv, m.dh), "kv")
            grp = m.Hq // m.Hkv
            O = np.zeros((T, m.Hq, m.dh))
            causal = np.tril(np.ones((T, T), dtype=bool))
            for h in range(m.Hq):
                S = Qr[:, h, :] @ Kr[:, h // grp, :].T / np.sqrt(m.dh)
                S = np.where(causal, S, -np.inf)
                P = np.exp(S - S.max(axis=1, keepdims=True))
                O[:, h, :] = (r(P, "p") @ Vr[:, h // grp, :]) / P.sum(axis=1, keepdims=True)
            X = X + r(O.reshape(T, -1), "o") @ W[p + "wo"].T
            H2 = r(rmsnorm(X, W[p + "mlp_norm"], m.rms_eps), "xn")
            X = X + r(silu(H2 @ W[p + "wg"].T) * (H2 @ W[p + "wu"].T), "act") @ W[p + "wd"].T
        Xf = X if positions is None else X[np.asarray(positions)]
        return r(rmsnorm(Xf, W["final_norm"], m.rms_eps), "xf") @ W["lm_head"].T


class ModelRunner:
    """Couples the model to oracle.sched.Controller: per-trajectory KV lists,
    (re)prefill of prompt + kept tokens on admission, sampling via
    oracle.sampler.  `weights_for(version)` supplies the policy of a version.

    teacher: optional dict traj_id -> list of forced token ids (teacher forcing:
    the oracle consumes those ids instead of its own samples, and records its
    own logits / sample for comparison in `self.log`)."""

    def __init__(self, m: ModelShape, weights_for, prompts, seed: int, temperature: float = 1.0,
                 teacher=None, record_logits=False, top_k: int = 0, top_p: float = 1.0):
        from .sampler import inv_temperature
        self.m = m
        self.top_k, self.top_p = top_k, top_p
        self.weights_for = weights_for
        self.prompts = prompts          # traj -> prompt token list  (callable)
        self.seed = seed
        self.invT = inv_temperature(temperature)
        self.kv = {}
        self.teacher = teacher
        self.record_logits = record_logits
        self.log = []
        self._models = {}
        self.k = 0           # steps served

    def model(self, version):
        if version not in self._models:
            self._models = {version: Model(self.m, self.weights_for(version))}
        return self._models[version]

    def admit(self, t, version):
        self.kv[t.tid] = self.model(version).new_kv()

    def prefill(self, t, a, b, version):
        """KV of positions [.., b) of prompt ++ kept tokens under `version` (the
        controller's chunked prefill, reading R30).  Positions below `a` not yet held
        -- a sample starting after its shared prompt pages (N4) -- are computed here
        too: the shared entry holds the same prompt under the same version."""
        mdl = self.model(version)
        kv = self.kv[t.tid]
        seq = list(self.prompts(t)) + list(t.tokens)
        for pos in range(len(kv[0][0]), b):
            mdl.decode_token(seq[pos], pos, kv)

    def release(self, t):
        self.kv.pop(t.tid, None)

    def step(self, batch, version):
        from .sampler import sample_row
        mdl = self.model(version)
        outs = []
        for g, t in batch:
            prompt = list(self.prompts(t))
            n = len(t.tokens)
            tok_in = t.tokens[-1] if n else prompt[-1]
            pos = len(prompt) + n - 1
            x = mdl.decode_token(tok_in, pos, self.kv[t.tid])
            z = mdl.logits(x).astype(np.float32)
            tok, lp, s = sample_row(z, self.invT, self.seed, n, t.tid, t.restarts, self.top_k, self.top_p)
            if self.record_logits:
                self.log.append(dict(k=self.k, g=g, tid=t.tid, n=n, restarts=t.restarts, logits=z, tok=tok, lp=lp,
                                     scores=s))
            if self.teacher is not None:
                tok = self.teacher[t.tid][n]
            outs.append((tok, lp))
        self.k += 1
        return outs
