"""Precision budget of the bf16 decode path at full width (reading R29).

A numpy fp64 forward of a 2-layer LLaMA-3.1-8B-shaped slice (same weights as
the engine, workload/weights.py), run once exactly and once with a bf16
(round-to-nearest-even) rounding at each point where the CUDA path stores a
bf16 value:
  xn   RMSNorm outputs (the QKV / gate-up GEMM activation operands)
  q    the query buffer            kv  the paged KV cache
  p    softmax weights before P.V   o   attention output (O-GEMM operand)
  act  silu(g)*u (down-GEMM operand) xf the final-norm output (LM-head operand)
Prints the logits relative L2 (per position, mean / max) with all roundings and
with each one alone.  Measured (r01): all 0.0083 mean / 0.0097 max; xn 0.0056,
kv 0.0039, o 0.0030, q 0.0023, act 0.0022, xf 0.0017, p 0.0011 -- they add in
quadrature.  Test tooling, not product code: imports oracle helpers.

  python tools/precision_budget.py        (~1 min on 8 cores, ~8 GB RAM)
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.model import rmsnorm, rope, silu  # noqa: E402
from workload.configs import LLAMA8B  # noqa: E402
from workload.prompts import make_prompts  # noqa: E402
from workload.weights import bf16_bits_to_f32, gen_weight_np, weight_names  # noqa: E402

m = LLAMA8B.with_layers(2)


def bf(x):
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def embed(t):
    return bf16_bits_to_f32(gen_weight_np(m, "embed", rows=[int(t)]))[0].astype(np.float64)


def forward(W, toks, emu):
    """emu: False (exact), True (every rounding) or a tuple of rounding-point names."""
    def r(a, k):
        return bf(a) if (emu is True or (emu and k in emu)) else a
    T = len(toks)
    X = np.stack([embed(t) for t in toks])
    f64 = lambda name: W[name].T.astype(np.float64)  # noqa: E731
    for l in range(m.L):
        p = f"L{l}."
        H = r(rmsnorm(X, W[p + "attn_norm"], m.rms_eps), "xn")
        Q, K, V = H @ f64(p + "wq"), H @ f64(p + "wk"), H @ f64(p + "wv")
        Qr = np.stack([rope(Q[t].reshape(m.Hq, m.dh), t, m.rope_theta) for t in range(T)])
        Kr = np.stack([rope(K[t].reshape(m.Hkv, m.dh), t, m.rope_theta) for t in range(T)])
        Qr, Kr, Vr = r(Qr, "q"), r(Kr, "kv"), r(V.reshape(T, m.Hkv, m.dh), "kv")
        g = m.Hq // m.Hkv
        O = np.zeros((T, m.Hq, m.dh))
        for h in range(m.Hq):
            S = Qr[:, h] @ Kr[:, h // g].T / np.sqrt(m.dh)
            S = np.where(np.tril(np.ones((T, T), bool)), S, -np.inf)
            P = np.exp(S - S.max(1, keepdims=True))
            O[:, h] = (r(P, "p") @ Vr[:, h // g]) / P.sum(1, keepdims=True)
        X = X + r(O.reshape(T, -1), "o") @ f64(p + "wo")
        H2 = r(rmsnorm(X, W[p + "mlp_norm"], m.rms_eps), "xn")
        A = r(silu(H2 @ f64(p + "wg")) * (H2 @ f64(p + "wu")), "act")
        X = X + A @ f64(p + "wd")
    Hf = r(rmsnorm(X, W["final_norm"], m.rms_eps), "xf")
    return Hf @ f64("lm_head")


def main():
    t0 = time.time()
    W = {n: bf16_bits_to_f32(gen_weight_np(m, n)).astype(np.float32) for n in weight_names(m) if n != "embed"}
    print(f"weights {time.time() - t0:.0f} s", flush=True)
    off, toks = make_prompts(1, 4, m.V, 4, 12)
    seq = list(toks[off[0]:off[1]]) + [5, 77, 1000, 42, 9]
    z64 = forward(W, seq, False)
    for keys in [True, ("xn",), ("q",), ("kv",), ("p",), ("o",), ("act",), ("xf",)]:
        z = forward(W, seq, keys)
        e = [np.linalg.norm(z[t] - z64[t]) / np.linalg.norm(z64[t]) for t in range(len(seq))]
        print(keys, f"mean {np.mean(e):.4f} max {np.max(e):.4f}", flush=True)


if __name__ == "__main__":
    main()
