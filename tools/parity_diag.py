"""Diagnostics for the full-width parity bars (test tooling; imports oracle/).

Runs the 8B-width 2-layer engine at Q_g = 256 for a few decode steps, keeps the
GPU logits of two rows, and measures the distance of the GPU logits to the
oracle's bf16-storage-point forward with each storage point left out in turn
(oracle.model.STORAGE_POINTS): the point whose removal brings the GPU closest
is the one the GPU does NOT round like the model.  Also prints the op-level
attention error / derived-bound ratios."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from oracle.model import STORAGE_POINTS, Model  # noqa: E402
from test_gpu_fullwidth import _oracle_weights  # noqa: E402
from workload.configs import K_INF, KV_BF16, LLAMA8B, SchedConfig  # noqa: E402
from workload.prompts import make_prompts  # noqa: E402


def main(m, Q_g, rows):
    from paper_2603_23414_b200.engine import RolloutEngine
    from workload.weights import fill_engine_weights
    steps = 3
    print("==", m.name, "Q_g", Q_g)
    cfg = SchedConfig(Q_g=Q_g, U=Q_g // 4, K=K_INF, pool_prompts=Q_g, cap=8, kv_pages=4 * Q_g, kv_dtype=KV_BF16)
    off, toks = make_prompts(1, Q_g, m.V, 4, 12)
    eng = RolloutEngine(m, cfg, max_traj=Q_g, max_prompt=16, prefill_chunk=4096)
    fill_engine_weights(eng, m, 0)
    eng.load_policy_weights(0)
    eng.submit_prompts(np.arange(Q_g, dtype=np.uint64) + 1, off, toks, np.full(Q_g, 8, np.int32))
    zs, infos = [], []
    for k in range(steps):
        st, info = eng.decode_step()
        infos.append((info.k, info.r_k, info.n_admitted, info.n_prefill_tokens))
        zs.append(eng.debug_logits()[rows].copy())
    tr, _ = eng.trace()
    eng.close()
    print("infos", infos)
    gen = {}
    for kind, a, b, c, d, e in tr:
        pass
    if m.d <= 512:
        from oracle.model import load_weights
        mdl = Model(m, load_weights(m))
    else:
        mdl = Model(m, _oracle_weights(m))
    # generated tokens: sampled ids are recoverable from the GPU logits (bit-exact sampler)
    from oracle.sampler import sample_row
    for j, s in enumerate(rows):
        prompt = [int(t) for t in toks[off[s]:off[s + 1]]]
        g = [sample_row(zs[n][j], np.float32(1.0), cfg.sample_seed, n, s, 0)[0] for n in range(steps)]
        seq = prompt + g[:steps - 1]
        pos = [len(prompt) - 1 + n for n in range(steps)]
        zx = mdl.full_forward(seq, positions=pos)
        ze = mdl.full_forward(seq, positions=pos, storage_bf16=True)
        # the same rounding model on a copy of the weights perturbed by 1e-7 relative:
        # how much of |gpu - emu| a tiny arithmetic difference alone produces
        for n in range(steps):
            nz = np.linalg.norm(zx[n])
            print(f"row {s} n {n}: |gpu-x| {np.linalg.norm(zs[n][j] - zx[n]) / nz:.5f} |emu-x| "
                  f"{np.linalg.norm(ze[n] - zx[n]) / nz:.5f} |gpu-emu| {np.linalg.norm(zs[n][j] - ze[n]) / nz:.5f}",
                  flush=True)
        Wp = dict(mdl.W)
        rng = np.random.default_rng(0)
        for k in list(Wp):
            if k != "embed" and isinstance(Wp[k], np.ndarray):
                Wp[k] = Wp[k] * (1 + 1e-7 * rng.standard_normal(Wp[k].shape))
        zq = Model(m, Wp).full_forward(seq, positions=pos, storage_bf16=True)
        for n in range(steps):
            nz = np.linalg.norm(zx[n])
            print(f"   emu vs emu(weights*(1+1e-7 N(0,1))): {np.linalg.norm(zq[n] - ze[n]) / nz:.5f}", flush=True)


if __name__ == "__main__":
    from workload.configs import TINY
    main(TINY, 16, [0, 5])
    main(LLAMA8B.with_layers(2), 16, [0, 5])
    main(LLAMA8B.with_layers(2), 256, [0, 129])
