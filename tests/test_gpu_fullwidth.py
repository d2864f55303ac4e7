"""Full-width parity: LLaMA-3.1-8B- and Qwen-2.5-32B-shaped policies (2-layer
slices at full width, SURVEY §8(c) "shape-faithful shallow slices") through the
C ABI with the launch configurations bench.py times (the GEMM picks its split
from M, N, K only; attention its split-KV plan from rows x kv heads).

Per checked (row, generated index n) -- teacher forcing on the GPU's own tokens,
oracle.model.Model.full_forward in fp64 (pinned against incremental decode and
a hand-derived example in test_oracle_model.py) -- two oracle logits vectors at
exactly that position:
  z_x  the plain fp64 definition,
  z_e  the same forward with bf16 rounding at the path's storage points
       (oracle.model.STORAGE_POINTS, reading R29).
z_e is one realisation of the rounding process the bf16 path runs: at 8B width
a 1e-7 relative perturbation of the weights (sub-ulp arithmetic differences,
like fp32 vs fp64 accumulation order) re-draws enough roundings to move z_e by
0.35-0.6% relative, as far as the GPU is from z_e (tools/parity_diag.py, r02).
So the GPU logits are another realisation of the same process, and the bars are:
* per position  rel(z_gpu, z_x) <= 1.2 rel(z_e, z_x): the GPU's deviation from
  the exact definition is the size the storage roundings produce AT THAT
  POSITION (measured ratio 0.96-1.04 over 12 positions at 8B width: the
  relative L2 of a 128k-long error vector concentrates) -- the per-position
  derived bound VERDICT r1 asked for, replacing the round-1 "mean <= 1e-2,
  max <= 1.5e-2" reading R29;
* per position  rel(z_gpu, z_e) <= rel(z_e, z_x): the GPU follows the rounding
  model more closely than the model follows exact arithmetic (a missing or
  extra rounding point would break this);
* the mean of rel(z_gpu, z_x) over checked positions <= 1e-2 (north star) in the
  batch tests; at 0.3-4k contexts the storage roundings alone exceed it (z_e
  ~1.1e-2), so there the per-position bound is the bar;
* sampled ids: the oracle's Gumbel-max on the GPU logits equals the GPU's token
  (bit-exact sampler); and at EVERY position (no near-tie exclusions) the GPU's
  token scores within 2 max|z_gpu - z_x| / T of the best perturbed score under
  the exact logits (same Gumbel noise) -- how often it is the oracle's own draw
  is reported;  behaviour logprobs within 4x max|z_gpu - z_x| + 1e-4 of the
  exact ones.

Weights: the workload generator's torch implementation (bit-identical to its
numpy one, pinned in test_oracle_model.py) evaluated on the GPU and copied to
host; the embedding table is never materialised (rows on demand).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.model import Model  # noqa: E402
from oracle.sampler import sample_row  # noqa: E402
from workload.configs import K_INF, KV_BF16, LLAMA8B, QWEN32B, SchedConfig  # noqa: E402
from workload.prompts import make_prompts  # noqa: E402
from workload.weights import bf16_bits_to_f32, gen_weight_np, gen_weight_torch, weight_names  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


class _EmbedRows:
    """W["embed"] stand-in: row `tok` generated on demand (fp64)."""

    def __init__(self, m):
        self.m = m

    def __getitem__(self, tok):
        return bf16_bits_to_f32(gen_weight_np(self.m, "embed", rows=[int(tok)]))[0].astype(np.float64)


def _oracle_weights(m):
    W = {"embed": _EmbedRows(m)}
    for name in weight_names(m):
        if name == "embed":
            continue
        t = gen_weight_torch(m, name, device="cuda")
        W[name] = t.float().cpu().numpy().astype(np.float64)
        del t
    return W


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def check_positions(mdl, cases, seed, invT=np.float32(1.0), label="", mean_bar=1e-2):
    """cases: list of (traj_id, prompt tokens, generated tokens, behaviour logprobs,
    {n: gpu logits row}).  Applies the bars of the module docstring at every n."""
    stats = dict(rel_x=[], rel_e=[], rel_ex=[], ratio=[], checked=0, violations=[])
    for tid, prompt, gen, lps, zg_by_n in cases:
        ns = sorted(zg_by_n)
        seq = list(prompt) + list(gen[:max(ns)])
        pos = [len(prompt) - 1 + n for n in ns]
        zx = mdl.full_forward(seq, positions=pos)
        ze = mdl.full_forward(seq, positions=pos, storage_bf16=True)
        for i, n in enumerate(ns):
            zg = zg_by_n[n].astype(np.float64)
            # bit-exact sampler on identical logits
            assert sample_row(zg_by_n[n], invT, seed, n, tid, 0)[0] == gen[n], (tid, n)
            rx, rex, rge = _rel(zg, zx[i]), _rel(ze[i], zx[i]), _rel(zg, ze[i])
            if rx > 1.2 * rex or rge > rex:
                stats["violations"].append((tid, n, round(rx, 5), round(rex, 5), round(rge, 5)))
            stats["rel_x"].append(rx)
            stats["rel_e"].append(rge)
            stats["ratio"].append(rx / rex)
            stats["rel_ex"].append(rex)
            err_x = float(np.abs(zg - zx[i]).max())
            tok_x, _, sc = sample_row(zx[i].astype(np.float32), invT, seed, n, tid, 0)
            # every position decided: the GPU's token maximises ITS perturbed scores, which
            # are within err_x * invT of the oracle's, so under the oracle's exact scores it
            # must be within 2 err_x * invT of the best (Gumbel noise identical on both sides)
            sc = sc.astype(np.float64)
            stats["checked"] += 1
            stats["agree"] = stats.get("agree", 0) + int(tok_x == gen[n])
            if sc[gen[n]] < sc.max() - 2 * err_x * float(invT) - 1e-6:
                stats["violations"].append((tid, n, "token", tok_x, gen[n], float(sc.max() - sc[gen[n]]), err_x))
            # the GPU's behaviour logprob is log-softmax of ITS logits at ITS token; the
            # exact one at the same token differs by at most 2 max|dz|
            lse = zx[i].max() + np.log(np.exp(zx[i] - zx[i].max()).sum())
            if abs(lps[n] - (zx[i][gen[n]] - lse)) > 4 * err_x + 1e-4:
                stats["violations"].append((tid, n, "logprob", lps[n], zx[i][gen[n]] - lse))
    rx = np.array(stats["rel_x"])
    print(f"{label}: rel-L2 vs exact mean {rx.mean():.2e} max {rx.max():.2e} (the bf16-storage model's own: mean "
          f"{np.mean(stats['rel_ex']):.2e} max {np.max(stats['rel_ex']):.2e}); ratio to the model's own "
          f"min {min(stats['ratio']):.3f} max {max(stats['ratio']):.3f}; vs the storage model mean "
          f"{np.mean(stats['rel_e']):.2e} max {np.max(stats['rel_e']):.2e}; ids checked {stats['checked']}, equal to "
          f"the oracle's own draw {stats.get('agree', 0)}; violations (tid, n, rel_x, rel_e_x, rel_gpu_e) {stats['violations']}",
          flush=True)
    assert not stats["violations"], stats["violations"]
    if mean_bar is not None:
        assert rx.mean() <= mean_bar
    return stats


STEPS = 6


def _drain(eng, Q_g):
    """Run to the end; every trajectory's tokens + behaviour logprobs from the groups."""
    gpu_tok, gpu_lp, v = {}, {}, 0
    while True:
        st, _ = eng.decode_step()
        if st == 2:
            break
        if st == 1:
            h = eng.harvest_finished(cap_recs=Q_g * 4)
            for r in h.records:
                seg = slice(r["tok_offset"], r["tok_offset"] + r["len"])
                gpu_tok[r["traj_id"]], gpu_lp[r["traj_id"]] = h.tokens[seg].tolist(), h.logprobs[seg].tolist()
            v += 1
            eng.load_policy_weights(v)
    return gpu_tok, gpu_lp


@pytest.mark.parametrize("shape,Q_g", [(LLAMA8B, 256), (QWEN32B, 64)], ids=["llama8b-L2-Q256", "qwen32b-L2-Q64"])
def test_fullwidth_teacher_forced(shape, Q_g):
    """The benchmark's batch (Q_g = 256 / 64 rows, the pair / single-CTA GEMM paths
    with their split-K decompositions), short prompts, 6 decode steps."""
    from paper_2603_23414_b200.engine import RolloutEngine
    from workload.weights import fill_engine_weights
    m = shape.with_layers(2)
    cap = STEPS + 2
    cfg = SchedConfig(Q_g=Q_g, U=Q_g // 4, K=K_INF, pool_prompts=Q_g, cap=cap, kv_pages=4 * Q_g, kv_dtype=KV_BF16)
    off, toks = make_prompts(1, Q_g, m.V, 4, 12)
    L = np.full(Q_g, cap, dtype=np.int32)              # nobody finishes inside the checked window
    eng = RolloutEngine(m, cfg, max_traj=Q_g, max_prompt=16, prefill_chunk=4096)
    fill_engine_weights(eng, m, 0)
    eng.load_policy_weights(0)
    eng.submit_prompts(np.arange(Q_g, dtype=np.uint64) + 1, off, toks, L)
    rows = sorted({0, 1, Q_g // 3, Q_g // 2 + 1, Q_g - 2, Q_g - 1})
    zs = []                                            # [step][row] fp32 logits
    for k in range(STEPS):
        st, info = eng.decode_step()
        assert info.k == k and info.r_k == Q_g          # pool = Q_g: slot s holds trajectory s
        z = eng.debug_logits()
        zs.append(z[rows].copy())
        del z
    gpu_tok, gpu_lp = _drain(eng, Q_g)
    eng.close()
    torch.cuda.empty_cache()
    assert sorted(gpu_tok) == list(range(Q_g)) and all(len(t) == cap for t in gpu_tok.values())
    mdl = Model(m, _oracle_weights(m))
    cases = [(s, [int(t) for t in toks[off[s]:off[s + 1]]], gpu_tok[s], gpu_lp[s], {n: zs[n][j] for n in range(STEPS)})
             for j, s in enumerate(rows)]
    st = check_positions(mdl, cases, cfg.sample_seed, label=m.name)


def test_fullwidth_long_context_split_kv_and_mixed_pass():
    """LLaMA-8B width, prefilled contexts of 0.3-4k tokens over 8 slots: the epoch-start
    prompts (10k tokens) run as separate prefill passes in 4096-row chunks (a prompt
    split across chunks attends to its earlier chunk through the page table); the
    decode steps run the 16-row bucket (graph-replayed from its second use) with
    split-KV attention (8 rows x 8 kv heads = 64 pairs < 148 SMs) in longest-first
    order; two trajectories finish early and the two remaining prompts are admitted
    in MIXED passes (their prompt rows ride in the decode forward).  Checked rows:
    the longest prompt, a 2k one, a short one, and a mixed-pass admission."""
    from paper_2603_23414_b200.engine import DONE, GROUP_READY, RolloutEngine
    from workload.weights import fill_engine_weights
    m = LLAMA8B.with_layers(2)
    plens = [4000, 2000, 700, 300, 1500, 64, 900, 500, 1200, 350]    # 8 slots, then 2 admitted later
    forced = [14, 14, 3, 14, 14, 5, 14, 14, 9, 9]
    n = len(plens)
    rng = np.random.default_rng(11)
    toks = [rng.integers(1, m.V, size=p).astype(np.int32) for p in plens]
    off = np.concatenate([[0], np.cumsum(plens)]).astype(np.int32)
    cfg = SchedConfig(Q_g=8, U=2, K=K_INF, pool_prompts=n, cap=16, kv_pages=260, kv_dtype=KV_BF16)
    eng = RolloutEngine(m, cfg, max_traj=n, max_prompt=4096, prefill_chunk=4096)
    fill_engine_weights(eng, m, 0)
    eng.load_policy_weights(0)
    eng.submit_prompts(np.arange(n, dtype=np.uint64) + 1, off, np.concatenate(toks), np.array(forced, np.int32))
    check_tids = [0, 1, 3, 8]
    slot_of, zrec = {}, {t: {} for t in check_tids}
    ntok = {t: 0 for t in range(n)}
    infos = []
    v = 0
    gpu_tok, gpu_lp = {}, {}
    while True:
        st, info = eng.decode_step()
        if st == DONE:
            break
        if info.k >= 0:
            infos.append(info)
            tr, _ = eng.trace()
            for kind, _k, slot, tid, _kept, _ in tr:
                if kind == 2:                        # ADMIT (srl.h SRL_EV_ADMIT): a=k, b=slot, c=traj
                    slot_of[tid] = slot
            z = eng.debug_logits()
            for t in check_tids:
                s = slot_of.get(t)
                if s is not None and ntok[t] < forced[t] and not np.isnan(z[s]).any():
                    zrec[t][ntok[t]] = z[s].copy()
            for t, s in list(slot_of.items()):
                if ntok[t] < forced[t]:
                    ntok[t] += 1
            del z
        if st == GROUP_READY:
            h = eng.harvest_finished(cap_recs=16)
            for r in h.records:
                seg = slice(r["tok_offset"], r["tok_offset"] + r["len"])
                gpu_tok[r["traj_id"]], gpu_lp[r["traj_id"]] = h.tokens[seg].tolist(), h.logprobs[seg].tolist()
            v += 1
            eng.load_policy_weights(v)
    eng.close()
    torch.cuda.empty_cache()
    assert sorted(gpu_tok) == list(range(n))
    assert [len(gpu_tok[t]) for t in range(n)] == forced
    # prefill rows = prompt tokens before the last one (that one is the admission's first decode row)
    assert any(i.n_prefill_tokens == plens[8] - 1 and i.n_admitted == 1 for i in infos), \
        [(i.k, i.n_admitted, i.n_prefill_tokens) for i in infos]                    # the mixed pass ran
    assert infos[0].n_prefill_tokens == sum(plens[:8]) - 8                           # chunked epoch-start prefill
    for t in check_tids:
        assert sorted(zrec[t]) == list(range(forced[t])), (t, sorted(zrec[t]))
    mdl = Model(m, _oracle_weights(m))
    cases = [(t, toks[t].tolist(), gpu_tok[t], gpu_lp[t], zrec[t]) for t in check_tids]
    # the north-star mean <= 1e-2 is not applied here: at 0.3-4k contexts the bf16 storage
    # roundings ALONE cost ~1.1e-2 mean rel-L2 (z_e vs z_x, measured r02); the per-position
    # derived bound above is the bar (R29)
    st = check_positions(mdl, cases, cfg.sample_seed, label="llama8b-L2 long context", mean_bar=None)
    assert np.mean(st["rel_x"]) <= 1.2 * np.mean(st["rel_ex"])


def test_fullwidth_qkv_finish_path():
    """The opt-in QKV handoff (srl_tuning.qkv_finish: split-K partials + the bias / RoPE /
    KV-append kernel) passes the same full-width parity test.  Subprocess: the
    test harness applies the setting at session start (tests/conftest.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SRL_TEST_TUNING="qkv_finish=1,qkv_attn=0")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                          "tests/test_gpu_fullwidth.py::test_fullwidth_teacher_forced[llama8b-L2-Q256]"],
                         cwd=root, capture_output=True, text=True, env=env, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]


def test_fullwidth_fused_kernel_paths():
    """The other kernel chain (srl_tuning qkv_attn = 0: bias, RoPE and the KV append in the
    QKV GEMM's own epilogue after its cluster split-K reduction; fuse_mlp = 1: gate/up and
    down as one persistent kernel) passes the same full-width parity test.  Subprocess:
    settings are applied at session start (tests/conftest.py)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SRL_TEST_TUNING="qkv_attn=0,fuse_mlp=1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                          "tests/test_gpu_fullwidth.py::test_fullwidth_teacher_forced[llama8b-L2-Q256]"],
                         cwd=root, capture_output=True, text=True, env=env, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
