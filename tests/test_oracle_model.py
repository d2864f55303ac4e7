"""Pins for oracle/model.py and oracle/attention.py (CPU only)."""
import numpy as np
import pytest

from oracle.attention import paged_attention
from oracle.model import Model, attention, load_weights, rmsnorm, rope
from workload.configs import TINY, ModelShape, QWEN32B
from workload.weights import bf16_bits_to_f32, gen_weight_np


def test_rmsnorm_unit_weight_gives_unit_rms():
    x = np.random.default_rng(0).normal(size=(5, 64)) * 7
    y = rmsnorm(x, np.ones(64), 0.0)
    np.testing.assert_allclose(np.sqrt((y * y).mean(-1)), 1.0, rtol=1e-12)


def test_rope_position_zero_identity_and_norm_preserving():
    x = np.random.default_rng(1).normal(size=(3, 32))
    np.testing.assert_array_equal(rope(x, 0, 1e4), x)
    y = rope(x, 37, 1e4)
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), np.linalg.norm(x, axis=1), rtol=1e-12)


def test_rope_relative_position_property():
    """<RoPE(q, m), RoPE(k, n)> depends only on m - n (the defining property)."""
    rng = np.random.default_rng(2)
    q, k = rng.normal(size=(1, 32)), rng.normal(size=(1, 32))
    a = (rope(q, 10, 1e4) * rope(k, 3, 1e4)).sum()
    b = (rope(q, 107, 1e4) * rope(k, 100, 1e4)).sum()
    assert abs(a - b) < 1e-9


def test_rope_rotate_half_pairs():
    """dims (i, i+dh/2) rotate together by pos * theta^(-2i/dh)."""
    x = np.zeros((1, 8))
    x[0, 1] = 1.0                    # pair (1, 5), frequency theta^(-2/8)
    pos, theta = 3, 100.0
    ang = pos * theta ** (-2.0 / 8)
    y = rope(x, pos, theta)
    np.testing.assert_allclose(y[0, [1, 5]], [np.cos(ang), np.sin(ang)], atol=1e-15)
    assert np.count_nonzero(np.abs(y) > 1e-15) == 2


def test_attention_ctx1_returns_v_and_identical_keys_average():
    rng = np.random.default_rng(3)
    q = rng.normal(size=(4, 16))
    K = rng.normal(size=(1, 2, 16))
    V = rng.normal(size=(1, 2, 16))
    o = attention(q, K, V)
    for h in range(4):
        np.testing.assert_allclose(o[h], V[0, h // 2], rtol=1e-14)
    K = np.repeat(rng.normal(size=(1, 2, 16)), 9, axis=0)
    V = rng.normal(size=(9, 2, 16))
    o = attention(q, K, V)
    for h in range(4):
        np.testing.assert_allclose(o[h], V[:, h // 2].mean(0), rtol=1e-10, atol=1e-15)


def test_attention_brute_force_and_gqa_mapping():
    """Against an explicit double loop with exp/normalise (no vectorised softmax)."""
    rng = np.random.default_rng(4)
    Hq, Hkv, dh, ctx = 6, 2, 8, 7
    q, K, V = rng.normal(size=(Hq, dh)), rng.normal(size=(ctx, Hkv, dh)), rng.normal(size=(ctx, Hkv, dh))
    o = attention(q, K, V)
    for h in range(Hq):
        kv = h // 3
        w = [np.exp(sum(q[h, d] * K[j, kv, d] for d in range(dh)) / np.sqrt(dh)) for j in range(ctx)]
        ref = sum(w[j] * V[j, kv] for j in range(ctx)) / sum(w)
        np.testing.assert_allclose(o[h], ref, rtol=1e-12)


def test_paged_attention_gathers_pages():
    rng = np.random.default_rng(5)
    P, Hkv, T, dh, Hq = 9, 2, 4, 8, 4
    kp, vp = rng.normal(size=(P, Hkv, T, dh)), rng.normal(size=(P, Hkv, T, dh))
    pt = np.array([[7, 2, 5], [1, 0, 8]])
    ctx = np.array([10, 3])
    q = rng.normal(size=(2, Hq, dh))
    o = paged_attention(q, kp, vp, pt, ctx)
    K0 = np.concatenate([kp[7].transpose(1, 0, 2), kp[2].transpose(1, 0, 2), kp[5].transpose(1, 0, 2)])[:10]
    V0 = np.concatenate([vp[7].transpose(1, 0, 2), vp[2].transpose(1, 0, 2), vp[5].transpose(1, 0, 2)])[:10]
    np.testing.assert_allclose(o[0], attention(q[0], K0, V0), rtol=1e-12)


def test_incremental_decode_equals_full_causal_forward():
    m = TINY
    mdl = Model(m, load_weights(m))
    toks = [5, 17, 300, 2, 99, 511, 1]
    full = mdl.full_forward(toks)
    kv = mdl.new_kv()
    for pos, t in enumerate(toks):
        x = mdl.decode_token(t, pos, kv)
        np.testing.assert_allclose(mdl.logits(x), full[pos], rtol=1e-9, atol=1e-12)


def test_incremental_decode_equals_full_forward_with_qkv_bias():
    m = ModelShape("tiny-bias", L=2, d=64, Hq=4, Hkv=2, dh=16, ff=96, V=64, rope_theta=1e6, qkv_bias=True)
    mdl = Model(m, load_weights(m))
    toks = [3, 9, 27, 1, 60]
    full = mdl.full_forward(toks)
    kv = mdl.new_kv()
    for pos, t in enumerate(toks):
        np.testing.assert_allclose(mdl.logits(mdl.decode_token(t, pos, kv)), full[pos], rtol=1e-9, atol=1e-12)


def test_zero_weights_residual_identity():
    m = TINY
    W = load_weights(m)
    for l in range(m.L):
        W[f"L{l}.wo"][:] = 0
        W[f"L{l}.wd"][:] = 0
    mdl = Model(m, W)
    kv = mdl.new_kv()
    x = mdl.decode_token(42, 0, kv)
    np.testing.assert_array_equal(x, W["embed"][42])


def test_weight_generator_recipe():
    """Values follow the documented recipe (bf16 of uniform with std 0.02 / norms near 1)."""
    w = bf16_bits_to_f32(gen_weight_np(TINY, "L0.wq"))
    assert w.shape == (TINY.Hq * TINY.dh, TINY.d)
    assert abs(w.std() - 0.02) < 0.001 and abs(w.mean()) < 0.001
    assert np.abs(w).max() <= 0.02 * np.sqrt(3) * (1 + 2 ** -8)
    n = bf16_bits_to_f32(gen_weight_np(TINY, "L1.mlp_norm"))
    assert (n >= 0.875 - 1e-3).all() and (n <= 1.125 + 1e-3).all()
    rows = gen_weight_np(QWEN32B, "lm_head", rows=[5, 152063])
    full_row = gen_weight_np(QWEN32B, "embed", rows=[5])
    assert rows.shape == (2, QWEN32B.d) and full_row.shape == (1, QWEN32B.d)


def test_weight_generator_numpy_equals_torch():
    torch = pytest.importorskip("torch")
    from workload.weights import gen_weight_torch
    for name in ("L0.wq", "L1.attn_norm", "embed"):
        for version in (0, 3):
            a = gen_weight_np(TINY, name, version=version)
            b = gen_weight_torch(TINY, name, version=version, device="cpu", chunk=1000)
            np.testing.assert_array_equal(a.view(np.int16), b.view(torch.int16).numpy())
    m = ModelShape("b", L=1, d=64, Hq=4, Hkv=2, dh=16, ff=96, V=64, rope_theta=1e6, qkv_bias=True)
    a = gen_weight_np(m, "L0.bk", version=2)
    b = gen_weight_torch(m, "L0.bk", version=2, device="cpu")
    np.testing.assert_array_equal(a.view(np.int16), b.view(torch.int16).numpy())


# ------------------------------------------------------------------ hand-derived pins
def _worked_example():
    import json
    import os
    d = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "model_worked_example.json")))
    m = ModelShape("worked", L=1, d=2, Hq=1, Hkv=1, dh=2, ff=1, V=2, rope_theta=1e4, rms_eps=0.0)
    W = {("L0." + k if k not in ("embed", "final_norm", "lm_head") else k): np.array(v, dtype=np.float64)
         for k, v in d["weights"].items()}
    return d, m, W


def test_model_hand_derived_worked_example():
    """silu on the GATE rows, the up rows as the multiplier, the final RMSNorm applied
    BEFORE the LM head: a 1-layer d=2 block derived by hand (tests/golden).  Each
    plausible misreading gives a logit at least 1e-2 away."""
    d, m, W = _worked_example()
    mdl = Model(m, W)
    x = mdl.decode_token(d["token"], 0, mdl.new_kv())
    z = mdl.logits(x)
    np.testing.assert_allclose(z, d["logits"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(mdl.full_forward([d["token"]])[0], d["logits"], rtol=0, atol=1e-12)
    for name, wrong in d["wrong_readings"].items():
        assert np.abs(np.asarray(wrong) - d["logits"]).max() > 1e-2, name


def test_silu_closed_forms():
    """silu(x) = x * sigmoid(x): silu(0) = 0, sigmoid(ln 3) = 3/4, silu(-x) = silu(x) - x."""
    from oracle.model import silu
    assert silu(0.0) == 0.0
    assert abs(silu(np.log(3.0)) - 0.75 * np.log(3.0)) < 1e-15
    x = np.linspace(-20, 20, 101)
    np.testing.assert_allclose(silu(-x), silu(x) - x, rtol=0, atol=1e-12)
    assert abs(silu(50.0) - 50.0) < 1e-15 and abs(silu(-50.0)) < 1e-18


def test_bf16_round_matches_torch_rne():
    """The storage-point rounding (reading R29) equals torch's float32 -> bfloat16
    conversion (round to nearest, ties to even) on random values, exact ties and
    subnormal / huge magnitudes."""
    import torch
    from oracle.model import bf16_round
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.normal(size=200000) * 10.0 ** rng.uniform(-30, 30, 200000),
                        np.array([1 + 2.0 ** -8, 1 + 3 * 2.0 ** -8, -(1 + 2.0 ** -8), 2.0 ** -130, 3e38, 0.0])])
    x32 = x.astype(np.float32)
    ref = torch.from_numpy(x32).to(torch.bfloat16).float().numpy().astype(np.float64)
    got = bf16_round(x32)
    assert np.array_equal(got, ref)
    assert bf16_round(1 + 2.0 ** -8) == 1.0 and bf16_round(1 + 3 * 2.0 ** -8) == 1 + 2.0 ** -6   # ties to even


def test_storage_rounding_points_each_act_and_positions_subset():
    """Every storage point of the rounding variant is used (each one alone changes the
    logits), none changes them by more than a few bf16 ulps' worth, and `positions`
    returns exactly those rows of the full output."""
    from oracle.model import STORAGE_POINTS
    W = load_weights(TINY)
    mdl = Model(TINY, W)
    toks = [5, 17, 300, 2, 99, 41, 7]
    z = mdl.full_forward(toks)
    np.testing.assert_array_equal(mdl.full_forward(toks, positions=[1, 4, 6]), z[[1, 4, 6]])
    rel = lambda a: np.linalg.norm(a - z, axis=1) / np.linalg.norm(z, axis=1)  # noqa: E731
    for p in STORAGE_POINTS:
        r = rel(mdl.full_forward(toks, storage_bf16=[p]))
        assert r.max() > 0, p
        assert r.max() < 2e-2, (p, r.max())
    r_all = rel(mdl.full_forward(toks, storage_bf16=True))
    assert 1e-4 < r_all.mean() < 2e-2


def test_runner_chunked_prefill_equals_whole_prefill():
    """oracle.model.ModelRunner under the N1 prefill budget (reading R30): with no policy
    update in between, a prompt prefilled in budget-sized chunks over several steps gives
    the same logits, token for token, as the unlimited (whole-prompt) prefill -- the
    incremental decode's KV is position-wise, so the chunking cannot change it -- and the
    schedule differs only in when decoding starts (first tokens later)."""
    import numpy as np
    from oracle.model import ModelRunner, load_weights
    from oracle.sched import Controller
    from workload.configs import TINY, SchedConfig
    plen, L = [40, 25, 33], [5, 4, 6]
    toks = [list(np.random.default_rng(i).integers(1, TINY.V, size=n)) for i, n in enumerate(plen)]
    W = load_weights(TINY)
    logs = []
    for C in (0, 7):
        cfg = SchedConfig(Q_g=3, U=3, pool_prompts=3, cap=8, prefill_budget=C)
        runner = ModelRunner(TINY, lambda v: W, lambda t: toks[t.tid], cfg.sample_seed, record_logits=True)
        c = Controller(cfg, runner)
        c.submit_prompts([1, 2, 3], plen, L)
        c.run()
        logs.append(({(e["tid"], e["n"]): e["logits"] for e in runner.log}, c.trace))
    (a, tr0), (b, tr7) = logs
    assert a.keys() == b.keys() and len(a) == sum(L)
    for key in a:
        assert np.array_equal(a[key], b[key]), key
    assert len(tr7) > len(tr0)                      # decoding starts later under the budget
