"""Compact weights (srl_model_cfg.weights_compact; include/srl.h): projection
matrices held only in the GEMM's packed layout, installed tensor by tensor with
srl_load_policy_tensor.  The packed bytes must equal those the staging path
produces, so a compact engine and a staging engine fed the same policy emit
bit-identical logits, tokens and logprobs, step by step -- including across a
policy refresh (version 1 weights) -- and the same schedule as the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from engine_harness import tiny_workload  # noqa: E402
from oracle.sched import Controller  # noqa: E402
from workload.configs import K_INF, KV_BF16, ModelShape, SchedConfig  # noqa: E402
from workload.weights import fill_engine_weights  # noqa: E402

# TINY with dh = 64 so q / k / v each cover whole 128-row tiles (compact_ok)
TINY64 = ModelShape("tiny64", L=2, d=128, Hq=4, Hkv=2, dh=64, ff=384, V=512, rope_theta=1e4, qkv_bias=True)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _install_by_tensor(eng, v):
    """srl_load_policy_tensor for every tensor (plain row-major sources), on an engine
    WITH a staging image: that image must come out in its own layout (wg / wu
    interleaved), because srl_load_policy_weights(NULL) re-packs from it."""
    from workload.weights import gen_weight_torch, weight_names
    for name in weight_names(TINY64):
        t = gen_weight_torch(TINY64, name, version=v, device=eng.W.device)
        eng.load_policy_tensor(name, t)
        eng.stream.synchronize()


def _run(compact, cfg, off, toks, L, by_tensor=False):
    from paper_2603_23414_b200.engine import DONE, GROUP_READY, RolloutEngine, events_to_oracle_form
    eng = RolloutEngine(TINY64, cfg, max_traj=64, max_prompt=16, prefill_chunk=256, compact_weights=compact)
    install = (lambda e, v: _install_by_tensor(e, v)) if by_tensor else (lambda e, v: fill_engine_weights(e, TINY64, v))
    install(eng, 0)
    eng.load_policy_weights(0)
    eng.submit_prompts(np.arange(len(off) - 1, dtype=np.uint64) + 1000, off, toks, L)
    logits, groups, v = [], [], 0
    while True:
        st, info = eng.decode_step()
        if st == DONE:
            break
        if info.k >= 0:
            logits.append(eng.debug_logits())
        if st == GROUP_READY:
            groups.append(eng.harvest_finished(cap_recs=64))
            v += 1
            install(eng, v)                         # a refreshed policy, installed the engine's way
            eng.load_policy_weights(v)
    ev, steps = events_to_oracle_form(eng.trace()[0])
    eng.close()
    return logits, groups, ev, steps


def test_compact_weights_bit_identical_to_staging_path():
    cfg = SchedConfig(Q_g=16, U=4, K=K_INF, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16)
    off, toks, L = tiny_workload(n_prompts=16)
    za, ga, eva, sa = _run(False, cfg, off, toks, L)
    zb, gb, evb, sb = _run(True, cfg, off, toks, L)
    assert eva == evb and sa == sb and len(za) == len(zb)
    for x, y in zip(za, zb):
        assert np.array_equal(x.view(np.int32), y.view(np.int32))
    for a, b in zip(ga, gb):
        assert np.array_equal(a.tokens, b.tokens) and np.array_equal(a.logprobs.view(np.int32), b.logprobs.view(np.int32))
    c = Controller(cfg)
    c.submit_prompts(np.arange(16) + 1000, np.diff(off), L)
    c.run()
    assert evb == c.events and sb == c.trace


def test_tensor_install_on_staging_engine_bit_identical():
    """srl_load_policy_tensor on a NON-compact engine must scatter
    wg / wu into the interleaved staging rows; srl_load_policy_weights(NULL) then
    re-packs from that image.  Same logits / tokens / logprobs bit for bit as the
    staging path, across policy refreshes."""
    cfg = SchedConfig(Q_g=16, U=4, K=K_INF, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16)
    off, toks, L = tiny_workload(n_prompts=16)
    za, ga, eva, sa = _run(False, cfg, off, toks, L)
    zb, gb, evb, sb = _run(False, cfg, off, toks, L, by_tensor=True)
    assert eva == evb and sa == sb and len(za) == len(zb)
    for x, y in zip(za, zb):
        assert np.array_equal(x.view(np.int32), y.view(np.int32))
    for a, b in zip(ga, gb):
        assert np.array_equal(a.tokens, b.tokens) and np.array_equal(a.logprobs.view(np.int32), b.logprobs.view(np.int32))


def test_compact_rejects_staging_calls():
    from paper_2603_23414_b200._lib import SRLError
    from paper_2603_23414_b200.engine import RolloutEngine
    cfg = SchedConfig(Q_g=4, U=2, pool_prompts=4, cap=8, kv_pages=32)
    eng = RolloutEngine(TINY64, cfg, max_traj=16, max_prompt=16, compact_weights=True)
    with pytest.raises(KeyError):
        eng.weight_view("L0.wq")
    eng.weight_view("L0.attn_norm")                 # non-packed tensors keep their staging storage
    with pytest.raises(SRLError):
        eng.load_policy_weights(0, torch.zeros(16, dtype=torch.uint8, device="cuda"))
    with pytest.raises(SRLError):
        eng.load_policy_tensor("nope", torch.zeros(16, dtype=torch.bfloat16, device="cuda"))
    eng.close()
