"""GPU parity of the learner-side consumer (include/srl_learner.h)
against oracle/learner.py (fp64), on seeded synthetic groups shaped like the
cfg2 update group (U = 64 trajectories, lognormal lengths up to 8192 tokens,
empty trajectories included) and on a real harvested group of the tiny engine.

Tolerances (the kernels compute in fp64 on fp32 inputs, in fixed orders, and
round the result to fp32 once):
* Eq. (3) and Eq. (1) per token: |gpu - oracle| <= 2^-24 |oracle| (the final fp32
  rounding) + 1e-12 (1 + |oracle|) (fp64 summation order);
* Eq. (2): |gpu - oracle| <= 2^-24 |A_t| + 1e-12 S_t, S_t = sum_l (gamma lambda)^l
  |delta_{t+l}| (the chunked affine scan reassociates an fp64 recursion);
* objective: |gpu - oracle| <= 1e-12 mean|term|; branch choices (which tokens are
  clipped) identical; staleness histograms and expansion bit-exact.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.learner import gae_advantages, ppo_terms, reinforcepp_advantages, token_staleness  # noqa: E402
from workload.lengths import LengthModel, sample_lengths  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _group(seed, n=64, cap=8192):
    L = sample_lengths(LengthModel(median=1600, sigma=0.55, tail=0.03, floor=1, cap=cap), seed, n).astype(np.int64)
    L[3] = 0          # an empty trajectory (allowed by the layout)
    L[5] = 1
    off = np.concatenate([[0], np.cumsum(L)]).astype(np.int64)
    return L, off


def test_reinforcepp_parity():
    from paper_2603_23414_b200 import learner
    rng = np.random.default_rng(0)
    for n in (2, 3, 64, 1024, 2048):
        R = rng.normal(0.3, 1.7, size=n).astype(np.float32)
        got = learner.reinforcepp(torch.from_numpy(R).cuda()).cpu().numpy().astype(np.float64)
        ref = reinforcepp_advantages(R.astype(np.float64))
        assert (np.abs(got - ref) <= 2.0 ** -24 * np.abs(ref) + 1e-12 * (1 + np.abs(ref))).all()
    np.testing.assert_array_equal(reinforcepp_advantages([1, 0, 1, 0]),
                                  learner.reinforcepp(torch.tensor([1., 0., 1., 0.], device="cuda")).cpu().numpy())
    z = learner.reinforcepp(torch.full((64,), 0.37, device="cuda")).cpu().numpy()
    assert (z == 0).all()                                        # sigma = 0 -> 0


def test_expand_bit_exact():
    from paper_2603_23414_b200 import learner
    L, off = _group(1)
    v = torch.randn(len(L), device="cuda")
    out = learner.expand(v, torch.from_numpy(off).cuda()).cpu().numpy()
    np.testing.assert_array_equal(out, np.repeat(v.cpu().numpy(), L))


@pytest.mark.parametrize("gamma,lam", [(1.0, 1.0), (0.99, 0.95), (1.0, 0.0), (0.9, 0.7)])
def test_gae_parity_ragged_group(gamma, lam):
    from paper_2603_23414_b200 import learner
    L, off = _group(2)
    rng = np.random.default_rng(3)
    r = rng.normal(size=off[-1]).astype(np.float32)
    r[rng.random(off[-1]) < 0.9] = 0.0                           # sparse, reward-at-the-end style
    V = rng.normal(size=off[-1] + len(L)).astype(np.float32)
    got = learner.gae(torch.from_numpy(r).cuda(), torch.from_numpy(V).cuda(), torch.from_numpy(off).cuda(),
                      gamma, lam).cpu().numpy().astype(np.float64)
    g32, l32 = float(np.float32(gamma)), float(np.float32(lam))
    worst = 0.0
    for i in range(len(L)):
        a, b = off[i], off[i + 1]
        ri, vi = r[a:b].astype(np.float64), V[a + i:b + i + 1].astype(np.float64)
        ref = gae_advantages(ri, vi, g32, l32)
        delta = ri + g32 * vi[1:] - vi[:-1]
        S = gae_advantages(np.abs(delta), np.zeros(len(ri) + 1), 1.0, g32 * l32)   # sum_l c^l |delta_{t+l}|
        err = np.abs(got[a:b] - ref)
        assert (err <= 2.0 ** -24 * np.abs(ref) + 1e-12 * S + 1e-30).all(), i
        if len(ref):
            worst = max(worst, float((err / (2.0 ** -24 * np.abs(ref) + 1e-12 * S + 1e-30)).max()))
    print(f"gae gamma={gamma} lambda={lam}: max err/bound {worst:.3f}")
    # the SPEC example exactly
    one = learner.gae(torch.tensor([1., 0., 2.], device="cuda"), torch.zeros(4, device="cuda"),
                      torch.tensor([0, 3], dtype=torch.int64, device="cuda"), 1.0, 1.0)
    assert one.cpu().tolist() == [3.0, 2.0, 2.0]


def test_ppo_objective_parity():
    from paper_2603_23414_b200 import learner
    L, off = _group(4)
    n = int(off[-1])
    rng = np.random.default_rng(5)
    old = (-rng.exponential(2.0, size=n)).astype(np.float32)
    new = (old + rng.normal(0, 0.3, size=n)).astype(np.float32)    # ratios spread over both clip bounds
    A = np.repeat(rng.normal(size=len(L)), L).astype(np.float32)
    ratio, dterm, obj = learner.ppo_objective(*(torch.from_numpy(x).cuda() for x in (new, old, A)), 0.2, 0.28)
    r_ref, t_ref, g_ref, o_ref = ppo_terms(new.astype(np.float64), old.astype(np.float64), A.astype(np.float64),
                                           float(np.float32(0.2)), float(np.float32(0.28)))
    ratio, dterm = ratio.cpu().numpy().astype(np.float64), dterm.cpu().numpy().astype(np.float64)
    assert (np.abs(ratio - r_ref) <= 2.0 ** -24 * r_ref + 1e-12 * (1 + r_ref)).all()
    assert np.array_equal(dterm == 0, g_ref == 0)                    # the same tokens clipped
    assert (np.abs(dterm - g_ref) <= 2.0 ** -24 * np.abs(g_ref) + 1e-12 * (1 + np.abs(g_ref))).all()
    assert abs(obj.item() - o_ref) <= 1e-12 * np.abs(t_ref).mean()
    assert 0.05 < (g_ref == 0).mean() < 0.95                          # both branches exercised


def test_staleness_bit_exact():
    from paper_2603_23414_b200 import learner
    rng = np.random.default_rng(6)
    ver = rng.integers(0, 40, size=100000).astype(np.int32)
    h = learner.staleness(torch.from_numpy(ver).cuda(), 39, nbins=16).cpu().numpy()
    ref = token_staleness(ver, 39)
    want = np.zeros(16, np.int64)
    for d, c in ref.items():
        want[min(d, 15)] += c
    np.testing.assert_array_equal(h, want)


def test_learner_on_a_harvested_group():
    """End to end on the tiny engine with refreshed policies: the device views of the
    harvested group equal the host harvest bit for bit (tokens, behaviour logprobs,
    versions); the GPU staleness histogram of every group equals the oracle
    controller's; with new = behaviour logprobs every ratio is exactly 1 and the
    objective is the mean advantage."""
    from engine_harness import fill_weights, make_engine, tiny_workload
    from oracle.sched import Controller
    from paper_2603_23414_b200 import learner
    from paper_2603_23414_b200.engine import DONE, GROUP_READY
    from workload.configs import K_INF, KV_BF16, TINY, SchedConfig
    cfg = SchedConfig(Q_g=8, U=4, K=K_INF, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16)
    off, toks, L = tiny_workload(n_prompts=16)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=16)
    eng.submit_prompts(np.arange(16, dtype=np.uint64) + 1000, off, toks, L)
    flat = torch.empty_like(eng.W)
    c = Controller(cfg)
    c.submit_prompts(np.arange(16) + 1000, np.diff(off), L)
    c.load_policy_weights(0)
    og = []
    while True:
        st = c.decode_step()
        if st == 2:
            break
        if st == GROUP_READY:
            og.append((c.harvest(), c.v))
            c.load_policy_weights(c.v + 1)
    v, gi = 0, 0
    while True:
        st, _ = eng.decode_step()
        if st == DONE:
            break
        if st != GROUP_READY:
            continue
        h = eng.harvest_finished(cap_recs=64)
        d = eng.harvest_device()
        assert d["n_records"] == len(h.records) and d["n_tokens"] == len(h.tokens)
        assert np.array_equal(d["tokens"].cpu().numpy(), h.tokens)
        assert np.array_equal(d["logprobs"].cpu().numpy().view(np.int32), h.logprobs.view(np.int32))
        assert np.array_equal(d["versions"].cpu().numpy(), h.versions)
        hist = learner.staleness(d["versions"], v, nbins=8).cpu().numpy()
        recs, v_or = og[gi]
        ref = token_staleness([x for r in recs for x in r["vers"]], v_or)
        assert {k: int(hist[k]) for k in range(8) if hist[k]} == ref
        toff = torch.tensor([0] + [r["tok_offset"] + r["len"] for r in h.records], dtype=torch.int64, device="cuda")
        R = torch.tensor([float(r["len"] % 7) for r in h.records], device="cuda")
        adv = learner.expand(learner.reinforcepp(R), toff)
        ratio, dterm, obj = learner.ppo_objective(d["logprobs"], d["logprobs"], adv, 0.2, 0.28)
        assert (ratio == 1).all()
        assert abs(obj.item() - adv.double().mean().item()) < 1e-12
        v += 1
        gi += 1
        fill_weights(eng, TINY, v, flat=flat)
        eng.load_policy_weights(v, flat)
    eng.close()
    assert gi == len(og) and gi >= 3
