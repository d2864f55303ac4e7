"""N1 on the GPU: per-step chunked prefill under a token budget
(srl_sched_cfg.prefill_budget; SURVEY §8(f) N1, P:32 Sarathi, P:180 prompt ++
kept tokens re-fed on resume; reading R30) against oracle/sched.py `_prefill`.

* scheduling: event log + (k, r_k) trace + groups BIT-EXACT, and this GPU's
  prefill tokens of every step equal the oracle's prefill_trace -- including
  REPREFILL resumes (whole prompt ++ kept tokens re-fed in chunks), preemption
  of a slot mid-prefill, K = 0 discards and steps where no slot decodes;
* model: teacher-forced logits within rel-L2 1e-2 of the fp64 oracle, whose
  ModelRunner prefills the same chunks under the version current at each step
  (a prompt prefilled across a policy update holds KV of two versions, KEEP_KV);
* replicas: R = 2 lockstep engines (in-process transport) with per-replica
  budgets, bit-exact against the R = 2 oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from engine_harness import make_engine, run_engine, tiny_workload  # noqa: E402
from oracle.model import ModelRunner, load_weights  # noqa: E402
from oracle.sampler import sample_row  # noqa: E402
from test_gpu_engine import _compare_schedule, _oracle  # noqa: E402
from workload.configs import K_INF, KV_BF16, KV_FP32, MODE_SYNC, RESUME_REPREFILL, TINY, SchedConfig  # noqa: E402
from workload.lengths import LengthModel  # noqa: E402

MAXP = 120


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _workload(n_prompts, cap=64, median=16, plen=(8, MAXP)):
    lm = LengthModel(median=median, sigma=0.6, tail=0.2, floor=1, cap=cap)
    return tiny_workload(n_prompts=n_prompts, cap=cap, lm=lm, plen=plen)


def _compare_prefill(res, c, rank=0):
    got = [(i.k, i.n_prefill_tokens) for i in res["infos"]]
    want = [(k, pre[rank]) for k, pre in c.prefill_trace]
    assert got == want


CASES = [
    ("C64", dict(prefill_budget=64)),
    ("C7", dict(prefill_budget=7)),
    ("C1", dict(prefill_budget=1, Q_g=4, pool_prompts=8)),
    ("C200_K1_reprefill", dict(prefill_budget=200, K=1, resume=RESUME_REPREFILL)),
    ("C50_Kinf_reprefill", dict(prefill_budget=50, K=K_INF, resume=RESUME_REPREFILL)),
    ("C40_K0", dict(prefill_budget=40, K=0)),
    ("C30_preempt", dict(prefill_budget=30, K=1, kv_pages=6, Q_g=8)),
    ("C100_sync", dict(prefill_budget=100, mode=MODE_SYNC, Q_g=8)),
    ("C0", dict(prefill_budget=0)),
]


@pytest.mark.parametrize("name,over", CASES, ids=[c[0] for c in CASES])
def test_prefill_budget_schedule_bit_exact(name, over):
    base = dict(Q_g=16, U=4, K=K_INF, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16)
    base.update(over)
    cfg = SchedConfig(**base)
    off, toks, L = _workload(16, cap=cfg.cap)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=MAXP)
    res = run_engine(eng, TINY, off, toks, L)
    eng.close()
    c, og = _oracle(cfg, off, toks, L)
    _compare_schedule(res, c, og)
    _compare_prefill(res, c)


@pytest.mark.parametrize("kv,over", [(KV_FP32, dict(prefill_budget=48, K=K_INF)),
                                     (KV_BF16, dict(prefill_budget=100, K=K_INF, resume=RESUME_REPREFILL)),
                                     (KV_BF16, dict(prefill_budget=13, K=K_INF, U=2))],
                         ids=["f32-C48", "bf16-C100-reprefill", "bf16-C13-U2"])
def test_prefill_budget_teacher_forced_logits(kv, over):
    """K = inf (no token is ever dropped: the harvested tokens are the ones every step
    sampled, so they teacher-force the oracle).  REPREFILL re-feeds prompt ++ kept tokens
    in budget-sized chunks after every update; KEEP_KV prefills cross updates."""
    cfg = SchedConfig(**{**dict(Q_g=8, U=4, pool_prompts=8, cap=48, kv_pages=256, kv_dtype=kv), **over})
    off, toks, L = _workload(8, cap=cfg.cap, median=12)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=MAXP)
    res = run_engine(eng, TINY, off, toks, L, record_logits=True)
    eng.close()
    teacher = {}
    for h, _ in res["groups"]:
        for r in h.records:
            teacher[r["traj_id"]] = h.tokens[r["tok_offset"]:r["tok_offset"] + r["len"]].tolist()
    prompts = lambda t: toks[off[t.tid]:off[t.tid + 1]]  # noqa: E731
    runner = ModelRunner(TINY, lambda v: load_weights(TINY, version=v), prompts, cfg.sample_seed,
                         teacher=teacher, record_logits=True)
    c, og = _oracle(cfg, off, toks, L, runner)
    _compare_schedule(res, c, og)
    _compare_prefill(res, c)
    worst = 0.0
    for e in runner.log:
        zg = res["logits"][e["k"]][e["g"]]
        zo = e["logits"].astype(np.float64)
        rel = np.linalg.norm(zg - zo) / np.linalg.norm(zo)
        worst = max(worst, rel)
        assert rel <= 1e-2, (e["k"], e["g"], e["tid"], rel)
        assert sample_row(zg, np.float32(1.0), cfg.sample_seed, e["n"], e["tid"], e["restarts"])[0] == \
            teacher[e["tid"]][e["n"]]
    assert len(runner.log) > 100
    print(f"worst logits rel-L2 {worst:.2e} over {len(runner.log)} rows")


def test_prefill_budget_replicas_bit_exact():
    from test_gpu_replicas import _run_replicas
    cfg = SchedConfig(R=2, Q_g=8, U=4, K=1, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16,
                      prefill_budget=40)
    off, toks, L = _workload(16, cap=cfg.cap)
    outs = _run_replicas(cfg, off, toks, L, max_prompt=MAXP)
    c, og = _oracle(cfg, off, toks, L)
    for rank, o in enumerate(outs):
        _compare_schedule(o, c, og)
        _compare_prefill(o, c, rank)
