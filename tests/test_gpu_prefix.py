"""N4 on the GPU: prompt-prefix KV page sharing among the G samples of a prompt
(P:235 several responses per prompt, P:387 RadixAttention) --
srl_sched_cfg.share_prefix against oracle/sched.py's page accounting
(`_prefix_pages`: per replica and prompt, refcounted, shared only within the
policy version the prefix was computed under).

* scheduling: event log + trace + groups BIT-EXACT against the oracle with
  sharing on, in page-limited configurations where sharing changes admissions
  and preemptions (the same runs without sharing give a different schedule);
* KV correctness: teacher-forced logits of every sample (which read the shared
  prompt pages written by another sample's prefill) within rel-L2 1e-2 of the
  fp64 oracle decode of its own full prompt, sampled ids bit-exact on identical
  logits;
* the prefill work actually shrinks: prompt rows processed per step equal what
  the sharing rule predicts (first holder: whole prompt; later holders: from the
  first unshared position)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from engine_harness import make_engine, run_engine, tiny_workload  # noqa: E402
from oracle.model import ModelRunner, load_weights  # noqa: E402
from oracle.sampler import sample_row  # noqa: E402
from test_gpu_engine import _compare_schedule, _oracle  # noqa: E402
from workload.configs import K_INF, KV_BF16, KV_FP32, RESUME_REPREFILL, TINY, SchedConfig  # noqa: E402
from workload.lengths import LengthModel  # noqa: E402

MAXP = 200


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _workload(n_prompts, G, cap=64, median=20):
    lm = LengthModel(median=median, sigma=0.6, tail=0.2, floor=1, cap=cap)
    return tiny_workload(n_prompts=n_prompts, G=G, cap=cap, lm=lm, plen=(60, MAXP))


CASES = [
    # (name, overrides): page-limited so the shared pages change who fits
    ("Kinf", dict(K=K_INF, kv_pages=24)),
    ("K0", dict(K=0, kv_pages=24)),
    ("K1", dict(K=1, kv_pages=20)),
    ("K1_reprefill", dict(K=1, kv_pages=24, resume=RESUME_REPREFILL)),
    ("preempt", dict(K=K_INF, kv_pages=14)),
    ("ample", dict(K=1, kv_pages=400)),
]


@pytest.mark.parametrize("name,over", CASES, ids=[c[0] for c in CASES])
def test_prefix_sharing_schedule_bit_exact(name, over):
    base = dict(Q_g=8, U=4, pool_prompts=4, G=4, cap=96, kv_dtype=KV_BF16, share_prefix=1)
    base.update(over)
    cfg = SchedConfig(**base)
    off, toks, L = _workload(8, cfg.G, cap=cfg.cap, median=30)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=MAXP)
    res = run_engine(eng, TINY, off, toks, L)
    eng.close()
    c, og = _oracle(cfg, off, toks, L)
    _compare_schedule(res, c, og)
    if name != "ample":
        # sharing mattered: the unshared oracle schedule differs
        import dataclasses
        c0, _ = _oracle(dataclasses.replace(cfg, share_prefix=0), off, toks, L)
        assert c0.events != c.events


def test_prefix_sharing_prefill_rows():
    """Ample pages, all 4 samples of each prompt admitted in step 0: the first holder
    prefills prompt_len - 1 rows, each later one prompt_len - 1 - 64 * floor((prompt_len - 1) / 64)."""
    cfg = SchedConfig(Q_g=16, U=4, K=K_INF, pool_prompts=4, G=4, cap=32, kv_pages=400, kv_dtype=KV_BF16,
                      share_prefix=1)
    off, toks, L = _workload(4, cfg.G, cap=cfg.cap)
    plen = np.diff(off)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=MAXP)
    eng.submit_prompts(np.arange(4, dtype=np.uint64) + 1000, off, toks, L)
    st, info = eng.decode_step()
    eng.close()
    want = sum(int(p) - 1 + 3 * (int(p) - 1 - 64 * ((int(p) - 1) // 64)) for p in plen)
    assert info.n_admitted == 16
    assert info.n_prefill_tokens == want, (info.n_prefill_tokens, want)
    assert want < 4 * int((plen - 1).sum())


@pytest.mark.parametrize("kv,over", [(KV_FP32, dict(K=K_INF, kv_pages=24)),
                                     (KV_BF16, dict(K=K_INF, kv_pages=20, resume=RESUME_REPREFILL)),
                                     (KV_BF16, dict(K=K_INF, kv_pages=400, prefill_chunk=96))],
                         ids=["f32-Kinf", "bf16-reprefill", "bf16-separate-prefill"])
def test_prefix_sharing_teacher_forced_logits(kv, over):
    """Every decoded row of every sample -- its attention reads the shared prompt pages --
    against the oracle's fp64 decode of its own whole prompt + tokens.  K = inf: no token
    is ever dropped, so the harvested tokens are the ones every step sampled (teacher
    forcing); REPREFILL re-admits every running sample after each update, under a new
    version, so entries are re-created and private copies taken (R31)."""
    over = dict(over)
    chunk = over.pop("prefill_chunk", 256)
    cfg = SchedConfig(Q_g=8, U=4, pool_prompts=4, G=4, cap=48, kv_dtype=kv, share_prefix=1, **over)
    off, toks, L = _workload(4, cfg.G, cap=cfg.cap, median=16)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=MAXP, prefill_chunk=chunk)
    res = run_engine(eng, TINY, off, toks, L, record_logits=True)
    eng.close()
    teacher = {}
    for h, _ in res["groups"]:
        for r in h.records:
            seg = slice(r["tok_offset"], r["tok_offset"] + r["len"])
            teacher[r["traj_id"]] = h.tokens[seg].tolist()
    G = cfg.G
    prompts = lambda t: toks[off[t.tid // G]:off[t.tid // G + 1]]  # noqa: E731
    runner = ModelRunner(TINY, lambda v: load_weights(TINY, version=v), prompts, cfg.sample_seed,
                         teacher=teacher, record_logits=True)
    c, og = _oracle(cfg, off, toks, L, runner)
    _compare_schedule(res, c, og)
    worst = 0.0
    for e in runner.log:
        zg = res["logits"][e["k"]][e["g"]]
        zo = e["logits"].astype(np.float64)
        rel = np.linalg.norm(zg - zo) / np.linalg.norm(zo)
        worst = max(worst, rel)
        assert rel <= 1e-2, (e["k"], e["g"], e["tid"], rel)
        t_same = sample_row(zg, np.float32(1.0), cfg.sample_seed, e["n"], e["tid"], e["restarts"])[0]
        assert t_same == teacher[e["tid"]][e["n"]]
    assert len(runner.log) > 100
    print(f"worst logits rel-L2 {worst:.2e} over {len(runner.log)} rows")


def test_prefix_sharing_replicas_bit_exact():
    """R = 2 lockstep replicas (in-process transport): every rank keeps every replica's
    prefix entries (refcounts, version tags) for the page accounting and only its own
    entries' page ids; schedules bit-exact against the R = 2 oracle on every rank."""
    from test_gpu_replicas import _run_replicas
    cfg = SchedConfig(R=2, Q_g=4, U=4, K=1, pool_prompts=4, G=4, cap=96, kv_pages=12, kv_dtype=KV_BF16,
                      share_prefix=1)
    off, toks, L = _workload(8, cfg.G, cap=cfg.cap, median=30)
    outs = _run_replicas(cfg, off, toks, L, max_prompt=MAXP)
    c, og = _oracle(cfg, off, toks, L)
    for o in outs:
        _compare_schedule(o, c, og)
    import dataclasses
    c0, _ = _oracle(dataclasses.replace(cfg, share_prefix=0), off, toks, L)
    assert c0.events != c.events
