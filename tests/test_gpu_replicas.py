"""GPU parity of the lockstep data-parallel replica path (rows a14
all-gather and a17 weight broadcast) against the CPU oracle's R-replica
controller (oracle/sched.py, global slot g = s*R + r, reading R24).

One B200 is available, so R engines share cuda:0 in one process, each driven
by its own host thread, exchanging through the in-process transport
(SRL_COMM_LOCAL); the NCCL transport runs as a one-rank communicator (the same
calls a multi-GPU launch makes).  Checked per rank:
* event log and (k, r_k) trace bit-exact vs oracle Controller(R, Q_g);
* every rank emits the same groups with identical tokens / logprobs / versions
  (the replicated state really is replicated);
* teacher-forced logits of every rank's rows within rel-L2 1e-2 of the oracle,
  sampled ids bit-exact on identical logits.
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from engine_harness import make_engine, run_engine, tiny_workload  # noqa: E402
from oracle.model import ModelRunner, load_weights  # noqa: E402
from oracle.sampler import sample_row  # noqa: E402
from oracle.sched import Controller  # noqa: E402
from workload.configs import (K_INF, KV_BF16, KV_FP32, MODE_SYNC, RESUME_REPREFILL, STOP_EOS, TINY,  # noqa: E402
                              SchedConfig)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _oracle(cfg, off, toks, L, runner=None):
    c = Controller(cfg, runner)
    c.submit_prompts(np.arange(len(off) - 1) + 1000, np.diff(off), L)
    groups = []
    c.run(on_group=lambda ctrl, recs: groups.append((recs, ctrl.v)))
    return c, groups


def _run_replicas(cfg, off, toks, L, *, record_logits=False, max_traj=64):
    """R engines on cuda:0, one thread each, in-process exchange."""
    from paper_2603_23414_b200.engine import LocalGroup
    R = cfg.R
    grp = LocalGroup(R)
    out, errs = [None] * R, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            eng = make_engine(TINY, cfg, max_traj=max_traj, max_prompt=16, rank=r, world=R, local_group=grp)
            out[r] = run_engine(eng, TINY, off, toks, L, record_logits=record_logits)
            out[r]["counters"] = eng.counters()
            eng.close()
        except Exception as ex:  # surfaced below
            errs.append((r, ex))

    th = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    assert not errs, errs
    return out


def _compare(res, c, og):
    assert res["steps"] == c.trace
    assert res["events"] == c.events
    assert len(res["groups"]) == len(og)
    for (h, v_gpu), (recs, v_or) in zip(res["groups"], og):
        assert v_gpu == v_or
        assert [r["traj_id"] for r in h.records] == [r["traj_id"] for r in recs]
        for r, o in zip(h.records, recs):
            assert (r["len"], r["v_first"], r["v_last"], r["lifecycle"], r["restarts"], r["finish_step"]) == \
                (o["len"], o["v_first"], o["v_last"], o["lifecycle"], o["restarts"], o["finish_step"])
            seg = slice(r["tok_offset"], r["tok_offset"] + r["len"])
            assert h.versions[seg].tolist() == o["vers"]


def _same_across_ranks(outs):
    ref = outs[0]
    for o in outs[1:]:
        assert o["events"] == ref["events"] and o["steps"] == ref["steps"]
        assert len(o["groups"]) == len(ref["groups"])
        for (h, _), (h0, _) in zip(o["groups"], ref["groups"]):
            assert [r["traj_id"] for r in h.records] == [r["traj_id"] for r in h0.records]
            assert np.array_equal(h.tokens, h0.tokens)
            assert np.array_equal(h.logprobs.view(np.int32), h0.logprobs.view(np.int32))   # bit-for-bit
            assert np.array_equal(h.versions, h0.versions)
        assert o["counters"]["raw_tokens"] == ref["counters"]["raw_tokens"]


CASES = [
    ("R2_partial", dict(R=2, Q_g=8, K=K_INF)),
    ("R2_onpolicy", dict(R=2, Q_g=8, K=0)),
    ("R3_K1_reprefill", dict(R=3, Q_g=4, K=1, resume=RESUME_REPREFILL)),
    ("R4_oversubscribed", dict(R=4, Q_g=2, K=K_INF, pool_prompts=16)),
    ("R2_preempt", dict(R=2, Q_g=6, K=1, kv_pages=5, pool_prompts=8, U=2)),
    ("R2_sync", dict(R=2, Q_g=8, mode=MODE_SYNC)),
    ("R2_eos", dict(R=2, Q_g=8, K=K_INF, stop=STOP_EOS, eos_id=7)),
]


@pytest.mark.parametrize("name,over", CASES, ids=[c[0] for c in CASES])
def test_replicas_schedule_bit_exact(name, over):
    base = dict(U=4, pool_prompts=16, G=1, cap=64, kv_pages=256, kv_dtype=KV_BF16)
    base.update(over)
    cfg = SchedConfig(**base)
    off, toks, L = tiny_workload(n_prompts=16)
    outs = _run_replicas(cfg, off, toks, L)
    _same_across_ranks(outs)
    if cfg.stop == STOP_EOS:
        # EOS stops depend on the sampled tokens: the oracle replays the GPU's tokens
        teacher = {}
        for h, _ in outs[0]["groups"]:
            for r in h.records:
                teacher[r["traj_id"]] = h.tokens[r["tok_offset"]:r["tok_offset"] + r["len"]].tolist()

        class Replay:
            def admit(self, t, v):
                pass

            def release(self, t):
                pass

            def step(self, batch, v):
                return [(teacher[t.tid][len(t.tokens)], 0.0) for _, t in batch]
        c, og = _oracle(cfg, off, toks, L, Replay())
    else:
        c, og = _oracle(cfg, off, toks, L)
    _compare(outs[0], c, og)


@pytest.mark.parametrize("K", [1, 0], ids=["K1", "K0"])
def test_replicas_preemption_bit_exact(K):
    """Per-replica KV exhaustion: every rank tracks every replica's free-page count
    and runs the same victim choice; only the owner moves its page ids."""
    from workload.lengths import LengthModel
    cfg = SchedConfig(R=2, Q_g=4, U=2, K=K, pool_prompts=16, cap=128, kv_pages=4, kv_dtype=KV_BF16)
    off, toks, L = tiny_workload(n_prompts=16, cap=128, lm=LengthModel(median=40, sigma=0.6, tail=0.3, floor=1, cap=128))
    outs = _run_replicas(cfg, off, toks, L)
    _same_across_ranks(outs)
    c, og = _oracle(cfg, off, toks, L)
    assert sum(1 for e in c.events if e[0] == "PREEMPT") > 0
    _compare(outs[0], c, og)


def test_replicas_qtot_above_one_ctl_block():
    """Q_tot = 2 x 600 slots > the controller CTA's 1024 threads: chunked scans."""
    cfg = SchedConfig(R=2, Q_g=600, U=64, K=K_INF, pool_prompts=1300, cap=8, kv_pages=700, kv_dtype=KV_BF16)
    off, toks, L = tiny_workload(n_prompts=1300, cap=8)
    outs = _run_replicas(cfg, off, toks, L, max_traj=1300)
    _same_across_ranks(outs)
    c, og = _oracle(cfg, off, toks, L)
    _compare(outs[0], c, og)


@pytest.mark.parametrize("kv", [KV_FP32, KV_BF16], ids=["f32", "bf16"])
def test_replicas_model_parity_teacher_forced(kv):
    cfg = SchedConfig(R=2, Q_g=8, U=4, K=K_INF, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=kv)
    off, toks, L = tiny_workload(n_prompts=16)
    outs = _run_replicas(cfg, off, toks, L, record_logits=True)
    _same_across_ranks(outs)
    teacher = {}
    for h, _ in outs[0]["groups"]:
        for r in h.records:
            teacher[r["traj_id"]] = h.tokens[r["tok_offset"]:r["tok_offset"] + r["len"]].tolist()
    prompts = lambda t: toks[off[t.tid]:off[t.tid + 1]]  # noqa: E731
    runner = ModelRunner(TINY, lambda v: load_weights(TINY, version=v), prompts, cfg.sample_seed,
                         teacher=teacher, record_logits=True)
    c, og = _oracle(cfg, off, toks, L, runner)
    _compare(outs[0], c, og)
    worst = 0.0
    for e in runner.log:
        g = e["g"]
        zg = outs[g % cfg.R]["logits"][e["k"]][g // cfg.R]       # row s of rank r holds global slot s*R + r
        zo = e["logits"].astype(np.float64)
        rel = np.linalg.norm(zg - zo) / np.linalg.norm(zo)
        worst = max(worst, rel)
        assert rel <= 1e-2, (e["k"], g, rel)
        assert sample_row(zg, np.float32(1.0), cfg.sample_seed, e["n"], e["tid"], e["restarts"])[0] == \
            teacher[e["tid"]][e["n"]]
    print(f"worst logits rel-L2 {worst:.2e}")


def test_nccl_transport_one_rank():
    """The NCCL transport (dlopen'd libnccl, in-place all-gather + grouped
    broadcasts) as a one-rank communicator: same schedule as the oracle."""
    from paper_2603_23414_b200.engine import nccl_unique_id
    cfg = SchedConfig(Q_g=16, U=4, K=1, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16)
    off, toks, L = tiny_workload(n_prompts=16)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=16, rank=0, world=1, nccl_id=nccl_unique_id())
    res = run_engine(eng, TINY, off, toks, L)
    prof = eng.profile()
    eng.close()
    c, og = _oracle(cfg, off, toks, L)
    _compare(res, c, og)
    assert prof is not None
