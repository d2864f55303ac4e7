"""GPU parity of the lockstep data-parallel replica path (rows a14
all-gather and a17 weight broadcast) against the CPU oracle's R-replica
controller (oracle/sched.py, global slot g = s*R + r, reading R24).

One B200 is available, so R engines share cuda:0 in one process, each driven
by its own host thread, exchanging through the in-process transport
(SRL_COMM_LOCAL); the NCCL transport runs as a one-rank communicator (the same
calls a multi-GPU launch makes); and R PROCESSES share cuda:0 exchanging through
the host-callback transport (SRL_COMM_HOST over a torch.distributed gloo group):
libsrl's replica protocol across process boundaries.  Checked per rank:
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


def _run_replicas(cfg, off, toks, L, *, record_logits=False, max_traj=64, max_prompt=16):
    """R engines on cuda:0, one thread each, in-process exchange."""
    from paper_2603_23414_b200.engine import LocalGroup
    R = cfg.R
    grp = LocalGroup(R)
    out, errs = [None] * R, []

    def work(r):
        try:
            torch.cuda.set_device(0)
            eng = make_engine(TINY, cfg, max_traj=max_traj, max_prompt=max_prompt, rank=r, world=R, local_group=grp)
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

            def prefill(self, t, a, b, v):
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


# ------------------------------------------------------------------ across processes (SRL_COMM_HOST + gloo)
def _w_host_replica(rank, port, world, over, outdir):
    import os
    import pickle

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2603_23414_b200.engine import HostGroup
    cfg = SchedConfig(**dict(dict(Q_g=8, U=4, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16, R=world),
                             **over))
    off, toks, L = tiny_workload(n_prompts=16)
    eng = make_engine(TINY, cfg, max_traj=64, max_prompt=16, rank=rank, world=world, host_group=HostGroup.gloo(dist))
    res = run_engine(eng, TINY, off, toks, L)           # refreshed weights broadcast from rank 0 every update
    cnt = eng.counters()
    eng.close()
    out = dict(events=res["events"], steps=res["steps"], counters=cnt,
               groups=[(v, [dict(r) for r in h.records], h.tokens, h.logprobs, h.versions) for h, v in res["groups"]])
    with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as fh:
        pickle.dump(out, fh)
    dist.destroy_process_group()


HOST_CASES = [("R2_partial", dict(K=K_INF)), ("R2_K1_eos", dict(K=1, stop=STOP_EOS, eos_id=7)),
              ("R3_onpolicy", dict(K=0, Q_g=4))]


@pytest.mark.parametrize("name,over", HOST_CASES, ids=[c[0] for c in HOST_CASES])
def test_replicas_across_processes_host_transport(tmp_path, name, over):
    """World-R processes, one engine each (all on cuda:0), exchanging the per-step
    [R][2][Q_g] rows and the refreshed policy through gloo: every rank's event log
    equals oracle Controller(R) bit for bit and the groups are identical on all
    ranks (tokens, logprob bits, versions)."""
    import pickle
    import socket

    import torch.multiprocessing as mp
    world = 3 if name.startswith("R3") else 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mp.start_processes(_w_host_replica, args=(port, world, over, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    outs = [pickle.load(open(tmp_path / f"r{r}.pkl", "rb")) for r in range(world)]
    cfg = SchedConfig(**dict(dict(Q_g=8, U=4, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16, R=world),
                             **over))
    off, toks, L = tiny_workload(n_prompts=16)
    if cfg.stop == STOP_EOS:   # EOS stops depend on the tokens: compare the ranks with each other and
        c = None               # the schedule with the single-process R-replica run instead
        ref = _run_replicas(cfg, off, toks, L)[0]
        assert outs[0]["events"] == ref["events"] and outs[0]["steps"] == ref["steps"]
    else:
        c, og = _oracle(cfg, off, toks, L)
        assert outs[0]["events"] == c.events and outs[0]["steps"] == c.trace
        assert [[r["traj_id"] for r in g[1]] for g in outs[0]["groups"]] == [[r["traj_id"] for r in recs]
                                                                              for recs, _ in og]
    for o in outs[1:]:
        assert o["events"] == outs[0]["events"] and o["steps"] == outs[0]["steps"]
        assert o["counters"]["raw_tokens"] == outs[0]["counters"]["raw_tokens"]
        for g, g0 in zip(o["groups"], outs[0]["groups"]):
            assert g[0] == g0[0] and [r["traj_id"] for r in g[1]] == [r["traj_id"] for r in g0[1]]
            assert np.array_equal(g[2], g0[2]) and np.array_equal(g[3].view(np.int32), g0[3].view(np.int32))
            assert np.array_equal(g[4], g0[4])


def test_replica_peer_failure_fails_fast_not_hang():
    """A rank that stops participating (dies) must not hang the others: with a 5 s
    transport timeout the surviving rank's srl_decode_step returns SRL_E_NCCL
    (communicator aborted) and every later call keeps failing."""
    import time

    from paper_2603_23414_b200._lib import SRLError
    from paper_2603_23414_b200.engine import LocalGroup
    cfg = SchedConfig(Q_g=8, U=4, R=2, pool_prompts=16, cap=64, kv_pages=256, kv_dtype=KV_BF16)
    off, toks, L = tiny_workload(n_prompts=16)
    grp = LocalGroup(2)
    res = {}

    def work(r):
        torch.cuda.set_device(0)
        eng = make_engine(TINY, cfg, max_traj=64, max_prompt=16, rank=r, world=2, local_group=grp,
                          comm_timeout_s=5)
        eng.submit_prompts(np.arange(16, dtype=np.uint64) + 1000, off, toks, L)
        for _ in range(3):
            eng.decode_step()
        if r == 1:
            res[1] = "stopped"     # rank 1 "dies": never calls again
            return
        t0 = time.time()
        try:
            for _ in range(100):
                eng.decode_step()
            res[0] = ("no error", time.time() - t0)
        except SRLError as ex:
            res[0] = (str(ex), time.time() - t0)
            try:
                eng.decode_step()
                res["after"] = "no error"
            except SRLError as ex2:
                res["after"] = str(ex2)
        eng.close()

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), "a rank hung"
    grp.close()
    msg, dt = res[0]
    assert "(-7)" in msg and dt < 60, res
    assert "(-7)" in res["after"], res
