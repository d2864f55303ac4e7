"""Scheduling parity at BASELINE.json's full scale (configs[1], cfg2): Q_g = 256
slots, U = 64, pools of 1024 prompts, 2 epochs = 2048 trajectories with the
cfg2 lognormal lengths up to the 8192-token cap -- ~29 k decode steps -- in
the launch configuration bench.py times (decode-row buckets, CUDA graphs,
PDL).  The policy is the tiny random-init decoder: under FORCED lengths the
schedule does not depend on the model, and the tiny model keeps the run to
seconds.  The whole event log (loads, admissions with slots, finishes in
compaction order, emitted groups with membership, versions) and the (k, r_k)
trace must equal the CPU oracle's bit for bit; the abstract bubble ratio
follows (Eq. (bubble)).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from engine_harness import make_engine, run_engine  # noqa: E402
from oracle.metrics import bubble_ratio  # noqa: E402
from oracle.sched import Controller  # noqa: E402
from workload.configs import (BARRIER_ADMITTED, BARRIER_TRAINED, K_INF, KV_BF16, MODE_SORTED, MODE_SYNC,  # noqa: E402
                              TINY, SchedConfig)
from workload.lengths import LengthModel, sample_lengths  # noqa: E402
from workload.prompts import make_prompts  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _cfg2_inputs(n=2048):
    off, toks = make_prompts(1, n, TINY.V, 256)
    L = sample_lengths(LengthModel(median=1600, sigma=0.55, tail=0.03, floor=1, cap=8192), 0, n)
    return off, toks, L


CASES = [("sorted_trained", dict(mode=MODE_SORTED, barrier=BARRIER_TRAINED)),
         ("sorted_admitted", dict(mode=MODE_SORTED, barrier=BARRIER_ADMITTED)),
         ("sync", dict(mode=MODE_SYNC))]


@pytest.mark.parametrize("name,over", CASES, ids=[c[0] for c in CASES])
def test_cfg2_scale_schedule_bit_exact(name, over):
    cfg = SchedConfig(Q_g=256, U=64, K=K_INF, pool_prompts=1024, G=1, cap=8192, kv_pages=11000, kv_dtype=KV_BF16,
                      **over)
    off, toks, L = _cfg2_inputs()
    eng = make_engine(TINY, cfg, max_traj=2048, max_prompt=256, prefill_chunk=4096)
    res = run_engine(eng, TINY, off, toks, L, refresh_weights=False)
    eng.close()
    c = Controller(cfg)
    c.submit_prompts(np.arange(len(L)) + 1000, np.diff(off), L)
    groups = c.run()
    assert res["steps"] == c.trace
    assert res["events"] == c.events
    assert [[r["traj_id"] for r in h.records] for h, _ in res["groups"]] == [[r["traj_id"] for r in g] for g in groups]
    B = bubble_ratio(c.trace, 256)
    print(f"{name}: {len(c.trace)} steps, {len(groups)} groups, abstract bubble {float(B):.4f}")
    if name == "sorted_trained":
        assert len(c.trace) == 28989   # bench.py --full measured the same schedule on the 8B engine
