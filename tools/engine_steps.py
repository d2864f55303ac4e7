"""Run a few decode steps of an 8B-width engine (L layers) for launch-list profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2603_23414_b200.engine import RolloutEngine
from workload.configs import LLAMA8B, SchedConfig, KV_BF16
from workload.lengths import LengthModel, sample_lengths
from workload.prompts import make_prompts
from workload.weights import fill_engine_weights
L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
m = LLAMA8B.with_layers(L)
cfg = SchedConfig(Q_g=256, U=64, pool_prompts=1024, cap=8192, kv_pages=3000, kv_dtype=KV_BF16)
eng = RolloutEngine(m, cfg, max_traj=1024, max_prompt=256, prefill_chunk=4096)
fill_engine_weights(eng, m, 0)
eng.load_policy_weights(0)
off, toks = make_prompts(1, 1024, m.V, 256)
eng.submit_prompts(np.arange(1024, dtype=np.uint64), off, toks, sample_lengths(LengthModel(cap=8192), 0, 1024))
for _ in range(steps):
    st, info = eng.decode_step()
    print("step", info.k, "dt_ms", round(info.dt_ms, 3), flush=True)
