"""The bench's cfg2 engine brought to mid-rollout (P decode steps, ~mean context
1700 at P = 1500), then ONE decode step bracketed by cudaProfilerStart/Stop for
`ncu --profile-from-start off` (direct launches: srl_tuning.graphs = 0).
usage: ncu_steady.py [P]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_23414_b200.engine import GROUP_READY, RolloutEngine  # noqa: E402
from paper_2603_23414_b200 import _lib  # noqa: E402
_lib.set_tuning(graphs=0)  # direct launches, one kernel per ncu record
from workload.configs import LLAMA8B  # noqa: E402
from workload.weights import fill_engine_weights  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1500
MIXED = len(sys.argv) > 2 and sys.argv[2] == "mixed"   # profile a step that admits prompts (mixed pass)
sched = bench.cfg2_sched(1)
off, toks, L = bench.workload_inputs(1, epochs=2)
eng = RolloutEngine(LLAMA8B, sched, max_traj=2048, max_prompt=256, prefill_chunk=4096)
fill_engine_weights(eng, LLAMA8B, 0)
eng.load_policy_weights(0)
eng.submit_prompts(np.arange(len(L), dtype=np.uint64) + 1, off, toks, L)
v = 0
k = 0
while k < P:
    st, info = eng.decode_step()
    k += info.k >= 0
    if st == GROUP_READY:
        eng.harvest_finished(cap_recs=2048)
        v += 1
        eng.load_policy_weights(v)
while True:   # a step without admissions (pure decode), or with them (mixed)
    # advance, unprofiled, to a step of the wanted kind: a decode step admits prompts
    # iff the previous step finished trajectories (slots free up at its END)
    st, info = eng.decode_step()
    if st == GROUP_READY:
        eng.harvest_finished(cap_recs=2048)
        v += 1
        eng.load_policy_weights(v)
        continue
    if (info.n_finished > 0) != MIXED:
        continue
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    st, info = eng.decode_step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled step", info.k, "r_k", info.r_k, "sum_ctx", info.sum_ctx, "prefill", info.n_prefill_tokens,
          "dt_ms", round(info.dt_ms, 3), flush=True)
    break
eng.close()
