"""Run an 8B-width engine (L layers) through prefill and a few decode steps, then
bracket ONE decode step with cudaProfilerStart/Stop (for ncu --profile-from-start off).
usage: ncu_engine.py [L] [warm_steps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2603_23414_b200.engine import RolloutEngine
from paper_2603_23414_b200 import _lib
_lib.set_tuning(graphs=0)  # direct launches, one kernel per ncu record
from workload.configs import LLAMA8B, SchedConfig, KV_BF16
from workload.lengths import LengthModel, sample_lengths
from workload.prompts import make_prompts
from workload.weights import fill_engine_weights

L = int(sys.argv[1]) if len(sys.argv) > 1 else 2
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 5
m = LLAMA8B.with_layers(L)
cfg = SchedConfig(Q_g=256, U=64, pool_prompts=1024, cap=8192, kv_pages=3000, kv_dtype=KV_BF16)
eng = RolloutEngine(m, cfg, max_traj=1024, max_prompt=256, prefill_chunk=4096)
fill_engine_weights(eng, m, 0)
eng.load_policy_weights(0)
off, toks = make_prompts(1, 1024, m.V, 256)
Ls = sample_lengths(LengthModel(cap=8192), 0, 1024)
eng.submit_prompts(np.arange(1024, dtype=np.uint64), off, toks, Ls)
for _ in range(warm):
    eng.decode_step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.decode_step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
