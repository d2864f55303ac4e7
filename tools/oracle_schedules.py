"""Abstract-time (dt = 1) schedules of the cfg2 workload under the scheduler
variants bench.py --full measures, from the CPU oracle: steps, groups,
Eq. (bubble), raw / discarded tokens, staleness.  Test tooling (imports
oracle/); the GPU runs must reproduce the step counts and abstract bubble
exactly (tests/test_gpu_fullscale_schedule.py pins three of them in-suite).

  python tools/oracle_schedules.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses  # noqa: E402

import bench  # noqa: E402
from oracle.metrics import bubble_ratio  # noqa: E402
from oracle.sched import Controller  # noqa: E402
from workload.configs import BARRIER_ADMITTED, MODE_POSTHOC, MODE_SYNC  # noqa: E402

VARIANTS = [("sortedrl K=inf TRAINED", {}), ("sortedrl K=inf ADMITTED", dict(barrier=BARRIER_ADMITTED)),
            ("sortedrl K=0 (on-policy)", dict(K=0)), ("sync baseline", dict(mode=MODE_SYNC)),
            ("post-hoc sorting", dict(mode=MODE_POSTHOC))]


def main():
    off, toks, L = bench.workload_inputs(1, epochs=2)
    for name, over in VARIANTS:
        cfg = dataclasses.replace(bench.cfg2_sched(1), **over)
        t = time.time()
        c = Controller(cfg)
        c.submit_prompts(np.arange(len(L)) + 1, np.diff(off), L)
        groups = c.run()
        stale = [g_v - r["v_first"] for g_v, g in enumerate(groups) for r in g]
        B = bubble_ratio(c.trace, cfg.Q_tot)
        print(f"{name:26s} steps {len(c.trace):6d} groups {len(groups):3d} bubble {float(B):.4f} "
              f"raw {c.raw_tokens} discarded {c.discarded_tokens} staleness mean {np.mean(stale):.2f} "
              f"max {max(stale)}  ({time.time() - t:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
