"""bench.py without a GPU: the reference arm (the CPU oracle, the tier's "reference")
prints one JSON line with the contract's keys, and `--gpus N` without a launcher
starts N ranks itself (CPU only)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, timeout=600):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _line(["--impl", "reference", "--steps", "2", "--warmup", "3"])
    assert d["impl"] == "reference" and d["unit"] == "tokens/s" and d["value"] > 0
    assert d["metric"].startswith("rollout tokens/s")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["single_thread_value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["steps"] == 2 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["ms_per_step"] > 0 and d["ranks"] == 1
    # BASELINE configs[0] end to end on the oracle (controller + tiny model)
    assert d["tiny_end_to_end"]["tokens"] > 100 and d["tiny_end_to_end"]["value"] > 0
    # same workload text as the GPU arm's config
    import bench
    assert d["config"]["workload"] == bench.WORKLOAD


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` run bare must start 2 ranks (one process per
    GPU, rendezvous on 127.0.0.1) -- here through the reference arm, whose ranks
    count themselves over a CPU process group before rank 0 reports."""
    d = _line(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert d["ranks"] == 2 and d["n_gpus"] == 2
