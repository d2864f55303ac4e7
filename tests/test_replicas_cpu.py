"""Host side of the N > 1 replica path on CPU (world_size 2, gloo).

* the NCCL unique id drawn by libsrl on rank 0 reaches every rank intact
  (engine.share_nccl_unique_id over torch.distributed);
* the lockstep protocol of rows a14/a12/a13: every rank holds the full
  controller state, produces tokens only for its own slots g = s*R + r, and
  all-gathers fixed [Q_g]-row (token, logprob) blocks laid out like the
  library's [R][2][Q_g] exchange buffer.  Under EOS stops (stops depend on the
  tokens) both ranks' event logs equal the single-process R = 2 oracle's --
  i.e. the exchanged rows are sufficient for the replicated state;
* bench.py's whole-job aggregation (sum of tokens over ranks / max time).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from oracle.sched import Controller  # noqa: E402
from workload.configs import K_INF, STOP_EOS, SchedConfig  # noqa: E402

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


def _spawn(fn, *args):
    port = _free_port()
    mp.start_processes(fn, args=(port, *args), nprocs=WORLD, join=True, start_method="spawn")


# ------------------------------------------------------------------ NCCL id sharing
def _w_share_id(rank, port, outdir):
    _init(rank, port)
    from paper_2603_23414_b200.engine import share_nccl_unique_id
    uid = share_nccl_unique_id(dist, rank)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    got = [torch.empty_like(t) for _ in range(WORLD)]
    dist.all_gather(got, t)
    np.save(os.path.join(outdir, f"id{rank}.npy"), torch.stack(got).numpy())
    dist.destroy_process_group()


def test_nccl_unique_id_shared_over_gloo(tmp_path):
    _spawn(_w_share_id, str(tmp_path))
    a = np.load(tmp_path / "id0.npy")
    b = np.load(tmp_path / "id1.npy")
    assert a.shape == (WORLD, 128) and np.array_equal(a, b)
    assert np.array_equal(a[0], a[1]) and a[0].any()


# ------------------------------------------------------------------ lockstep protocol
V, EOS = 97, 5


def _token(tid, n, version):
    """A deterministic stand-in policy: token of trajectory `tid` at generated index n."""
    h = (tid * 0x9E3779B1 + n * 0x85EBCA77 + version * 0xC2B2AE3D) & 0xFFFFFFFF
    h ^= h >> 15
    h = (h * 0x2C1B3C6D) & 0xFFFFFFFF
    h ^= h >> 12
    return int(h % V), float(-(h % 1000) / 100.0)


class _GlobalRunner:
    def admit(self, t, v):
        pass

    def prefill(self, t, a, b, v):
        pass

    def release(self, t):
        pass

    def step(self, batch, version):
        return [_token(t.tid, len(t.tokens), version) for _, t in batch]


class _ShardedRunner(_GlobalRunner):
    """Rank r computes its own slots only, then all-gathers [2][Q_g] blocks."""

    def __init__(self, cfg, rank):
        self.cfg, self.rank = cfg, rank

    def step(self, batch, version):
        Q, R = self.cfg.Q_g, self.cfg.R
        tok = torch.zeros(Q, dtype=torch.int32)
        lp = torch.zeros(Q, dtype=torch.float32)
        for g, t in batch:
            if g % R == self.rank:
                a, b = _token(t.tid, len(t.tokens), version)
                tok[g // R], lp[g // R] = a, b
        blk = torch.cat([tok, lp.view(torch.int32)])          # this rank's [2][Q_g] block
        allb = [torch.empty_like(blk) for _ in range(R)]
        dist.all_gather(allb, blk)
        out = []
        for g, _ in batch:
            b = allb[g % R]
            out.append((int(b[g // R]), float(b[Q + g // R].view(torch.float32))))
        return out


def _cfg():
    return SchedConfig(R=WORLD, Q_g=6, U=4, K=K_INF, pool_prompts=12, cap=40, kv_pages=64, stop=STOP_EOS,
                       eos_id=EOS)


def _run(cfg, runner):
    c = Controller(cfg, runner)
    n = 30
    c.submit_prompts(np.arange(n) + 100, np.full(n, 8), None)
    c.run()
    return c


def _w_lockstep(rank, port, outdir):
    _init(rank, port)
    cfg = _cfg()
    c = _run(cfg, _ShardedRunner(cfg, rank))
    import pickle
    with open(os.path.join(outdir, f"ev{rank}.pkl"), "wb") as fh:
        pickle.dump((c.events, c.trace, c.raw_tokens), fh)
    dist.destroy_process_group()


def test_lockstep_protocol_matches_single_process_oracle(tmp_path):
    import pickle
    _spawn(_w_lockstep, str(tmp_path))
    ref = _run(_cfg(), _GlobalRunner())
    finishes = [e for e in ref.events if e[0] == "FINISH"]
    assert any(e[4] < _cfg().cap for e in finishes), "EOS never fired: the test would not depend on tokens"
    for r in range(WORLD):
        with open(tmp_path / f"ev{r}.pkl", "rb") as fh:
            ev, tr, raw = pickle.load(fh)
        assert ev == ref.events and tr == ref.trace and raw == ref.raw_tokens


# ------------------------------------------------------------------ bench aggregation
def _w_aggregate(rank, port, outdir):
    _init(rank, port)
    import bench
    raw, useful, ms = [(1000.0, 400.0, 10.0), (3000.0, 600.0, 20.0)][rank]
    tok_s, useful_s, mx = bench.aggregate_over_ranks(dist, raw, useful, ms, device="cpu")
    np.save(os.path.join(outdir, f"agg{rank}.npy"), np.array([tok_s, useful_s, mx]))
    dist.destroy_process_group()


def test_bench_whole_job_aggregation(tmp_path):
    _spawn(_w_aggregate, str(tmp_path))
    for r in range(WORLD):
        tok_s, useful_s, mx = np.load(tmp_path / f"agg{r}.npy")
        assert mx == 20.0                                     # max over ranks
        assert tok_s == pytest.approx(4000.0 / 20e-3)         # all ranks' tokens / slowest rank's time
        assert useful_s == pytest.approx(1000.0 / 20e-3)


# ------------------------------------------------------------------ SRL_COMM_HOST callbacks over gloo
def _w_host_transport(rank, port, outdir):
    """The srl_host_transport callbacks HostGroup.gloo builds, invoked exactly as
    libsrl invokes them (through the C function pointers, on a raw byte buffer)."""
    import ctypes as C
    _init(rank, port)
    from paper_2603_23414_b200.engine import HostGroup
    hg = HostGroup.gloo(dist)
    seg = 24
    buf = (C.c_uint8 * (seg * WORLD))()
    for i in range(seg):
        buf[rank * seg + i] = (rank * 37 + i) & 0xFF
    rc = hg.t.allgather(None, C.cast(buf, C.c_void_p), seg)
    gathered = bytes(buf)
    bbuf = (C.c_uint8 * 10)()
    if rank == 0:
        for i in range(10):
            bbuf[i] = 200 + i
    rc2 = hg.t.broadcast(None, C.cast(bbuf, C.c_void_p), 10)
    np.save(os.path.join(outdir, f"host{rank}.npy"), np.frombuffer(gathered + bytes(bbuf) + bytes([rc, rc2]), np.uint8))
    dist.destroy_process_group()


def test_host_transport_callbacks_over_gloo(tmp_path):
    _spawn(_w_host_transport, str(tmp_path))
    want = bytes(((r * 37 + i) & 0xFF) for r in range(WORLD) for i in range(24)) + bytes(range(200, 210)) + b"\0\0"
    for r in range(WORLD):
        assert np.load(tmp_path / f"host{r}.npy").tobytes() == want
