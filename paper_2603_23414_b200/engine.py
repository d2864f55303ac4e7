"""Thin Python binding of the SortedRL rollout engine (include/srl.h).

Argument marshalling only: device memory comes from torch and is lent to the
C library; every step of the rollout path runs in libsrl.so.  Names follow the
C ABI: submit_prompts, decode_step, harvest_finished, load_policy_weights.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (COMM_HOST, COMM_LOCAL, COMM_NCCL, HOST_FN, Arena, Comm, HostTransport, ModelCfg, SchedCfg,
                   StepInfo, TraceRec, TrajRec, check)

OK, GROUP_READY, DONE = 0, 1, 2
EV_NAMES = {0: "STEP", 1: "LOAD", 2: "ADMIT", 3: "PREEMPT", 4: "FINISH", 5: "EMIT", 6: "DISCARD", 7: "SCAVENGE",
            8: "EMIT_MEMBER"}


def _i32p(a):
    return a.ctypes.data_as(C.c_void_p)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for srl_comm (call on rank 0, share with the others)."""
    buf = (C.c_uint8 * 128)()
    check(_lib.load().srl_nccl_unique_id(C.cast(buf, C.c_void_p)), "srl_nccl_unique_id")
    return bytes(buf)


def share_nccl_unique_id(dist, rank: int) -> bytes:
    """Rank 0 draws the id, torch.distributed broadcasts it (any backend)."""
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


class HostGroup:
    """SRL_COMM_HOST: the replica exchange through caller callbacks.  `allgather(buf)`
    receives a uint8 numpy view of `world` equal segments (this rank's filled) and
    must fill the rest; `broadcast(buf)` a uint8 view that rank 0 filled.  Each
    returns nothing and raises on failure (the engine then reports SRL_E_NCCL).
    `gloo(dist)` builds one over a torch.distributed (e.g. gloo) process group."""

    def __init__(self, allgather, broadcast):
        def wrap(fn):
            def cb(ctx, buf, n):
                try:
                    fn(np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)), shape=(int(n) if fn is broadcast
                                                                                     else int(n) * self.world,)))
                    return 0
                except Exception as exc:   # noqa: BLE001 -- reported through the C status
                    self.error = exc
                    return 1
            return HOST_FN(cb)
        self.world = None
        self.error = None
        self._cbs = (wrap(allgather), wrap(broadcast))      # kept alive with the group
        self.t = HostTransport(self._cbs[0], self._cbs[1], None)

    @classmethod
    def gloo(cls, dist):
        import torch
        world = dist.get_world_size()
        rank = dist.get_rank()

        def allgather(buf):
            seg = buf.size // world
            mine = torch.from_numpy(buf[rank * seg:(rank + 1) * seg].copy())
            outs = [torch.empty(seg, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, mine)
            for r in range(world):
                buf[r * seg:(r + 1) * seg] = outs[r].numpy()

        def broadcast(buf):
            t = torch.from_numpy(buf.copy()) if rank == 0 else torch.empty(buf.size, dtype=torch.uint8)
            dist.broadcast(t, src=0)
            buf[:] = t.numpy()
        g = cls(allgather, broadcast)
        g.world = world
        return g


class LocalGroup:
    """An in-process replica group (SRL_COMM_LOCAL): `world` engines, one host
    thread each, exchanging through peer copies.  Close after its engines."""

    def __init__(self, world: int):
        self.lib = _lib.load()
        self.world = world
        self.h = C.c_void_p()
        check(self.lib.srl_local_group_create(world, C.byref(self.h)), "srl_local_group_create")

    def close(self):
        if self.h:
            self.lib.srl_local_group_destroy(self.h)
            self.h = C.c_void_p()


@dataclass
class Harvest:
    records: list          # dicts per trajectory (group order)
    tokens: np.ndarray     # int32, concatenated
    logprobs: np.ndarray   # float32
    versions: np.ndarray   # int32


class RolloutEngine:
    """One engine per GPU.  `model` / `sched` are duck-typed records with the
    srl_model_cfg / srl_sched_cfg field names (workload.configs provides them)."""

    def __init__(self, model, sched, *, max_traj: int, max_prompt: int, prefill_chunk: int = 2048,
                 device: int = 0, stream=None, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 local_group: LocalGroup | None = None, host_group: HostGroup | None = None,
                 compact_weights: bool = False, comm_timeout_s: int = 0):
        """world > 1 (or an explicit nccl_id / local_group) makes this engine rank
        `rank` of a lockstep replica group: NCCL when `nccl_id` is given (one process
        per GPU), in-process when `local_group` is."""
        import torch
        self.torch = torch
        self.lib = _lib.load()
        self.model, self.sched = model, sched
        self.dev = torch.device("cuda", device)
        self.compact = bool(compact_weights)
        self.m = ModelCfg(model.L, model.d, model.Hq, model.Hkv, model.dh, model.ff, model.V,
                          float(model.rope_theta), float(model.rms_eps), int(model.qkv_bias), int(self.compact))
        self.s = SchedCfg(sched.Q_g, sched.U, sched.K, sched.pool_prompts, sched.G, sched.cap, sched.page_tokens,
                          sched.kv_pages, sched.mode, sched.resume, sched.barrier, sched.stop, sched.eos_id,
                          sched.kv_dtype, float(sched.temperature), int(sched.sample_seed), max_traj, max_prompt,
                          prefill_chunk, int(getattr(sched, "top_k", 0)), float(getattr(sched, "top_p", 1.0)),
                          int(getattr(sched, "share_prefix", 0)), int(getattr(sched, "prefill_budget", 0)))
        wb, kb, sb = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(self.lib.srl_arena_sizes(C.byref(self.m), C.byref(self.s), world, C.byref(wb), C.byref(kb),
                                       C.byref(sb)), "srl_arena_sizes")
        self.bytes = (wb.value, kb.value, sb.value)
        self.W = torch.empty(wb.value, dtype=torch.uint8, device=self.dev)
        self.KV = torch.empty(kb.value, dtype=torch.uint8, device=self.dev)
        self.S = torch.empty(sb.value, dtype=torch.uint8, device=self.dev)
        # a dedicated stream: the decode tail is captured into a CUDA graph, which the
        # legacy default stream does not allow
        self.stream = stream if stream is not None else torch.cuda.Stream(self.dev)
        arena = Arena(self.W.data_ptr(), self.KV.data_ptr(), self.S.data_ptr(), wb.value, kb.value, sb.value)
        comm = None
        transports = [x for x in (nccl_id, local_group, host_group) if x is not None]
        if world > 1 or transports:
            if len(transports) != 1:
                raise ValueError("a replica engine needs exactly one of nccl_id / local_group / host_group")
            comm = Comm()
            comm.rank, comm.world, comm.timeout_s = rank, world, int(comm_timeout_s)
            if nccl_id is not None:
                comm.kind = COMM_NCCL
                C.memmove(comm.nccl_unique_id, nccl_id, 128)
            elif local_group is not None:
                comm.kind = COMM_LOCAL
                comm.local_group = local_group.h
            else:
                comm.kind = COMM_HOST
                host_group.world = world
                comm.host = C.pointer(host_group.t)
                self._host_group = host_group      # the callbacks must outlive the engine
        self.h = C.c_void_p()
        check(self.lib.srl_create(C.byref(self.m), C.byref(self.s), device, C.c_void_p(self.stream.cuda_stream),
                                  C.byref(arena), C.byref(comm) if comm else None, C.byref(self.h)), "srl_create")
        self.max_traj = max_traj
        self.Q_g, self.V = sched.Q_g, model.V

    # ------------------------------------------------------------------ weights
    def weight_view(self, name: str):
        """bf16 view of a named tensor in the flat weight region: [rows, cols] for dense
        tensors, [rows/16, 16, cols] for the block-interleaved gate/up weights."""
        off, rows, cols, rb, bs = (C.c_int64() for _ in range(5))
        if self.lib.srl_weight_layout(C.byref(self.m), name.encode(), C.byref(off), C.byref(rows), C.byref(cols),
                                      C.byref(rb), C.byref(bs)) != 0:
            raise KeyError(name)
        W16 = self.W.view(self.torch.bfloat16)
        o, r, c, rb, bs = off.value // 2, rows.value, cols.value, rb.value, bs.value
        if rb == r:
            return W16[o:o + r * c].view(r, c) if c > 1 else W16[o:o + r]
        return W16.as_strided((r // rb, rb, c), (bs * c, c, 1), o)

    def load_policy_tensor(self, name: str, src):
        """Install one tensor of the next policy (row-major bf16 device tensor)."""
        self._sync_in()
        return check(self.lib.srl_load_policy_tensor(self.h, name.encode(), C.c_void_p(src.data_ptr())),
                     "srl_load_policy_tensor")

    def _sync_in(self):
        """Order the engine stream after work torch queued on the current stream."""
        self.stream.wait_stream(self.torch.cuda.current_stream(self.dev))

    def harvest_device(self):
        """Device views (torch tensors, no copy) of the last harvested group: tokens,
        behaviour logprobs, generating versions (srl_harvest_device), the record
        count and the token count; the records' tok_offset / len (from the host
        harvest of the same group) give the ragged offsets."""
        import torch
        t, lp, ver, recs = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        n, ntok = C.c_int32(), C.c_int64()
        check(self.lib.srl_harvest_device(self.h, C.byref(t), C.byref(lp), C.byref(ver), C.byref(recs), C.byref(n),
                                          C.byref(ntok)), "srl_harvest_device")

        class _View:
            def __init__(self, ptr, typestr, count, dev):
                self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                                 "version": 3, "strides": None}
        dev = self.dev
        mk = lambda ptr, ts: torch.as_tensor(_View(ptr.value or 0, ts, ntok.value, dev), device=dev)  # noqa: E731
        return dict(tokens=mk(t, "<i4"), logprobs=mk(lp, "<f4"), versions=mk(ver, "<i4"), n_records=n.value,
                    n_tokens=ntok.value)

    def load_policy_weights(self, version: int, flat=None):
        self._sync_in()
        ptr = C.c_void_p(flat.data_ptr()) if flat is not None else None
        return check(self.lib.srl_load_policy_weights(self.h, ptr, int(version)), "srl_load_policy_weights")

    # ------------------------------------------------------------------ rollout
    def submit_prompts(self, prompt_ids, tok_off, toks, forced_len=None):
        ids = np.ascontiguousarray(prompt_ids, dtype=np.uint64)
        off = np.ascontiguousarray(tok_off, dtype=np.int32)
        tk = np.ascontiguousarray(toks, dtype=np.int32)
        fl = None if forced_len is None else np.ascontiguousarray(forced_len, dtype=np.int32)
        self._sync_in()
        return check(self.lib.srl_submit_prompts(self.h, len(ids), _i32p(ids), _i32p(off), _i32p(tk),
                                                 _i32p(fl) if fl is not None else None), "srl_submit_prompts")

    def decode_step(self):
        self._sync_in()
        info = StepInfo()
        rc = check(self.lib.srl_decode_step(self.h, C.byref(info)), "srl_decode_step")
        return rc, info

    def harvest_finished(self, cap_recs: int = 4096, cap_toks: int | None = None) -> Harvest:
        cap_toks = cap_toks if cap_toks is not None else cap_recs * self.sched.cap
        recs = (TrajRec * cap_recs)()
        n = C.c_int32()
        toks = np.empty(cap_toks, dtype=np.int32)
        lps = np.empty(cap_toks, dtype=np.float32)
        vers = np.empty(cap_toks, dtype=np.int32)
        check(self.lib.srl_harvest_finished(self.h, cap_recs, recs, C.byref(n), _i32p(toks), _i32p(lps), _i32p(vers),
                                            cap_toks), "srl_harvest_finished")
        out = []
        total = 0
        for i in range(n.value):
            r = recs[i]
            out.append({f: getattr(r, f) for f, _ in TrajRec._fields_})
            total = max(total, r.tok_offset + r.len)
        return Harvest(out, toks[:total].copy(), lps[:total].copy(), vers[:total].copy())

    def set_cache_bound(self, K: int):
        return check(self.lib.srl_set_cache_bound(self.h, int(K)), "srl_set_cache_bound")

    # ------------------------------------------------------------------ introspection
    def trace(self, start: int = 0, cap: int = 1 << 20):
        recs = (TraceRec * cap)()
        n, tot = C.c_int32(), C.c_int64()
        check(self.lib.srl_get_trace(self.h, start, cap, recs, C.byref(n), C.byref(tot)), "srl_get_trace")
        return [(recs[i].kind, recs[i].a, recs[i].b, recs[i].c, recs[i].d, recs[i].e) for i in range(n.value)], tot.value

    def counters(self):
        v = [C.c_int64() for _ in range(5)]
        check(self.lib.srl_get_counters(self.h, *[C.byref(x) for x in v]), "srl_get_counters")
        return dict(zip(["raw_tokens", "discarded_tokens", "emitted", "groups", "kernel_launches"], [x.value for x in v]))

    def set_profiling(self, on: bool, classes=None):
        """classes: iterable of _lib.KERNEL_CLASSES names to bracket (default all)."""
        mask = 0xFFFFFFFF if classes is None else sum(1 << _lib.KERNEL_CLASSES.index(c) for c in classes)
        check(self.lib.srl_set_profile_mask(self.h, mask), "srl_set_profile_mask")
        return check(self.lib.srl_set_profiling(self.h, 1 if on else 0), "srl_set_profiling")

    def set_profile_mask(self, classes=None):
        """Bracket only `classes` (default all) from the next step on; the decode graphs
        are cached per class set, so switching is free after each set's first capture."""
        mask = 0xFFFFFFFF if classes is None else sum(1 << _lib.KERNEL_CLASSES.index(c) for c in classes)
        return check(self.lib.srl_set_profile_mask(self.h, mask), "srl_set_profile_mask")

    def profile(self):
        """{class: (device ms, launches)} accumulated since set_profiling(True)."""
        ms = (C.c_double * len(_lib.KERNEL_CLASSES))()
        nl = (C.c_int64 * len(_lib.KERNEL_CLASSES))()
        check(self.lib.srl_get_profile(self.h, ms, nl), "srl_get_profile")
        return {k: (ms[i], nl[i]) for i, k in enumerate(_lib.KERNEL_CLASSES)}

    def debug_logits(self) -> np.ndarray:
        out = np.full((self.Q_g, self.V), np.nan, dtype=np.float32)   # rows of idle slots stay NaN
        check(self.lib.srl_debug_copy_logits(self.h, _i32p(out), out.size), "srl_debug_copy_logits")
        return out

    def close(self):
        if self.h:
            self.lib.srl_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def events_to_oracle_form(trace):
    """Convert the engine's trace records into the oracle's event tuples
    (oracle/sched.py) and the (k, r_k) step trace."""
    ev, steps = [], []
    i = 0
    while i < len(trace):
        kind, a, b, c, d, e = trace[i]
        name = EV_NAMES[kind]
        if name == "STEP":
            steps.append((a, b))
        elif name == "LOAD":
            ev.append(("LOAD", a, b, c, d))
        elif name in ("ADMIT", "PREEMPT", "FINISH"):
            ev.append((name, a, b, c, d))
        elif name == "EMIT":
            members = tuple(trace[i + 1 + j][3] for j in range(c))
            ev.append(("EMIT", a, b, members, d))
            i += c
        elif name == "DISCARD":
            ev.append(("DISCARD", a, b, {1: "pending", 2: "running", 3: "ready"}[c]))
        elif name == "SCAVENGE":
            ev.append(("SCAVENGE", a, b, c))
        i += 1
    return ev, steps
