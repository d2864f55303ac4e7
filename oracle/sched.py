"""The SortedRL controller + stateful rollout buffer, step by step (CPU oracle).

TEST INFRASTRUCTURE ONLY (oracle/__init__.py).  Written from PAPER.md:
  P:163–167 §3.1  oversubscription: feed more prompts than the queue capacity Q
  P:169           early termination on a batching threshold (reading R4: |ready| >= U)
  P:171–173       grouped rollout + cache-aware loading ("no new prompts are loaded
                  ... until all cached prompts have been consumed")
  P:177           selective batching: ready trajectories fed "in a dedicated order"
                  (reading R6: ascending (response length, traj_id))
  P:180 §3.2      fully on-policy (terminate + scavenge prompts) vs partial mode
                  (scavenge tokens + logprobs, concatenate on resume)
  P:196–200 §3.3  state manager and buffer entry {prompt, partial trajectory,
                  logprobs, completion flag, lifecycle}
  P:353 §4.4.3    group size n: pool of n*b prompts, no reload until every sample
                  of the current buffer has been fed to the trainer
  P:338–342       Eq. (bubble) trace records (k, r_k)
  P:235, P:387    G > 1 responses per prompt; RadixAttention-style sharing of the
                  prompt's KV pages among them (`share_prefix`)
  P:32, P:180     chunked prefill (Sarathi) of admitted prompts (+ the kept
                  tokens a resumed trajectory re-feeds) under a per-step,
                  per-replica token budget (`prefill_budget`,
                  reading R30)
and the DESIGN.md readings R1–R28 (SURVEY §8(c) O-C pseudo-code).  The two
paper modes are the cache bound K (policy versions) at its extremes: K = 0 is
fully on-policy, K = inf is partial mode; intermediate K generalises them.

Everything here is integer bookkeeping; the token values come from a pluggable
`runner` (a dummy one for pure scheduling, oracle.model for end-to-end runs).
"""
from __future__ import annotations

import bisect
from dataclasses import dataclass, field
from typing import List, Optional

from workload.configs import (BARRIER_ADMITTED, BARRIER_TRAINED, MODE_POSTHOC, MODE_SORTED, MODE_SYNC,
                              RESUME_REPREFILL, STOP_EOS, STOP_FORCED, SchedConfig)

# status codes (match include/srl.h)
OK, GROUP_READY, DONE = 0, 1, 2


class SchedError(Exception):
    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclass
class Traj:
    tid: int
    prompt_id: int
    sample: int
    prompt_len: int
    forced_len: int
    epoch: int = -1
    tokens: List[int] = field(default_factory=list)
    lps: List[float] = field(default_factory=list)
    vers: List[int] = field(default_factory=list)
    v_first: Optional[int] = None
    lifecycle: int = 0
    restarts: int = 0
    admit_step: int = -1
    finish_step: int = -1
    state: str = "stream"       # stream | pending | running | ready | emitted
    slot: int = -1
    pages: int = 0
    shared: int = 0             # prompt-prefix pages held through the replica's shared entry
    fresh: bool = True
    pre_next: int = -1          # N1: next prefill position (-1: prefill not started since admission)
    pre_end: int = 0            # N1: prefill positions [.., pre_end) = prompt ++ kept tokens minus the last


class DummyRunner:
    """Token source for pure scheduling runs: token 0, logprob 0."""

    def admit(self, t: Traj, version: int):
        pass

    def prefill(self, t: Traj, a: int, b: int, version: int):
        pass

    def release(self, t: Traj):
        pass

    def step(self, batch, version):
        return [(0, 0.0) for _ in batch]


class Controller:
    def __init__(self, cfg: SchedConfig, runner=None):
        if cfg.Q_g <= 0 or cfg.R <= 0 or cfg.U <= 0 or cfg.G <= 0 or cfg.cap <= 0 or cfg.pool_prompts <= 0:
            raise SchedError("INVALID_ARG", "Q_g, R, U, G, cap, pool_prompts must be positive")
        if cfg.page_tokens <= 0 or cfg.kv_pages <= 0:
            raise SchedError("INVALID_ARG", "page_tokens and kv_pages must be positive")
        if cfg.mode in (MODE_SORTED, MODE_POSTHOC) and cfg.U > cfg.pool_prompts * cfg.G:
            raise SchedError("INVALID_ARG", "U larger than the prompt pool (S:252)")
        if cfg.stop == STOP_EOS and cfg.eos_id < 0:
            raise SchedError("INVALID_ARG", "EOS stop needs eos_id")
        if cfg.prefill_budget < 0:
            raise SchedError("INVALID_ARG", "prefill_budget must be >= 0 (0 = unlimited)")
        if cfg.prefill_budget > 0 and cfg.share_prefix and cfg.G > 1:
            # a shared prefix prefilled across a version bump would mix versions (R30)
            raise SchedError("INVALID_ARG", "prefill_budget and share_prefix are exclusive")
        self.cfg = cfg
        self.runner = runner or DummyRunner()
        Q = cfg.Q_tot
        self.slots: List[Optional[Traj]] = [None] * Q
        self.free_pages = [cfg.kv_pages] * cfg.R
        self.stream: List[Traj] = []
        self.prompt_ids = set()
        self.next_stream = 0
        self.epoch = 0
        self.epoch_of_latest = -1
        self.resumed: List[tuple] = []   # sorted keys (-lifecycle, tid) of non-fresh pending
        self.fresh: List[Traj] = []      # FIFO of fresh pending (ascending tid)
        self.fresh_head = 0
        self.ready: List[Traj] = []
        self.v: Optional[int] = None
        self.k = 0
        self.group: Optional[List[Traj]] = None
        self.group_final = False
        self.harvested = False
        self.n_groups = 0
        self.trace: List[tuple] = []     # (k, r_k)
        self.events: List[tuple] = []
        self.raw_tokens = 0
        self.discarded_tokens = 0
        self.loaded = 0                  # trajectories loaded so far
        self.emitted = 0
        self.work_conserving: List[bool] = []
        self._page_blocked = False
        # N4 prompt-prefix sharing: per (replica, prompt index) the shared entry's
        # holder count and the policy version its KV was computed under
        self.pfx_ref = {}
        self.pfx_tag = {}
        self.pfx_done = {}               # the entry's shared positions have been prefilled
        self.prefill_trace: List[tuple] = []   # (k, per-replica prefill tokens of step k)

    # ------------------------------------------------------------ submission
    def submit_prompts(self, prompt_ids, prompt_lens, forced_len=None):
        """Append prompts to the dataloader stream (traj_id = prompt_index*G + sample)."""
        cfg = self.cfg
        prompt_ids = list(prompt_ids)
        n = len(prompt_ids)
        if len(set(prompt_ids)) != n or any(p in self.prompt_ids for p in prompt_ids):
            raise SchedError("DUPLICATE_ID", "prompt id submitted twice (S:114)")
        if forced_len is not None:
            if len(forced_len) != n * cfg.G or any(not (1 <= int(L) <= cfg.cap) for L in forced_len):
                raise SchedError("INVALID_ARG", "forced_len must have n*G entries in [1, cap]")
        elif cfg.stop == STOP_FORCED:
            raise SchedError("INVALID_ARG", "FORCED stop mode needs forced_len")
        if any(int(p) < 1 for p in prompt_lens):
            raise SchedError("INVALID_ARG", "empty prompt")
        base = len(self.prompt_ids)
        for i in range(n):
            for s in range(cfg.G):
                tid = (base + i) * cfg.G + s
                L = int(forced_len[i * cfg.G + s]) if forced_len is not None else cfg.cap
                self.stream.append(Traj(tid, int(prompt_ids[i]), s, int(prompt_lens[i]), L))
        self.prompt_ids.update(prompt_ids)

    # ------------------------------------------------------------ helpers
    def _push_pending(self, t: Traj):
        t.state = "pending"
        t.slot = -1
        if t.fresh:
            self.fresh.append(t)
        else:
            bisect.insort(self.resumed, (-t.lifecycle, t.tid, t))

    def _pending_empty(self) -> bool:
        return not self.resumed and self.fresh_head >= len(self.fresh)

    def _peek_pending(self) -> Traj:
        if self.resumed:
            return self.resumed[0][2]
        return self.fresh[self.fresh_head]

    def _pop_pending(self) -> Traj:
        if self.resumed:
            return self.resumed.pop(0)[2]
        t = self.fresh[self.fresh_head]
        self.fresh_head += 1
        return t

    def _remove_pending(self, t: Traj):
        for i, e in enumerate(self.resumed):
            if e[2] is t:
                del self.resumed[i]
                return
        raise AssertionError("not in resumed pending")

    def _occupied(self):
        return [g for g, t in enumerate(self.slots) if t is not None]

    def _pages_needed(self, t: Traj) -> int:
        # positions 0 .. prompt_len + n - 1 hold KV after this step
        P = self.cfg.page_tokens
        return (t.prompt_len + len(t.tokens) + P - 1) // P

    def _prefix_pages(self, t: Traj) -> int:
        """N4 (P:387 RadixAttention, within an epoch): with share_prefix and G > 1 the
        full pages of prompt positions that every sample prefills -- [0, prompt_len - 1),
        the last prompt token being each sample's own first decode row -- are held
        once per replica and prompt, refcounted.  A new holder shares them only if
        they were computed under the current policy version (weights shift after
        every update); otherwise it keeps a private copy of the whole prompt."""
        cfg = self.cfg
        if not cfg.share_prefix or cfg.G <= 1:
            return 0
        return (t.prompt_len - 1) // cfg.page_tokens

    def _free_slot(self, g: int):
        t = self.slots[g]
        r = g % self.cfg.R
        self.free_pages[r] += t.pages
        if t.shared:
            key = (r, t.tid // self.cfg.G)
            self.pfx_ref[key] -= 1
            if self.pfx_ref[key] == 0:
                self.free_pages[r] += t.shared
            t.shared = 0
        t.pages = 0
        t.slot = -1
        self.slots[g] = None
        self.runner.release(t)

    def _load_possible(self) -> bool:
        cfg = self.cfg
        if self.next_stream >= len(self.stream):
            return False
        if self.loaded == 0:
            return True
        if cfg.mode in (MODE_SYNC, MODE_POSTHOC) or cfg.barrier == BARRIER_TRAINED:
            return self.emitted == self.loaded
        # ADMITTED: no trajectory of the latest epoch still pending
        for e in self.resumed:
            if e[2].epoch == self.epoch_of_latest:
                return False
        for t in self.fresh[self.fresh_head:]:
            if t.epoch == self.epoch_of_latest:
                return False
        return True

    def _drop_tokens(self, t: Traj):
        self.discarded_tokens += len(t.tokens)
        t.tokens, t.lps, t.vers = [], [], []
        t.v_first = None
        t.restarts += 1

    # ------------------------------------------------------------ controller steps
    def _maybe_load(self):
        cfg = self.cfg
        if not self._load_possible():
            return
        n = cfg.Q_tot if cfg.mode == MODE_SYNC else cfg.pool_prompts * cfg.G
        chunk = self.stream[self.next_stream:self.next_stream + n]
        self.next_stream += len(chunk)
        for t in chunk:
            t.epoch = self.epoch
            self._push_pending(t)
        self.events.append(("LOAD", self.k, self.epoch, chunk[0].tid, len(chunk)))
        self.epoch_of_latest = self.epoch
        self.epoch += 1
        self.loaded += len(chunk)

    def _refill(self):
        cfg = self.cfg
        self._page_blocked = False
        for g in range(cfg.Q_tot):
            if self.slots[g] is not None:
                continue
            if self._pending_empty():
                break
            t = self._peek_pending()
            need = self._pages_needed(t)
            r = g % cfg.R
            S = self._prefix_pages(t)
            key = (r, t.tid // cfg.G)
            ref = self.pfx_ref.get(key, 0)
            share = S > 0 and (ref == 0 or self.pfx_tag[key] == self.v)
            cost = need - S if (share and ref > 0) else need
            if self.free_pages[r] < cost:
                self._page_blocked = True
                break
            self._pop_pending()
            self.free_pages[r] -= cost
            t.pages = need - S if share else need
            t.shared = S if share else 0
            if share:
                if ref == 0:
                    self.pfx_tag[key] = self.v
                    self.pfx_done[key] = False
                self.pfx_ref[key] = ref + 1
            t.pre_next = -1
            t.pre_end = t.prompt_len + len(t.tokens) - 1
            t.slot = g
            t.state = "running"
            t.fresh = False
            if t.v_first is None:
                t.v_first = self.v
            t.admit_step = self.k
            self.slots[g] = t
            self.events.append(("ADMIT", self.k, g, t.tid, len(t.tokens)))
            self.runner.admit(t, self.v)

    def _preempt(self, g: int):
        t = self.slots[g]
        keep = self.cfg.K != 0 or self.cfg.mode == MODE_SYNC
        self._free_slot(g)
        t.lifecycle += 1
        if not keep:
            self._drop_tokens(t)
        elif not t.tokens:
            t.v_first = None          # admitted this step, nothing generated yet
        self.events.append(("PREEMPT", self.k, g, t.tid, int(keep)))
        self._push_pending(t)

    def _grow_pages(self):
        cfg = self.cfg
        for g in range(cfg.Q_tot):
            t = self.slots[g]
            if t is None:
                continue
            need = self._pages_needed(t) - t.shared
            r = g % cfg.R
            while t.pages < need and self.slots[g] is t:
                if self.free_pages[r] > 0:
                    self.free_pages[r] -= 1
                    t.pages += 1
                    continue
                cands = [h for h in range(r, cfg.Q_tot, cfg.R) if self.slots[h] is not None]
                if cands == [g]:
                    # alone on its replica and still short of pages: preempting itself
                    # cannot help (with K = 0 it would restart forever) -- reading R25
                    raise SchedError("CAPACITY", "a trajectory outgrows its replica's KV pool")
                victim = max(cands, key=lambda h: (self.slots[h].admit_step, h))
                self._preempt(victim)

    def _prefill(self):
        """N1 (reading R30): each replica prefills its admitted slots strictly in
        admission order (admit_step, then global slot), at most `prefill_budget`
        positions per step (0 = unlimited: every admission is prefilled in its own
        step, R13).  A slot starts at position 0, or -- N4 -- after its shared prompt
        pages when the entry's first holder has already prefilled them; a slot that is
        still short of its prefill after the budget stops the walk (later ones wait).
        A slot decodes in a step only once its prefill is complete (in that step or
        an earlier one).  Returns the per-replica prefill tokens of this step."""
        cfg = self.cfg
        C = cfg.prefill_budget if cfg.prefill_budget > 0 else None
        used = [0] * cfg.R
        for r in range(cfg.R):
            slots = sorted((self.slots[g].admit_step, g) for g in range(r, cfg.Q_tot, cfg.R)
                           if self.slots[g] is not None and self.slots[g].pre_next < self.slots[g].pre_end)
            for _, g in slots:
                t = self.slots[g]
                key = (r, t.tid // cfg.G)
                if t.pre_next < 0:
                    t.pre_next = t.shared * cfg.page_tokens if (t.shared and self.pfx_done[key]) else 0
                n = t.pre_end - t.pre_next
                if C is not None:
                    n = min(n, C - used[r])
                if n > 0:
                    self.runner.prefill(t, t.pre_next, t.pre_next + n, self.v)
                    t.pre_next += n
                    used[r] += n
                if t.shared and t.pre_next >= t.shared * cfg.page_tokens:
                    self.pfx_done[key] = True
                if t.pre_next < t.pre_end:
                    break
        return used

    def _emission_check(self) -> bool:
        cfg = self.cfg
        occupied = any(t is not None for t in self.slots)
        if cfg.mode == MODE_SYNC:
            if not self.ready or occupied or not self._pending_empty():
                return False
            group = self.ready[:cfg.U]
            self.ready = self.ready[cfg.U:]
            final = not self.ready
        else:
            # post-hoc sorting (ablation): nothing is emitted before the whole
            # loaded batch has finished; then sorted groups of U as in SortedRL
            if cfg.mode == MODE_POSTHOC and (occupied or not self._pending_empty()):
                return False
            drain = self._pending_empty() and not occupied and not self._load_possible()
            if len(self.ready) >= cfg.U:
                group = sorted(self.ready, key=lambda t: (len(t.tokens), t.tid))[:cfg.U]
                final = False
            elif drain and self.ready:
                group = sorted(self.ready, key=lambda t: (len(t.tokens), t.tid))
                final = True
            else:
                return False
            ids = {t.tid for t in group}
            self.ready = [t for t in self.ready if t.tid not in ids]
        for t in group:
            t.state = "emitted"
        self.emitted += len(group)
        self.group = group
        self.group_final = final
        self.harvested = False
        self.events.append(("EMIT", self.n_groups, self.v, tuple(t.tid for t in group), int(final)))
        self.n_groups += 1
        return True

    # ------------------------------------------------------------ public API
    def decode_step(self) -> int:
        cfg = self.cfg
        if self.group is not None:
            raise SchedError("STATE", "a group awaits harvest/load_policy_weights (P:30)")
        if self.v is None:
            raise SchedError("STATE", "no policy weights loaded")
        if self._emission_check():
            return GROUP_READY
        self._maybe_load()
        self._refill()
        self._grow_pages()
        pre = self._prefill()
        occ = self._occupied()
        # work conservation record: a free slot only if nothing is admissible
        self.work_conserving.append(len(occ) == cfg.Q_tot or self._pending_empty() or self._page_blocked)
        if not occ:
            if not self._pending_empty():
                raise SchedError("CAPACITY", "KV pool cannot hold the next admission")
            if not self.stream:
                raise SchedError("EMPTY", "nothing submitted (S:124)")
            return DONE
        # decode rows: the occupied slots whose prefill is complete (N1; all of them
        # without a budget)
        batch = [(g, self.slots[g]) for g in occ if self.slots[g].pre_next >= self.slots[g].pre_end]
        r_k = len(batch)
        self.prefill_trace.append((self.k, tuple(pre)))
        outs = self.runner.step(batch, self.v)
        finished = []
        for (g, t), (tok, lp) in zip(batch, outs):
            t.tokens.append(int(tok))
            t.lps.append(lp)
            t.vers.append(self.v)
            n = len(t.tokens)
            if ((cfg.stop == STOP_FORCED and n == t.forced_len) or
                    (cfg.stop == STOP_EOS and int(tok) == cfg.eos_id) or n == cfg.cap):
                finished.append(g)
        self.raw_tokens += r_k
        for g in finished:                       # ascending global slot order
            t = self.slots[g]
            t.finish_step = self.k
            self.events.append(("FINISH", self.k, g, t.tid, len(t.tokens)))
            self._free_slot(g)
            t.state = "ready"
            self.ready.append(t)
        self.trace.append((self.k, r_k))
        self.k += 1
        if self._emission_check():
            return GROUP_READY
        return OK

    def harvest(self):
        if self.group is None or self.harvested:
            raise SchedError("STATE", "no group is ready")
        recs = []
        for t in self.group:
            recs.append(dict(traj_id=t.tid, prompt_id=t.prompt_id, sample=t.sample, len=len(t.tokens),
                             v_first=t.v_first, v_last=t.vers[-1], finish_step=t.finish_step,
                             lifecycle=t.lifecycle, restarts=t.restarts, final=self.group_final,
                             tokens=list(t.tokens), lps=list(t.lps), vers=list(t.vers)))
        self.harvested = True
        return recs

    def load_policy_weights(self, version: int):
        cfg = self.cfg
        if self.group is not None and not self.harvested:
            raise SchedError("STATE", "harvest the ready group first")
        if self.v is not None and version <= self.v:
            raise SchedError("STATE", "policy version must increase")
        first = self.v is None
        self.v = int(version)
        self.group = None
        if first or cfg.mode == MODE_SYNC:
            return
        live = [t for t in self.stream[:self.next_stream] if t.state in ("running", "ready", "pending")]
        live.sort(key=lambda t: t.tid)
        for t in live:
            if cfg.K >= 0 and t.v_first is not None and self.v - t.v_first > cfg.K:
                where = t.state
                self.events.append(("DISCARD", self.v, t.tid, where))
                if where == "running":
                    self._free_slot(t.slot)
                elif where == "ready":
                    self.ready = [x for x in self.ready if x is not t]
                else:
                    self._remove_pending(t)
                self._drop_tokens(t)
                t.lifecycle += 1
                self._push_pending(t)
            elif cfg.resume == RESUME_REPREFILL and t.state == "running":
                self.events.append(("SCAVENGE", self.v, t.tid, t.slot))
                self._free_slot(t.slot)
                t.lifecycle += 1
                self._push_pending(t)

    # ------------------------------------------------------------ convenience
    def run(self, version0: int = 0, max_steps: int = 10 ** 9, on_group=None):
        """Drive the loop of SURVEY §3 item 2 to completion; returns the list of groups."""
        if self.v is None:
            self.load_policy_weights(version0)
        groups = []
        steps = 0
        while steps < max_steps:
            st = self.decode_step()
            if st == DONE:
                break
            if st == GROUP_READY:
                recs = self.harvest()
                groups.append(recs)
                if on_group:
                    on_group(self, recs)
                self.load_policy_weights(self.v + 1)
            else:
                steps += 1
        return groups
