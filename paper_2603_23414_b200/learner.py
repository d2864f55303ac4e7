"""Thin binding of include/srl_learner.h (argument marshalling only): the update
group's consumer on the GPU -- PAPER.md Eq. (1) clipped objective, Eq. (2) GAE,
Eq. (3) Reinforce++ advantages, token staleness.  Inputs / outputs are torch
CUDA tensors; every computation runs in libsrl.so."""
from __future__ import annotations

import ctypes as C

from . import _lib
from ._lib import check


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(t):
    import torch
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def reinforcepp(rewards):
    """Eq. (3): float32 [n] -> advantages [n]."""
    import torch
    adv = torch.empty_like(rewards)
    check(_lib.load().srl_learner_reinforcepp(_p(rewards), rewards.numel(), _p(adv), _stream(rewards)),
          "srl_learner_reinforcepp")
    return adv


def expand(per_traj, tok_off):
    """per-trajectory values -> per token (tok_off int64 [n + 1])."""
    import torch
    out = torch.empty(int(tok_off[-1].item()), dtype=torch.float32, device=per_traj.device)
    check(_lib.load().srl_learner_expand(_p(per_traj), _p(tok_off), per_traj.numel(), _p(out), _stream(per_traj)),
          "srl_learner_expand")
    return out


def gae(rewards, values, tok_off, gamma: float, lam: float):
    """Eq. (2): per-token rewards, values with one bootstrap entry per trajectory."""
    import torch
    adv = torch.empty_like(rewards)
    check(_lib.load().srl_learner_gae(_p(rewards), _p(values), _p(tok_off), tok_off.numel() - 1, float(gamma),
                                      float(lam), _p(adv), _stream(rewards)), "srl_learner_gae")
    return adv


def ppo_objective(new_lp, old_lp, adv, eps_low: float, eps_high: float):
    """Eq. (1): (ratio [n], d term / d new_lp [n], objective 0-dim float64 tensor)."""
    import torch
    lib = _lib.load()
    n = new_lp.numel()
    ratio, dterm = torch.empty_like(new_lp), torch.empty_like(new_lp)
    obj = torch.empty((), dtype=torch.float64, device=new_lp.device)
    ws = torch.empty(lib.srl_learner_ppo_workspace(n), dtype=torch.uint8, device=new_lp.device)
    check(lib.srl_learner_ppo_objective(_p(new_lp), _p(old_lp), _p(adv), n, float(eps_low), float(eps_high),
                                        _p(ratio), _p(dterm), _p(obj), _p(ws), _stream(new_lp)),
          "srl_learner_ppo_objective")
    return ratio, dterm, obj


def staleness(versions, v_update: int, nbins: int = 64):
    """int32 [nbins] histogram of v_update - version over tokens (last bin: >= nbins - 1)."""
    import torch
    hist = torch.empty(nbins, dtype=torch.int32, device=versions.device)
    check(_lib.load().srl_learner_staleness(_p(versions), versions.numel(), int(v_update), nbins, _p(hist),
                                            _stream(versions)), "srl_learner_staleness")
    return hist
