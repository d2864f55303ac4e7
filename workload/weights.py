"""Counter-based random-init policy weights (bf16), identical on CPU and GPU.

Every element is a pure function of (seed, tensor name, policy version,
element index), computed with 32-bit integer hashing and exactly-rounded fp32
operations, then rounded to bf16 (round-to-nearest-even).  The numpy and the
torch implementations below therefore produce the same bits, so the oracle and
the GPU path consume identical weights without shipping gigabytes around.

Recipe (SURVEY §8(c) O-W and reading Q28):
  matrices     uniform, std 0.02          (a = 0.02*sqrt(3))
  qkv biases   uniform, std 0.5           (so the bias path is visible)
  norm weights 1 + uniform(-0.125, 0.125)
  version v    W_v = bf16(base + v * delta), delta = 0.1 * (independent draw)
"""
from __future__ import annotations

import math
import zlib

import numpy as np

from .configs import ModelShape

_A_MAT = np.float32(0.02 * math.sqrt(3.0))
_A_BIAS = np.float32(0.5 * math.sqrt(3.0))
_A_NORM = np.float32(0.125)
_DELTA = np.float32(0.1)
_M32 = 0xFFFFFFFF


def weight_names(m: ModelShape):
    names = ["embed"]
    for l in range(m.L):
        p = f"L{l}."
        names += [p + "attn_norm", p + "wq", p + "wk", p + "wv"]
        if m.qkv_bias:
            names += [p + "bq", p + "bk", p + "bv"]
        names += [p + "wo", p + "mlp_norm", p + "wg", p + "wu", p + "wd"]
    names += ["final_norm", "lm_head"]
    return names


def weight_shape(m: ModelShape, name: str):
    base = name.split(".")[-1]
    return {
        "embed": (m.V, m.d), "lm_head": (m.V, m.d), "final_norm": (m.d,),
        "attn_norm": (m.d,), "mlp_norm": (m.d,),
        "wq": (m.Hq * m.dh, m.d), "wk": (m.Hkv * m.dh, m.d), "wv": (m.Hkv * m.dh, m.d),
        "bq": (m.Hq * m.dh,), "bk": (m.Hkv * m.dh,), "bv": (m.Hkv * m.dh,),
        "wo": (m.d, m.Hq * m.dh), "wg": (m.ff, m.d), "wu": (m.ff, m.d), "wd": (m.d, m.ff),
    }[base]


def _kind(name: str) -> str:
    base = name.split(".")[-1]
    if base.endswith("norm"):
        return "norm"
    if base in ("bq", "bk", "bv"):
        return "bias"
    return "mat"


def _key(seed: int, name: str, stream: int) -> int:
    return (zlib.crc32(name.encode()) ^ (seed * 0x9E3779B1) ^ (stream * 0x85EBCA77)) & _M32


# ------------------------------------------------------------------ numpy
def _lowbias32_np(h: np.ndarray) -> np.ndarray:
    h = h ^ (h >> np.uint32(16))
    h = h * np.uint32(0x7FEB352D)
    h = h ^ (h >> np.uint32(15))
    h = h * np.uint32(0x846CA68B)
    h = h ^ (h >> np.uint32(16))
    return h


def _u24_np(idx: np.ndarray, key: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = _lowbias32_np(idx.astype(np.uint32) ^ np.uint32(key))
        h = _lowbias32_np(h ^ np.uint32((key * 0x9E3779B9) & _M32))
    # signed uniform in [-1, 1): exact in fp32
    return ((h >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -23)) - np.float32(1.0)


def _f32_to_bf16_bits_np(x: np.ndarray) -> np.ndarray:
    b = x.astype(np.float32).view(np.uint32)
    b = (b + (np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1)))) >> np.uint32(16)
    return b.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def _value_np(kind: str, idx: np.ndarray, seed: int, name: str, version: int) -> np.ndarray:
    s = _u24_np(idx, _key(seed, name, 0))
    if kind == "norm":
        v = np.float32(1.0) + s * _A_NORM
    else:
        v = s * (_A_MAT if kind == "mat" else _A_BIAS)
    if version:
        dlt = _u24_np(idx, _key(seed, name, 1)) * (_A_MAT if kind != "bias" else _A_BIAS) * _DELTA
        v = v + np.float32(version) * dlt
    return v.astype(np.float32)


def gen_weight_np(m: ModelShape, name: str, seed: int = 2, version: int = 0, rows=None) -> np.ndarray:
    """bf16 bit pattern (uint16) of weight `name`; `rows` selects a subset of rows."""
    shape = weight_shape(m, name)
    ncol = shape[1] if len(shape) == 2 else 1
    if rows is None:
        idx = np.arange(int(np.prod(shape)), dtype=np.int64)
        out_shape = shape
    else:
        rows = np.asarray(rows, dtype=np.int64)
        idx = (rows[:, None] * ncol + np.arange(ncol, dtype=np.int64)[None, :]).reshape(-1)
        out_shape = (len(rows), ncol) if len(shape) == 2 else (len(rows),)
    v = _value_np(_kind(name), idx, seed, name, version)
    return _f32_to_bf16_bits_np(v).reshape(out_shape)


def fill_engine_weights(eng, m: ModelShape, version: int = 0, seed: int = 2, flat=None):
    """Write the version-`version` policy into an engine's flat weight region
    (`eng.weight_view(name)` gives each tensor), or into `flat`, a uint8 tensor
    with the same layout."""
    import torch
    if getattr(eng, "compact", False) and flat is None:
        # compact engines hold projections only packed: install tensor by tensor
        for name in weight_names(m):
            t = gen_weight_torch(m, name, seed=seed, version=version, device=eng.W.device)
            eng.load_policy_tensor(name, t)
            eng.stream.synchronize()
            del t
        return
    for name in weight_names(m):
        view = eng.weight_view(name)
        if flat is not None:   # same layout inside `flat`
            base = flat.view(torch.bfloat16)
            view = base.as_strided(view.shape, view.stride(), view.storage_offset())
        if view.is_contiguous():
            gen_weight_torch(m, name, seed=seed, version=version, device=view.device,
                             out=view.view(*weight_shape(m, name)))
        else:                  # block-interleaved gate/up rows
            tmp = gen_weight_torch(m, name, seed=seed, version=version, device=view.device)
            view.copy_(tmp.view(view.shape))
            del tmp


# ------------------------------------------------------------------ torch (same bits, on device)
def _lowbias32_t(h):
    h = h ^ (h >> 16)
    h = (h * 0x7FEB352D) & _M32
    h = h ^ (h >> 15)
    h = (h * 0x846CA68B) & _M32
    h = h ^ (h >> 16)
    return h


def _u24_t(idx, key: int):
    import torch
    h = _lowbias32_t((idx & _M32) ^ key)
    h = _lowbias32_t(h ^ ((key * 0x9E3779B9) & _M32))
    return (h >> 8).to(torch.float32) * (2.0 ** -23) - 1.0


def gen_weight_torch(m: ModelShape, name: str, seed: int = 2, version: int = 0, device="cuda",
                     out=None, chunk: int = 1 << 26):
    """Same values as gen_weight_np, as a torch.bfloat16 tensor on `device`."""
    import torch
    shape = weight_shape(m, name)
    n = int(np.prod(shape))
    if out is None:
        out = torch.empty(shape, dtype=torch.bfloat16, device=device)
    flat = out.view(-1)
    kind = _kind(name)
    a = float(_A_MAT if kind == "mat" else (_A_BIAS if kind == "bias" else _A_NORM))
    ad = float(_A_MAT if kind != "bias" else _A_BIAS)
    k0, k1 = _key(seed, name, 0), _key(seed, name, 1)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = torch.arange(s, e, dtype=torch.int64, device=device)
        u = _u24_t(idx, k0)
        # fp32 ops, each exactly rounded, in the same order as _value_np
        if kind == "norm":
            v = torch.mul(u, torch.tensor(a, dtype=torch.float32, device=device))
            v = torch.add(v, torch.tensor(1.0, dtype=torch.float32, device=device))
        else:
            v = torch.mul(u, torch.tensor(a, dtype=torch.float32, device=device))
        if version:
            d = torch.mul(_u24_t(idx, k1), torch.tensor(ad, dtype=torch.float32, device=device))
            d = torch.mul(d, torch.tensor(float(_DELTA), dtype=torch.float32, device=device))
            d = torch.mul(d, torch.tensor(float(version), dtype=torch.float32, device=device))
            v = torch.add(v, d)
        flat[s:e] = v.to(torch.bfloat16)
        del idx, u, v
    return out
