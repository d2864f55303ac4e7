"""ctypes loader for ``libsrl.so`` — argument marshalling only.

Every computation behind these names runs in the sm_100a library; if the
library is missing this module raises instead of falling back to anything.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsrl.so")

_P = C.c_void_p
_I32 = C.c_int32
_I64 = C.c_int64
_U64 = C.c_uint64
_F32P = C.POINTER(C.c_float)

class ModelCfg(C.Structure):
    _fields_ = [("L", _I32), ("d", _I32), ("Hq", _I32), ("Hkv", _I32), ("dh", _I32), ("ff", _I32), ("V", _I32),
                ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("qkv_bias", _I32), ("weights_compact", _I32)]


class SchedCfg(C.Structure):
    _fields_ = [("Q_g", _I32), ("U", _I32), ("K", _I32), ("pool_prompts", _I32), ("G", _I32), ("cap", _I32),
                ("page_tokens", _I32), ("kv_pages", _I32), ("mode", _I32), ("resume", _I32), ("barrier", _I32),
                ("stop", _I32), ("eos_id", _I32), ("kv_dtype", _I32), ("temperature", C.c_float),
                ("sample_seed", _U64), ("max_traj", _I32), ("max_prompt", _I32), ("prefill_chunk", _I32),
                ("top_k", _I32), ("top_p", C.c_float), ("share_prefix", _I32), ("prefill_budget", _I32)]


COMM_NCCL, COMM_LOCAL, COMM_HOST = 0, 1, 2   # srl.h SRL_COMM_*

# srl_host_transport callbacks: int32 (*)(void* ctx, void* buf, uint64 bytes)
HOST_FN = C.CFUNCTYPE(_I32, _P, _P, _U64)


class HostTransport(C.Structure):
    _fields_ = [("allgather", HOST_FN), ("broadcast", HOST_FN), ("ctx", _P)]


class Comm(C.Structure):
    _fields_ = [("rank", _I32), ("world", _I32), ("kind", _I32), ("timeout_s", _I32), ("local_group", _P),
                ("host", C.POINTER(HostTransport)), ("nccl_unique_id", C.c_uint8 * 128)]


class Arena(C.Structure):
    _fields_ = [("weights", _P), ("kv", _P), ("scratch", _P), ("weights_bytes", _U64), ("kv_bytes", _U64),
                ("scratch_bytes", _U64)]


class StepInfo(C.Structure):
    _fields_ = [("k", _I64), ("r_k", _I32), ("n_finished", _I32), ("n_ready", _I32), ("n_admitted", _I32),
                ("n_prefill_tokens", _I32), ("v", _I32), ("dt_ms", C.c_float), ("sum_ctx", _I64),
                ("r_local", _I32), ("pad_", _I32)]


KERNEL_CLASSES = ["gemm_qkv", "gemm_o", "gemm_gate_up", "gemm_down", "lm_head", "attention", "elementwise",
                  "sample", "controller", "prefill", "exchange"]


class TrajRec(C.Structure):
    _fields_ = [("prompt_id", _I64), ("tok_offset", _I64), ("traj_id", _I32), ("sample", _I32), ("len", _I32),
                ("v_first", _I32), ("v_last", _I32), ("finish_step", _I32), ("lifecycle", _I32),
                ("restarts", _I32), ("final_group", _I32), ("epoch", _I32)]


class TraceRec(C.Structure):
    _fields_ = [("kind", _I32), ("a", _I32), ("b", _I32), ("c", _I32), ("d", _I32), ("e", _I32)]


class Tuning(C.Structure):
    """srl.h srl_tuning: process-wide kernel selection (defaults = production)."""
    _fields_ = [(n, _I32) for n in ("gemm_split", "gemm_pair", "gemm_h", "gemm_stages", "gemm_xstages",
                                    "partial_norm", "partial_small_m", "qkv_finish", "fused_sample",
                                    "attn_min_items", "attn_target_items", "attn_l2_prefetch", "pdl", "graphs",
                                    "mixed_prefill", "verbose", "fuse_mlp", "mlp_splits", "attn_stages", "qkv_attn",
                                    "pair_h2")]


_MP, _SP, _AP, _CP = C.POINTER(ModelCfg), C.POINTER(SchedCfg), C.POINTER(Arena), C.POINTER(Comm)
_U64P, _I64P, _I32P = C.POINTER(_U64), C.POINTER(_I64), C.POINTER(_I32)

# name -> (restype, argtypes)
SIGNATURES = {
    "srl_last_error": (C.c_char_p, []),
    "srl_op_gemm_bf16": (_I32, [_P, _I32, _P, _I32, _I32, _I32, _P, _P, _P]),
    "srl_op_gemm_workspace": (_I64, [_I32, _I32, _I32, _I32]),
    "srl_op_packed_weight_bytes": (_I64, [_I32, _I32]),
    "srl_op_mlp_bf16": (_I32, [_P, _I32, _P, _P, _I32, _I32, _I32, _P, _P, _P, _P]),
    "srl_op_pack_weight": (_I32, [_P, _I32, _I32, _P, _P]),
    "srl_op_attention_workspace": (_I64, [_I32, _I32, _I32, _I32, _I32]),
    "srl_op_attention": (_I32, [_P, _P, _P, _I32, _P, _I32, _P, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P, _P]),
    "srl_op_sample": (_I32, [_P, _I32, _I32, _P, _P, _P, C.c_float, _U64, _P, _P, _P, _P]),
    "srl_op_sample_trunc": (_I32, [_P, _I32, _I32, _P, _P, _P, C.c_float, _U64, _I32, C.c_float, _P, _P, _P, _P]),
    "srl_arena_sizes": (_I32, [_MP, _SP, _I32, _U64P, _U64P, _U64P]),
    "srl_weight_offset": (_I64, [_MP, C.c_char_p, _I64P]),
    "srl_weight_layout": (_I32, [_MP, C.c_char_p, _I64P, _I64P, _I64P, _I64P, _I64P]),
    "srl_create": (_I32, [_MP, _SP, _I32, _P, _AP, _CP, C.POINTER(_P)]),
    "srl_destroy": (_I32, [_P]),
    "srl_submit_prompts": (_I32, [_P, _I32, _P, _P, _P, _P]),
    "srl_decode_step": (_I32, [_P, C.POINTER(StepInfo)]),
    "srl_harvest_finished": (_I32, [_P, _I32, C.POINTER(TrajRec), _I32P, _P, _P, _P, _I64]),
    "srl_load_policy_weights": (_I32, [_P, _P, _I64]),
    "srl_get_trace": (_I32, [_P, _I64, _I32, C.POINTER(TraceRec), _I32P, _I64P]),
    "srl_get_counters": (_I32, [_P, _I64P, _I64P, _I64P, _I64P, _I64P]),
    "srl_set_cache_bound": (_I32, [_P, _I32]),
    "srl_debug_copy_logits": (_I32, [_P, _P, _I64]),
    "srl_set_profiling": (_I32, [_P, _I32]),
    "srl_set_profile_mask": (_I32, [_P, C.c_uint32]),
    "srl_get_profile": (_I32, [_P, C.POINTER(C.c_double), _I64P]),
    "srl_nccl_unique_id": (_I32, [_P]),
    "srl_load_policy_tensor": (_I32, [_P, C.c_char_p, _P]),
    "srl_local_group_create": (_I32, [_I32, C.POINTER(_P)]),
    "srl_local_group_destroy": (_I32, [_P]),
    "srl_harvest_device": (_I32, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), _I32P, _I64P]),
    "srl_learner_reinforcepp": (_I32, [_P, _I32, _P, _P]),
    "srl_learner_expand": (_I32, [_P, _P, _I32, _P, _P]),
    "srl_learner_gae": (_I32, [_P, _P, _P, _I32, C.c_float, C.c_float, _P, _P]),
    "srl_learner_ppo_workspace": (_I64, [_I64]),
    "srl_learner_ppo_objective": (_I32, [_P, _P, _P, _I64, C.c_float, C.c_float, _P, _P, _P, _P, _P]),
    "srl_learner_staleness": (_I32, [_P, _I64, _I32, _I32, _P, _P]),
    "srl_default_tuning": (None, [C.POINTER(Tuning)]),
    "srl_get_tuning": (_I32, [C.POINTER(Tuning)]),
    "srl_set_tuning": (_I32, [C.POINTER(Tuning)]),
}

GEMM_W_PACKED = 0x100   # srl_ops.h SRL_GEMM_W_PACKED

_lib = None


class SRLError(RuntimeError):
    pass


def load():
    """Load the library (building it first if absent and nvcc is present)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> int:
    if rc < 0:
        raise SRLError(f"{what} failed ({rc}): {load().srl_last_error().decode()}")
    return rc


def get_tuning() -> dict:
    t = Tuning()
    check(load().srl_get_tuning(C.byref(t)), "srl_get_tuning")
    return {n: getattr(t, n) for n, _ in Tuning._fields_}


def set_tuning(**fields) -> dict:
    """Change some srl_tuning fields (the rest keep their values); returns the
    previous settings, so `set_tuning(**old)` restores them.  defaults=True first
    resets every field to srl_default_tuning."""
    lib = load()
    old = get_tuning()
    t = Tuning()
    if fields.pop("defaults", False):
        lib.srl_default_tuning(C.byref(t))
    else:
        check(lib.srl_get_tuning(C.byref(t)), "srl_get_tuning")
    for k, v in fields.items():
        if k not in old:
            raise KeyError(f"unknown srl_tuning field {k}")
        setattr(t, k, int(v))
    check(lib.srl_set_tuning(C.byref(t)), "srl_set_tuning")
    return old
