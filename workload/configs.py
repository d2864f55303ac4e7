"""Configuration records (plain data) for the model shapes and the scheduler.

Model shapes are the public LLaMA-3.1-8B / Qwen-2.5-32B configurations named
by the paper ("LLaMA-3.1-8B", "Qwen-2.5-32B"); the paper
itself prints no dimensions (reading R19).  Weights are random-init.
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict


@dataclass(frozen=True)
class ModelShape:
    name: str
    L: int          # layers
    d: int          # hidden size
    Hq: int         # query heads
    Hkv: int        # key/value heads (GQA)
    dh: int         # head dim
    ff: int         # MLP intermediate size
    V: int          # vocabulary
    rope_theta: float
    rms_eps: float = 1e-5
    qkv_bias: bool = False

    @property
    def qkv_out(self) -> int:
        return (self.Hq + 2 * self.Hkv) * self.dh

    def with_layers(self, L: int) -> "ModelShape":
        d = asdict(self)
        d["L"] = L
        d["name"] = f"{self.name}-L{L}"
        return ModelShape(**d)


TINY = ModelShape("tiny", L=2, d=128, Hq=4, Hkv=2, dh=32, ff=384, V=512, rope_theta=1e4)
LLAMA8B = ModelShape("llama3.1-8b", L=32, d=4096, Hq=32, Hkv=8, dh=128, ff=14336, V=128256,
                     rope_theta=5e5)
QWEN32B = ModelShape("qwen2.5-32b", L=64, d=5120, Hq=40, Hkv=8, dh=128, ff=27648, V=152064,
                     rope_theta=1e6, qkv_bias=True)


def model_by_name(name: str) -> ModelShape:
    for m in (TINY, LLAMA8B, QWEN32B):
        if m.name == name:
            return m
    raise KeyError(name)


# Scheduler enums (values match include/srl.h)
MODE_SORTED, MODE_SYNC, MODE_POSTHOC = 0, 1, 2
RESUME_KEEP_KV, RESUME_REPREFILL = 0, 1
BARRIER_TRAINED, BARRIER_ADMITTED = 0, 1
STOP_FORCED, STOP_EOS = 0, 1
KV_BF16, KV_FP32 = 0, 1
K_INF = -1


@dataclass
class SchedConfig:
    """SortedRL controller parameters (SURVEY §8(b) srl_sched_cfg).

    Q_g  running-queue slots per GPU ("Q ... running queue size")
    R    data-parallel replicas; Q_tot = R * Q_g
    U    update-group size ("update batch size")
    K    off-policy cache bound in policy versions, -1 = infinity
    pool_prompts  n*b prompts loaded per epoch
    G    responses per prompt
    cap  max generation length
    """
    Q_g: int = 16
    R: int = 1
    U: int = 4
    K: int = K_INF
    pool_prompts: int = 16
    G: int = 1
    cap: int = 64
    page_tokens: int = 64
    kv_pages: int = 1 << 20          # pages per replica
    mode: int = MODE_SORTED
    resume: int = RESUME_KEEP_KV
    barrier: int = BARRIER_TRAINED
    stop: int = STOP_FORCED
    eos_id: int = -1
    kv_dtype: int = KV_FP32
    temperature: float = 1.0
    sample_seed: int = 3
    top_k: int = 0                   # N4: 0 = no top-k truncation
    top_p: float = 1.0               # N4: 1 = no nucleus truncation
    share_prefix: int = 0            # N4: G > 1 samples of a prompt share its prompt-prefix KV pages
    prefill_budget: int = 0          # N1: prefill tokens per replica per step (0 = unlimited)

    @property
    def Q_tot(self) -> int:
        return self.R * self.Q_g
