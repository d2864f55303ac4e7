"""Seeded synthetic input generators shared by the CPU oracle and the GPU path.

This package holds NONE of the method's arithmetic (no decode math, no
sampling, no scheduling): only configuration records and counter-based
generators of the inputs both sides consume (response-length targets, prompt
tokens, model weights).  See DESIGN.md "Input recipe".
"""
from .configs import ModelShape, SchedConfig, TINY, LLAMA8B, QWEN32B, model_by_name  # noqa: F401
from .lengths import LengthModel, sample_lengths  # noqa: F401
from .prompts import make_prompts  # noqa: F401
from .weights import weight_names, weight_shape, gen_weight_np, gen_weight_torch, bf16_bits_to_f32  # noqa: F401
