"""Seeded synthetic inputs shared by the tests, the bench and the oracle's callers.

This package holds NO arithmetic of the method (no FLOPs model, no scheduling,
no packing, no attention). It only draws random sequence lengths and random
tensors, so that the CPU oracle (`oracle/`) and the CUDA path
(`paper_2505_19609_b200/`) can be fed the same inputs without sharing code.

Recipe:
  * lengths: numpy PCG64 `default_rng(seed)`; presets calibrated to PAPER.md
    Table 1 and the Llama-3 / Qwen2.5 mix statistics.
  * tensors: Q, K, V, dO ~ N(0, 1) per sequence from
    `default_rng((seed, seq_idx, tensor_id))`, rounded to bf16 (RNE).
"""
from .lengths import (PRESETS, gen_lengths, quantiles, forced_tail_batch)  # noqa: F401
from .configs import CONFIGS, get_config, Shape  # noqa: F401
from .tensors import seq_tensors, round_bf16  # noqa: F401
