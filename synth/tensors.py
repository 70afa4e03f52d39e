"""Seeded per-sequence attention inputs (SURVEY.md §8(d) "Tensor values").

Q, K, V, dO ~ N(0, sigma^2) fp32 drawn from `default_rng((seed, seq_idx, tensor_id))`
and rounded to bf16 by round-to-nearest-even. Inputs are per sequence, so they
do not depend on the plan (a sequence's tensors are identical whether it ends up
local or distributed).
"""
from __future__ import annotations

import numpy as np

TENSOR_IDS = {"q": 0, "k": 1, "v": 2, "do": 3}


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def seq_tensors(seed: int, seq_idx: int, length: int, hq: int, hkv: int, d: int,
                bf16: bool = True, sigma_qk: float = 1.0):
    """Return dict q [S,hq,d], k [S,hkv,d], v [S,hkv,d], do [S,hq,d] as float32 arrays.

    `sigma_qk` > 1 gives the "peaky" variant that stresses online-softmax rescaling.
    """
    out = {}
    for name, tid in TENSOR_IDS.items():
        h = hq if name in ("q", "do") else hkv
        rng = np.random.default_rng((seed, seq_idx, tid))
        a = rng.standard_normal((length, h, d), dtype=np.float32)
        if name in ("q", "k") and sigma_qk != 1.0:
            a = a * np.float32(sigma_qk)
        out[name] = round_bf16(a) if bf16 else a
    return out
