"""Workload configurations C1-C5 and S4 (BASELINE.json `configs`).

Each config fixes the attention shape (PAPER.md evaluates Qwen2.5-0.5B and
Qwen2.5-7B; Llama-3-8B is the P:33 mix's model), the CP degree N, the
BucketSize C (readings R33) and a seeded global batch of lengths.
Only lengths and shapes live here -- no scheduling or FLOPs arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .lengths import forced_tail_batch, gen_lengths


@dataclass(frozen=True)
class Shape:
    hq: int
    hkv: int
    d: int

    @property
    def hidden(self) -> int:      # h of Eq. 12: Hq * d
        return self.hq * self.d

    @property
    def kv_hidden(self) -> int:   # h_kv of Eq. 12/14: Hkv * d
        return self.hkv * self.d


QWEN05 = Shape(14, 2, 64)     # Qwen2.5-0.5B attention
QWEN7 = Shape(28, 4, 128)     # Qwen2.5-7B attention
LLAMA8 = Shape(32, 8, 128)    # Llama-3-8B attention
TOY = Shape(2, 2, 64)         # C1 (GQA variant: Shape(2, 1, 64))


@dataclass
class Config:
    name: str
    shape: Shape
    cp: int
    dp: int
    bucket: int
    dtype: str
    lengths_fn: object = field(repr=False)
    note: str = ""

    def lengths(self, seed: int = 0) -> np.ndarray:
        return np.asarray(self.lengths_fn(seed), dtype=np.int64)


TOY_LENGTHS = [17, 33, 64, 90, 128, 200, 256, 300]


def _c2(seed):
    return forced_tail_batch("longtail", 63, [32768], seed, max_len=32768)


def _c3(seed):
    return forced_tail_batch("longtail", 63, [131072], seed, max_len=32768)


def _c4(seed):
    return forced_tail_batch("short1k", 511, [131072], seed)


def _c5(n_per_gpu, n):
    return lambda seed: gen_lengths("bimodal", n_per_gpu * n, seed)


def _build():
    cfgs = {
        "C1": Config("C1", TOY, 2, 1, 600, "fp32", lambda seed: TOY_LENGTHS,
                     "toy: 8 seqs, 2 heads, d=64, fp32, CP=2 plan"),
        "C1g": Config("C1g", Shape(2, 1, 64), 2, 1, 600, "fp32", lambda seed: TOY_LENGTHS,
                      "toy GQA variant (Hkv=1)"),
        "C2": Config("C2", QWEN05, 1, 1, 65536, "bf16", _c2,
                     "Qwen2.5-0.5B shape, Long-SFT mix up to 32K, 1 GPU"),
        "C3n2": Config("C3n2", QWEN7, 2, 1, 131072, "bf16", _c3, "Qwen2.5-7B, tail 128K, CP=2"),
        "C3n4": Config("C3n4", QWEN7, 4, 1, 65536, "bf16", _c3, "Qwen2.5-7B, tail 128K, CP=4"),
        "C4": Config("C4", QWEN7, 8, 1, 65536, "bf16", _c4,
                     "Qwen2.5-7B, 512 seqs 99.8% <1K + 128K, CP=8"),
    }
    for n in (1, 2, 4, 8):
        cfgs[f"C5n{n}"] = Config(f"C5n{n}", LLAMA8, n, 1, 65536, "bf16", _c5(16, n),
                                 f"Llama-3-8B bimodal, 16 seqs/GPU, CP={n}")
        cfgs[f"C5Hn{n}"] = Config(f"C5Hn{n}", LLAMA8, n, 1, 65536, "bf16", _c5(256, n),
                                  f"Llama-3-8B bimodal, 256 seqs/GPU, CP={n}")
    for n, c in ((1, 524288), (2, 98304), (4, 49152), (8, 24576)):
        cfgs[f"S4n{n}"] = Config(f"S4n{n}", QWEN7, n, 1, c, "bf16", _c4,
                                 f"Qwen2.5-7B strong scaling, C4 batch, CP={n}")
    return cfgs


CONFIGS = _build()


def get_config(name: str) -> Config:
    return CONFIGS[name]
