"""Sequence-length generators shaped like the paper's Long-SFT datasets.

PAPER.md Table 1 gives the quantiles these presets are calibrated to:
  Wikipedia      <1K 87.88 %  <4K 99.34 %  <8K 99.92 %            longest 78K
  ChatQA2-Long   <1K 21.92 %  <4K 31.48 %  <8K 40.43 %  <32K 99.86 %
and P:33 gives the Llama-3 mix (99.89 % short, avg < 1K; 0.11 % long, ~37K).

A single lognormal never produces the 32K-128K tail at batch sizes of a few
hundred, so the configs append explicit long sequences (`forced_tail_batch`).
"""
from __future__ import annotations

import math

import numpy as np

# name -> (kind, params). Parameters from SURVEY.md §8(d) "Length presets".
PRESETS = {
    # lognormal(mu, sigma), rounded, clamped to [16, max]
    "longtail": ("lognormal", dict(mu=5.6700, sigma=1.0588, lo=16)),
    # longtail resampled (rejection) into [16, 1023]: the "99.9 % < 1K" mixes
    "short1k": ("lognormal_trunc", dict(mu=5.6700, sigma=1.0588, lo=16, hi=1023)),
    # 0.40 x lognormal(ln 900, 1.6) + 0.60 x lognormal(ln 13000, 0.30), clamp [16, 32768]
    "bimodal": ("mixture", dict(w=0.40, mu1=math.log(900.0), s1=1.6,
                                mu2=math.log(13000.0), s2=0.30, lo=16, hi=32768)),
}


def gen_lengths(preset: str, n: int, seed: int, max_len: int | None = None) -> np.ndarray:
    """Draw `n` int64 lengths from `preset`, deterministic in (preset, n, seed)."""
    kind, p = PRESETS[preset]
    rng = np.random.default_rng(seed)
    if kind == "lognormal":
        x = np.rint(rng.lognormal(p["mu"], p["sigma"], n))
        hi = max_len if max_len is not None else np.iinfo(np.int64).max
        x = np.clip(x, p["lo"], hi)
    elif kind == "lognormal_trunc":
        out = np.empty(0)
        while out.size < n:
            y = np.rint(rng.lognormal(p["mu"], p["sigma"], 2 * n + 16))
            y = y[(y >= p["lo"]) & (y <= p["hi"])]
            out = np.concatenate([out, y])
        x = out[:n]
    elif kind == "mixture":
        pick = rng.random(n) < p["w"]
        a = rng.lognormal(p["mu1"], p["s1"], n)
        b = rng.lognormal(p["mu2"], p["s2"], n)
        x = np.rint(np.where(pick, a, b))
        hi = p["hi"] if max_len is None else min(p["hi"], max_len)
        x = np.clip(x, p["lo"], hi)
    else:  # pragma: no cover
        raise ValueError(kind)
    return x.astype(np.int64)


def forced_tail_batch(preset: str, n_short: int, tail: list[int], seed: int,
                      max_len: int | None = None) -> np.ndarray:
    """`n_short` draws from `preset` followed by the explicit long sequences `tail`."""
    body = gen_lengths(preset, n_short, seed, max_len=max_len)
    return np.concatenate([body, np.asarray(tail, dtype=np.int64)])


def quantiles(lengths, thresholds):
    """Fraction of lengths strictly below each threshold (Table 1's "<1K" columns)."""
    a = np.asarray(lengths)
    return [float(np.mean(a < t)) for t in thresholds], int(a.max()) if a.size else 0
