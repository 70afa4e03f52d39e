"""Oracle: useful-work accounting for the bench metric and the plan floor.

Test infrastructure only (see oracle/__init__.py).

R32: Eq. 12's 4hS^2 is the non-causal forward only; the bench counts
useful causal pairs S(S+1)/2 per sequence at 4*d*Hq flop per pair forward and
2.5x that backward (FlashAttention convention, P:101/P:228 family), i.e.
14*d*Hq*S(S+1)/2 per sequence, counted once however it is sharded.
"""
from __future__ import annotations

from .pack import chunk_bounds


def causal_pairs(S: int) -> int:
    return S * (S + 1) // 2


def useful_flops(lens, hq: int, d: int, bwd_factor_x2: int = 5) -> int:
    """fwd+bwd useful FLOP (R32): (1 + bwd_factor_x2/2) * 4*d*Hq per causal pair."""
    per_pair_fwd = 4 * d * hq
    return sum(per_pair_fwd * causal_pairs(int(S)) for S in lens) * (2 + bwd_factor_x2) // 2


def rank_pairs(lens, assign, N: int):
    """Causal (query, key) pairs each CP rank computes under the zigzag layout (R20)."""
    out = [0] * N
    for S, a in zip(lens, assign):
        S = int(S)
        if a == -1:
            for c in range(2 * N):
                lo, hi = chunk_bounds(S, c, N)
                owner = c if c < N else 2 * N - 1 - c
                out[owner] += causal_pairs(hi) - causal_pairs(lo)
        else:
            out[a] += causal_pairs(S)
    return out


def plan_floor(mb_list, N: int):
    """Plan-inherent imbalance: sum over micro-batches of max-rank pairs
    divided by the sum of mean-rank pairs (Eq. 8-style, attention only; Eq. 1)."""
    smax = smean = 0
    for lens, assign in mb_list:
        p = rank_pairs(lens, assign, N)
        smax += max(p)
        smean += sum(p) / N
    return smax / smean if smean else 1.0
