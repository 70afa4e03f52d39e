"""Oracle: Skrull's performance model (Appendix C).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass(frozen=True)
class Model:
    """Eq. 12/14 parameters: hidden h, KV hidden h_kv, pack batch b."""
    hidden: int
    kv_hidden: int
    pack_batch: int = 1


@dataclass(frozen=True)
class Fit:
    """A LinearFit: slope alpha, intercept beta / T_fixed."""
    slope: float
    intercept: float


def flops(S: int, m: Model) -> int:
    """Eq. 12: FLOPs(S) = 20*b*h^2*S + 4*b*h*h_kv*S + 4*b*h*S^2, exact integer."""
    b, h, hkv = m.pack_batch, m.hidden, m.kv_hidden
    return 20 * b * h * h * S + 4 * b * h * hkv * S + 4 * b * h * S * S


def volume(S: int, m: Model) -> int:
    """Eq. 14: Volume(S) = b * S * hidden_kv, in elements (R25)."""
    return m.pack_batch * S * m.kv_hidden


def t_comp(f, fit: Fit):
    """Eq. 13: T_comp = alpha * FLOPs + beta. Zero work costs zero (R36)."""
    if f == 0:
        return 0
    return fit.slope * f + fit.intercept


def t_comm(v, fit: Fit):
    """Eq. 15: T_comm = alpha * V + T_fixed; 0 when V = 0 (R26)."""
    if v == 0:
        return 0
    return fit.slope * v + fit.intercept


def fit_linear(xs, ys, min_x: float = 0.0) -> Fit:
    """Ordinary least squares over points with x >= min_x (P:567 'latency is
    approximately proportional to communication volumes'). Negative intercept -> 0."""
    pts = [(float(x), float(y)) for x, y in zip(xs, ys) if x >= min_x]
    if len(pts) < 2:
        raise ValueError("insufficient profile points")
    n = len(pts)
    mx = sum(p[0] for p in pts) / n
    my = sum(p[1] for p in pts) / n
    sxx = sum((p[0] - mx) ** 2 for p in pts)
    sxy = sum((p[0] - mx) * (p[1] - my) for p in pts)
    slope = sxy / sxx
    icpt = my - slope * mx
    return Fit(slope, max(0.0, icpt))


def bucket_size(budget: float, mem: Fit) -> int:
    """Appendix C.1: Memory(S) = alpha*S + beta, so C = floor((budget - beta)/alpha)."""
    if budget <= mem.intercept or mem.slope <= 0:
        raise ValueError("infeasible budget")
    return int(math.floor((budget - mem.intercept) / mem.slope))
