#!/usr/bin/env python
"""Fit the degree-3 polynomial of ex2_poly (csrc/cuda/sm100.cuh): 2^f ~ 1 + c1 f + c2 f^2 + c3 f^3
on f in [0, 1), minimax in RELATIVE error with p(0) = 1 fixed (exact at integer x), solved as a
linear program on a dense grid (scipy HiGHS). Prints the fp32-rounded coefficients and the
relative error of the fp32 Horner evaluation; tests/test_ex2_poly.py pins that bound.

    python tools/fit_ex2_poly.py
"""
import numpy as np
from scipy.optimize import linprog


def fit(n=20001):
    f = np.linspace(0.0, 1.0, n)
    y = 2.0 ** f
    A = np.stack([f / y, f ** 2 / y, f ** 3 / y], 1)
    b0 = 1.0 / y - 1.0
    ones = np.ones((n, 1))
    A_ub = np.vstack([np.hstack([A, -ones]), np.hstack([-A, -ones])])
    b_ub = np.concatenate([-b0, b0])
    r = linprog([0, 0, 0, 1], A_ub=A_ub, b_ub=b_ub, bounds=[(None, None)] * 3 + [(0, None)], method="highs")
    assert r.status == 0
    return r.x[:3].astype(np.float32), float(r.x[3])


if __name__ == "__main__":
    c, t = fit()
    print("c1, c2, c3 =", ", ".join(repr(float(x)) for x in c), f"(LP minimax rel err {t:.3e})")
