"""CPU: the FMA-pipe exp2 of the attention kernels (ex2_poly, csrc/cuda/sm100.cuh) against 2^x.

The kernels compute a share of the softmax exponentials 2^x (x = scale*log2(e)*s - m <= 0) with a
degree-3 polynomial instead of MUFU ex2. Its coefficients are read from the CUDA
source and the fp32 evaluation (range reduction by the 1.5*2^23 round-down add, Horner with fused
multiply-adds, exponent add) is emulated bit for bit in numpy float32 and compared with the exact
2^x: the relative error bound 8.6e-5 (tools/fit_ex2_poly.py) is far below the bf16 half-ulp 2^-9
that P is rounded to before the PV GEMM (R31).
"""
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _coeffs():
    src = open(os.path.join(ROOT, "paper_2505_19609_b200", "csrc", "cuda", "sm100.cuh")).read()
    body = src[src.index("float ex2_poly(float x)"):]
    body = body[:body.index("}")]
    c3, c2 = (np.float32(v) for v in re.search(r"fmaf\(f, ([0-9.e-]+)f, ([0-9.e-]+)f\)", body).groups())
    c1 = np.float32(re.search(r"fmaf\(p, f, ([0-9.e-]+)f\)", body).group(1))
    return c1, c2, c3


def _fma32(a, b, c):
    # fp32 fused multiply-add: the exact product+sum (float64 holds a 24x24-bit product exactly,
    # the sum with c to within fp32 resolution) rounded once to fp32
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def ex2_poly_emulated(x):
    c1, c2, c3 = _coeffs()
    x = np.maximum(np.asarray(x, np.float32), np.float32(-126.0))
    # __fadd_rd(x, 1.5*2^23): for x in [-126, 0] the exact sum lies in [2^23, 2^24), where fp32
    # spacing is 1, so round-down gives 12582912 + floor(x)
    i = np.floor(x.astype(np.float64)).astype(np.int64)
    f = (x.astype(np.float64) - i).astype(np.float32)           # exact (Sterbenz)
    p = _fma32(f, np.full_like(f, c3), np.full_like(f, c2))
    p = _fma32(p, f, np.full_like(f, c1))
    p = _fma32(p, f, np.ones_like(f))
    bits = p.view(np.int32).astype(np.int64) + (i << 23)
    return bits.astype(np.int32).view(np.float32)


def test_ex2_poly_relative_error_bound():
    x = np.concatenate([np.linspace(-126.0, 0.0, 2_000_001, dtype=np.float32),
                        -np.arange(0, 127, dtype=np.float32),                  # integers: exact
                        np.float32(-1.0) + np.arange(1, 4096, dtype=np.float32) * np.float32(2.0 ** -12)])
    got = ex2_poly_emulated(x).astype(np.float64)
    ref = np.exp2(x.astype(np.float64))
    rel = np.abs(got / ref - 1.0)
    assert rel.max() <= 8.6e-5
    assert rel.max() < 2.0 ** -9 / 10          # an order of magnitude below bf16's half-ulp
    ints = -np.arange(0, 127, dtype=np.float32)
    assert np.array_equal(ex2_poly_emulated(ints), np.exp2(ints.astype(np.float64)).astype(np.float32))


def test_ex2_poly_monotone_on_fraction_grid():
    # the softmax row max is taken before the exponentials; a non-monotone 2^f would reorder the
    # largest probabilities. Check on every fp32 value of f in [0, 1) at 2^-16 resolution.
    f = np.arange(0, 1 << 16, dtype=np.float64) / (1 << 16)
    x = (f - 1.0).astype(np.float32)
    y = ex2_poly_emulated(x)
    assert np.all(np.diff(y.astype(np.float64)) >= 0)
