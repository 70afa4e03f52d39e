"""CPU checks of the parity tolerance's own pieces (tests/attn_harness, DESIGN.md §9 R34' / R34''):
the bf16 half-ulp and the operand-rounding allowance are test infrastructure, so they are pinned
here against what they must equal by construction (not against the GPU)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from synth import seq_tensors  # noqa: E402
from tests import attn_harness  # noqa: E402
from tests.attn_harness import halfulp_bf16, operand_rounding_dev, tol_ok  # noqa: E402


def test_halfulp_bf16_is_half_the_grid_spacing():
    for x in (1.0, 1.5, 3.99, 4.0, 0.3, 1e-3, 200.0):
        e = np.floor(np.log2(x))
        assert halfulp_bf16(x) == 2.0 ** (e - 8)
        # rounding any value of the binade to bf16 moves it by at most the half-ulp
        v = np.float32(x * (1 + 2 ** -9 * 0.999))
        r = torch.tensor(v).to(torch.bfloat16).double().item()
        assert abs(r - float(v)) <= halfulp_bf16(x)
    assert halfulp_bf16(0.0) == 0.0


def test_operand_rounding_dev_vanishes_when_operands_are_exact():
    # one key: P = 1 and O = v (bf16 inputs) are exact in bf16, dP - D = 0 -> dS = 0: no deviation
    x = seq_tensors(3, 0, 1, 4, 2, 64)
    for e in operand_rounding_dev(x["q"], x["k"], x["v"], x["do"]):
        assert np.all(e == 0.0)


def test_operand_rounding_dev_within_the_a_priori_bound():
    # |sum_q (rb(P) - P) dO| <= 2^-8 sum_q P |dO| per dV element (round-to-nearest bf16: relative
    # error <= half an ulp of 2^-7 relative spacing at the bottom of a binade)
    S, hq, hkv, d = 97, 6, 2, 64
    x = seq_tensors(5, 1, S, hq, hkv, d)
    _, _, eV = operand_rounding_dev(x["q"], x["k"], x["v"], x["do"])
    q, k, do = (np.asarray(x[n], np.float64) for n in ("q", "k", "do"))
    bound = np.zeros((S, hkv, d))
    for h in range(hq):
        g = h * hkv // hq
        A = q[:, h] @ k[:, g].T / np.sqrt(d)
        A[np.triu_indices(S, 1)] = -np.inf
        P = np.exp(A - A.max(1, keepdims=True))
        P /= P.sum(1, keepdims=True)
        bound[:, g] += 2.0 ** -8 * P.T @ np.abs(do[:, h])
    assert np.all(eV <= bound * (1 + 1e-9))
    assert eV.max() > 0     # not trivially zero: P is not bf16-exact in general


def test_operand_rounding_dev_query_block_equals_whole_rows():
    # q_pos convention (as oracle.attn_bwd): the tail block's dK / dV rows >= j0 and its dQ rows are
    # the whole sequence's
    S, j0 = 70, 33
    x = seq_tensors(7, 2, S, 4, 2, 64)
    eQ, eK, eV = operand_rounding_dev(x["q"], x["k"], x["v"], x["do"])
    tQ, tK, tV = operand_rounding_dev(x["q"][j0:], x["k"], x["v"], x["do"][j0:], q_pos=j0)
    np.testing.assert_allclose(tK[j0:], eK[j0:], rtol=0, atol=1e-15)
    np.testing.assert_allclose(tV[j0:], eV[j0:], rtol=0, atol=1e-15)
    np.testing.assert_allclose(tQ, eQ[j0:], rtol=0, atol=1e-15)


def test_tol_ok_allowance_is_additive():
    n0 = len(attn_harness.STATS)      # synthetic comparisons: kept out of the parity summary
    ref = np.array([1.0, 0.1])
    got = ref + np.array([0.0235, 0.0])          # within 2e-2 + halfulp(1) = 0.0239
    assert tol_ok(got, ref, False)[0]
    got = ref + np.array([0.025, 0.0])           # beyond R34'
    assert not tol_ok(got, ref, False)[0]
    assert tol_ok(got, ref, False, allow=np.array([0.002, 0.0]))[0]
    assert not tol_ok(got, ref, False, allow=np.array([0.0005, 0.0]))[0]
    # a callable allowance is evaluated only when some element exceeds R34'
    calls = []
    allow = lambda: calls.append(1) or np.array([0.002, 0.0])  # noqa: E731
    assert tol_ok(ref + np.array([0.01, 0.0]), ref, False, allow=allow)[0] and not calls
    assert tol_ok(got, ref, False, allow=allow)[0] and len(calls) == 1
    del attn_harness.STATS[n0:]
