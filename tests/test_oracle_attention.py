"""Pins for oracle/attention.py: worked example, closed forms, invariants, library and FD checks."""
import math

import numpy as np
import pytest

from oracle.attention import attn_bwd, attn_bwd_kv_group, attn_fwd


def _rand(rng, S, hq, hkv, d, sd=1.0):
    return (rng.standard_normal((S, hq, d)) * sd, rng.standard_normal((S, hkv, d)) * sd,
            rng.standard_normal((S, hkv, d)), rng.standard_normal((S, hq, d)))


def _num(x):
    return {"ln3": math.log(3), "ln4": math.log(4), "0.75*ln3": 0.75 * math.log(3)}.get(x, x) \
        if isinstance(x, str) else x


def test_worked_example_w1(golden):
    g = golden("attn_w1.json")
    q = np.array([_num(x) for x in g["q"]]).reshape(2, 1, 1)
    k = np.array([_num(x) for x in g["k"]]).reshape(2, 1, 1)
    v = np.array([_num(x) for x in g["v"]]).reshape(2, 1, 1)
    do = np.array([_num(x) for x in g["do"]]).reshape(2, 1, 1)
    O, LSE = attn_fwd(q, k, v, scale=1.0)
    dQ, dK, dV = attn_bwd(q, k, v, do, scale=1.0)
    np.testing.assert_allclose(O[:, 0, 0], [_num(x) for x in g["O"]], atol=1e-12)
    np.testing.assert_allclose(LSE[0], [_num(x) for x in g["LSE"]], atol=1e-12)
    np.testing.assert_allclose(dQ[:, 0, 0], [_num(x) for x in g["dQ"]], atol=1e-12)
    np.testing.assert_allclose(dK[:, 0, 0], g["dK"], atol=1e-12)
    np.testing.assert_allclose(dV[:, 0, 0], g["dV"], atol=1e-12)


def test_rows_sum_to_one_and_causality():
    rng = np.random.default_rng(0)
    q, k, v, do = _rand(rng, 37, 4, 2, 8)
    ones = np.ones_like(v)
    O1, _ = attn_fwd(q, k, ones)
    np.testing.assert_allclose(O1, 1.0, atol=1e-12)            # sum_j P_ij = 1
    O, L = attn_fwd(q, k, v)
    dQ, dK, dV = attn_bwd(q, k, v, do)
    t = 20
    q2, k2, v2 = q.copy(), k.copy(), v.copy()
    q2[t + 1:] += 3.0
    k2[t + 1:] -= 2.0
    v2[t + 1:] *= 5.0
    O2, L2 = attn_fwd(q2, k2, v2)
    dQ2, _, _ = attn_bwd(q2, k2, v2, do)
    np.testing.assert_array_equal(O2[:t + 1], O[:t + 1])
    np.testing.assert_array_equal(L2[:, :t + 1], L[:, :t + 1])
    np.testing.assert_array_equal(dQ2[:t + 1], dQ[:t + 1])


def test_single_token_closed_form():
    rng = np.random.default_rng(1)
    q, k, v, do = _rand(rng, 1, 4, 2, 8)
    O, LSE = attn_fwd(q, k, v)
    dQ, dK, dV = attn_bwd(q, k, v, do)
    np.testing.assert_allclose(O[0, :2], np.broadcast_to(v[0, 0], (2, 8)), atol=1e-14)
    np.testing.assert_allclose(O[0, 2:], np.broadcast_to(v[0, 1], (2, 8)), atol=1e-14)
    np.testing.assert_allclose(dV[0, 0], do[0, 0] + do[0, 1], atol=1e-14)
    np.testing.assert_allclose(dV[0, 1], do[0, 2] + do[0, 3], atol=1e-14)
    assert np.abs(dQ).max() < 1e-14 and np.abs(dK).max() < 1e-14


def test_uniform_queries_give_cumulative_mean():
    rng = np.random.default_rng(2)
    _, k, v, do = _rand(rng, 25, 2, 1, 4)
    q = np.zeros((25, 2, 4))
    O, LSE = attn_fwd(q, k, v)
    cm = np.cumsum(v[:, 0], axis=0) / np.arange(1, 26)[:, None]
    np.testing.assert_allclose(O[:, 0], cm, atol=1e-12)
    np.testing.assert_allclose(LSE[0], np.log(np.arange(1, 26)), atol=1e-12)
    _, dK, _ = attn_bwd(q, k, v, do)
    assert np.abs(dK).max() < 1e-12


def test_gradient_identities_and_shift_invariance():
    rng = np.random.default_rng(3)
    q, k, v, do = _rand(rng, 30, 6, 2, 8)
    dQ, dK, dV = attn_bwd(q, k, v, do)
    np.testing.assert_allclose(dK.sum(axis=0), 0.0, atol=1e-10)            # sum_j dS_ij = 0
    np.testing.assert_allclose(dV[:, 0].sum(axis=0), do[:, 0:3].sum(axis=(0, 1)), atol=1e-10)
    np.testing.assert_allclose(dV[:, 1].sum(axis=0), do[:, 3:6].sum(axis=(0, 1)), atol=1e-10)
    c = rng.standard_normal((1, 2, 8))
    O, _ = attn_fwd(q, k, v)
    Os, _ = attn_fwd(q, k + c, v)
    dQs, dKs, dVs = attn_bwd(q, k + c, v, do)
    np.testing.assert_allclose(Os, O, atol=1e-10)
    np.testing.assert_allclose(dQs, dQ, atol=1e-10)
    np.testing.assert_allclose(dKs, dK, atol=1e-10)
    np.testing.assert_allclose(dVs, dV, atol=1e-10)


def test_gqa_equals_mha_with_repeated_kv():
    rng = np.random.default_rng(4)
    q, k, v, do = _rand(rng, 19, 6, 2, 8)
    kr, vr = np.repeat(k, 3, axis=1), np.repeat(v, 3, axis=1)     # HF repeat_kv (R30)
    O, L = attn_fwd(q, k, v)
    Om, Lm = attn_fwd(q, kr, vr)
    np.testing.assert_allclose(O, Om, atol=1e-12)
    dQ, dK, dV = attn_bwd(q, k, v, do)
    dQm, dKm, dVm = attn_bwd(q, kr, vr, do)
    np.testing.assert_allclose(dQ, dQm, atol=1e-12)
    np.testing.assert_allclose(dK, dKm.reshape(19, 2, 3, 8).sum(2), atol=1e-12)
    np.testing.assert_allclose(dV, dVm.reshape(19, 2, 3, 8).sum(2), atol=1e-12)
    dQg, dKg, dVg, heads = attn_bwd_kv_group(q, k, v, do, 1)
    assert heads == [3, 4, 5]
    np.testing.assert_allclose(dKg, dK[:, 1], atol=1e-12)
    np.testing.assert_allclose(dVg, dV[:, 1], atol=1e-12)


def test_matches_library_sdpa_fp64():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(5)
    q, k, v, do = _rand(rng, 45, 4, 4, 16)
    O, _ = attn_fwd(q, k, v)
    dQ, dK, dV = attn_bwd(q, k, v, do)
    tq, tk, tv = (torch.tensor(x.transpose(1, 0, 2), requires_grad=True) for x in (q, k, v))
    to = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=True)
    to.backward(torch.tensor(do.transpose(1, 0, 2)))
    np.testing.assert_allclose(O, to.detach().numpy().transpose(1, 0, 2), atol=1e-12)
    np.testing.assert_allclose(dQ, tq.grad.numpy().transpose(1, 0, 2), atol=1e-12)
    np.testing.assert_allclose(dK, tk.grad.numpy().transpose(1, 0, 2), atol=1e-12)
    np.testing.assert_allclose(dV, tv.grad.numpy().transpose(1, 0, 2), atol=1e-12)


def test_finite_differences():
    rng = np.random.default_rng(6)
    S, hq, hkv, d = 5, 2, 1, 3
    q, k, v, do = _rand(rng, S, hq, hkv, d)
    dQ, dK, dV = attn_bwd(q, k, v, do)

    def loss(q_, k_, v_):
        return float((attn_fwd(q_, k_, v_)[0] * do).sum())

    h = 1e-6
    for X, G, which in ((q, dQ, 0), (k, dK, 1), (v, dV, 2)):
        num = np.zeros_like(X)
        for idx in np.ndindex(X.shape):
            Xp, Xm = X.copy(), X.copy()
            Xp[idx] += h
            Xm[idx] -= h
            args_p = [q, k, v]
            args_m = [q, k, v]
            args_p[which], args_m[which] = Xp, Xm
            num[idx] = (loss(*args_p) - loss(*args_m)) / (2 * h)
        np.testing.assert_allclose(G, num, rtol=1e-6, atol=1e-8)


def test_query_chunk_with_offset_equals_full_rows():
    # sharded == unsharded at the oracle level: a query chunk [a,b) with q_pos=a against
    # the K/V prefix [0,b) reproduces rows a..b-1 of the whole-sequence result (R23)
    rng = np.random.default_rng(7)
    q, k, v, do = _rand(rng, 50, 4, 2, 8)
    O, L = attn_fwd(q, k, v)
    dQ, dK, dV = attn_bwd(q, k, v, do)
    a, b = 13, 31
    Oc, Lc = attn_fwd(q[a:b], k[:b], v[:b], q_pos=a)
    np.testing.assert_allclose(Oc, O[a:b], atol=1e-12)
    np.testing.assert_allclose(Lc, L[:, a:b], atol=1e-12)
    # dK/dV of the full sequence = sum over query chunks of per-chunk partials
    parts = [(0, 13), (13, 31), (31, 50)]
    sk, sv = np.zeros_like(dK), np.zeros_like(dV)
    for a, b in parts:
        dq, dk, dv = attn_bwd(q[a:b], k[:b], v[:b], do[a:b], q_pos=a)
        np.testing.assert_allclose(dq, dQ[a:b], atol=1e-12)
        sk[:b] += dk
        sv[:b] += dv
    np.testing.assert_allclose(sk, dK, atol=1e-12)
    np.testing.assert_allclose(sv, dV, atol=1e-12)
