"""Oracle: fp64 naive masked causal attention, forward and analytic backward.

Test infrastructure only (see oracle/__init__.py).

PAPER.md runs attention through FlashAttention and
states no formula; the method reaches exactly the plain result, so this is the
plain definition (readings R29 scale 1/sqrt(d), no dropout /
bias / window; R30 GQA head map g = floor(h*Hkv/Hq)):

  A_ij = scale * q_i . k_j  for j <= i, else -inf;   P = softmax_row(A)
  O_i = sum_j P_ij v_j;     LSE_i = log sum_j exp(A_ij)
  dV_j = sum_{h in g} sum_i P_ij dO_i;   dP_ij = dO_i . v_j;   D_i = sum_j P_ij dP_ij
  dS_ij = P_ij (dP_ij - D_i);  dQ_i = scale sum_j dS_ij k_j;  dK_j = scale sum_{h in g} sum_i dS_ij q_i

No online softmax and no tiling trick: the scores of a block of query rows are
materialised in full up to the causal bound (blocking only bounds memory).
"""
from __future__ import annotations

import numpy as np

_BLOCK = 2048


def _group(h: int, hq: int, hkv: int) -> int:
    """R30: contiguous GQA groups, g = floor(h * Hkv / Hq)."""
    return (h * hkv) // hq


def attn_fwd(q, k, v, scale=None, q_pos: int = 0):
    """One sequence. q [Sq,Hq,d] holds query positions q_pos..q_pos+Sq-1; k, v [Sk,Hkv,d]
    hold key positions 0..Sk-1 (Sk >= q_pos+Sq). Returns O [Sq,Hq,d], LSE [Hq,Sq] (natural log)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    Sq, hq, d = q.shape
    hkv = k.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    O = np.zeros((Sq, hq, d))
    LSE = np.zeros((hq, Sq))
    for h in range(hq):
        g = _group(h, hq, hkv)
        for r0 in range(0, Sq, _BLOCK):
            r1 = min(Sq, r0 + _BLOCK)
            kend = q_pos + r1                       # causal bound of the block's last row
            A = scale * (q[r0:r1, h, :] @ k[:kend, g, :].T)
            pos = q_pos + np.arange(r0, r1)[:, None]
            A = np.where(np.arange(kend)[None, :] <= pos, A, -np.inf)
            mx = A.max(axis=1, keepdims=True)
            E = np.exp(A - mx)
            s = E.sum(axis=1, keepdims=True)
            P = E / s
            O[r0:r1, h, :] = P @ v[:kend, g, :]
            LSE[h, r0:r1] = (mx + np.log(s))[:, 0]
    return O, LSE


def attn_bwd(q, k, v, do, scale=None, q_pos: int = 0):
    """Analytic backward of `attn_fwd` for one sequence (or one query chunk with q_pos).
    Returns dQ [Sq,Hq,d], dK [Sk,Hkv,d], dV [Sk,Hkv,d] in fp64 (dK/dV summed over the group)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    do = np.asarray(do, np.float64)
    Sq, hq, d = q.shape
    Sk, hkv = k.shape[0], k.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    dQ = np.zeros((Sq, hq, d))
    dK = np.zeros((Sk, hkv, d))
    dV = np.zeros((Sk, hkv, d))
    for h in range(hq):
        g = _group(h, hq, hkv)
        for r0 in range(0, Sq, _BLOCK):
            r1 = min(Sq, r0 + _BLOCK)
            kend = q_pos + r1
            A = scale * (q[r0:r1, h, :] @ k[:kend, g, :].T)
            pos = q_pos + np.arange(r0, r1)[:, None]
            A = np.where(np.arange(kend)[None, :] <= pos, A, -np.inf)
            mx = A.max(axis=1, keepdims=True)
            E = np.exp(A - mx)
            P = E / E.sum(axis=1, keepdims=True)
            dO = do[r0:r1, h, :]
            dV[:kend, g, :] += P.T @ dO
            dP = dO @ v[:kend, g, :].T
            D = (P * dP).sum(axis=1, keepdims=True)
            dS = P * (dP - D)
            dQ[r0:r1, h, :] = scale * (dS @ k[:kend, g, :])
            dK[:kend, g, :] += scale * (dS.T @ q[r0:r1, h, :])
    return dQ, dK, dV


def attn_fwd_bwd(q, k, v, do, scale=None):
    """Convenience: forward and backward of one whole sequence."""
    O, LSE = attn_fwd(q, k, v, scale)
    dQ, dK, dV = attn_bwd(q, k, v, do, scale)
    return O, LSE, dQ, dK, dV


def attn_bwd_kv_group(q, k, v, do, g: int, scale=None):
    """dK, dV of KV head g only (all q-heads of the group, all queries): the parity slice
    used at full sizes ('restricted to one KV-head group')."""
    q = np.asarray(q)
    hq = q.shape[1]
    hkv = k.shape[1]
    heads = [h for h in range(hq) if _group(h, hq, hkv) == g]
    dQ, dK, dV = attn_bwd(q[:, heads, :], k[:, g:g + 1, :], v[:, g:g + 1, :],
                          do[:, heads, :], scale)
    return dQ, dK[:, 0, :], dV[:, 0, :], heads
