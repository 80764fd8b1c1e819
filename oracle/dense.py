"""Dense softmax attention in fp64 -- the plain definition (TEST INFRASTRUCTURE).

Forward, PAPER.md:101-105 (§2.1, Eq. 1):
    Attention(Q, K, V) = softmax(Q K^T / sqrt(d_k)) V,  d_k = head dim.
Mask (reading c14): a (q, k) pair is allowed iff the
mask is full, or global position of k <= global position of q.  A query row
with no allowed key has O = 0 and LSE = -inf (reading c1).
LSE is the natural-log log-sum-exp of the scaled logits (reading c16).

Backward: the paper only says it "mirrors the backward computation method used
in flash-attention".  The oracle computes the exact gradient of
Eq. 1; written out (the standard identities, pinned by finite differences in
tests/test_oracle_dense.py):
    P  = exp(S - LSE)          dV = P^T dO
    dP = dO V^T                D  = rowsum(dO o O)
    dS = P o (dP - D)          dQ = dS K / sqrt(d),   dK = dS^T Q / sqrt(d)

Per head; query rows are processed ``row_chunk`` at a time only to bound the
memory of the N x N logits (rows are independent; for dK/dV the sum over query
rows is grouped by chunk).
"""
from __future__ import annotations

import numpy as np

__all__ = ["attention_fwd", "attention_bwd", "allowed_mask"]


def allowed_mask(qpos, kpos, causal: bool):
    """Boolean [len(qpos), len(kpos)]: True where key j may be attended by query i."""
    qpos = np.asarray(qpos)
    kpos = np.asarray(kpos)
    if not causal:
        return np.ones((qpos.size, kpos.size), dtype=bool)
    return kpos[None, :] <= qpos[:, None]


def _scores(qh, kh, qpos, kpos, causal, scale):
    s = (qh @ kh.T) * scale
    if causal:
        s = np.where(allowed_mask(qpos, kpos, True), s, -np.inf)
    return s


def _lse_rows(s):
    m = np.max(s, axis=1)
    finite = np.isfinite(m)
    m_safe = np.where(finite, m, 0.0)
    with np.errstate(divide="ignore"):
        lse = m_safe + np.log(np.sum(np.exp(s - m_safe[:, None]), axis=1))
    return np.where(finite, lse, -np.inf)


def attention_fwd(q, k, v, qpos=None, kpos=None, causal=False, scale=None, row_chunk=2048):
    """q: [nq, h, d], k/v: [nk, h, d] float64.  Returns (O [nq,h,d], LSE [h,nq])."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    nq, h, d = q.shape
    nk = k.shape[0]
    if qpos is None:
        qpos = np.arange(nq)
    if kpos is None:
        kpos = np.arange(nk)
    qpos = np.asarray(qpos)
    kpos = np.asarray(kpos)
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    out = np.zeros((nq, h, v.shape[2]), dtype=np.float64)
    lse = np.full((h, nq), -np.inf, dtype=np.float64)
    if nk == 0:
        return out, lse
    for hh in range(h):
        kh = k[:, hh, :]
        vh = v[:, hh, :]
        for r0 in range(0, nq, row_chunk):
            r1 = min(nq, r0 + row_chunk)
            s = _scores(q[r0:r1, hh, :], kh, qpos[r0:r1], kpos, causal, scale)
            l = _lse_rows(s)
            p = np.exp(s - np.where(np.isfinite(l), l, 0.0)[:, None])
            p[~np.isfinite(l)] = 0.0
            out[r0:r1, hh, :] = p @ vh
            lse[hh, r0:r1] = l
    return out, lse


def attention_bwd(q, k, v, do, qpos=None, kpos=None, causal=False, scale=None, row_chunk=2048):
    """Exact gradients of Eq. 1 w.r.t. Q, K, V for upstream gradient dO.

    Returns (dQ, dK, dV, O, LSE); O and LSE are recomputed by attention_fwd.
    """
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    do = np.asarray(do, dtype=np.float64)
    nq, h, d = q.shape
    nk = k.shape[0]
    if qpos is None:
        qpos = np.arange(nq)
    if kpos is None:
        kpos = np.arange(nk)
    qpos = np.asarray(qpos)
    kpos = np.asarray(kpos)
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    o, lse = attention_fwd(q, k, v, qpos, kpos, causal, scale, row_chunk)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for hh in range(h):
        kh = k[:, hh, :]
        vh = v[:, hh, :]
        for r0 in range(0, nq, row_chunk):
            r1 = min(nq, r0 + row_chunk)
            qh = q[r0:r1, hh, :]
            doh = do[r0:r1, hh, :]
            l = lse[hh, r0:r1]
            s = _scores(qh, kh, qpos[r0:r1], kpos, causal, scale)
            p = np.exp(s - np.where(np.isfinite(l), l, 0.0)[:, None])
            p[~np.isfinite(l)] = 0.0
            dv[:, hh, :] += p.T @ doh
            dp = doh @ vh.T
            dd = np.sum(doh * o[r0:r1, hh, :], axis=1)
            ds = p * (dp - dd[:, None])
            dq[r0:r1, hh, :] = (ds @ kh) * scale
            dk[:, hh, :] += (ds.T @ qh) * scale
    return dq, dk, dv, o, lse
