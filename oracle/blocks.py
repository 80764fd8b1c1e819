"""Per-block primitives of the WallFacer loop, fp64 (TEST INFRASTRUCTURE).

* ``init_state``        Alg. 1 l.4 "initialize ... O, lse to zero";
                        read as lse = -inf, O = 0 (reading c1).
* ``block_attn``        attention of a query block against one K/V block (Eq. 1
                        restricted to that block), returning the block's (O, lse).
* ``forward_iteration`` Alg. 1 l.9: merge a block into the running
                        state by online softmax:
                          new_lse = logaddexp(lse, lse_blk)
                          out = exp(lse - new_lse) out + exp(lse_blk - new_lse) out_blk
* ``combine``           Alg. 1 l.11 ReduceScatter_combine:
                        L = logsumexp_a lse_a ; O = sum_a exp(lse_a - L) O_a.
* ``block_bwd``         the flash-attention backward step for one (query block,
                        K/V block) pair, given the FINAL forward
                        statistics LSE and D = rowsum(dO o O) of the query rows.
"""
from __future__ import annotations

import numpy as np

from .dense import attention_fwd, allowed_mask

__all__ = ["init_state", "block_attn", "forward_iteration", "combine", "block_bwd"]


def init_state(nq, h, d):
    return np.zeros((nq, h, d)), np.full((h, nq), -np.inf)


def block_attn(q, k, v, qpos, kpos, causal, scale=None):
    """(O_blk [nq,h,d], lse_blk [h,nq]) of q against the K/V block alone."""
    return attention_fwd(q, k, v, qpos, kpos, causal, scale)


def _logaddexp(a, b):
    # np.logaddexp(-inf, -inf) = -inf, as the reading c1 requires.
    return np.logaddexp(a, b)


def forward_iteration(state, q, k, v, qpos, kpos, causal, scale=None):
    """Alg. 1 l.9: merge the block (q vs k,v) into ``state`` = (O, lse)."""
    out, lse = state
    ob, lb = block_attn(q, k, v, qpos, kpos, causal, scale)
    new = _logaddexp(lse, lb)
    safe = np.where(np.isfinite(new), new, 0.0)
    wa = np.where(np.isfinite(lse), np.exp(lse - safe), 0.0)  # [h, nq]
    wb = np.where(np.isfinite(lb), np.exp(lb - safe), 0.0)
    out = wa.T[:, :, None] * out + wb.T[:, :, None] * ob
    return out, new


def combine(outs, lses):
    """ReduceScatter_combine of C partial states for the same query rows."""
    L = lses[0]
    for l in lses[1:]:
        L = _logaddexp(L, l)
    safe = np.where(np.isfinite(L), L, 0.0)
    o = np.zeros_like(outs[0])
    for oa, la in zip(outs, lses):
        w = np.where(np.isfinite(la), np.exp(la - safe), 0.0)
        o = o + w.T[:, :, None] * oa
    return o, L


def block_bwd(q, k, v, do, lse, dd, qpos, kpos, causal, scale=None):
    """Partial (dQ, dK, dV) of one block pair; sums over blocks give the exact gradient.

    lse: [h, nq] final forward LSE of the query rows; dd: [h, nq] D = rowsum(dO o O).
    """
    nq, h, d = q.shape
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    allow = allowed_mask(qpos, kpos, causal)
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    for hh in range(h):
        s = (q[:, hh, :] @ k[:, hh, :].T) * scale
        l = lse[hh]
        p = np.where(allow & np.isfinite(l)[:, None], np.exp(s - np.where(np.isfinite(l), l, 0.0)[:, None]), 0.0)
        dv[:, hh, :] = p.T @ do[:, hh, :]
        dp = do[:, hh, :] @ v[:, hh, :].T
        ds = p * (dp - dd[hh][:, None])
        dq[:, hh, :] = (ds @ k[:, hh, :]) * scale
        dk[:, hh, :] = (ds.T @ q[:, hh, :]) * scale
    return dq, dk, dv
