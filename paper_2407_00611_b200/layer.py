"""A WallFacer Transformer layer: the GPT-7B-style block the
paper trains — RMSNorm, QKV projection fused with the team
all-gather (wf_qkv_proj, Alg. 1 l.1), WallFacer attention (wf_attn_fwd/bwd), output
projection, residual, RMSNorm, SwiGLU MLP, residual — forward and backward on this
library's kernels only (tcgen05 GEMMs, the attention kernels and the layer operators of
csrc/layer_ops.cu).  This module only sequences C-ABI calls and owns the activations.

Attention-output checkpointing (DistFlashAttn's scheme the paper adopts):
with ``checkpoint=True`` the forward keeps only the layer input and the attention output
(O, LSE); the backward recomputes the cheap parts (norms, projections, MLP) but never the
attention forward.  Weight gradients are this rank's partial sums (data parallel over the
sequence: the caller all-reduces them); in emulated mode the P ranks' rows are stacked, so
they are the full sums.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import wf


@dataclass
class LayerWeights:
    """bf16 weights, nn.Linear layout ([out, in]); the three attention projections and the
    MLP gate/up are stacked."""
    norm1: torch.Tensor   # [H]
    wqkv: torch.Tensor    # [3E, H]
    wo: torch.Tensor      # [H, E]
    norm2: torch.Tensor   # [H]
    w13: torch.Tensor     # [2F, H]  (gate | up)
    w2: torch.Tensor      # [H, F]

    @staticmethod
    def random(hidden, heads, head_dim, ffn, seed=0, device="cuda"):
        g = torch.Generator().manual_seed(seed)
        E = heads * head_dim

        def lin(o, i):
            return (torch.randn((o, i), generator=g) * i ** -0.5).to(torch.bfloat16).to(device)

        def nrm(n):
            return (1.0 + 0.1 * torch.randn((n,), generator=g)).to(torch.bfloat16).to(device)

        return LayerWeights(nrm(hidden), lin(3 * E, hidden), lin(hidden, E), nrm(hidden), lin(2 * ffn, hidden),
                            lin(hidden, ffn))


class WallFacerLayer:
    def __init__(self, ctx: wf.Context, weights: LayerWeights, heads: int, head_dim: int, causal: bool = True,
                 eps: float = 1e-5, checkpoint: bool = True):
        self.ctx, self.w, self.h, self.d = ctx, weights, heads, head_dim
        self.causal, self.eps, self.checkpoint = causal, eps, checkpoint

    # ------------------------------------------------------------------ pieces
    def _attn_in(self, x0, N):
        a, r1 = wf.rmsnorm_fwd(x0, self.w.norm1, self.eps)
        q, k, v = self.ctx.qkv_proj(a, self.w.wqkv, N, self.h, self.d, self.causal)
        return a, r1, q, k, v

    def _after_attn(self, x0, o):
        rows = x0.shape[0]
        o2 = wf.gemm_bf16(o.view(rows, -1), self.w.wo)
        x1 = wf.add_bf16(x0, o2)
        b, r2 = wf.rmsnorm_fwd(x1, self.w.norm2, self.eps)
        gu = wf.gemm_bf16(b, self.w.w13)
        hh = wf.swiglu_fwd(gu)
        return x1, b, r2, gu, hh

    # ------------------------------------------------------------------ API
    def forward(self, x0, N):
        """x0 bf16 [rows, H] (this rank's shard; emulated: all ranks stacked) -> (x2, saved)."""
        a, r1, q, k, v = self._attn_in(x0, N)
        o, lse = self.ctx.fwd(q, k, v, N, self.causal)
        x1, b, r2, gu, hh = self._after_attn(x0, o)
        m = wf.gemm_bf16(hh, self.w.w2)
        x2 = wf.add_bf16(x1, m)
        if self.checkpoint:
            saved = dict(x0=x0, o=o, lse=lse)
        else:
            saved = dict(x0=x0, o=o, lse=lse, a=a, r1=r1, q=q, k=k, v=v, x1=x1, b=b, r2=r2, gu=gu, hh=hh)
        return x2, saved

    def backward(self, dx2, saved, N):
        """-> (dx0, grads dict of fp32/bf16 weight gradients)."""
        w = self.w
        x0, o, lse = saved["x0"], saved["o"], saved["lse"]
        rows = x0.shape[0]
        if self.checkpoint:  # recompute everything except the attention forward
            a, r1, q, k, v = self._attn_in(x0, N)
            x1, b, r2, gu, hh = self._after_attn(x0, o)
        else:
            a, r1, q, k, v = (saved[n] for n in ("a", "r1", "q", "k", "v"))
            x1, b, r2, gu, hh = (saved[n] for n in ("x1", "b", "r2", "gu", "hh"))
        dhh = wf.gemm_bf16(dx2, w.w2, b_mn=True)
        dw2 = wf.gemm_bf16(dx2, hh, a_mn=True, b_mn=True)
        dgu = wf.swiglu_bwd(dhh, gu)
        db = wf.gemm_bf16(dgu, w.w13, b_mn=True)
        dw13 = wf.gemm_bf16(dgu, b, a_mn=True, b_mn=True)
        dn2 = torch.zeros_like(w.norm2, dtype=torch.float32)
        dx1 = wf.rmsnorm_bwd(db, x1, w.norm2, r2, dn2, dres=dx2)
        do = wf.gemm_bf16(dx1, w.wo, b_mn=True).view(rows, self.h, self.d)
        dwo = wf.gemm_bf16(dx1, o.view(rows, -1), a_mn=True, b_mn=True)
        dq, dk, dv = self.ctx.bwd(do, q, k, v, o, lse, N, self.causal)
        dqkv = wf.pack3(dq, dk, dv)
        da = wf.gemm_bf16(dqkv, w.wqkv, b_mn=True)
        dwqkv = wf.gemm_bf16(dqkv, a, a_mn=True, b_mn=True)
        dn1 = torch.zeros_like(w.norm1, dtype=torch.float32)
        dx0 = wf.rmsnorm_bwd(da, x0, w.norm1, r1, dn1, dres=dx1)
        return dx0, dict(norm1=dn1, wqkv=dwqkv, wo=dwo, norm2=dn2, w13=dw13, w2=dw2)


def layer_flops(N, hidden, heads, head_dim, ffn, causal):
    """Model FLOPs of one layer, fwd + bwd (GEMMs 3x their forward; attention in the
    FlashAttention convention)."""
    E = heads * head_dim
    gemm_fwd = 2.0 * N * hidden * (3 * E + E + 3 * ffn)
    att_fwd = 4.0 * N * N * heads * head_dim * (0.5 if causal else 1.0)
    return 3 * gemm_fwd + 3.5 * att_fwd
