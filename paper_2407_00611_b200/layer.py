"""A WallFacer Transformer layer: the block P:199 describes --
the attention output "is finalized after a standard LayerNorm and FeedForward layer
process" -- as a pre-LN GPT block (reading c22): LayerNorm, QKV projection fused with the
team all-gather (wf_qkv_proj, Alg. 1 l.1), WallFacer attention (wf_attn_fwd/bwd), output
projection, residual, LayerNorm, FeedForward (Linear H->F, exact GELU, Linear F->H),
residual -- forward and backward on this library's kernels only (tcgen05 GEMMs, the
attention kernels and the layer operators of csrc/layer_ops.cu).  This module only
sequences C-ABI calls and owns the activations.

Attention-output checkpointing (DistFlashAttn's scheme the paper adopts):
with ``checkpoint=True`` the forward keeps only the layer input and the attention output
(O, LSE); the backward recomputes the cheap parts (norms, projections, FFN) but never the
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
    """bf16 weights, nn.Linear layout ([out, in]); the three attention projections are stacked."""
    ln1_w: torch.Tensor   # [H]
    ln1_b: torch.Tensor   # [H]
    wqkv: torch.Tensor    # [3E, H]
    wo: torch.Tensor      # [H, E]
    ln2_w: torch.Tensor   # [H]
    ln2_b: torch.Tensor   # [H]
    w1: torch.Tensor      # [F, H]
    w2: torch.Tensor      # [H, F]

    @staticmethod
    def random(hidden, heads, head_dim, ffn, seed=0, device="cuda"):
        g = torch.Generator().manual_seed(seed)
        E = heads * head_dim

        def lin(o, i):
            return (torch.randn((o, i), generator=g) * i ** -0.5).to(torch.bfloat16).to(device)

        def vec(n, c, s):
            return (c + s * torch.randn((n,), generator=g)).to(torch.bfloat16).to(device)

        return LayerWeights(vec(hidden, 1.0, 0.1), vec(hidden, 0.0, 0.1), lin(3 * E, hidden), lin(hidden, E),
                            vec(hidden, 1.0, 0.1), vec(hidden, 0.0, 0.1), lin(ffn, hidden), lin(hidden, ffn))


class WallFacerLayer:
    def __init__(self, ctx: wf.Context, weights: LayerWeights, heads: int, head_dim: int, causal: bool = True,
                 eps: float = 1e-5, checkpoint: bool = True):
        self.ctx, self.w, self.h, self.d = ctx, weights, heads, head_dim
        self.causal, self.eps, self.checkpoint = causal, eps, checkpoint

    # ------------------------------------------------------------------ pieces
    def _attn_in(self, x0, N):
        a, m1, r1 = wf.layernorm_fwd(x0, self.w.ln1_w, self.w.ln1_b, self.eps)
        q, k, v = self.ctx.qkv_proj(a, self.w.wqkv, N, self.h, self.d, self.causal)
        return a, m1, r1, q, k, v

    def _after_attn(self, x0, o):
        rows = x0.shape[0]
        o2 = wf.gemm_bf16(o.view(rows, -1), self.w.wo)
        x1 = wf.add_bf16(x0, o2)
        b, m2, r2 = wf.layernorm_fwd(x1, self.w.ln2_w, self.w.ln2_b, self.eps)
        u = wf.gemm_bf16(b, self.w.w1)
        hh = wf.gelu_fwd(u)
        return x1, b, m2, r2, u, hh

    # ------------------------------------------------------------------ API
    def forward(self, x0, N):
        """x0 bf16 [rows, H] (this rank's shard; emulated: all ranks stacked) -> (x2, saved)."""
        a, m1, r1, q, k, v = self._attn_in(x0, N)
        o, lse = self.ctx.fwd(q, k, v, N, self.causal)
        x1, b, m2, r2, u, hh = self._after_attn(x0, o)
        m = wf.gemm_bf16(hh, self.w.w2)
        x2 = wf.add_bf16(x1, m)
        if self.checkpoint:
            saved = dict(x0=x0, o=o, lse=lse)
        else:
            saved = dict(x0=x0, o=o, lse=lse, a=a, m1=m1, r1=r1, q=q, k=k, v=v, x1=x1, b=b, m2=m2, r2=r2, u=u,
                         hh=hh)
        return x2, saved

    def backward(self, dx2, saved, N):
        """-> (dx0, grads dict of fp32/bf16 weight gradients, keyed like LayerWeights)."""
        w = self.w
        x0, o, lse = saved["x0"], saved["o"], saved["lse"]
        rows = x0.shape[0]
        if self.checkpoint:  # recompute everything except the attention forward
            a, m1, r1, q, k, v = self._attn_in(x0, N)
            x1, b, m2, r2, u, hh = self._after_attn(x0, o)
        else:
            a, m1, r1, q, k, v = (saved[n] for n in ("a", "m1", "r1", "q", "k", "v"))
            x1, b, m2, r2, u, hh = (saved[n] for n in ("x1", "b", "m2", "r2", "u", "hh"))
        dhh = wf.gemm_bf16(dx2, w.w2, b_mn=True)
        dw2 = wf.gemm_bf16(dx2, hh, a_mn=True, b_mn=True)
        du = wf.gelu_bwd(dhh, u)
        db = wf.gemm_bf16(du, w.w1, b_mn=True)
        dw1 = wf.gemm_bf16(du, b, a_mn=True, b_mn=True)
        dl2w = torch.zeros_like(w.ln2_w, dtype=torch.float32)
        dl2b = torch.zeros_like(w.ln2_b, dtype=torch.float32)
        dx1 = wf.layernorm_bwd(db, x1, w.ln2_w, m2, r2, dl2w, dl2b, dres=dx2)
        do = wf.gemm_bf16(dx1, w.wo, b_mn=True).view(rows, self.h, self.d)
        dwo = wf.gemm_bf16(dx1, o.view(rows, -1), a_mn=True, b_mn=True)
        dq, dk, dv = self.ctx.bwd(do, q, k, v, o, lse, N, self.causal)
        dqkv = wf.pack3(dq, dk, dv)
        da = wf.gemm_bf16(dqkv, w.wqkv, b_mn=True)
        dwqkv = wf.gemm_bf16(dqkv, a, a_mn=True, b_mn=True)
        dl1w = torch.zeros_like(w.ln1_w, dtype=torch.float32)
        dl1b = torch.zeros_like(w.ln1_b, dtype=torch.float32)
        dx0 = wf.layernorm_bwd(da, x0, w.ln1_w, m1, r1, dl1w, dl1b, dres=dx1)
        return dx0, dict(ln1_w=dl1w, ln1_b=dl1b, wqkv=dwqkv, wo=dwo, ln2_w=dl2w, ln2_b=dl2b, w1=dw1, w2=dw2)


def layer_flops(N, hidden, heads, head_dim, ffn, causal):
    """Model FLOPs of one layer, fwd + bwd (GEMMs 3x their forward; attention in the
    FlashAttention convention)."""
    E = heads * head_dim
    gemm_fwd = 2.0 * N * hidden * (3 * E + E + 2 * ffn)
    att_fwd = 4.0 * N * N * heads * head_dim * (0.5 if causal else 1.0)
    return 3 * gemm_fwd + 3.5 * att_fwd
