"""Seeded synthetic inputs shared by the oracle, the tests and the bench.

This module holds NO arithmetic of the method (no attention, no sharding, no
merge): it only draws the random tensors both sides consume, so that the CUDA
path and the fp64 oracle see the same bf16 bytes.

Recipe: Q, K, V, dO drawn i.i.d. N(0, 1) in fp32 from
``torch.Generator().manual_seed(seed)`` on the CPU, in that order, then cast to
bf16.  The "peaky" variant multiplies Q by 4 before the cast, so logits have
std ~4 and attention is concentrated (the 2e-2 bound on O is then not
vacuous).  Layout is global ``[N, heads, head_dim]`` (B = 1).
"""
from __future__ import annotations

import torch

__all__ = ["make_qkv_do", "make_x_w", "to_f64"]


def make_qkv_do(N: int, heads: int, head_dim: int, seed: int = 0, peaky: bool = False):
    """Return (Q, K, V, dO) as CPU bf16 tensors of shape [N, heads, head_dim]."""
    g = torch.Generator().manual_seed(int(seed))
    shape = (N, heads, head_dim)
    q = torch.randn(shape, generator=g, dtype=torch.float32)
    k = torch.randn(shape, generator=g, dtype=torch.float32)
    v = torch.randn(shape, generator=g, dtype=torch.float32)
    do = torch.randn(shape, generator=g, dtype=torch.float32)
    if peaky:
        q = q * 4.0
    return tuple(t.to(torch.bfloat16).contiguous() for t in (q, k, v, do))


def make_x_w(rows: int, hidden: int, heads: int, head_dim: int, seed: int = 0):
    """Return (X, W) CPU bf16 for the QKV projection (Alg. 1 l.1): X [rows, hidden] ~ N(0, 1),
    W [3 heads head_dim, hidden] ~ N(0, 1/hidden) (nn.Linear-style scale, so Q/K/V ~ N(0, 1))."""
    g = torch.Generator().manual_seed(int(seed) + 1000)
    x = torch.randn((rows, hidden), generator=g, dtype=torch.float32)
    w = torch.randn((3 * heads * head_dim, hidden), generator=g, dtype=torch.float32) * hidden ** -0.5
    return x.to(torch.bfloat16).contiguous(), w.to(torch.bfloat16).contiguous()


def to_f64(t):
    """Widen a (bf16) torch tensor to a float64 numpy array (exact)."""
    return t.detach().to("cpu").to(torch.float64).numpy()
