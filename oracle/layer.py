"""fp64 oracle of the WallFacer Transformer layer.

PAPER.md:199: "The output of this forward attention block is finalized after a standard
LayerNorm and FeedForward layer process"; P:337 places the checkpoint at the end of the
self-attention phase.  Reading c22: a pre-LN GPT block --
    a  = LayerNorm1(x)                          (nn.LayerNorm: affine weight and bias)
    x1 = x + Attention(a Wqkv^T) Wo^T           (exact attention, Eq. 1)
    b  = LayerNorm2(x1)
    y  = x1 + GELU(b W1^T) W2^T                 (FeedForward: Linear H->F, GELU, Linear F->H)
with the exact (erf) GELU, F = 4H by default, and no linear biases (the paper names none).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Written as the plain definitions in PyTorch fp64 CPU ops, gradients by torch.autograd (a
library primitive).  The sequence parallelism does not change the function: the oracle
is the layer on the whole sequence.  Pins (tests/test_oracle_layer.py): the attention
part equals oracle.dense.attention_fwd, LayerNorm / GELU closed forms and textbook values,
and central finite differences of the whole layer's gradients.
"""
import math

import numpy as np
import torch

WEIGHTS = ("ln1_w", "ln1_b", "wqkv", "wo", "ln2_w", "ln2_b", "w1", "w2")


def layernorm(x, w, b, eps):
    """(x - mean) / sqrt(var + eps) * w + b, mean and biased variance over the last axis."""
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + eps) * w + b


def gelu(u):
    """u * Phi(u), Phi the standard normal CDF (exact form)."""
    return u * 0.5 * (1.0 + torch.erf(u / math.sqrt(2.0)))


def attention(q, k, v, causal):
    """Eq. 1 per head: q, k, v [N, h, d] -> [N, h, d]."""
    N, h, d = q.shape
    s = torch.einsum("qhd,khd->hqk", q, k) / np.sqrt(d)
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(N, N, dtype=torch.bool), 1), float("-inf"))
    return torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v)


def layer_forward(x, W, heads, head_dim, causal, eps=1e-5):
    """x [N, H] fp64 torch; W dict of fp64 torch weights (WEIGHTS)."""
    N = x.shape[0]
    E = heads * head_dim
    a = layernorm(x, W["ln1_w"], W["ln1_b"], eps)
    qkv = a @ W["wqkv"].T
    q, k, v = (qkv[:, i * E:(i + 1) * E].reshape(N, heads, head_dim) for i in range(3))
    o = attention(q, k, v, causal).reshape(N, E)
    x1 = x + o @ W["wo"].T
    b = layernorm(x1, W["ln2_w"], W["ln2_b"], eps)
    return x1 + gelu(b @ W["w1"].T) @ W["w2"].T


def layer_grads(x, W, dy, heads, head_dim, causal, eps=1e-5):
    """Returns (y, dx, {name: dW}) in fp64 numpy."""
    xt = torch.tensor(np.asarray(x, dtype=np.float64), requires_grad=True)
    Wt = {k: torch.tensor(np.asarray(v, dtype=np.float64), requires_grad=True) for k, v in W.items()}
    y = layer_forward(xt, Wt, heads, head_dim, causal, eps)
    y.backward(torch.tensor(np.asarray(dy, dtype=np.float64)))
    return y.detach().numpy(), xt.grad.numpy(), {k: v.grad.numpy() for k, v in Wt.items()}
