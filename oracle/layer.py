"""fp64 oracle of the WallFacer Transformer layer (the GPT-7B-style
block of P:337/P:407: RMSNorm -> QKV projection -> exact attention (Eq. 1) -> output
projection -> residual -> RMSNorm -> SwiGLU MLP -> residual).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Written as the plain definitions in PyTorch fp64 CPU ops, gradients by torch.autograd (a
library primitive).  The sequence parallelism does not change the function: the oracle
is the layer on the whole sequence.  Pins (tests/test_oracle_layer.py): the attention
part equals oracle.dense.attention_fwd, RMSNorm / SwiGLU closed forms, and central finite
differences of the whole layer's gradients.
"""
import numpy as np
import torch


def rmsnorm(x, w, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * w


def swiglu(gu):
    F = gu.shape[-1] // 2
    g, u = gu[..., :F], gu[..., F:]
    return g * torch.sigmoid(g) * u


def attention(q, k, v, causal):
    """Eq. 1 per head: q, k, v [N, h, d] -> [N, h, d]."""
    N, h, d = q.shape
    s = torch.einsum("qhd,khd->hqk", q, k) / np.sqrt(d)
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(N, N, dtype=torch.bool), 1), float("-inf"))
    return torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v)


def layer_forward(x, W, heads, head_dim, causal, eps=1e-5):
    """x [N, H] fp64 torch; W dict of fp64 torch weights (norm1, wqkv, wo, norm2, w13, w2)."""
    N = x.shape[0]
    E = heads * head_dim
    a = rmsnorm(x, W["norm1"], eps)
    qkv = a @ W["wqkv"].T
    q, k, v = (qkv[:, i * E:(i + 1) * E].reshape(N, heads, head_dim) for i in range(3))
    o = attention(q, k, v, causal).reshape(N, E)
    x1 = x + o @ W["wo"].T
    b = rmsnorm(x1, W["norm2"], eps)
    return x1 + swiglu(b @ W["w13"].T) @ W["w2"].T


def layer_grads(x, W, dy, heads, head_dim, causal, eps=1e-5):
    """Returns (y, dx, {name: dW}) in fp64 numpy."""
    xt = torch.tensor(np.asarray(x, dtype=np.float64), requires_grad=True)
    Wt = {k: torch.tensor(np.asarray(v, dtype=np.float64), requires_grad=True) for k, v in W.items()}
    y = layer_forward(xt, Wt, heads, head_dim, causal, eps)
    y.backward(torch.tensor(np.asarray(dy, dtype=np.float64)))
    return y.detach().numpy(), xt.grad.numpy(), {k: v.grad.numpy() for k, v in Wt.items()}
