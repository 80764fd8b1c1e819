"""Pins of the layer oracle (oracle/layer.py): attention vs the dense oracle, LayerNorm and
GELU against closed forms and textbook values, and central finite differences of every
gradient of the whole layer (reading c22)."""
import math

import numpy as np
import torch

from oracle.dense import attention_fwd
from oracle.layer import WEIGHTS, attention, gelu, layer_forward, layer_grads, layernorm


def _weights(rng, H, E, F):
    return dict(ln1_w=1 + 0.1 * rng.standard_normal(H), ln1_b=0.1 * rng.standard_normal(H),
                wqkv=rng.standard_normal((3 * E, H)) / np.sqrt(H), wo=rng.standard_normal((H, E)) / np.sqrt(E),
                ln2_w=1 + 0.1 * rng.standard_normal(H), ln2_b=0.1 * rng.standard_normal(H),
                w1=rng.standard_normal((F, H)) / np.sqrt(H), w2=rng.standard_normal((H, F)) / np.sqrt(F))


def test_attention_matches_dense_oracle():
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((9, 2, 4)) for _ in range(3))
    for causal in (False, True):
        o = attention(*(torch.tensor(t) for t in (q, k, v)), causal).numpy()
        o_ref, _ = attention_fwd(q, k, v, causal=causal)
        assert np.abs(o - o_ref).max() < 1e-12


def test_layernorm_closed_forms():
    # [1, -1, 1, -1]: mean 0, variance 1 -> unchanged (eps -> 0); affine applies after
    x = torch.tensor([[1.0, -1.0, 1.0, -1.0]], dtype=torch.float64)
    w = torch.tensor([2.0, 3.0, 4.0, 5.0], dtype=torch.float64)
    b = torch.tensor([0.5, 0.0, -0.5, 1.0], dtype=torch.float64)
    assert torch.allclose(layernorm(x, w, b, 0.0), x * w + b)
    # shift and scale invariance: LN(a x + c) = LN(x) for a > 0
    r = torch.tensor(np.random.default_rng(3).standard_normal((3, 16)))
    one, zero = torch.ones(16, dtype=torch.float64), torch.zeros(16, dtype=torch.float64)
    assert torch.allclose(layernorm(7.0 * r - 2.5, one, zero, 0.0), layernorm(r, one, zero, 0.0))
    # output rows have mean 0 and (biased) variance 1
    y = layernorm(r, one, zero, 0.0)
    assert torch.allclose(y.mean(-1), torch.zeros(3, dtype=torch.float64), atol=1e-12)
    assert torch.allclose((y * y).mean(-1), torch.ones(3, dtype=torch.float64))
    # a constant row normalises to 0: the output is the bias
    assert torch.allclose(layernorm(torch.full((1, 4), 3.0, dtype=torch.float64), w, b, 1e-5), b)


def test_gelu_values():
    u = torch.tensor([0.0, 1.0, -1.0, 8.0, -8.0], dtype=torch.float64)
    g = gelu(u)
    phi1 = 0.8413447460685429  # standard normal CDF at 1 (table value)
    assert g[0] == 0 and abs(g[1] - phi1) < 1e-15 and abs(g[2] + (1 - phi1)) < 1e-15
    assert abs(g[3] - 8.0) < 1e-13 and abs(g[4]) < 1e-13
    # gelu(u) - gelu(-u) = u (Phi(u) + Phi(-u) = 1)
    r = torch.tensor(np.random.default_rng(4).standard_normal(32))
    assert torch.allclose(gelu(r) - gelu(-r), r)
    # agrees with math.erf written independently
    assert abs(float(gelu(torch.tensor(0.3, dtype=torch.float64))) - 0.3 * 0.5 * (1 + math.erf(0.3 / math.sqrt(2)))) < 1e-16


def test_layer_grads_finite_differences():
    rng = np.random.default_rng(1)
    N, H, h, d, F = 6, 8, 2, 4, 12
    W = _weights(rng, H, h * d, F)
    assert set(W) == set(WEIGHTS)
    x = rng.standard_normal((N, H))
    dy = rng.standard_normal((N, H))
    for causal in (True, False):
        _, dx, dW = layer_grads(x, W, dy, h, d, causal)

        def f(xx, WW):
            with torch.no_grad():
                y = layer_forward(torch.tensor(xx), {k: torch.tensor(v) for k, v in WW.items()}, h, d, causal)
            return float((y.numpy() * dy).sum())

        eps = 1e-6
        for (i, j) in ((0, 0), (3, 5), (5, 7)):
            xp, xm = x.copy(), x.copy()
            xp[i, j] += eps
            xm[i, j] -= eps
            assert abs((f(xp, W) - f(xm, W)) / (2 * eps) - dx[i, j]) < 1e-6
        for name, idx in (("wqkv", (5, 3)), ("wo", (2, 1)), ("w1", (7, 4)), ("w2", (3, 9)), ("ln1_w", (2,)),
                          ("ln1_b", (5,)), ("ln2_w", (6,)), ("ln2_b", (0,))):
            Wp = {k: v.copy() for k, v in W.items()}
            Wm = {k: v.copy() for k, v in W.items()}
            Wp[name][idx] += eps
            Wm[name][idx] -= eps
            assert abs((f(x, Wp) - f(x, Wm)) / (2 * eps) - dW[name][idx]) < 1e-6, name
