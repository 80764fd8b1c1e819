"""Pins of the layer oracle (oracle/layer.py)."""
import numpy as np
import torch

from oracle.dense import attention_fwd
from oracle.layer import attention, layer_forward, layer_grads, rmsnorm, swiglu


def _weights(rng, H, E, F):
    return dict(norm1=1 + 0.1 * rng.standard_normal(H), wqkv=rng.standard_normal((3 * E, H)) / np.sqrt(H),
                wo=rng.standard_normal((H, E)) / np.sqrt(E), norm2=1 + 0.1 * rng.standard_normal(H),
                w13=rng.standard_normal((2 * F, H)) / np.sqrt(H), w2=rng.standard_normal((H, F)) / np.sqrt(F))


def test_attention_matches_dense_oracle():
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((9, 2, 4)) for _ in range(3))
    for causal in (False, True):
        o = attention(*(torch.tensor(t) for t in (q, k, v)), causal).numpy()
        o_ref, _ = attention_fwd(q, k, v, causal=causal)
        assert np.abs(o - o_ref).max() < 1e-12


def test_rmsnorm_swiglu_closed_forms():
    # constant row c: mean(x^2) = c^2 -> y = w sign(c) (eps -> 0)
    x = torch.full((1, 6), -3.0, dtype=torch.float64)
    w = torch.arange(1.0, 7.0, dtype=torch.float64)
    assert torch.allclose(rmsnorm(x, w, 0.0), -w)
    # swiglu([g | u]) = g sigmoid(g) u: zero gate -> 0, u = 1, g -> large: ~g
    gu = torch.tensor([[0.0, 50.0, 2.0, 1.0]], dtype=torch.float64)
    out = swiglu(gu)
    assert out[0, 0] == 0 and abs(out[0, 1] - 50.0) < 1e-12


def test_layer_grads_finite_differences():
    rng = np.random.default_rng(1)
    N, H, h, d, F = 6, 8, 2, 4, 12
    W = _weights(rng, H, h * d, F)
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
        for name, idx in (("wqkv", (5, 3)), ("wo", (2, 1)), ("w13", (7, 4)), ("w2", (3, 9)), ("norm1", (2,)),
                          ("norm2", (6,))):
            Wp = {k: v.copy() for k, v in W.items()}
            Wm = {k: v.copy() for k, v in W.items()}
            Wp[name][idx] += eps
            Wm[name][idx] -= eps
            assert abs((f(x, Wp) - f(x, Wm)) / (2 * eps) - dW[name][idx]) < 1e-6, name
