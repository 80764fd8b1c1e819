"""GPU parity of the layer's non-GEMM operators (wf_layernorm_fwd/bwd, wf_gelu_fwd/bwd) against
the fp64 oracle (oracle/layer.py's LayerNorm and exact GELU, gradients by torch.autograd in
fp64), at hidden sizes that exercise every vector count per thread and a ragged tail
(hidden % 2048 != 0), and row counts that do not fill the grid."""
import math

import numpy as np
import pytest
import torch

from oracle.layer import gelu as gelu_ref
from oracle.layer import layernorm as layernorm_ref

pytestmark = pytest.mark.gpu


def _wf():
    from paper_2407_00611_b200 import wf
    return wf


def _inputs(rows, H, seed):
    g = torch.Generator().manual_seed(seed)
    x = (torch.randn(rows, H, generator=g) * 2.0 + 0.5).to(torch.bfloat16)
    w = (1.0 + 0.1 * torch.randn(H, generator=g)).to(torch.bfloat16)
    b = (0.1 * torch.randn(H, generator=g)).to(torch.bfloat16)
    dy = torch.randn(rows, H, generator=g).to(torch.bfloat16)
    dres = torch.randn(rows, H, generator=g).to(torch.bfloat16)
    return x, w, b, dy, dres


@pytest.mark.parametrize("rows,H", [(1, 8), (3, 520), (37, 1032), (300, 4096), (64, 8192), (1000, 2048)])
def test_layernorm_fwd_bwd(rows, H):
    wf = _wf()
    eps = 1e-5
    x, w, b, dy, dres = _inputs(rows, H, seed=rows + H)
    xg, wg, bg, dyg, dresg = (t.cuda() for t in (x, w, b, dy, dres))
    y, mean, rstd = wf.layernorm_fwd(xg, wg, bg, eps)
    dw = torch.zeros(H, dtype=torch.float32, device="cuda")
    db = torch.zeros(H, dtype=torch.float32, device="cuda")
    dx = wf.layernorm_bwd(dyg, xg, wg, mean, rstd, dw, db, dres=dresg)
    dx0 = wf.layernorm_bwd(dyg, xg, wg, mean, rstd, dw, db)  # accumulates into the same dw, db
    torch.cuda.synchronize()
    # fp64 reference (autograd through the oracle's definition)
    xt = x.double().requires_grad_(True)
    wt = w.double().requires_grad_(True)
    bt = b.double().requires_grad_(True)
    yt = layernorm_ref(xt, wt, bt, eps)
    yt.backward(dy.double())
    mu = x.double().mean(-1)
    rs = 1.0 / torch.sqrt(((x.double() - mu[:, None]) ** 2).mean(-1) + eps)
    assert torch.allclose(mean.cpu().double(), mu, atol=1e-5, rtol=1e-5)
    assert torch.allclose(rstd.cpu().double(), rs, atol=1e-5, rtol=1e-4)
    ymax = yt.detach().abs().max().item()
    assert (y.cpu().double() - yt.detach()).abs().max().item() <= 1e-2 * ymax
    gx = xt.grad
    gmax = gx.abs().max().item()
    assert (dx0.cpu().double() - gx).abs().max().item() <= 1e-2 * gmax
    assert (dx.cpu().double() - (gx + dres.double())).abs().max().item() <= 1e-2 * (gx + dres.double()).abs().max().item()
    # dw, db accumulated over both calls with dres and without: 2x the single gradient
    for got, ref in ((dw, wt.grad), (db, bt.grad)):
        assert torch.allclose(got.cpu().double(), 2 * ref, atol=1e-3 * (1 + ref.abs().max().item()), rtol=1e-3)


@pytest.mark.parametrize("n", [8, 4096, 3 * 1000 * 8, 1 << 20])
def test_gelu_fwd_bwd(n):
    wf = _wf()
    g = torch.Generator().manual_seed(n)
    u = (torch.randn(n, generator=g) * 3.0).to(torch.bfloat16)
    u[:8] = torch.tensor([0.0, -0.0, 1.0, -1.0, 6.0, -6.0, 12.0, -12.0]).to(torch.bfloat16)
    dh = torch.randn(n, generator=g).to(torch.bfloat16)
    h = wf.gelu_fwd(u.cuda())
    du = wf.gelu_bwd(dh.cuda(), u.cuda())
    torch.cuda.synchronize()
    ut = u.double().requires_grad_(True)
    ht = gelu_ref(ut)
    ht.backward(dh.double())
    # bf16 outputs: half an ulp (2^-9 relative) of rounding plus the kernel's erf / exp error
    hr, dur = ht.detach(), ut.grad
    assert ((h.cpu().double() - hr).abs() <= 4e-3 * hr.abs() + 1e-5).all()
    assert ((du.cpu().double() - dur).abs() <= 4e-3 * dur.abs() + 1e-4 * dh.double().abs() + 1e-6).all()
    # textbook values: GELU(1) = Phi(1) = 0.8413447, GELU(-1) = -0.1586553
    assert abs(h[2].item() - 0.8413447) <= 4e-3 and abs(h[3].item() + 0.1586553) <= 1e-3
    assert h[0].item() == 0.0 and h[6].item() == 12.0 and h[7].item() == 0.0
    assert math.isfinite(du.cpu().double().abs().max().item())
