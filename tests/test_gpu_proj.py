"""GPU parity of the QKV projection GEMM (wf_gemm_bf16 / wf_qkv_proj, Alg. 1 l.1)
against the fp64 oracle (oracle/proj.py), and of the fused projection + team gather: the
forward after wf_qkv_proj must equal the forward with the separate gather, bit for bit,
with the same CommTrace as the oracle's schedule."""
from collections import Counter

import numpy as np
import pytest
import torch

from oracle.proj import gemm, qkv_projection
from oracle.sharding import unit_positions
from wf_inputs import make_x_w, to_f64

pytestmark = pytest.mark.gpu


def _wf():
    import paper_2407_00611_b200 as wf
    return wf


def _close(y, ref):
    # bf16 output of an fp32-accumulated product: half an ulp of bf16 (2^-9 relative) plus
    # accumulation-order noise well below 1e-3 of the largest entry
    err = np.abs(y - ref)
    bound = 2.0 ** -8 * np.abs(ref) + 1e-3 * np.abs(ref).max()
    return bool((err <= bound).all()), float((err / (np.abs(ref) + 1e-3 * np.abs(ref).max())).max())


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 512, 128), (384, 384, 192), (1024, 3456, 1152),
                                   (2048, 768, 4096)])
def test_gemm_parity(M, N, K):
    wf = _wf()
    g = torch.Generator().manual_seed(M + N + K)
    a = torch.randn((M, K), generator=g).to(torch.bfloat16)
    b = (torch.randn((N, K), generator=g) * K ** -0.5).to(torch.bfloat16)
    y = wf.gemm_bf16(a.cuda(), b.cuda())
    torch.cuda.synchronize()
    ok, worst = _close(to_f64(y), gemm(to_f64(a), to_f64(b)))
    assert ok, worst


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 512, 192), (384, 1152, 256), (512, 768, 320), (1024, 512, 4096)])
def test_gemm_transposed_layouts(a_mn, b_mn, M, N, K):
    # the backward products of a projection: dX = dY W (b_mn), dW = dY^T X (a_mn, b_mn)
    wf = _wf()
    g = torch.Generator().manual_seed(M + 3 * N + K + a_mn)
    a = torch.randn((K, M) if a_mn else (M, K), generator=g).to(torch.bfloat16)
    b = (torch.randn((K, N) if b_mn else (N, K), generator=g) * K ** -0.5).to(torch.bfloat16)
    y = wf.gemm_bf16(a.cuda(), b.cuda(), a_mn=bool(a_mn), b_mn=bool(b_mn))
    torch.cuda.synchronize()
    A = to_f64(a).T if a_mn else to_f64(a)
    B = to_f64(b).T if b_mn else to_f64(b)
    ok, worst = _close(to_f64(y), gemm(A, B))
    assert ok, worst


def test_gemm_large_sampled_rows():
    # the GPT-7B projection shape of one rank at P = 8 (16K rows, 4096 -> 3 x 4096)
    wf = _wf()
    M, N, K = 16384, 12288, 4096
    x, w = make_x_w(M, K, 32, 128, seed=3)
    y = wf.gemm_bf16(x.cuda(), w.cuda()).cpu()
    rows = np.array([0, 1, 127, 128, 5000, 8191, 16383])
    ok, worst = _close(to_f64(y[rows]), gemm(to_f64(x[rows]), to_f64(w)))
    assert ok, worst


def test_gemm_rejects_bad_shapes():
    wf = _wf()
    a = torch.zeros((100, 64), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(wf.WFError, match="status 2"):
        wf.gemm_bf16(a, torch.zeros((128, 64), dtype=torch.bfloat16, device="cuda"))


def _shards(P, N, causal):
    return np.concatenate([unit_positions(r, P, N, causal) for r in range(P)])


@pytest.mark.parametrize("P,C,sched", [(1, 1, 0), (2, 2, 0), (4, 2, 0), (4, 4, 0), (8, 2, 0), (8, 4, 0), (4, 2, 1),
                                        (8, 2, 1)])
@pytest.mark.parametrize("causal", [True, False])
def test_qkv_proj_fused_gather(P, C, sched, causal):
    wf = _wf()
    h, d, H = 2, 128, 192
    N = 256 * P
    x, w = make_x_w(N, H, h, d, seed=P * 10 + C)
    idx = torch.from_numpy(_shards(P, N, causal))
    xs = x[idx].contiguous().cuda()
    ctx = wf.Context(P, C, emulated=P > 1)
    if sched:
        ctx.set_schedule(sched)
    q, k, v = ctx.qkv_proj(xs, w.cuda(), N, h, d, causal)
    o1, l1 = ctx.fwd(q, k, v, N, causal)
    torch.cuda.synchronize()
    tr = Counter(e for e in ctx.trace() if e[0] == 0)
    ctx.close()
    # projection values
    Q, K, V = qkv_projection(to_f64(x[idx]), to_f64(w), h, d)
    for got, ref in ((q, Q), (k, K), (v, V)):
        ok, worst = _close(to_f64(got).reshape(N, -1), ref.reshape(N, -1))
        assert ok, worst
    # the fused gather delivers exactly what the separate gather copies
    ctx2 = wf.Context(P, C, emulated=P > 1)
    if sched:
        ctx2.set_schedule(sched)
    o2, l2 = ctx2.fwd(q.clone(), k.clone(), v.clone(), N, causal)
    torch.cuda.synchronize()
    tr2 = Counter(e for e in ctx2.trace() if e[0] == 0)
    ctx2.close()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    assert tr == tr2


def test_qkv_proj_dit_shape():
    # DiT-XL-like: 16 heads x 72 (E = 1152: 128-wide N tiles), hidden 1152, P = 4, C = 2
    wf = _wf()
    P, C, h, d, H, N = 4, 2, 16, 72, 1152, 2048
    x, w = make_x_w(N, H, h, d, seed=5)
    ctx = wf.Context(P, C, emulated=True)
    q, k, v = ctx.qkv_proj(x.cuda(), w.cuda(), N, h, d, False)
    o1, _ = ctx.fwd(q, k, v, N, False)
    torch.cuda.synchronize()
    ctx.close()
    Q, _, V = qkv_projection(to_f64(x), to_f64(w), h, d)
    assert _close(to_f64(q).reshape(N, -1), Q.reshape(N, -1))[0]
    assert _close(to_f64(v).reshape(N, -1), V.reshape(N, -1))[0]
    ctx2 = wf.Context(P, C, emulated=True)
    o2, _ = ctx2.fwd(q.clone(), k.clone(), v.clone(), N, False)
    torch.cuda.synchronize()
    ctx2.close()
    assert torch.equal(o1, o2)
