"""GPU parity at BASELINE.json's full size in the launch configuration bench.py times
(GPT-style 32 heads x 128, causal, N = 32K, P = 1), against the fp64 oracle on sampled
outputs it can compute one by one, and on properties that hold at any size:

* O, LSE and dQ of sampled query rows: each row needs only its own logits (Eq. 1);
* dK, dV of sampled key rows of one head: needs that head's LSE of all rows (one oracle
  pass over the head);
* sum_j dV_j = sum_i dO_i and sum_j dK_j = 0 for every head (rows of P sum to 1; pinned in
  tests/test_oracle_dense.py).
Plus edge cases: the smallest N per mask, a single head, head_dim 64, and the C ABI's
error paths.
"""
import numpy as np
import pytest
import torch

from oracle.dense import attention_fwd
from wf_inputs import make_qkv_do, to_f64

pytestmark = pytest.mark.gpu


def _wf():
    import paper_2407_00611_b200 as wf
    return wf


@pytest.fixture(scope="module")
def gpt32k():
    wf = _wf()
    N, h, d = 32768, 32, 128
    q, k, v, do = make_qkv_do(N, h, d, seed=2, peaky=True)
    dev = torch.device("cuda")
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    ctx = wf.Context(1, 1)
    o, lse = ctx.fwd(qd, kd, vd, N, True)
    dq, dk, dv = ctx.bwd(dod, qd, kd, vd, o, lse, N, True)
    torch.cuda.synchronize()
    ctx.close()
    return dict(q=q, k=k, v=v, do=do, o=o.cpu(), lse=lse.cpu(), dq=dq.cpu(), dk=dk.cpu(), dv=dv.cpu(), N=N, h=h, d=d)


def test_fullsize_sampled_rows(gpt32k):
    g = gpt32k
    N, h, d = g["N"], g["h"], g["d"]
    rng = np.random.default_rng(0)
    rows = np.unique(np.concatenate([[0, 1, 127, 128, N // 2, N - 1], rng.integers(0, N, 26)]))
    K, V = to_f64(g["k"]), to_f64(g["v"])
    Q, dO = to_f64(g["q"])[rows], to_f64(g["do"])[rows]
    o_ref, l_ref = attention_fwd(Q, K, V, qpos=rows, kpos=np.arange(N), causal=True)
    eo = np.abs(to_f64(g["o"])[rows] - o_ref).max()
    el = np.abs(g["lse"].double().numpy()[:, rows] - l_ref).max()
    assert eo <= 2e-2 and el <= 1e-2, (eo, el)
    # dQ of the sampled rows: dQ_i = sum_j P_ij (dP_ij - D_i) k_j / sqrt(d), D_i = dO_i . O_i
    sc = 1 / np.sqrt(d)
    dq_ref = np.zeros_like(Q)
    for hh in range(h):
        s = Q[:, hh] @ K[:, hh].T * sc
        s = np.where(np.arange(N)[None, :] <= rows[:, None], s, -np.inf)
        p = np.exp(s - l_ref[hh][:, None])
        dp = dO[:, hh] @ V[:, hh].T
        dd = np.sum(dO[:, hh] * o_ref[:, hh], axis=1)
        dq_ref[:, hh] = (p * (dp - dd[:, None])) @ K[:, hh] * sc
    edq = np.abs(to_f64(g["dq"])[rows] - dq_ref).max() / np.abs(dq_ref).max()
    assert edq <= 2e-2, edq


def test_fullsize_sampled_key_rows_one_head(gpt32k):
    g = gpt32k
    N, d, hh = g["N"], g["d"], 5
    sc = 1 / np.sqrt(d)
    Q, K, V, dO = (to_f64(g[x])[:, hh] for x in ("q", "k", "v", "do"))
    o_ref, l_ref = attention_fwd(Q[:, None], K[:, None], V[:, None], causal=True, row_chunk=1024)
    o_ref, l_ref = o_ref[:, 0], l_ref[0]
    cols = np.array([0, 1, 2, 1000, 16383, 16384, 30000, N - 1])
    dk_ref = np.zeros((cols.size, d))
    dv_ref = np.zeros((cols.size, d))
    dd = np.sum(dO * o_ref, axis=1)
    for c0 in range(0, N, 4096):
        qi = np.arange(c0, min(N, c0 + 4096))
        s = Q[qi] @ K[cols].T * sc
        s = np.where(cols[None, :] <= qi[:, None], s, -np.inf)
        p = np.exp(s - l_ref[qi][:, None])
        dp = dO[qi] @ V[cols].T
        ds = p * (dp - dd[qi][:, None])
        dv_ref += p.T @ dO[qi]
        dk_ref += ds.T @ Q[qi] * sc
    edk = np.abs(to_f64(g["dk"])[cols, hh] - dk_ref).max() / np.abs(dk_ref).max()
    edv = np.abs(to_f64(g["dv"])[cols, hh] - dv_ref).max() / np.abs(dv_ref).max()
    assert edk <= 2e-2 and edv <= 2e-2, (edk, edv)


def test_fullsize_gradient_identities(gpt32k):
    g = gpt32k
    dv, dk, do = to_f64(g["dv"]), to_f64(g["dk"]), to_f64(g["do"])
    # bf16 outputs summed over 32K rows: compare to the magnitude of the summands
    ev = np.abs(dv.sum(0) - do.sum(0)).max() / np.abs(do).sum(0).max()
    ek = np.abs(dk.sum(0)).max() / np.abs(dk).sum(0).max()
    assert ev < 2e-3 and ek < 2e-3, (ev, ek)


@pytest.mark.parametrize("causal,N,h,d", [(True, 256, 1, 128), (False, 128, 1, 64), (True, 512, 3, 64),
                                          (False, 384, 2, 72)])
def test_edge_shapes_single_gpu(causal, N, h, d):
    from oracle.dense import attention_bwd
    wf = _wf()
    q, k, v, do = make_qkv_do(N, h, d, seed=9, peaky=True)
    ctx = wf.Context(1, 1)
    o, lse = ctx.fwd(q.cuda(), k.cuda(), v.cuda(), N, causal)
    dq, dk, dv = ctx.bwd(do.cuda(), q.cuda(), k.cuda(), v.cuda(), o, lse, N, causal)
    torch.cuda.synchronize()
    ctx.close()
    dq_r, dk_r, dv_r, o_r, l_r = attention_bwd(to_f64(q), to_f64(k), to_f64(v), to_f64(do), causal=causal)
    assert np.abs(to_f64(o) - o_r).max() <= 2e-2
    for gg, rr in ((dq, dq_r), (dk, dk_r), (dv, dv_r)):
        assert np.abs(to_f64(gg) - rr).max() / np.abs(rr).max() <= 2e-2


def test_error_paths():
    wf = _wf()
    ctx = wf.Context(1, 1)
    q = torch.zeros((200, 2, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(wf.WFError, match="status 2"):  # N not a multiple of 256 (causal)
        ctx.fwd(q, q, q, 200, True)
    q = torch.zeros((256, 2, 96), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(wf.WFError, match="status 2"):  # head_dim not compiled
        ctx.fwd(q, q, q, 256, True)
    ctx.close()
    with pytest.raises(wf.WFError, match="status 2"):  # C does not divide P
        wf.Context(8, 3, emulated=True)


@pytest.mark.slow
@pytest.mark.parametrize("N", [262144, 524288])
def test_max_length_sampled(N):
    # the longest BASELINE sequence lengths on one GPU (2^31 elements per tensor at 512K):
    # sampled query rows of two heads against the oracle, and the dV column-sum identity
    wf = _wf()
    h, d = 32, 128
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v, do = (torch.randn((N, h, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    ctx = wf.Context(1, 1)
    o, lse = ctx.fwd(q, k, v, N, True)
    dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, True)
    torch.cuda.synchronize()
    ctx.close()
    rows = np.array([0, 777, N // 2 + 5, N - 1])
    for hh in (0, h - 1):
        K, V = to_f64(k[:, hh:hh + 1].cpu()), to_f64(v[:, hh:hh + 1].cpu())
        Q = to_f64(q[rows, hh:hh + 1].cpu())
        o_ref, l_ref = attention_fwd(Q, K, V, qpos=rows, kpos=np.arange(N), causal=True)
        assert np.abs(to_f64(o[rows, hh:hh + 1].cpu()) - o_ref).max() <= 2e-2
        assert np.abs(lse[hh, rows].double().cpu().numpy() - l_ref[0]).max() <= 1e-2
    s_dv = dv.float().sum(0)
    s_do = do.float().sum(0)
    assert (s_dv - s_do).abs().max().item() <= 2e-3 * do.float().abs().sum(0).max().item()


@pytest.mark.slow
@pytest.mark.parametrize("C", [4, 2])
def test_target_config_emulated_p8(C, monkeypatch):
    # BASELINE's target: GPT 32 x 128 causal, N = 128K, P = 8 (C = 4: extension regime with
    # the real-mode unit-pipelined decomposition, two key units per slice; C = 2: paper regime,
    # R = 2 ring), all eight ranks emulated on one GPU: sampled rows of two heads against the
    # oracle, and the dV column-sum identity over the whole sequence
    monkeypatch.setenv("WF_EMU_UNITPIPE", "1")
    wf = _wf()
    from oracle.sharding import unit_positions
    P, N, h, d = 8, 131072, 32, 128
    g = torch.Generator(device="cuda").manual_seed(21)
    q, k, v, do = (torch.randn((N, h, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    idx = torch.from_numpy(np.concatenate([unit_positions(r, P, N, True) for r in range(P)])).cuda()
    qs, ks, vs, dos = (t[idx].contiguous() for t in (q, k, v, do))
    ctx = wf.Context(P, C, emulated=True)
    o, lse = ctx.fwd(qs, ks, vs, N, True)
    dq, dk, dv = ctx.bwd(dos, qs, ks, vs, o, lse, N, True)
    torch.cuda.synchronize()
    ctx.close()
    inv = torch.argsort(idx)
    o_g = o[inv]
    lse_g = lse.reshape(P, h, N // P).permute(1, 0, 2).reshape(h, N)[:, inv]
    rows = np.array([0, 4097, N // 2 - 1, N // 2 + 3, N - 1])
    for hh in (0, h - 1):
        K, V = to_f64(k[:, hh:hh + 1].cpu()), to_f64(v[:, hh:hh + 1].cpu())
        Q = to_f64(q[rows, hh:hh + 1].cpu())
        o_ref, l_ref = attention_fwd(Q, K, V, qpos=rows, kpos=np.arange(N), causal=True)
        assert np.abs(to_f64(o_g[rows, hh:hh + 1].cpu()) - o_ref).max() <= 2e-2
        assert np.abs(lse_g[hh, rows].double().cpu().numpy() - l_ref[0]).max() <= 1e-2
    s_dv, s_do = dv.float().sum(0), do.float().sum(0)
    assert (s_dv - s_do).abs().max().item() <= 2e-3 * do.float().abs().sum(0).max().item()


@pytest.mark.slow
@pytest.mark.parametrize("C", [1, 2, 4])
def test_dit_config_emulated_p8(C, monkeypatch):
    # BASELINE's DiT config: 16 heads x 72, full mask, N = 64K, P = 8, every C; all ranks
    # emulated on one GPU (C = 4 unit-pipelined): sampled rows of two heads, dV identity
    monkeypatch.setenv("WF_EMU_UNITPIPE", "1")
    wf = _wf()
    P, N, h, d = 8, 65536, 16, 72
    g = torch.Generator(device="cuda").manual_seed(31 + C)
    q, k, v, do = (torch.randn((N, h, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    ctx = wf.Context(P, C, emulated=True)
    o, lse = ctx.fwd(q, k, v, N, False)        # full mask: contiguous shards, rank-major = global order
    dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, False)
    torch.cuda.synchronize()
    ctx.close()
    lse_g = lse.reshape(P, h, N // P).permute(1, 0, 2).reshape(h, N)
    rows = np.array([0, 999, N // 2, N - 1])
    for hh in (0, h - 1):
        K, V = to_f64(k[:, hh:hh + 1].cpu()), to_f64(v[:, hh:hh + 1].cpu())
        Q = to_f64(q[rows, hh:hh + 1].cpu())
        o_ref, l_ref = attention_fwd(Q, K, V, qpos=rows, kpos=np.arange(N), causal=False)
        assert np.abs(to_f64(o[rows, hh:hh + 1].cpu()) - o_ref).max() <= 2e-2
        assert np.abs(lse_g[hh, rows].double().cpu().numpy() - l_ref[0]).max() <= 1e-2
    s_dv, s_do = dv.float().sum(0), do.float().sum(0)
    assert (s_dv - s_do).abs().max().item() <= 2e-3 * do.float().abs().sum(0).max().item()
