"""GPU parity at BASELINE.json's full sizes against the fp64 oracle (oracle/dense.py,
oracle/blocks.py), on sampled outputs the oracle computes one by one:

* O, LSE and dQ of >= 16 sampled query rows, every head: `attention_bwd` on those rows
  against all keys (each row's O, LSE, D and dQ depend only on its own logits, Eq. 1);
* dK, dV of 8 sampled key rows of one head, spread over every rank's units: the head's
  LSE of all rows from `attention_fwd` (causal: row chunks against their key prefix, the
  keys after a chunk's last row being masked anyway), D = rowsum(dO o O), then
  `block_bwd` of all query rows against those keys (the FA2 identities);
* the kernel's fp32 output before the bf16 rounding (`wf_block_fwd` o_out_f32) against
  a bound derived from the arithmetic: P is rounded to bf16 for the P.V MMA (relative
  error <= 2^-9 per weight) and l may be summed from the rounded or unrounded weights,
  so |O_f32 - O| <= 2^-8 (P|V|)_i + 1e-5 row by row, (P|V|)_i = sum_j P_ij |V_j|
  evaluated by the oracle itself (attention_fwd with |V|).  This separates kernel
  error from the bf16 output rounding, which alone spends up to 2^-9 |O| (1.6e-2 of the
  2e-2 O bound at |O| in [4, 8)); measured (GPT 32K, peaky): fp32 max error 5.9e-3, i.e.
  bf16 P's 2^-9 per weight on rows dominated by a few keys -- a fixed absolute 2e-3 is
  not a property of any kernel that multiplies bf16 P, the per-row bound is.

Configurations (inputs: wf_inputs "peaky", Q x 4, so attention concentrates and the O
bound is not vacuous): BASELINE configs[1]'s GPT 32x128 causal N = 32K at P = 1 (the
launch bench.py times); configs[2]'s target, GPT 128K causal at P = 8 for C = 1 (ring),
2 (paper regime, R = 2) and 4 (extension, unit-pipelined); configs[3]'s DiT 16x72 full
mask N = 64K at P = 8 for C = 1, 2, 4 -- P = 8 with all ranks emulated on one GPU (the
same kernels and schedule; the real transport is tested in tests/test_multi.py).  Plus
edge cases: the smallest N per mask, a single head, head_dim 64, the C ABI's error
paths, and the longest sequences (256K, 512K) on one GPU.
"""
import numpy as np
import pytest
import torch

from oracle.blocks import block_bwd, combine
from oracle.dense import attention_bwd, attention_fwd
from oracle.sharding import unit_positions
from wf_inputs import make_qkv_do, to_f64

pytestmark = pytest.mark.gpu

O_TOL, LSE_TOL, G_TOL = 2e-2, 1e-2, 2e-2


def _wf():
    import paper_2407_00611_b200 as wf
    return wf


# ---------------------------------------------------------------------- oracle side
def _sample_rows(N, seed, k=10):
    rng = np.random.default_rng(seed)
    fixed = [0, 1, 127, 128, N // 2 - 1, N // 2, N - 1]
    return np.unique(np.concatenate([fixed, rng.choice(N, k, replace=False)]))


def _sample_keys(N, P, causal):
    """8 key rows spread over the units of all P ranks (zigzag chunks when causal: chunk ch
    belongs to rank ch or 2P - 1 - ch; the even chunks 0, 2, ..., 2P - 2 cover every rank)."""
    if causal:
        c = N // (2 * P)
        return np.array([(i * 2 * P // 8) * c + (37 * i + 11) % c for i in range(8)])
    n = N // P
    return np.array([(i * P // 8) * n + (53 * i + 7) % n for i in range(8)])


class Reference:
    """fp64 oracle values of one configuration on its sampled rows / key rows / head."""

    def __init__(self, N, h, d, causal, seed, P, head, key_tail=None):
        self.N, self.h, self.d, self.causal, self.head = N, h, d, causal, head
        self.q, self.k, self.v, self.do = make_qkv_do(N, h, d, seed=seed, peaky=True)
        self.rows = _sample_rows(N, seed)
        if key_tail:  # causal: 8 keys in the last key_tail positions need only those rows' LSE
            self.keys = N - key_tail + (np.arange(8) * (key_tail // 8) + 5)
        else:
            self.keys = _sample_keys(N, P, causal)
        Q, K, V, dO = (to_f64(t) for t in (self.q, self.k, self.v, self.do))
        # query rows: O, LSE, dQ on every head
        dq, _, _, o, lse = attention_bwd(Q[self.rows], K, V, dO[self.rows], qpos=self.rows, kpos=np.arange(N),
                                         causal=causal)
        self.o_rows, self.lse_rows, self.dq_rows = o, lse, dq
        # key rows of one head: LSE and D of all rows, then the block backward
        Qh, Kh, Vh, dOh = (x[:, head:head + 1] for x in (Q, K, V, dO))
        del Q, K, V, dO
        oh = np.zeros_like(Qh)
        lh = np.zeros((1, N))
        step = 2048
        first = (int(self.keys.min()) // step) * step if causal else 0  # rows before see none of the keys
        for r0 in range(first, N, step):
            r1 = min(N, r0 + step)
            qp = np.arange(r0, r1)
            if not causal:
                oh[r0:r1], lh[:, r0:r1] = attention_fwd(Qh[r0:r1], Kh, Vh, qpos=qp, causal=False)
                continue
            # causal: the keys before the chunk are all visible (no mask), the chunk's own keys
            # form the masked diagonal block; the two partial states are LSE-combined (Alg. 1
            # l.11, oracle.blocks.combine), the keys after the chunk are masked out entirely
            parts = [attention_fwd(Qh[r0:r1], Kh[r0:r1], Vh[r0:r1], qpos=qp, kpos=qp, causal=True)]
            if r0 > 0:
                parts.append(attention_fwd(Qh[r0:r1], Kh[:r0], Vh[:r0], qpos=qp, kpos=np.arange(r0), causal=False))
            oh[r0:r1], lh[:, r0:r1] = combine([x[0] for x in parts], [x[1] for x in parts])
        dd = np.sum(dOh * oh, axis=2).T
        rr = np.arange(first, N)
        _, dk, dv = block_bwd(Qh[first:], Kh[self.keys], Vh[self.keys], dOh[first:], lh[:, first:], dd[:, first:], rr,
                              self.keys, causal)
        self.dk_keys, self.dv_keys = dk[:, 0], dv[:, 0]


def check(ref, o, lse, dq, dk, dv):
    """o, dq, dk, dv: global-order [N, h, d] results (CPU, bf16); lse [h, N] fp32."""
    rows, keys, hh = ref.rows, ref.keys, ref.head
    errs = {
        "o": np.abs(to_f64(o[rows]) - ref.o_rows).max(),
        "lse": np.abs(lse[:, rows].double().numpy() - ref.lse_rows).max(),
        "dq": np.abs(to_f64(dq[rows]) - ref.dq_rows).max() / np.abs(ref.dq_rows).max(),
        "dk": np.abs(to_f64(dk[keys, hh]) - ref.dk_keys).max() / np.abs(ref.dk_keys).max(),
        "dv": np.abs(to_f64(dv[keys, hh]) - ref.dv_keys).max() / np.abs(ref.dv_keys).max(),
    }
    tol = {"o": O_TOL, "lse": LSE_TOL, "dq": G_TOL, "dk": G_TOL, "dv": G_TOL}
    return all(errs[k] <= tol[k] for k in errs), errs


def run_emulated(ref, P, C):
    """All P ranks of one configuration emulated on this GPU; results in global order."""
    wf = _wf()
    N, h = ref.N, ref.h
    idx = torch.from_numpy(np.concatenate([unit_positions(r, P, N, ref.causal) for r in range(P)]))
    qs, ks, vs, dos = (t[idx].contiguous().cuda() for t in (ref.q, ref.k, ref.v, ref.do))
    ctx = wf.Context(P, C, emulated=P > 1)
    o, lse = ctx.fwd(qs, ks, vs, N, ref.causal)
    dq, dk, dv = ctx.bwd(dos, qs, ks, vs, o, lse, N, ref.causal)
    torch.cuda.synchronize()
    ctx.close()
    del qs, ks, vs, dos
    inv = torch.argsort(idx)
    lse_g = lse.cpu().reshape(P, h, N // P).permute(1, 0, 2).reshape(h, N)[:, inv]
    return tuple(x.cpu()[inv] for x in (o, dq, dk, dv)) + (lse_g,)


# ---------------------------------------------------------------------- GPT 32K, P = 1
@pytest.fixture(scope="module")
def gpt32k():
    return Reference(32768, 32, 128, True, seed=2, P=1, head=5)


def test_gpt32k_p1_sampled(gpt32k):
    o, dq, dk, dv, lse = run_emulated(gpt32k, 1, 1)
    ok, errs = check(gpt32k, o, lse, dq, dk, dv)
    assert ok, errs
    # dV column sums: sum_j dV_j = sum_i dO_i per head (rows of P sum to 1)
    s_dv, s_do = dv.float().sum(0), gpt32k.do.float().sum(0)
    assert (s_dv - s_do).abs().max().item() <= 2e-3 * gpt32k.do.float().abs().sum(0).max().item()


@pytest.mark.parametrize("cfg", ["gpt32k", "dit64k"])
def test_fp32_output_before_rounding(cfg):
    """The block kernel's fp32 O (one launch over the whole sequence, as bench.py's P = 1
    step) within the bf16-P bound of the module docstring, and its fp32 LSE within 1e-3."""
    wf = _wf()
    N, h, d, causal, seed = (32768, 32, 128, True, 2) if cfg == "gpt32k" else (65536, 16, 72, False, 6)
    q, k, v, _ = make_qkv_do(N, h, d, seed=seed, peaky=True)
    of, _, lse = wf.block_fwd(q.cuda(), k.cuda(), v.cuda(), causal=causal, chunk=N if causal else 0,
                              qstart=[0] if causal else None, kstart=[0] if causal else None, out_f32=True,
                              out_bf16=False)
    torch.cuda.synchronize()
    rows = _sample_rows(N, seed + 1, k=9)
    Q, K, V = to_f64(q[rows]), to_f64(k), to_f64(v)
    o_ref, l_ref = attention_fwd(Q, K, V, qpos=rows, kpos=np.arange(N), causal=causal)
    pv_abs, _ = attention_fwd(Q, K, np.abs(V), qpos=rows, kpos=np.arange(N), causal=causal)
    err = np.abs(of[rows].double().cpu().numpy() - o_ref)
    bound = 2.0 ** -8 * pv_abs + 1e-5
    assert (err <= bound).all(), (err.max(), (err / bound).max())
    # the kernel error leaves room for the bf16 output rounding (<= 2^-9 |O|) in the 2e-2 bound
    assert (err + 2.0 ** -9 * np.abs(o_ref)).max() <= O_TOL, err.max()
    el = np.abs(lse[:, rows].double().cpu().numpy() - l_ref).max()
    assert el <= 1e-3, el


# ---------------------------------------------------------------------- target: GPT 128K, P = 8
@pytest.fixture(scope="module")
def gpt128k():
    # dK/dV key rows in the last 8192 positions (rank 0's second zigzag chunk): their LSE
    # needs only the last 8192 query rows; the other ranks' dK/dV are covered by the
    # dV column-sum identity and by the 32K/DiT configurations' spread key rows
    return Reference(131072, 32, 128, True, seed=21, P=8, head=3, key_tail=8192)


@pytest.mark.slow
@pytest.mark.parametrize("C", [1, 2, 4])
def test_target_config_emulated_p8(gpt128k, C):
    """BASELINE configs[2]: GPT 32x128 causal, N = 128K, P = 8; C = 1 is the ring baseline,
    C = 2 the paper regime (R = 2 ring of two-unit blocks), C = 4 the extension
    (unit-pipelined, two key units per slice)."""
    o, dq, dk, dv, lse = run_emulated(gpt128k, 8, C)
    ok, errs = check(gpt128k, o, lse, dq, dk, dv)
    assert ok, (C, errs)
    s_dv, s_do = dv.float().sum(0), gpt128k.do.float().sum(0)
    assert (s_dv - s_do).abs().max().item() <= 2e-3 * gpt128k.do.float().abs().sum(0).max().item()


# ---------------------------------------------------------------------- DiT 64K, P = 8
@pytest.fixture(scope="module")
def dit64k():
    return Reference(65536, 16, 72, False, seed=31, P=8, head=11)


@pytest.mark.slow
@pytest.mark.parametrize("C", [1, 2, 4])
def test_dit_config_emulated_p8(dit64k, C):
    """BASELINE configs[3]: DiT 16x72, full mask, N = 64K, P = 8, every C."""
    o, dq, dk, dv, lse = run_emulated(dit64k, 8, C)
    ok, errs = check(dit64k, o, lse, dq, dk, dv)
    assert ok, (C, errs)


# ---------------------------------------------------------------------- edges
@pytest.mark.parametrize("causal,N,h,d", [(True, 256, 1, 128), (False, 128, 1, 64), (True, 512, 3, 64),
                                          (False, 384, 2, 72)])
def test_edge_shapes_single_gpu(causal, N, h, d):
    wf = _wf()
    q, k, v, do = make_qkv_do(N, h, d, seed=9, peaky=True)
    ctx = wf.Context(1, 1)
    o, lse = ctx.fwd(q.cuda(), k.cuda(), v.cuda(), N, causal)
    dq, dk, dv = ctx.bwd(do.cuda(), q.cuda(), k.cuda(), v.cuda(), o, lse, N, causal)
    torch.cuda.synchronize()
    ctx.close()
    dq_r, dk_r, dv_r, o_r, l_r = attention_bwd(to_f64(q), to_f64(k), to_f64(v), to_f64(do), causal=causal)
    assert np.abs(to_f64(o) - o_r).max() <= O_TOL
    for gg, rr in ((dq, dq_r), (dk, dk_r), (dv, dv_r)):
        assert np.abs(to_f64(gg) - rr).max() / np.abs(rr).max() <= G_TOL


def test_error_paths():
    wf = _wf()
    ctx = wf.Context(1, 1)
    q = torch.zeros((256, 2, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(wf.WFError, match="status 2"):  # N not a multiple of 256 (causal)
        ctx.fwd(q[:200].contiguous(), q[:200].contiguous(), q[:200].contiguous(), 200, True)
    q = torch.zeros((256, 2, 96), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(wf.WFError, match="status 2"):  # head_dim not compiled
        ctx.fwd(q, q, q, 256, True)
    q = torch.zeros((256, 2, 128), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(wf.WFError, match="rows"):  # shard rows inconsistent with N / P
        ctx.fwd(q, q, q, 512, True)
    with pytest.raises(wf.WFError, match="bf16"):  # dtype checked before the C ABI
        ctx.fwd(q.float(), q, q, 256, True)
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
        assert np.abs(to_f64(o[rows, hh:hh + 1].cpu()) - o_ref).max() <= O_TOL
        assert np.abs(lse[hh, rows].double().cpu().numpy() - l_ref[0]).max() <= LSE_TOL
    s_dv = dv.float().sum(0)
    s_do = do.float().sum(0)
    assert (s_dv - s_do).abs().max().item() <= 2e-3 * do.float().abs().sum(0).max().item()
