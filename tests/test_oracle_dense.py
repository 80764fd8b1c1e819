"""Pins for oracle/dense.py and oracle/blocks.py against brute force, special
cases and finite differences (never against the oracle's own formula)."""
import math

import numpy as np
import pytest

from oracle.dense import attention_fwd, attention_bwd
from oracle.blocks import init_state, block_attn, forward_iteration, combine, block_bwd


def brute_attention(q, k, v, qpos, kpos, causal):
    """Pure-Python double loop of Eq. 1, one head at a time."""
    nq, h, d = q.shape
    nk = k.shape[0]
    out = [[[0.0] * v.shape[2] for _ in range(h)] for _ in range(nq)]
    lse = [[-math.inf] * nq for _ in range(h)]
    sc = 1.0 / math.sqrt(d)
    for hh in range(h):
        for i in range(nq):
            logits = []
            for j in range(nk):
                if causal and kpos[j] > qpos[i]:
                    continue
                s = sum(float(q[i, hh, t]) * float(k[j, hh, t]) for t in range(d)) * sc
                logits.append((j, s))
            if not logits:
                continue
            mx = max(s for _, s in logits)
            z = sum(math.exp(s - mx) for _, s in logits)
            lse[hh][i] = mx + math.log(z)
            for j, s in logits:
                w = math.exp(s - mx) / z
                for t in range(v.shape[2]):
                    out[i][hh][t] += w * float(v[j, hh, t])
    return np.array(out), np.array(lse)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("shape", [(4, 1, 2), (7, 2, 3), (16, 2, 8)])
def test_dense_matches_brute_force(causal, shape):
    # 4-token causal case vs a literal double loop.
    rng = np.random.default_rng(1)
    n, h, d = shape
    q, k, v = (rng.standard_normal((n, h, d)) for _ in range(3))
    pos = rng.permutation(n) if causal else np.arange(n)
    o, l = attention_fwd(q, k, v, pos, pos, causal)
    ob, lb = brute_attention(q, k, v, pos, pos, causal)
    assert np.allclose(o, ob, atol=1e-12, rtol=0)
    assert np.allclose(l, lb, atol=1e-12, rtol=0)


def test_single_key_returns_v():
    # softmax over one key is 1, output = V.
    q = np.array([[[1.0]]]); k = np.array([[[1.0]]]); v = np.array([[[1.0]]])
    o, l = attention_fwd(q, k, v)
    assert o[0, 0, 0] == 1.0 and l[0, 0] == 1.0  # lse = logit = 1*1/sqrt(1)
    rng = np.random.default_rng(2)
    q = rng.standard_normal((5, 2, 4)); k = rng.standard_normal((1, 2, 4)); v = rng.standard_normal((1, 2, 4))
    o, _ = attention_fwd(q, k, v)
    assert np.allclose(o, np.broadcast_to(v, o.shape), atol=1e-15)


def test_identical_v_rows():
    # convex combination of identical rows is that row.
    rng = np.random.default_rng(3)
    q = rng.standard_normal((9, 2, 4)) * 3; k = rng.standard_normal((11, 2, 4))
    c = rng.standard_normal((1, 2, 4)); v = np.repeat(c, 11, axis=0)
    o, _ = attention_fwd(q, k, v)
    assert np.allclose(o, np.broadcast_to(c, o.shape), atol=1e-13)


def test_fully_masked_row_is_zero_minus_inf():
    # reading c1 / SPEC.md:88: fully masked rows -> O = 0, lse = -inf, never NaN.
    rng = np.random.default_rng(4)
    q, k, v = (rng.standard_normal((3, 1, 2)) for _ in range(3))
    o, l = attention_fwd(q, k, v, qpos=[0, 1, 2], kpos=[5, 6, 7], causal=True)
    assert np.all(o == 0) and np.all(np.isneginf(l))


def test_key_permutation_invariance_full_mask():
    rng = np.random.default_rng(5)
    q, k, v = (rng.standard_normal((6, 2, 4)) for _ in range(3))
    perm = rng.permutation(6)
    o1, l1 = attention_fwd(q, k, v)
    o2, l2 = attention_fwd(q, k[perm], v[perm])
    assert np.allclose(o1, o2, atol=1e-14) and np.allclose(l1, l2, atol=1e-14)


def _loss(q, k, v, g, pos, causal):
    o, _ = attention_fwd(q, k, v, pos, pos, causal)
    return float(np.sum(o * g))


@pytest.mark.parametrize("causal", [False, True])
def test_gradients_match_finite_differences(causal):
    # central differences, step 1e-6, fp64, 1e-5 relative, random 8x4.
    rng = np.random.default_rng(6)
    n, h, d = 8, 1, 4
    q, k, v, g = (rng.standard_normal((n, h, d)) for _ in range(4))
    pos = np.arange(n)
    dq, dk, dv, _, _ = attention_bwd(q, k, v, g, pos, pos, causal)
    eps = 1e-6
    for name, x, ana in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        num = np.zeros_like(x)
        for idx in np.ndindex(x.shape):
            xp = x.copy(); xp[idx] += eps
            xm = x.copy(); xm[idx] -= eps
            args = dict(q=q, k=k, v=v)
            args[name] = xp
            fp = _loss(args["q"], args["k"], args["v"], g, pos, causal)
            args[name] = xm
            fm = _loss(args["q"], args["k"], args["v"], g, pos, causal)
            num[idx] = (fp - fm) / (2 * eps)
        rel = np.abs(num - ana).max() / max(np.abs(num).max(), 1e-12)
        assert rel < 1e-5, (name, rel)


def test_zero_upstream_gradient():
    # d_out = 0 -> all gradients zero.
    rng = np.random.default_rng(7)
    q, k, v = (rng.standard_normal((6, 2, 4)) for _ in range(3))
    dq, dk, dv, _, _ = attention_bwd(q, k, v, np.zeros_like(q), causal=True)
    assert not dq.any() and not dk.any() and not dv.any()


@pytest.mark.parametrize("causal", [False, True])
def test_gradient_column_sum_identities(causal):
    # Rows of P sum to 1 => sum_j dV_j = sum_i dO_i and sum_j dK_j = 0 (any mask).
    # These are the properties the full-size GPU tests use; pinned here too.
    rng = np.random.default_rng(8)
    q, k, v, do = (rng.standard_normal((32, 2, 8)) for _ in range(4))
    dq, dk, dv, _, _ = attention_bwd(q, k, v, do, causal=causal)
    assert np.allclose(dv.sum(0), do.sum(0), atol=1e-12)
    assert np.allclose(dk.sum(0), 0, atol=1e-12)


# ---- blocks -------------------------------------------------------------

def test_merge_into_initial_state_is_identity():
    # SPEC.md:58
    rng = np.random.default_rng(9)
    q, k, v = (rng.standard_normal((5, 2, 3)) for _ in range(3))
    pos = np.arange(5)
    o, l = forward_iteration(init_state(5, 2, 3), q, k, v, pos, pos, False)
    ob, lb = block_attn(q, k, v, pos, pos, False)
    assert np.array_equal(o, ob) and np.array_equal(l, lb)


@pytest.mark.parametrize("causal", [False, True])
def test_two_block_merge_equals_concatenation_any_order(causal):
    # associativity / order independence within 1e-10.
    rng = np.random.default_rng(10)
    n = 12
    q, k, v = (rng.standard_normal((n, 2, 4)) for _ in range(3))
    pos = np.arange(n)
    o, l = attention_fwd(q, k, v, pos, pos, causal)
    a, b = slice(0, 5), slice(5, n)
    for order in ((a, b), (b, a)):
        st = init_state(n, 2, 4)
        for blk in order:
            st = forward_iteration(st, q, k[blk], v[blk], pos, pos[blk], causal)
        assert np.abs(st[0] - o).max() < 1e-10 and np.abs(st[1] - l).max() < 1e-10


def test_fully_masked_block_is_noop():
    # SPEC.md:60
    rng = np.random.default_rng(11)
    q, k, v = (rng.standard_normal((4, 1, 2)) for _ in range(3))
    st = forward_iteration(init_state(4, 1, 2), q, k, v, [4, 5, 6, 7], [0, 1, 2, 3], True)
    st2 = forward_iteration(st, q, k, v, [4, 5, 6, 7], [8, 9, 10, 11], True)
    assert np.array_equal(st[0], st2[0]) and np.array_equal(st[1], st2[1])


def test_combine_disjoint_halves_and_masked_member():
    # SPEC.md:305-306
    rng = np.random.default_rng(12)
    n = 10
    q, k, v = (rng.standard_normal((n, 2, 4)) for _ in range(3))
    pos = np.arange(n)
    o, l = attention_fwd(q, k, v)
    p1 = block_attn(q, k[:4], v[:4], pos, pos[:4], False)
    p2 = block_attn(q, k[4:], v[4:], pos, pos[4:], False)
    oc, lc = combine([p1[0], p2[0]], [p1[1], p2[1]])
    assert np.abs(oc - o).max() < 1e-12 and np.abs(lc - l).max() < 1e-12
    empty = init_state(n, 2, 4)
    oc, lc = combine([p1[0], empty[0]], [p1[1], empty[1]])
    assert np.array_equal(oc, p1[0]) and np.array_equal(lc, p1[1])


@pytest.mark.parametrize("causal", [False, True])
def test_block_bwd_split_sums_to_dense(causal):
    # two-block split equals the single block within 1e-10.
    rng = np.random.default_rng(13)
    n = 16
    q, k, v, do = (rng.standard_normal((n, 2, 4)) for _ in range(4))
    pos = np.arange(n)
    dq, dk, dv, o, lse = attention_bwd(q, k, v, do, pos, pos, causal)
    dd = np.sum(do * o, axis=2).T
    a, b = slice(0, 7), slice(7, n)
    g1 = block_bwd(q, k[a], v[a], do, lse, dd, pos, pos[a], causal)
    g2 = block_bwd(q, k[b], v[b], do, lse, dd, pos, pos[b], causal)
    assert np.abs(g1[0] + g2[0] - dq).max() < 1e-10
    assert np.abs(np.concatenate([g1[1], g2[1]]) - dk).max() < 1e-10
    assert np.abs(np.concatenate([g1[2], g2[2]]) - dv).max() < 1e-10
