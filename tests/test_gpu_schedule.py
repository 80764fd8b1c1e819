"""GPU parity of the whole WallFacer path (wf_attn_fwd / wf_attn_bwd through the C ABI)
against the fp64 dense oracle, and of its CommTrace against the oracle's literal
schedule simulation.

Multi-rank configurations run in the library's emulated mode (all P ranks on one
GPU, same schedule and kernels, messages as device copies); the real peer-memory path is
covered by tests/test_multi.py (P processes sharing one GPU, and one process per GPU
under gpurun --gpus N).
"""
from collections import Counter

import numpy as np
import pytest
import torch

from oracle.dense import attention_bwd, attention_fwd
from oracle.schedule import simulate_backward, simulate_forward
from oracle.sharding import unit_positions
from wf_inputs import make_qkv_do, to_f64

pytestmark = pytest.mark.gpu

O_TOL, LSE_TOL, G_TOL = 2e-2, 1e-2, 2e-2


def _wf():
    import paper_2407_00611_b200 as wf
    return wf


def shard_index(P, N, causal):
    return np.concatenate([unit_positions(r, P, N, causal) for r in range(P)])


def run_path(P, C, N, h, d, causal, seed=0, peaky=True, emulated=True, sched=0):
    wf = _wf()
    q, k, v, do = make_qkv_do(N, h, d, seed=seed, peaky=peaky)
    idx = torch.from_numpy(shard_index(P, N, causal))
    dev = torch.device("cuda")
    qs, ks, vs, dos = (t[idx].contiguous().to(dev) for t in (q, k, v, do))
    ctx = wf.Context(P, C, emulated=emulated)
    if sched:
        ctx.set_schedule(sched)
    o, lse = ctx.fwd(qs, ks, vs, N, causal)
    dq, dk, dv = ctx.bwd(dos, qs, ks, vs, o, lse, N, causal)
    torch.cuda.synchronize()
    trace = ctx.trace()
    ctx.close()
    inv = np.argsort(shard_index(P, N, causal))
    n = N // P
    lse_g = lse.reshape(P, h, n).permute(1, 0, 2).reshape(h, N).cpu().double().numpy()[:, inv]
    outs = dict(o=to_f64(o)[inv], lse=lse_g, dq=to_f64(dq)[inv], dk=to_f64(dk)[inv], dv=to_f64(dv)[inv])
    return (q, k, v, do), outs, trace


def check_values(inputs, outs, causal):
    q, k, v, do = (to_f64(t) for t in inputs)
    dq, dk, dv, o, lse = attention_bwd(q, k, v, do, causal=causal)
    errs = dict(o=np.abs(outs["o"] - o).max(), lse=np.abs(outs["lse"] - lse).max())
    for name, ref in (("dq", dq), ("dk", dk), ("dv", dv)):
        errs[name] = np.abs(outs[name] - ref).max() / np.abs(ref).max()
    ok = errs["o"] <= O_TOL and errs["lse"] <= LSE_TOL and max(errs["dq"], errs["dk"], errs["dv"]) <= G_TOL
    return ok, errs


def oracle_trace(P, C, N, h, d, causal, direct=False):
    _, _, ef, _ = simulate_forward(N, None, None, P, C, causal, compute=False, heads=h, head_dim=d, direct=direct)
    _, _, _, eb = simulate_backward(N, None, None, None, None, None, P, C, causal, compute=False, heads=h, head_dim=d,
                                    direct=direct)
    return Counter((e.pas, e.kind, e.step, e.src, e.dst, e.block, e.nbytes) for e in ef + eb)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("d", [128, 72])
def test_single_gpu_real_context(causal, d):
    inputs, outs, trace = run_path(1, 1, 1024, 2, d, causal, emulated=False)
    ok, errs = check_values(inputs, outs, causal)
    assert ok, errs
    assert trace == []


EMU = [(2, 1), (2, 2), (4, 1), (4, 2), (4, 4), (8, 1), (8, 2), (8, 4)]


@pytest.mark.parametrize("P,C", EMU)
@pytest.mark.parametrize("causal", [False, True])
def test_emulated_schedule(P, C, causal):
    N = 256 * P if causal else 128 * P * 2
    h, d = 2, 128
    inputs, outs, trace = run_path(P, C, N, h, d, causal, seed=P + C)
    ok, errs = check_values(inputs, outs, causal)
    assert ok, (P, C, causal, errs)
    assert Counter(trace) == oracle_trace(P, C, N, h, d, causal)


# P = 16: the ring (C = 1, R = 16), R = 4 sub-rings (C = 2), the paper's C = sqrt(P) (R = 1,
# init shuffle only) and the extension C = 8 (C^2 > P): Alg. 2/3 at a size where the init
# pairs and the ring neighbours are no longer all adjacent ranks.  Plain N(0,1) inputs: with
# the peaky recipe |O| reaches ~4.5, where the bf16 rounding of the output alone is up to
# 2^-6 and the max-abs check sits at the edge of the north_star 2e-2 bound (measured 0.0205
# at C = 2 with LSE exact to 7e-6 and gradients at 8e-3); the peaky recipe runs at P <= 8
# above and at full size, with the kernel error separated from the output rounding by
# test_gpu_fullsize.py::test_fp32_output_before_rounding.
@pytest.mark.parametrize("P,C,causal", [(16, 1, True), (16, 2, True), (16, 4, True), (16, 8, True), (16, 4, False)])
def test_emulated_schedule_p16(P, C, causal):
    N = 256 * P if causal else 128 * P * 2
    h, d = 2, 128
    inputs, outs, trace = run_path(P, C, N, h, d, causal, seed=P + C, peaky=False)
    ok, errs = check_values(inputs, outs, causal)
    assert ok, (P, C, causal, errs)
    assert Counter(trace) == oracle_trace(P, C, N, h, d, causal)


def test_emulated_dit_shape():
    # DiT-style head_dim 72, full mask (BASELINE configs[3] shape, small N)
    inputs, outs, _ = run_path(4, 2, 1024, 3, 72, False, seed=7)
    ok, errs = check_values(inputs, outs, False)
    assert ok, errs


@pytest.mark.parametrize("P,C", [(2, 2), (4, 4), (8, 4)])
@pytest.mark.parametrize("causal", [False, True])
def test_emulated_unit_pipelined_extension(P, C, causal):
    # the real-mode decomposition of the extension regime (one launch per (query unit, key
    # unit), W = P / C key units per slice; W = 2 at P = 8, C = 4), run for every virtual rank
    N = 256 * P if causal else 128 * P * 2
    h, d = 2, 128
    inputs, outs, trace = run_path(P, C, N, h, d, causal, seed=P + C + 1)
    ok, errs = check_values(inputs, outs, causal)
    assert ok, (P, C, causal, errs)
    assert Counter(trace) == oracle_trace(P, C, N, h, d, causal)


@pytest.mark.parametrize("P,C", [(4, 2), (8, 2)])
@pytest.mark.parametrize("causal", [False, True])
def test_emulated_direct_pull(P, C, causal):
    # DIRECT-PULL init (wf_set_schedule, reading c21): values, and the trace of the variant
    N = 256 * P if causal else 128 * P * 2
    h, d = 2, 128
    inputs, outs, trace = run_path(P, C, N, h, d, causal, seed=P + C + 5, sched=1)
    ok, errs = check_values(inputs, outs, causal)
    assert ok, (P, C, causal, errs)
    assert Counter(trace) == oracle_trace(P, C, N, h, d, causal, direct=True)
