"""GPU parity of the WallFacer Transformer layer (paper_2407_00611_b200/layer.py, SURVEY.md
§8(f) item 3) against the fp64 layer oracle (oracle/layer.py): output, input gradient and
every weight gradient, single GPU and emulated multi-rank, with and without
attention-output checkpointing (which must not change any result)."""
import numpy as np
import pytest
import torch

from oracle.layer import WEIGHTS, layer_grads
from oracle.sharding import unit_positions
from wf_inputs import to_f64

pytestmark = pytest.mark.gpu

# north_star's bound (max-abs / max |ref|) for the output, the input gradient and every
# weight gradient; every activation is stored in bf16 between ~12 operators
Y_TOL, G_TOL = 2e-2, 2e-2


def _run(P, C, N, H, h, d, F, causal, checkpoint, seed=0):
    import paper_2407_00611_b200 as wf
    from paper_2407_00611_b200.layer import LayerWeights, WallFacerLayer
    W = LayerWeights.random(H, h, d, F, seed=seed)
    g = torch.Generator().manual_seed(seed + 7)
    x = torch.randn((N, H), generator=g).to(torch.bfloat16)
    dy = torch.randn((N, H), generator=g).to(torch.bfloat16)
    idx = np.concatenate([unit_positions(r, P, N, causal) for r in range(P)])
    ti = torch.from_numpy(idx)
    ctx = wf.Context(P, C, emulated=P > 1)
    layer = WallFacerLayer(ctx, W, h, d, causal=causal, checkpoint=checkpoint)
    y, saved = layer.forward(x[ti].contiguous().cuda(), N)
    dx, grads = layer.backward(dy[ti].contiguous().cuda(), saved, N)
    torch.cuda.synchronize()
    ctx.close()
    inv = np.argsort(idx)
    out = dict(y=to_f64(y)[inv], dx=to_f64(dx)[inv])
    out.update({k: (v.double().cpu().numpy() if v.dtype == torch.float32 else to_f64(v)) for k, v in grads.items()})
    Wn = {k: to_f64(getattr(W, k)) for k in WEIGHTS}
    return out, (to_f64(x), Wn, to_f64(dy))


def _check(out, ref_in, h, d, causal):
    x, W, dy = ref_in
    y_r, dx_r, dW_r = layer_grads(x, W, dy, h, d, causal)
    errs = {"y": np.abs(out["y"] - y_r).max() / np.abs(y_r).max(),
            "dx": np.abs(out["dx"] - dx_r).max() / np.abs(dx_r).max()}
    for k, ref in dW_r.items():
        errs[k] = np.abs(out[k] - ref).max() / np.abs(ref).max()
    ok = errs["y"] <= Y_TOL and all(v <= G_TOL for k, v in errs.items() if k != "y")
    return ok, errs


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("checkpoint", [True, False])
def test_layer_single_gpu(causal, checkpoint):
    h, d = 2, 128
    out, ref_in = _run(1, 1, 512, 256, h, d, 1024, causal, checkpoint)
    ok, errs = _check(out, ref_in, h, d, causal)
    assert ok, errs


@pytest.mark.parametrize("P,C", [(4, 2), (4, 4), (2, 1)])
def test_layer_emulated(P, C):
    h, d = 2, 128
    out, ref_in = _run(P, C, 256 * P, 256, h, d, 1024, True, True, seed=P + C)
    ok, errs = _check(out, ref_in, h, d, True)
    assert ok, errs


def test_checkpointing_is_exact():
    # the forward is deterministic: identical; gradients differ only by the order of the
    # fp32 dQ reductions (TMA reduce-add) and of the norm-weight atomics
    a, _ = _run(4, 2, 1024, 256, 2, 128, 1024, True, True, seed=3)
    b, _ = _run(4, 2, 1024, 256, 2, 128, 1024, True, False, seed=3)
    assert np.array_equal(a["y"], b["y"])
    for k in a:
        assert np.abs(a[k] - b[k]).max() <= 1e-2 * np.abs(b[k]).max(), k
