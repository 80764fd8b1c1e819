"""Non-authoritative sanity: the single-GPU path against torch's
scaled_dot_product_attention (the library attention in this image) on the same bf16 inputs.
The oracle (tests/test_gpu_*.py) is the reference; this only guards against a shared
misreading of the attention definition between the oracle and the kernels."""
import pytest
import torch

from wf_inputs import make_qkv_do

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("d", [128, 64])
def test_matches_torch_sdpa(causal, d):
    import paper_2407_00611_b200 as wf
    N, h = 2048, 4
    q, k, v, do = (t.cuda() for t in make_qkv_do(N, h, d, seed=5, peaky=False))
    ctx = wf.Context(1, 1)
    o, lse = ctx.fwd(q, k, v, N, causal)
    dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, causal)
    torch.cuda.synchronize()
    ctx.close()
    # torch reference in fp32 from the same bf16 values, layout [batch, heads, tokens, d]
    qt, kt, vt = (t.float().permute(1, 0, 2).unsqueeze(0).requires_grad_(True) for t in (q, k, v))
    ot = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, is_causal=causal)
    ot.backward(do.float().permute(1, 0, 2).unsqueeze(0))
    ref = {"o": ot, "dq": qt.grad, "dk": kt.grad, "dv": vt.grad}
    got = {"o": o, "dq": dq, "dk": dk, "dv": dv}
    for name, r in ref.items():
        r = r.detach().squeeze(0).permute(1, 0, 2)
        err = (got[name].float() - r).abs().max().item() / max(r.abs().max().item(), 1e-6)
        assert err <= 2e-2, (name, err)
