"""GPU-box helper: small invocations of every kernel for compute-sanitizer
(memcheck / synccheck / racecheck):

    compute-sanitizer --tool memcheck  python tools/sanitize.py [--multi]
    compute-sanitizer --tool synccheck python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py

Covers the block forward (d = 64, 72, 128; contiguous, zigzag, with an incoming state),
the block backward, the projection GEMM (single-CTA and CTA-pair, three layouts), the
layer operators, and the emulated schedule at P = 4 (C = 1 ring, C = 2 paper regime,
C = 4 unit-pipelined extension: merge, D, sum kernels).  --multi adds a two-process real
run on this GPU (gloo bootstrap): the signal/wait kernel, IPC pulls and pushes.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00611_b200 as wf  # noqa: E402
from wf_inputs import make_qkv_do  # noqa: E402


def blocks():
    for d in (64, 72, 128):
        q, k, v, do = (t.cuda() for t in make_qkv_do(512, 2, d, seed=1))
        of, ob, lse = wf.block_fwd(q, k, v, causal=False, out_f32=True)
        wf.block_fwd(q, k, v, causal=True, chunk=256, qstart=[0, 768], kstart=[256, 512], o_in=of, lse_in=lse,
                     out_f32=True)
        dsum = (do.float() * ob.float()).sum(-1).t().contiguous()
        dq = torch.zeros(q.shape, dtype=torch.float32, device="cuda")
        dk, dv = torch.zeros_like(dq), torch.zeros_like(dq)
        wf.block_bwd(q, k, v, do, lse, dsum, dq, dk, dv, causal=True, chunk=256, qstart=[0, 768],
                     kstart=[0, 768])
    torch.cuda.synchronize()


def gemms():
    a = torch.randn((256, 128), device="cuda").to(torch.bfloat16)
    b = torch.randn((512, 128), device="cuda").to(torch.bfloat16)
    wf.gemm_bf16(a, b)
    wf.gemm_bf16(a, b[:384].contiguous())
    wf.gemm_bf16(a.t().contiguous(), b, a_mn=True)
    wf.gemm_bf16(a, b.t().contiguous(), b_mn=True)
    torch.cuda.synchronize()


def layer_ops():
    x = torch.randn((256, 512), device="cuda").to(torch.bfloat16)
    w = torch.ones(512, device="cuda").to(torch.bfloat16)
    y, m, r = wf.layernorm_fwd(x, w, w)
    dw = torch.zeros(512, device="cuda")
    db = torch.zeros(512, device="cuda")
    wf.layernorm_bwd(y, x, w, m, r, dw, db, dres=x)
    h = wf.gelu_fwd(x)
    wf.gelu_bwd(h, x)
    wf.add_bf16(x, h)
    e = x[:, :256].contiguous()
    wf.pack3(e, e, e)
    torch.cuda.synchronize()


def schedule():
    from oracle.sharding import unit_positions  # noqa: F401  (input layout only)
    for P, C, causal in ((4, 1, True), (4, 2, True), (4, 4, True), (4, 2, False)):
        N, h, d = 512 * P, 2, 128
        q, k, v, do = (t.cuda() for t in make_qkv_do(N, h, d, seed=P + C))
        ctx = wf.Context(P, C, emulated=True)
        o, lse = ctx.fwd(q, k, v, N, causal)
        ctx.bwd(do, q, k, v, o, lse, N, causal)
        torch.cuda.synchronize()
        ctx.close()


def multi():
    import torch.multiprocessing as mp
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    from test_multi import _spawn  # noqa: E402
    res = _spawn(2, True, [("attn", 1, 1024, True, 2), ("attn", 2, 1024, True, 2)])
    assert len(res) == 2
    del mp


if __name__ == "__main__":
    blocks()
    gemms()
    layer_ops()
    schedule()
    if "--multi" in sys.argv:
        multi()
    print("sanitize workload done")
