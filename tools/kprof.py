"""GPU-box helper: one warm fwd+bwd at the bench workload (GPT 32K causal, P=1) for ncu
kernel captures:  ncu --metrics ... -k regex:wf_block -s 2 -c 2 python tools/kprof.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_00611_b200 as wf  # noqa: E402
from wf_inputs import make_qkv_do  # noqa: E402

N, h, d = 32768, 32, 128
q, k, v, do = (x.cuda() for x in make_qkv_do(N, h, d, seed=0, peaky=True))
ctx = wf.Context(1, 1)
for _ in range(2):
    o, lse = ctx.fwd(q, k, v, N, True)
    dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, True)
torch.cuda.synchronize()
print("ok")
