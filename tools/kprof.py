"""GPU-box helper: one warm fwd+bwd at a bench workload (P=1) for ncu kernel captures:
  ncu --metrics ... -k regex:wf_block -s 2 -c 2 python tools/kprof.py          # GPT 32K causal
  WL=dit ncu ... python tools/kprof.py                                           # DiT 64K full 16x72
"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_00611_b200 as wf  # noqa: E402
from wf_inputs import make_qkv_do  # noqa: E402

if os.environ.get("WL", "gpt") == "dit":
    N, h, d, causal = 65536, 16, 72, False
else:
    N, h, d, causal = 32768, 32, 128, True
q, k, v, do = (x.cuda() for x in make_qkv_do(N, h, d, seed=0, peaky=True))
ctx = wf.Context(1, 1)
for _ in range(2):
    o, lse = ctx.fwd(q, k, v, N, causal)
    dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, causal)
torch.cuda.synchronize()
print("ok")
