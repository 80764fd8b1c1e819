"""Record the block kernels' warp-role timelines (clock64 stamps of one CTA) at the
bench workload and save them to gpurun_out/timeline_{fwd,bwd}.npy (GPU box helper)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2407_00611_b200 as wf  # noqa: E402
from paper_2407_00611_b200._lib import lib  # noqa: E402

# WL=dit: the DiT 64K full 16x72 workload instead of GPT 32K causal 32x128
DIT = os.environ.get("WL") == "dit"
N, h, d = (65536, 16, 72) if DIT else (32768, 32, 128)
causal = not DIT
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
dev = torch.device("cuda")
q, k, v, do = (torch.randn((N, h, d), device=dev).to(torch.bfloat16) for _ in range(4))
ctx = wf.Context(1, 1)
o, lse = ctx.fwd(q, k, v, N, causal)
dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, causal)
torch.cuda.synchronize()
n = 4 * 1024 * 8
for name in ("fwd", "bwd"):
    assert lib().wf_debug_timeline(cta) == 0
    if name == "fwd":
        ctx.fwd(q, k, v, N, causal, o=o, lse=lse)
    else:
        ctx.bwd(do, q, k, v, o, lse, N, causal, dq=dq, dk=dk, dv=dv)
    buf = (ctypes.c_uint64 * n)()
    assert lib().wf_debug_timeline_read(buf, n) == 0
    np.save(f"gpurun_out/timeline_{name}{os.environ.get('TLTAG', '')}.npy", np.frombuffer(buf, dtype=np.uint64).reshape(4, 1024, 8))
    lib().wf_debug_timeline(-1)
print("saved")
