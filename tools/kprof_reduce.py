"""GPU-box helper: the HBM-bound kernels around the block kernels (team LSE-merge, dQ team sum /
dK-dV owner sums, D preprocess) at C > 1, in emulated mode (all P ranks on one GPU, so a
"peer" partial is read from this GPU's HBM), for ncu captures:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:'wf_(merge|sum|dsum)' python tools/kprof_reduce.py      # GPT shape, P=4, C=2

P, C and N from the environment (P, C, N); GPT heads 32 x 128, causal.  After the warm-up
call it prints, per kernel, the algorithmic bytes of one launch."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2407_00611_b200 as wf  # noqa: E402
from wf_inputs import make_qkv_do  # noqa: E402

P = int(os.environ.get("P", "4"))
C = int(os.environ.get("C", "2"))
N = int(os.environ.get("N", "65536"))
h, d, causal = 32, 128, True
n, E = N // P, h * d
q, k, v, do = (x.cuda() for x in make_qkv_do(N, h, d, seed=0, peaky=False))
ctx = wf.Context(P, C, emulated=True)
for _ in range(2):
    o, lse = ctx.fwd(q, k, v, N, causal)
    dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, causal)
torch.cuda.synchronize()
ctx.close()
# algorithmic bytes per launch (one rank's rows): merge reads C fp32 partials of O and C LSE
# rows, writes bf16 O and fp32 LSE; D reads dO and O (bf16) and writes two fp32 stats rows
merge = C * n * E * 4 + C * n * h * 4 + n * E * 2 + n * h * 4
dsum = 2 * n * E * 2 + 2 * n * h * 4
print(f"P={P} C={C} N={N}: algorithmic bytes per launch: merge {merge / 1e6:.1f} MB, dsum {dsum / 1e6:.1f} MB; "
      f"sum: (parts x 4 + 2) x n x E = {(4 + 2) * n * E / 1e6:.1f} MB per fp32 part")
