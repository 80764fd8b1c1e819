"""GPU-box helper: the target configuration's compute in emulation -- all P ranks of a
(P, C) job on one GPU (messages become device copies), timed with CUDA events.  The time
per step divided by P estimates one rank's compute-bound step at that launch
configuration (no NVLink transfers, no cross-rank waits).

    python tools/emu_bench.py [--P 8] [--N 131072 ...] [--C 1 4] [--workload gpt|dit]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_00611_b200 as wf  # noqa: E402
from paper_2407_00611_b200.scheduler import candidates  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=8)
    ap.add_argument("--N", type=int, nargs="+", default=[131072])
    ap.add_argument("--C", type=int, nargs="*", default=None)
    ap.add_argument("--workload", default="gpt", choices=["gpt", "dit"])
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    P = a.P
    h, d, causal = (32, 128, True) if a.workload == "gpt" else (16, 72, False)
    for N in a.N:
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v, do = (torch.randn((N, h, d), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
        fl = 3.5 * 4.0 * N * N * h * d * (0.5 if causal else 1.0)
        for C in (a.C or candidates(P)):
            ctx = wf.Context(P, C, emulated=True)
            o, lse = ctx.fwd(q, k, v, N, causal)
            dq, dk, dv = ctx.bwd(do, q, k, v, o, lse, N, causal)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                ctx.fwd(q, k, v, N, causal, o=o, lse=lse)
                ctx.bwd(do, q, k, v, o, lse, N, causal, dq=dq, dk=dk, dv=dv)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            ctx.close()
            torch.cuda.empty_cache()
            print(json.dumps({"workload": a.workload, "P": P, "C": C, "N": N, "emulated_ms_all_ranks": ms,
                              "est_rank_ms": ms / P, "est_tflops_per_gpu": fl / P / (ms / P / 1e3) / 1e12}),
                  flush=True)
        del q, k, v, do
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
