"""Communication Topology Scheduler (§3.4, Eq. 8).

    Config = argmax_{C, placement} Profile(C in [1, sqrt(P)], placement in [P2P_intra, Collect_intra])

"The scheduler requires only a few iterations to profile the performance of
automatically generated configurations".  On one NVSwitch node every GPU
pair has the same bandwidth, so placement has no effect and the search is
over the team size C.  The candidate set follows reading c2: every C with C | P and
(C^2 <= P => C^2 | P), i.e. the paper's range plus our C^2 > P extension; for the
paper-regime team sizes both schedules of the first K/V block are profiled (the paper's
gather + init shuffle, and the DIRECT-PULL variant, reading c21).

Every rank profiles the same candidates in the same order through the C ABI (wf_attn_fwd
+ wf_attn_bwd), the per-candidate time is the max over ranks (all_reduce MAX), and all
ranks take the same argmax.
"""
from __future__ import annotations

import torch

from .wf import Context


def candidates(P: int, cmax: int = 4):
    """Valid team sizes up to cmax (BASELINE.json's metric sweeps C in {1, 2, 4})."""
    out = []
    for C in range(1, min(P, cmax) + 1):
        if P % C:
            continue
        if C * C <= P and P % (C * C):
            continue
        out.append(C)
    return out


def variants(P, cmax=4):
    """(C, schedule) pairs: every valid C, and for the paper-regime team sizes (1 < C, C^2 <= P)
    also the DIRECT-PULL init variant (wf_set_schedule, reading c21)."""
    out = []
    for C in candidates(P, cmax):
        out.append((C, 0))
        if 1 < C and C * C <= P:
            out.append((C, 1))
    return out


def label(C, sched):
    return f"{C}" + ("/direct" if sched else "")


def search(P, rank, N, heads, head_dim, causal, steps=2, warmup=1, cands=None, group=None):
    """Profile each candidate (C, schedule); returns (best_C, best_schedule, {label: ms_per_step})."""
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    n = N // P
    g = torch.Generator(device=dev).manual_seed(777 + rank)
    q, k, v, do = (torch.randn((n, heads, head_dim), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty((heads, n), dtype=torch.float32, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    table, keys = {}, {}
    for C, sched in cands or variants(P):
        ctx = Context(P, C, rank=rank, group=group)
        if sched:
            ctx.set_schedule(sched)
        for _ in range(warmup):
            ctx.fwd(q, k, v, N, causal, o=o, lse=lse)
            ctx.bwd(do, q, k, v, o, lse, N, causal, dq=dq, dk=dk, dv=dv)
        if P > 1:
            dist.barrier(group=group)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            ctx.fwd(q, k, v, N, causal, o=o, lse=lse)
            ctx.bwd(do, q, k, v, o, lse, N, causal, dq=dq, dk=dk, dv=dv)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
        if P > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        table[label(C, sched)] = float(t.item())
        keys[label(C, sched)] = (C, sched)
        ctx.close()
    best = min(table, key=table.get)
    return keys[best][0], keys[best][1], table
