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


def search(P, rank, N, heads, head_dim, causal, steps=5, warmup=2, rounds=3, cands=None, group=None,
           emulated=False):
    """Profile each candidate (C, schedule); returns (best_C, best_schedule, table) with
    table[label] = {"ms": median over rounds of the per-step time (max over ranks),
    "spread": (max - min) / median over the rounds}.

    Every candidate gets its own context (kept alive for the whole search) and `warmup`
    untimed steps; then `rounds` interleaved rounds time `steps` steps of every candidate
    in turn, so slow drifts of the clock (power cap) hit all candidates alike.  emulated:
    all P ranks on this GPU (wf_init_emulated; tests), inputs stacked rank-major."""
    import statistics
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device())
    dist_on = P > 1 and not emulated
    rows = N if emulated else N // P
    g = torch.Generator(device=dev).manual_seed(777 + rank)
    q, k, v, do = (torch.randn((rows, heads, head_dim), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty((P, heads, rows // P) if emulated else (heads, rows), dtype=torch.float32, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    cands = list(cands or variants(P))
    ctxs = []
    try:
        for C, sched in cands:
            ctx = Context(P, C, rank=rank, group=group, emulated=emulated)
            ctxs.append(ctx)
            if sched:
                ctx.set_schedule(sched)

        def run(ctx, n):
            for _ in range(n):
                ctx.fwd(q, k, v, N, causal, o=o, lse=lse)
                ctx.bwd(do, q, k, v, o, lse, N, causal, dq=dq, dk=dk, dv=dv)

        for ctx in ctxs:
            run(ctx, warmup)
        times = {label(C, s): [] for C, s in cands}
        for _ in range(rounds):
            for (C, sched), ctx in zip(cands, ctxs):
                if dist_on:
                    dist.barrier(group=group)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run(ctx, steps)
                e1.record()
                torch.cuda.synchronize()
                t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
                if dist_on:
                    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
                times[label(C, sched)].append(float(t.item()))
    finally:
        for ctx in ctxs:
            ctx.close()
    table = {}
    for key, ts in times.items():
        med = statistics.median(ts)
        table[key] = {"ms": med, "spread": (max(ts) - min(ts)) / med}
    best = min(table, key=lambda x: table[x]["ms"])
    C, sched = dict((label(c, s), (c, s)) for c, s in cands)[best]
    return C, sched, table
