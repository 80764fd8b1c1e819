"""Analytic cost and memory model (Eqs. 2-7).

Two layers:

* the paper's closed forms, as printed: Eq. 2 (Ring Attention P2P time), Eq. 3 (WallFacer
  all-gather + reduce-scatter), Eq. 4 (WallFacer ring P2P), Eq. 5 (one activation A),
  Eqs. 6-7 (peak memory, in units of A);
* a prediction for THIS library: bytes per phase from the library's own plan trace
  (wf_plan_trace, the same schedule the GPU path runs), block-kernel time from the
  kernel rates, transfer time from a link bandwidth, combined with the overlap the
  runtime implements (ring transfers of step s+1 hide behind the block kernel of step s;
  gathers, init shuffle and reductions are exposed except in the unit-pipelined
  extension regime, where each unit's kernel waits only for its own unit).

The prediction is host logic (no oracle, no GPU).  bench.py prints it next to the measured
step time; tools/cost_report.py prints the table for the BASELINE configurations.
"""
from __future__ import annotations

from collections import defaultdict

from .wf import plan, plan_trace, workspace_bytes

# ----------------------------------------------------------------- the paper's equations


def eq2_ring(B, N, H, P, W=1.0, L=0.0):
    """Eq. 2: Ring Attention P2P cost per forward block = 2BNH/W + P L.
    W in elements per unit time; returns elements/W + latency."""
    return P * (2 * B * N * H / (P * W) + L)


def eq3_collective(B, N, H, P, C, W=1.0):
    """Eq. 3: WallFacer all-gather + reduce-scatter = 4BNH(C-1)/(PW)."""
    return 4 * B * N * H * (C - 1) / (P * W)


def eq4_p2p(B, N, H, P, C, W=1.0, L=0.0):
    """Eq. 4: WallFacer ring P2P = P/C^2 (2CBNH/(PW) + L)."""
    return P / (C * C) * (2 * C * B * N * H / (P * W) + L)


def eq5_activation(B, N, H, P):
    """Eq. 5: one activation of a sub-sequence on one GPU, A = BNH/P."""
    return B * N * H / P


def eq6_peak_ring(Y):
    """Eq. 6: PM_Ring - M_{m+o} = (Y + 4) A; returns the multiple of A."""
    return Y + 4


def eq7_peak_wall(Y, C):
    """Eq. 7: PM_Wall - M_{m+o} = (Y + 3C + 1) A."""
    return Y + 3 * C + 1


# ----------------------------------------------------------------- this library's schedule

def schedule_bytes(P, C, N, heads, head_dim):
    """Bytes each rank RECEIVES per (pass, kind), from the library's plan trace.
    Returns {rank: {(pass, kind): bytes}}; pass 0 = forward, 1 = backward."""
    out = {r: defaultdict(int) for r in range(P)}
    for pas, kind, _step, _src, dst, _blk, nbytes in plan_trace(P, C, N, heads, head_dim, -1):
        out[dst][(pas, kind)] += nbytes
    return out


def per_step_bytes(P, C, N, heads, head_dim):
    """Bytes of one ring hop, forward (K/V block) and backward (Q-package + dQ)."""
    n, E = N // P, heads * head_dim
    fwd = 2 * C * n * E * 2
    bwd = 2 * C * n * E * 2 + 2 * C * n * heads * 4 + C * n * E * 4
    return fwd, bwd


def flops(N, heads, head_dim, causal):
    """FlashAttention convention: fwd 4 N^2 h d (x 1/2 causal), bwd 2.5 x fwd."""
    f = 4.0 * N * N * heads * head_dim * (0.5 if causal else 1.0)
    return f, 2.5 * f


_RING = {"RING_KV", "RING_QPKG", "RING_DQ"}
_PRE = {"AG_Q", "AG_KV", "AG_QDO", "AG_STATS", "INIT_KV", "SLICE_KV"}
_POST = {"RS_O", "RS_LSE", "RET_DQ", "REV_DKV", "RS_DQ"}


def predict(P, C, N, heads, head_dim, causal, fwd_tflops, bwd_tflops, link_gbps=700.0, latency_us=10.0):
    """Predicted per-rank step time (ms) of wf_attn_fwd + wf_attn_bwd.

    fwd_tflops / bwd_tflops: block-kernel rates (algorithmic TFLOP/s of one GPU's kernels);
    link_gbps: per-GPU receive bandwidth of a peer copy; latency_us: per message phase.
    Returns a dict with the per-phase terms, the totals and the exposed-comm prediction;
    the max over ranks is taken for every byte count (the slowest rank sets the step)."""
    ff, fb = flops(N, heads, head_dim, causal)
    comp_f = ff / P / (fwd_tflops * 1e12) * 1e3
    comp_b = fb / P / (bwd_tflops * 1e12) * 1e3
    pl = plan(P, C, 0)
    R, ext = pl["R"], pl["regime"] == "ext"
    step_f, step_b = per_step_bytes(P, C, N, heads, head_dim)
    by = schedule_bytes(P, C, N, heads, head_dim)

    def phase_ms(pas, kinds, byte_share=1.0):
        """Slowest rank's bytes of these kinds at link_gbps (times byte_share) plus one
        latency per message kind present."""
        worst = max(sum(b for (p, k), b in d.items() if p == pas and k in kinds) for d in by.values())
        nmsg = len([k for k in kinds if any(d.get((pas, k), 0) for d in by.values())])
        return byte_share * worst / (link_gbps * 1e9) * 1e3 + (latency_us * 1e-3 * nmsg if worst else 0.0)

    lat = latency_us * 1e-3
    res = {"P": P, "C": C, "R": R, "regime": "ext" if ext else "paper"}
    for pas, comp, hop in ((0, comp_f, step_f), (1, comp_b, step_b)):
        pre, post = phase_ms(pas, _PRE), phase_ms(pas, _POST)
        if ext and C > 1:
            # unit-pipelined (the peer-memory transport, the library's only real-mode one): of
            # the C-1 member partials a rank receives, all but the one its sender finishes last
            # were pushed during later units; only that one's bytes are exposed, while every
            # message kind still pays its latency
            rs = {"RS_O", "RS_LSE", "RS_DQ"}
            post = phase_ms(pas, _POST - rs) + phase_ms(pas, rs, byte_share=1.0 / (C - 1))
        if R > 1:
            per = comp / R
            ring = per + (R - 1) * max(per, hop / (link_gbps * 1e9) * 1e3 + lat)
        else:
            ring = comp
        if ext and C > 1:
            # unit-pipelined: the first unit's kernel waits for one of the P units, the rest overlap
            units = P
            pre_exposed = pre / units
            pre_total = max(pre, comp) - comp + pre_exposed
        else:
            pre_total = pre
        name = "fwd" if pas == 0 else "bwd"
        res[name] = {"compute_ms": comp, "pre_ms": pre_total, "ring_ms": ring, "post_ms": post,
                     "total_ms": pre_total + ring + post}
    res["total_ms"] = res["fwd"]["total_ms"] + res["bwd"]["total_ms"]
    res["compute_ms"] = comp_f + comp_b
    res["exposed_comm_frac"] = 1.0 - res["compute_ms"] / res["total_ms"]
    res["recv_bytes_max"] = max(sum(d.values()) for d in by.values())
    return res


def memory(P, C, N, heads, head_dim, causal, Y=None):
    """Device memory of one rank: the library workspace and the caller's tensors, beside the
    paper's activation accounting (Eq. 5-7).  Y (layers) adds the paper's checkpoint term."""
    n, E = N // P, heads * head_dim
    A = n * E * 2  # Eq. 5 in bytes (bf16)
    ws = workspace_bytes(P, C, N, heads, head_dim, causal)
    io = 8 * n * E * 2 + n * heads * 4  # Q K V O dO dQ dK dV + LSE
    out = {"A_bytes": A, "workspace_bytes": ws, "caller_bytes": io, "workspace_over_A": ws / A,
           "paper_team_3CA_bytes": 3 * C * A}
    if Y is not None:
        out["paper_peak_ring_A"] = eq6_peak_ring(Y)
        out["paper_peak_wall_A"] = eq7_peak_wall(Y, C)
    return out
