"""Literal simulation of WallFacer's P/C schedule with fp64 payloads (TEST INFRASTRUCTURE).

Forward = Alg. 1, rank by rank:
  l.1  team all-gather of Q, K, V (AllGather_QKVmatmul; the projection itself is
       outside the path)                      -> AG_Q, AG_KV
  l.2  send the team K/V block to r_send, receive from r_recv -> INIT_KV
  l.3  get_P2P_ranks -> next / last (Alg. 3)
  l.4  O = 0, lse = -inf (reading c1)
  l.5-10 for i in 1..P/C^2: forward_iteration on the current block, and pass the
       block to `next` (double buffer) -> RING_KV; the wasted send after the last
       iteration (l.8 at i = P/C^2) is not performed (reading c3)
  l.11 ReduceScatter_combine inside the team              -> RS_O, RS_LSE
Backward = §3.2.1 "Backward Propagation": K/V outer loop
stationary on the init-shuffle block, Q inner loop: the Q-package (Q, dO, LSE, D)
and its dQ circulate along the sub-ring (RING_QPKG, RING_DQ), then one extra P2P
returns dQ home (RET_DQ; reading c10).  The paper is silent on where dK/dV go
(reading c11, revised): each holder of a stationary block sends every unit's rows of
its dK/dV partial straight to the unit's owner, who sums the C replicas (REV_DKV);
dQ is summed by a team reduce-scatter (RS_DQ).
Extension regime C^2 > P (reading c2, ours): R = 1, only Q (and dO, stats) are
team-gathered; member a pulls K/V slice a = units [a P/C, (a+1) P/C) from their
owners (SLICE_KV); dK/dV partials go straight back to the owners (REV_DKV).

Messages go through a mailbox network: every receive must match a send with the
same (kind, step, src, dst) and the network must be empty at the end
(quiescence).  A record (pass, kind, step, src, dst, block, bytes)
is emitted for every message with src != dst (self-sends are local, reading c4).
Byte widths (reading c17): Q/K/V/dO bf16 (2 B); partial O, LSE, D and the
dQ/dK/dV partials fp32 (4 B).  Step numbering: -1 gathers and init shuffle;
s in [0, R-2] for the hop after compute step s; R-1 for RET_DQ; R for the
post-loop reductions.  Block ids: see DESIGN.md "CommTrace".

Pinned by tests/test_oracle_schedule.py: assembled outputs equal the dense
oracle (<= 1e-10) for P <= 16, C in {1,2,4}, both masks; byte totals equal the
paper's Eqs. 2-4 and its model-M numbers.
"""
from __future__ import annotations

from collections import namedtuple

import numpy as np

from .blocks import init_state, forward_iteration, combine, block_bwd
from .sharding import unit_positions, team_positions
from .topology import build_plan

__all__ = ["Event", "KINDS", "Network", "simulate_forward", "simulate_backward", "trace_totals"]

Event = namedtuple("Event", "pas kind step src dst block nbytes")

KINDS = ["AG_Q", "AG_KV", "INIT_KV", "SLICE_KV", "RING_KV", "RS_O", "RS_LSE",
         "AG_QDO", "AG_STATS", "RING_QPKG", "RING_DQ", "RET_DQ", "REV_DKV", "RS_DKV", "RS_DQ"]


class Network:
    def __init__(self):
        self.box = {}
        self.events = []

    def send(self, pas, kind, step, src, dst, block, nbytes, payload=None):
        key = (kind, step, src, dst)
        if key in self.box:
            raise RuntimeError(f"duplicate message {key}")
        self.box[key] = (block, payload)
        if src != dst:
            self.events.append(Event(pas, kind, step, src, dst, block, int(nbytes)))

    def recv(self, kind, step, src, dst):
        key = (kind, step, src, dst)
        if key not in self.box:
            raise RuntimeError(f"unmatched receive {key} (deadlock)")
        return self.box.pop(key)

    def assert_quiescent(self):
        if self.box:
            raise RuntimeError(f"unconsumed messages: {sorted(self.box)[:4]}")


def _slice_units(a, P, C):
    w = P // C
    return list(range(a * w, (a + 1) * w))


def _rows_of_member(arr, j, n):
    return arr[j * n:(j + 1) * n]


def simulate_forward(Q, K, V, P, C, causal, compute=True, heads=None, head_dim=None, net=None, direct=False):
    """Q/K/V: global [N, h, d] float64 (or None with compute=False).

    direct: the DIRECT-PULL init variant (SURVEY.md §8(a) "Schedule variants", reading
    c21): in the paper regime the K/V team all-gather and the init shuffle are replaced by
    one message per unit from its owner to every rank whose initial block contains it
    (kind SLICE_KV, as in the extension regime); the ring itself is unchanged.

    Returns (O [N,h,d], LSE [h,N], events, ctx) -- outputs in global token order.
    """
    plan = build_plan(P, C)
    if compute:
        N, h, d = Q.shape
    else:
        N, h, d = Q, heads, head_dim  # Q carries N in trace-only mode
    n = N // P
    E = h * d
    T, R = plan["T"], plan["R"]
    net = net or Network()
    pos = {u: unit_positions(u, P, N, causal) for u in range(P)}
    local = {u: ((Q[pos[u]], K[pos[u]], V[pos[u]]) if compute else None) for u in range(P)}

    # Alg. 1 l.1: team all-gather (every rank sends its unit to each teammate).
    for r in range(P):
        t = r // C
        for p in range(t * C, t * C + C):
            net.send(0, "AG_Q", -1, r, p, r, n * E * 2, local[r][0] if compute else None)
            if plan["regime"] == "paper" and not direct:
                net.send(0, "AG_KV", -1, r, p, r, 2 * n * E * 2, local[r][1:] if compute else None)
    team = {}
    for r in range(P):
        t = r // C
        members = list(range(t * C, t * C + C))
        qs, kvs = [], []
        for p in members:
            _, q = net.recv("AG_Q", -1, p, r)
            qs.append(q)
            if plan["regime"] == "paper" and not direct:
                _, kv = net.recv("AG_KV", -1, p, r)
                kvs.append(kv)
        entry = dict(qpos=team_positions(members, P, N, causal))
        if compute:
            entry["q"] = np.concatenate(qs)
            if kvs:
                entry["k"] = np.concatenate([x[0] for x in kvs])
                entry["v"] = np.concatenate([x[1] for x in kvs])
        team[r] = entry

    partial = {}
    if plan["regime"] == "paper":
        send, recv, nxt, lst = plan["send"], plan["recv"], plan["next"], plan["last"]
        cur = {}
        if direct:
            # the units of the initial block team(recv[r]) straight from their owners
            for r in range(P):
                blk = recv[r] // C
                for u in range(blk * C, blk * C + C):
                    net.send(0, "SLICE_KV", -1, u, r, u, 2 * n * E * 2, local[u][1:] if compute else None)
            for r in range(P):
                blk = recv[r] // C
                kvs = [net.recv("SLICE_KV", -1, u, r)[1] for u in range(blk * C, blk * C + C)]
                kv = ((np.concatenate([x[0] for x in kvs]), np.concatenate([x[1] for x in kvs])) if compute else None)
                cur[r] = (blk, kv)
        else:
            # Alg. 1 l.2: init shuffle of the team K/V block.
            for r in range(P):
                t = r // C
                kv = (team[r]["k"], team[r]["v"]) if compute else None
                net.send(0, "INIT_KV", -1, r, send[r], t, 2 * C * n * E * 2, kv)
            for r in range(P):
                blk, kv = net.recv("INIT_KV", -1, recv[r], r)
                cur[r] = (blk, kv)
        state = {r: (init_state(C * n, h, d) if compute else None) for r in range(P)}
        for s in range(R):                                         # Alg. 1 l.5
            for r in range(P):
                blk, kv = cur[r]
                if compute:                                        # l.9
                    kpos = team_positions(range(blk * C, blk * C + C), P, N, causal)
                    state[r] = forward_iteration(state[r], team[r]["q"], kv[0], kv[1], team[r]["qpos"], kpos, causal)
                if s < R - 1:                                      # l.8, no wasted final send
                    net.send(0, "RING_KV", s, r, nxt[r], blk, 2 * C * n * E * 2, kv)
            if s < R - 1:
                for r in range(P):
                    cur[r] = net.recv("RING_KV", s, lst[r], r)
        partial = state
    else:
        for r in range(P):
            a = r % C
            for u in _slice_units(a, P, C):
                net.send(0, "SLICE_KV", -1, u, r, u, 2 * n * E * 2, local[u][1:] if compute else None)
        for r in range(P):
            a = r % C
            units = _slice_units(a, P, C)
            kvs = [net.recv("SLICE_KV", -1, u, r)[1] for u in units]
            if compute:
                k = np.concatenate([x[0] for x in kvs])
                v = np.concatenate([x[1] for x in kvs])
                kpos = team_positions(units, P, N, causal)
                partial[r] = forward_iteration(init_state(C * n, h, d), team[r]["q"], k, v, team[r]["qpos"], kpos, causal)
            else:
                partial[r] = None

    # Alg. 1 l.11: ReduceScatter_combine inside the team.
    for r in range(P):
        t = r // C
        for j, p in enumerate(range(t * C, t * C + C)):
            if compute:
                o, l = partial[r]
                po, pl = _rows_of_member(o, j, n), l[:, j * n:(j + 1) * n]
            else:
                po = pl = None
            net.send(0, "RS_O", R, r, p, p, n * E * 4, po)
            net.send(0, "RS_LSE", R, r, p, p, n * h * 4, pl)
    O = np.zeros((N, h, d)) if compute else None
    LSE = np.full((h, N), -np.inf) if compute else None
    for r in range(P):
        t = r // C
        outs, lses = [], []
        for p in range(t * C, t * C + C):
            outs.append(net.recv("RS_O", R, p, r)[1])
            lses.append(net.recv("RS_LSE", R, p, r)[1])
        if compute:
            o, l = combine(outs, lses)
            O[pos[r]] = o
            LSE[:, pos[r]] = l
    net.assert_quiescent()
    return O, LSE, net.events, dict(plan=plan, n=n, E=E)


def simulate_backward(Q, K, V, dO, O, LSE, P, C, causal, compute=True, heads=None, head_dim=None, net=None,
                      direct=False, log=None):
    """Backward of the schedule.  O, LSE: final forward outputs (global order).
    direct: the DIRECT-PULL init variant (see simulate_forward) for the stationary block.
    log: optional dict; receives the bookkeeping the coverage pins check:
      "visits"  list of (rank, step, query team, key units) of every block_bwd call;
      "dq_home" list of (rank, team) of every dQ partial that reached its final holder;
      "dkv"     {unit: number of dK/dV replica partials its owner summed}.

    Returns (dQ, dK, dV, events).
    """
    plan = build_plan(P, C)
    if compute:
        N, h, d = Q.shape
    else:
        N, h, d = Q, heads, head_dim
    n = N // P
    E = h * d
    T, R = plan["T"], plan["R"]
    net = net or Network()
    pos = {u: unit_positions(u, P, N, causal) for u in range(P)}
    loc = {}
    for u in range(P):
        if compute:
            p = pos[u]
            dd = np.sum(dO[p] * O[p], axis=2).T                 # D = rowsum(dO o O) [h, n] (reading c12)
            loc[u] = dict(q=Q[p], k=K[p], v=V[p], do=dO[p], lse=LSE[:, p], dd=dd)
        else:
            loc[u] = None

    # Team gathers: Q+dO, LSE+D, and (paper regime) K+V.
    for r in range(P):
        t = r // C
        for p in range(t * C, t * C + C):
            x = loc[r]
            net.send(1, "AG_QDO", -1, r, p, r, 2 * n * E * 2, (x["q"], x["do"]) if compute else None)
            net.send(1, "AG_STATS", -1, r, p, r, 2 * n * h * 4, (x["lse"], x["dd"]) if compute else None)
            if plan["regime"] == "paper" and not direct:
                net.send(1, "AG_KV", -1, r, p, r, 2 * n * E * 2, (x["k"], x["v"]) if compute else None)
    team = {}
    for r in range(P):
        t = r // C
        members = list(range(t * C, t * C + C))
        qd = [net.recv("AG_QDO", -1, p, r)[1] for p in members]
        st = [net.recv("AG_STATS", -1, p, r)[1] for p in members]
        kv = [net.recv("AG_KV", -1, p, r)[1] for p in members] if plan["regime"] == "paper" and not direct else []
        e = dict(qpos=team_positions(members, P, N, causal), t=t)
        if compute:
            e["q"] = np.concatenate([x[0] for x in qd])
            e["do"] = np.concatenate([x[1] for x in qd])
            e["lse"] = np.concatenate([x[0] for x in st], axis=1)
            e["dd"] = np.concatenate([x[1] for x in st], axis=1)
            if kv:
                e["k"] = np.concatenate([x[0] for x in kv])
                e["v"] = np.concatenate([x[1] for x in kv])
        team[r] = e

    dq_part = {}   # rank -> dQ partial for its own team's C*n rows (after return hop)
    dkv_part = {}  # rank -> (dK, dV) replica partial for its own team block / or per-unit dict (ext)
    if plan["regime"] == "paper":
        send, recv, nxt, lst = plan["send"], plan["recv"], plan["next"], plan["last"]
        if direct:
            for r in range(P):
                b = recv[r] // C
                for u in range(b * C, b * C + C):
                    x = loc[u]
                    net.send(1, "SLICE_KV", -1, u, r, u, 2 * n * E * 2, (x["k"], x["v"]) if compute else None)
        else:
            for r in range(P):
                t = r // C
                net.send(1, "INIT_KV", -1, r, send[r], t, 2 * C * n * E * 2,
                         (team[r]["k"], team[r]["v"]) if compute else None)
        stat = {}
        for r in range(P):
            if direct:
                b = recv[r] // C
                kvs = [net.recv("SLICE_KV", -1, u, r)[1] for u in range(b * C, b * C + C)]
                kv = ((np.concatenate([x[0] for x in kvs]), np.concatenate([x[1] for x in kvs])) if compute else None)
            else:
                b, kv = net.recv("INIT_KV", -1, recv[r], r)
            stat[r] = dict(b=b, kv=kv, kpos=team_positions(range(b * C, b * C + C), P, N, causal),
                           dk=np.zeros((C * n, h, d)) if compute else None,
                           dv=np.zeros((C * n, h, d)) if compute else None)
        pkg = {}
        for r in range(P):
            e = team[r]
            pkg[r] = dict(team=e["t"], qpos=e["qpos"],
                          data=(e["q"], e["do"], e["lse"], e["dd"]) if compute else None,
                          dq=np.zeros((C * n, h, d)) if compute else None)
        for s in range(R):
            for r in range(P):
                pk, st = pkg[r], stat[r]
                if log is not None:
                    log.setdefault("visits", []).append((r, s, pk["team"], tuple(range(st["b"] * C, st["b"] * C + C))))
                if compute:
                    q, do, lse, dd = pk["data"]
                    dq, dk, dv = block_bwd(q, st["kv"][0], st["kv"][1], do, lse, dd, pk["qpos"], st["kpos"], causal)
                    pk["dq"] = pk["dq"] + dq
                    st["dk"] = st["dk"] + dk
                    st["dv"] = st["dv"] + dv
                if s < R - 1:
                    net.send(1, "RING_QPKG", s, r, nxt[r], pk["team"], 2 * C * n * E * 2 + 2 * C * n * h * 4,
                             (pk["team"], pk["qpos"], pk["data"]))
                    net.send(1, "RING_DQ", s, r, nxt[r], pk["team"], C * n * E * 4, pk["dq"])
            if s < R - 1:
                new = {}
                for r in range(P):
                    _, (tm, qp, data) = net.recv("RING_QPKG", s, lst[r], r)
                    _, dq = net.recv("RING_DQ", s, lst[r], r)
                    new[r] = dict(team=tm, qpos=qp, data=data, dq=dq)
                pkg = new
        if R > 1:
            for r in range(P):
                net.send(1, "RET_DQ", R - 1, r, nxt[r], pkg[r]["team"], C * n * E * 4, (pkg[r]["team"], pkg[r]["dq"]))
            for r in range(P):
                _, (tm, dq) = net.recv("RET_DQ", R - 1, lst[r], r)
                if tm != r // C:
                    raise RuntimeError("return hop did not bring dQ home")
                if log is not None:
                    log.setdefault("dq_home", []).append((r, tm))
                dq_part[r] = dq
        else:
            for r in range(P):
                if pkg[r]["team"] != r // C:
                    raise RuntimeError("R=1 package is not the own team")
                if log is not None:
                    log.setdefault("dq_home", []).append((r, pkg[r]["team"]))
                dq_part[r] = pkg[r]["dq"]
        # dK/dV (reading c11, revised): every holder of a stationary team block sends each
        # unit's rows of its fp32 partial straight to the unit's owner, which sums the C
        # replicas (one per team member that held the block).
        contrib = {u: [] for u in range(P)}
        for r in range(P):
            st = stat[r]
            b = st["b"]
            for j, u in enumerate(range(b * C, b * C + C)):
                piece = (_rows_of_member(st["dk"], j, n), _rows_of_member(st["dv"], j, n)) if compute else None
                net.send(1, "REV_DKV", R, r, u, u, 2 * n * E * 4, piece)
        for u in range(P):
            for r in range(P):
                if recv[r] // C == u // C:
                    contrib[u].append(net.recv("REV_DKV", R, r, u)[1])
        dkv_part = contrib
    else:
        for r in range(P):
            a = r % C
            for u in _slice_units(a, P, C):
                net.send(1, "SLICE_KV", -1, u, r, u, 2 * n * E * 2, (loc[u]["k"], loc[u]["v"]) if compute else None)
        contrib = {u: [] for u in range(P)}
        for r in range(P):
            a = r % C
            units = _slice_units(a, P, C)
            kvs = [net.recv("SLICE_KV", -1, u, r)[1] for u in units]
            e = team[r]
            if log is not None:
                log.setdefault("visits", []).append((r, 0, r // C, tuple(units)))
                log.setdefault("dq_home", []).append((r, r // C))
            if compute:
                k = np.concatenate([x[0] for x in kvs])
                v = np.concatenate([x[1] for x in kvs])
                kpos = team_positions(units, P, N, causal)
                dq, dk, dv = block_bwd(e["q"], k, v, e["do"], e["lse"], e["dd"], e["qpos"], kpos, causal)
            else:
                dq = dk = dv = None
            dq_part[r] = dq
            for j, u in enumerate(units):
                piece = (_rows_of_member(dk, j, n), _rows_of_member(dv, j, n)) if compute else None
                net.send(1, "REV_DKV", R, r, u, u, 2 * n * E * 4, piece)
        for u in range(P):
            # every rank whose member index owns u's slice sent a partial
            a = u // (P // C)
            for r in range(P):
                if r % C == a:
                    contrib[u].append(net.recv("REV_DKV", R, r, u)[1])
        dkv_part = contrib

    if log is not None:
        log["dkv"] = {u: len(contrib[u]) for u in range(P)}
    # Team reduce-scatter sum of dQ.
    for r in range(P):
        t = r // C
        for j, p in enumerate(range(t * C, t * C + C)):
            net.send(1, "RS_DQ", R, r, p, p, n * E * 4, _rows_of_member(dq_part[r], j, n) if compute else None)
    dQ = np.zeros((N, h, d)) if compute else None
    dK = np.zeros((N, h, d)) if compute else None
    dV = np.zeros((N, h, d)) if compute else None
    for r in range(P):
        t = r // C
        members = range(t * C, t * C + C)
        dqs = [net.recv("RS_DQ", R, p, r)[1] for p in members]
        dkvs = dkv_part[r]
        if compute:
            dQ[pos[r]] = sum(dqs)
            dK[pos[r]] = sum(x[0] for x in dkvs)
            dV[pos[r]] = sum(x[1] for x in dkvs)
    net.assert_quiescent()
    return dQ, dK, dV, net.events


def trace_totals(events, rank=None, pas=None):
    """Bytes received per kind (optionally for one destination rank / one pass)."""
    tot = {}
    for e in events:
        if rank is not None and e.dst != rank:
            continue
        if pas is not None and e.pas != pas:
            continue
        tot[e.kind] = tot.get(e.kind, 0) + e.nbytes
    return tot
