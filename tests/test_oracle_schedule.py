"""Pins for oracle/topology.py, oracle/sharding.py and oracle/schedule.py:
hand traces of Alg. 2/3, exhaustive structural invariants, the paper's
closed-form volumes (Eqs. 2-4) and its model-M numbers, and value equality of
the literal schedule with dense attention (brute-force-pinned)."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle.dense import attention_fwd, attention_bwd
from oracle.schedule import simulate_forward, simulate_backward, trace_totals
from oracle.sharding import causal_pairs, unit_positions
from oracle.topology import ConfigError, build_plan, get_init_recv, get_init_send, get_p2p_config, regime

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PV = json.load(open(os.path.join(GOLD, "paper_values.json")))


def valid_pairs(maxP):
    for P in range(1, maxP + 1):
        for C in range(1, P + 1):
            try:
                regime(P, C)
            except ConfigError:
                continue
            yield P, C


# ---- topology -----------------------------------------------------------

def test_alg_hand_traces():
    g = PV["alg_hand_traces"]
    assert get_init_send(5, 2, 16, 4) == g["init_send_5_2_16_4"]
    assert get_init_recv(9, 1, 16, 4) == g["init_recv_9_1_16_4"]
    assert list(get_p2p_config(5, 2, 16, 4)) == g["p2p_5_2_16_4"]
    assert get_p2p_config(4, 2, 16, 4)[1] == g["p2p_4_2_16_4_last"]


def test_P8_C2_golden_table():
    gold = json.load(open(os.path.join(GOLD, "topology_P8_C2.json")))
    plan = build_plan(8, 2)
    assert plan["R"] == gold["R"]
    for key in ("init_send", "init_recv", "next", "last"):
        assert plan[key.replace("init_", "")] == gold[key], key
    for r in range(8):
        blocks, x = [], r
        for s in range(plan["R"]):
            blocks.append(plan["recv"][x] // 2)
            x = plan["last"][x]
        assert blocks == gold["blocks"][r]
    cycles = set()
    for r in range(8):
        cyc, x = [r], plan["next"][r]
        while x != r:
            cyc.append(x); x = plan["next"][x]
        cycles.add(tuple(sorted(cyc)))
    assert len(cycles) == gold["n_subrings"]


def test_C1_is_ring_attention():
    # PAPER.md:167 "When C equals one, the algorithm falls back to Ring Attention".
    for P in (1, 2, 5, 8, 16):
        plan = build_plan(P, 1)
        assert plan["send"] == list(range(P)) and plan["recv"] == list(range(P))
        assert plan["next"] == [(r + 1) % P for r in range(P)] and plan["R"] == P


def test_invalid_configs():
    for P, C in ((8, 3), (8, 16), (6, 2), (0, 1), (4, 0)):
        with pytest.raises(ConfigError):
            regime(P, C)
    assert regime(12, 2) == "paper" and regime(8, 4) == "ext" and regime(2, 2) == "ext"


def test_topology_invariants_exhaustive():
    # permutation, C^2 disjoint cycles of length P/C^2 sharing r_a and
    # group, and full coverage of (query team, K/V team block) pairs exactly once.
    count = 0
    for P, C in valid_pairs(256):
        if regime(P, C) != "paper":
            continue
        count += 1
        plan = build_plan(P, C)
        T, R = plan["T"], plan["R"]
        assert sorted(plan["send"]) == list(range(P))
        assert all(plan["send"][plan["recv"][r]] == r for r in range(P))
        seen, ncyc = set(), 0
        g = T // C
        for r in range(P):
            if r in seen:
                continue
            cyc, x = [], r
            while x not in cyc:
                cyc.append(x); x = plan["next"][x]
            assert x == r and len(cyc) == R
            assert len({y % C for y in cyc}) == 1 and len({(y // C) // g for y in cyc}) == 1
            assert all(plan["last"][plan["next"][y]] == y for y in cyc)
            seen.update(cyc); ncyc += 1
        assert ncyc == C * C
        pairs = []
        for r in range(P):
            x = r
            for s in range(R):
                pairs.append((r // C, plan["recv"][x] // C))
                x = plan["last"][x]
        assert sorted(pairs) == sorted(itertools.product(range(T), range(T)))
    assert count >= 400  # 402 valid paper-regime pairs with P <= 256


# ---- sharding -----------------------------------------------------------

def test_zigzag_golden():
    z = PV["zigzag"]
    assert causal_pairs(2, 8, True) == z["N8_P2_zigzag"]
    assert causal_pairs(2, 8, False) == z["N8_P2_naive"]
    assert causal_pairs(4, 16, True) == z["N16_P4_zigzag"]
    assert list(unit_positions(0, 2, 8, True)) == z["N8_P2_dev0_tokens"]


def test_zigzag_balance_and_permutation():
    # SPEC.md:235-236
    for P in (1, 2, 3, 4, 8, 16):
        for mult in (1, 3):
            N = 2 * P * mult
            c = causal_pairs(P, N, True)
            assert max(c) == min(c)
            allpos = np.concatenate([unit_positions(u, P, N, True) for u in range(P)])
            assert sorted(allpos) == list(range(N))


# ---- schedule values ----------------------------------------------------

def _rand(N, h, d, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((N, h, d)) for _ in range(4)]


CONFIGS = [(P, C) for P in (1, 2, 4, 8, 16) for C in (1, 2, 4) if C <= P and P % C == 0
           and (C * C > P or P % (C * C) == 0)]


@pytest.mark.parametrize("P,C", CONFIGS)
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("N", [64, 256])
def test_schedule_equals_dense(P, C, causal, N):
    # for all valid (P <= 16, C in {1,2,4}, both masks, N in {64,256}) <= 1e-10.
    h, d = 2, 4
    Q, K, V, dO = _rand(N, h, d, seed=P * 100 + C * 10 + causal)
    O, L, ev, _ = simulate_forward(Q, K, V, P, C, causal)
    Od, Ld = attention_fwd(Q, K, V, causal=causal)
    assert np.abs(O - Od).max() < 1e-10 and np.abs(L - Ld).max() < 1e-10
    dq, dk, dv, _ = simulate_backward(Q, K, V, dO, O, L, P, C, causal)
    dqd, dkd, dvd, _, _ = attention_bwd(Q, K, V, dO, causal=causal)
    for a, b in ((dq, dqd), (dk, dkd), (dv, dvd)):
        assert np.abs(a - b).max() < 1e-10


@pytest.mark.parametrize("C", [1, 2])
def test_tiny_config(C):
    # BASELINE.json configs[0]: N=256, 2 heads x 32, non-causal, P=4 simulated, C in {1,2}.
    from wf_inputs import make_qkv_do, to_f64
    q, k, v, do = (to_f64(t) for t in make_qkv_do(256, 2, 32, seed=0))
    O, L, _, _ = simulate_forward(q, k, v, 4, C, False)
    Od, Ld = attention_fwd(q, k, v)
    assert np.abs(O - Od).max() < 1e-10 and np.abs(L - Ld).max() < 1e-10


# ---- schedule bookkeeping ----------------------------------------------

def _p2p_paper_convention(P, C, N, E, rank):
    """Received P2P elements per rank counting the self-held init block (reading c4)."""
    _, _, ev, ctx = simulate_forward(N, None, None, P, C, False, compute=False, heads=1, head_dim=E)
    plan = ctx["plan"]
    tot = trace_totals(ev, rank=rank)
    n = N // P
    if plan["regime"] == "paper":
        wire = tot.get("INIT_KV", 0) + tot.get("RING_KV", 0)
        self_held = 2 * C * n * E * 2 if plan["send"][rank] == rank else 0
    else:
        wire = tot.get("SLICE_KV", 0)
        a = rank % C
        self_held = 2 * n * E * 2 if a * (P // C) <= rank < (a + 1) * (P // C) else 0
    return (wire + self_held) // 2, ev, plan


@pytest.mark.parametrize("P,C", [(P, C) for P, C in valid_pairs(16)])
def test_p2p_volume_is_eq2_eq4(P, C):
    # Eq. 2: ring 2NE per GPU; Eq. 4: WallFacer 2NE/C.
    N, E = 2 * P * 8, 4
    for r in range(P):
        elems, _, _ = _p2p_paper_convention(P, C, N, E, r)
        assert elems * C == 2 * N * E


@pytest.mark.parametrize("P,C", [(P, C) for P, C in valid_pairs(16) if C * C <= P])
def test_collective_volume_is_eq3(P, C):
    # Eq. 3: 4 N E (C-1) / P per GPU (AG of Q,K,V + RS of O; reading c18).
    N, E = 2 * P * 8, 4
    _, _, ev, _ = simulate_forward(N, None, None, P, C, False, compute=False, heads=1, head_dim=E)
    for r in range(P):
        t = trace_totals(ev, rank=r)
        elems = (t.get("AG_Q", 0) + t.get("AG_KV", 0)) // 2 + t.get("RS_O", 0) // 4  # bf16 gathers, fp32 partials
        assert elems * P == 4 * N * E * (C - 1)


def test_eq2_eq3_toys():
    e2 = PV["eq2_toy"]
    elems, ev, plan = _p2p_paper_convention(e2["P"], 1, e2["N"], e2["H"], 0)
    msgs = sum(1 for x in ev if x.dst == 0 and x.kind in ("RING_KV",)) + 1  # + the self-held init (reading c4)
    assert elems / 1 + msgs * 1 == e2["value"]   # W = L = 1
    e3 = PV["eq3_toy"]
    _, _, ev, _ = simulate_forward(e3["N"], None, None, e3["P"], e3["C"], False, compute=False, heads=1, head_dim=e3["H"])
    t = trace_totals(ev, rank=0)
    assert (t["AG_Q"] + t["AG_KV"]) // 2 + t["RS_O"] // 4 == e3["value"]


def test_model_M_volumes():
    # 1.625 GB ring vs 0.152 (collective) + 0.406 (P2P) GB, per device, bf16.
    m = PV["model_M"]
    N, P, C, E = m["N"], m["P"], m["C"], m["H"]
    ring, _, _ = _p2p_paper_convention(P, 1, N, E, 5)
    wall, ev, _ = _p2p_paper_convention(P, C, N, E, 5)
    t = trace_totals(ev, rank=5)
    coll = (t["AG_Q"] + t["AG_KV"]) // 2 + t["RS_O"] // 4  # elements (paper: activation precision)
    assert ring * 2 == m["ring_p2p_bytes"] and wall * 2 == m["wall_p2p_bytes"] and coll * 2 == m["wall_collective_bytes"]
    gib = 2 ** 30
    assert round(ring * 2 / gib, 3) == m["ring_p2p_gib"]
    assert round(wall * 2 / gib, 3) == m["wall_p2p_gib"]
    assert round(coll * 2 / gib, 3) == m["wall_collective_gib"]
    # the paper adds its rounded terms: 0.152 + 0.406 = 0.558 (exact total 0.5586)
    assert round(round(wall * 2 / gib, 3) + round(coll * 2 / gib, 3), 3) == m["wall_total_gib"]


def test_fig1_savings():
    f = PV["fig1_savings"]
    for C, key in ((2, "C2"), (4, "C4")):
        P, N, E = 16, 256, 2
        ring, _, _ = _p2p_paper_convention(P, 1, N, E, 3)
        wall, _, _ = _p2p_paper_convention(P, C, N, E, 3)
        assert 1 - wall / ring == f[key]


def test_C1_trace_is_plain_ring():
    P, N, E = 8, 128, 4
    _, _, ev, _ = simulate_forward(N, None, None, P, 1, True, compute=False, heads=1, head_dim=E)
    assert {e.kind for e in ev} == {"RING_KV"}
    for r in range(P):
        mine = [e for e in ev if e.src == r]
        assert len(mine) == P - 1 and all(e.dst == (r + 1) % P for e in mine)


def test_C_sqrtP_has_no_ring():
    for P, C in ((4, 2), (16, 4)):
        _, _, ev, _ = simulate_forward(2 * P * 4, None, None, P, C, False, compute=False, heads=1, head_dim=2)
        assert not any(e.kind.startswith("RING") for e in ev)
        _, _, _, ev2 = simulate_backward(2 * P * 4, None, None, None, None, None, P, C, False, compute=False, heads=1, head_dim=2)
        assert not any(e.kind.startswith("RING") or e.kind == "RET_DQ" for e in ev2)


def test_trace_mask_independent_and_deterministic():
    # SPEC.md:321-322
    P, C, N = 8, 2, 64
    Q, K, V, dO = _rand(N, 2, 4, 3)
    a = simulate_forward(Q, K, V, P, C, False)[2]
    b = simulate_forward(Q, K, V, P, C, True)[2]
    c = simulate_forward(Q, K, V, P, C, True)[2]
    assert a == b == c


@pytest.mark.parametrize("P,C", [(4, 2), (8, 2), (16, 4), (16, 2)])
def test_direct_pull_variant_equals_dense(P, C):
    # DIRECT-PULL init (reading c21): same values as dense attention and as the default
    # schedule; no K/V team gather and no init shuffle on the wire, each rank receives the
    # units of its initial block team(init_recv) from their owners (minus its own unit).
    N, h, d = 128 * P, 2, 8
    rng = np.random.default_rng(P * 7 + C)
    Q, K, V, dO = (rng.standard_normal((N, h, d)) for _ in range(4))
    for causal in (False, True):
        O, L, ev_f, _ = simulate_forward(Q, K, V, P, C, causal, direct=True)
        dq, dk, dv, o, l = attention_bwd(Q, K, V, dO, causal=causal)
        assert np.abs(O - o).max() < 1e-10 and np.abs(L - l).max() < 1e-10
        gq, gk, gv, ev_b = simulate_backward(Q, K, V, dO, O, L, P, C, causal, direct=True)
        assert max(np.abs(gq - dq).max(), np.abs(gk - dk).max(), np.abs(gv - dv).max()) < 1e-10
    kinds = {e.kind for e in ev_f + ev_b}
    assert "AG_KV" not in kinds and "INIT_KV" not in kinds
    plan = build_plan(P, C)
    for r in range(P):
        blk = plan["recv"][r] // C
        want = {u for u in range(blk * C, blk * C + C) if u != r}
        got = {e.src for e in ev_f if e.kind == "SLICE_KV" and e.dst == r}
        assert got == want


# ---- backward bookkeeping pins (independent of the oracle's own byte formulas) -----

def _mib_by_kind(ev, rank, pas):
    t = trace_totals(ev, rank=rank, pas=pas)
    assert all(v % 2 ** 20 == 0 for v in t.values())
    return {k: v // 2 ** 20 for k, v in t.items()}


def test_backward_bytes_golden_gpt128k_p8():
    # SURVEY.md:512-519: received MiB per rank at GPT-128K, P=8 (C=2 and C=1), from an
    # independent emulator of PAPER.md:169-188 / 201-205.  Fails if dQ travels as bf16,
    # if the dQ return hop is dropped, or if the package loses LSE/D.
    gold = json.load(open(os.path.join(GOLD, "bytes_gpt128k_p8.json")))
    cfg = gold["config"]
    N, h, d, P = cfg["N"], cfg["heads"], cfg["head_dim"], cfg["P"]
    for C, key in ((2, "C2"), (1, "C1")):
        g = gold[key]
        _, _, evf, _ = simulate_forward(N, None, None, P, C, True, compute=False, heads=h, head_dim=d)
        _, _, _, evb = simulate_backward(N, None, None, None, None, None, P, C, True, compute=False, heads=h,
                                         head_dim=d)
        for r in range(P):
            f = _mib_by_kind(evf, r, 0)
            b = _mib_by_kind(evb, r, 1)
            for kind, mib in g["fwd"].items():
                assert f.get(kind, 0) == mib, (C, r, "fwd", kind, f.get(kind))
            for kind, mib in g["bwd"].items():
                assert b.get(kind, 0) == mib, (C, r, "bwd", kind, b.get(kind))
            if "INIT_KV" in g:
                want = 0 if r in g["INIT_KV"]["ranks_zero"] else g["INIT_KV"]["other"]
                assert f.get("INIT_KV", 0) == want and b.get("INIT_KV", 0) == want, (C, r)


@pytest.mark.parametrize("P,C", [(P, C) for P, C in valid_pairs(16)] + [(32, 4), (64, 4), (64, 8)])
def test_backward_coverage_invariants(P, C):
    # every (query team, key unit) pair is visited exactly once over the
    # ring (the backward "mirrors" the forward's coverage), every team's dQ ends at its home
    # once per member (P:205's return hop), and each unit owner sums exactly C dK/dV
    # replicas in the paper regime (one per team member holding the stationary block,
    # reading c11) or T = P/C in the extension (one per team, reading c2).
    log = {}
    simulate_backward(2 * P * 4, None, None, None, None, None, P, C, True, compute=False, heads=1, head_dim=2,
                      log=log)
    T = P // C
    seen = {}
    for r, s, team, units in log["visits"]:
        for u in units:
            seen[(team, u)] = seen.get((team, u), 0) + 1
    # each team has C members; each member covers its share of the keys, so every
    # (team, unit) pair is visited once by the team as a whole
    assert sorted(seen) == [(t, u) for t in range(T) for u in range(P)]
    assert set(seen.values()) == {1}, (P, C)
    assert sorted(log["dq_home"]) == [(r, r // C) for r in range(P)]
    want = C if C * C <= P else T
    assert log["dkv"] == {u: want for u in range(P)}
