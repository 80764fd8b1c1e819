"""Host tests of the analytic cost/memory model (paper_2407_00611_b200/costmodel.py):
the paper's equations against the values the paper prints (tests/golden/paper_values.json),
the library's plan-trace bytes against those closed forms, and sanity of the prediction."""
import json
import os

import pytest

from paper_2407_00611_b200 import costmodel as cm
from paper_2407_00611_b200.wf import plan

PV = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_eq2_eq3_toys():
    t = PV["eq2_toy"]
    assert cm.eq2_ring(1, t["N"], t["H"], t["P"], W=1, L=1) == t["value"]
    t = PV["eq3_toy"]
    assert cm.eq3_collective(1, t["N"], t["H"], t["P"], t["C"]) == t["value"]


def test_model_M_printed_volumes():
    m = PV["model_M"]
    N, H, P, C = m["N"], m["H"], m["P"], m["C"]
    gib = 2 ** 30
    assert round(cm.eq2_ring(1, N, H, P) * 2 / gib, 3) == m["ring_p2p_gib"]
    assert round(cm.eq3_collective(1, N, H, P, C) * 2 / gib, 3) == m["wall_collective_gib"]
    assert round(cm.eq4_p2p(1, N, H, P, C) * 2 / gib, 3) == m["wall_p2p_gib"]
    assert cm.eq4_p2p(1, N, H, P, C) * 2 == m["wall_p2p_bytes"]
    mm = PV["model_M_memory"]
    assert cm.eq6_peak_ring(64) == mm["ring_A"] and cm.eq7_peak_wall(64, C) == mm["wall_A"]


@pytest.mark.parametrize("P,C", [(4, 1), (4, 2), (8, 1), (8, 2), (16, 2), (16, 4), (32, 2)])
def test_library_bytes_match_eq3_eq4_paper_regime(P, C):
    h, d = 2, 64
    N = 256 * P
    n, E = N // P, h * d
    H = E
    by = cm.schedule_bytes(P, C, N, h, d)
    for r, t in by.items():
        ring = t[(0, "INIT_KV")] + t[(0, "RING_KV")]
        recv = plan(P, C, r)["recv"]
        # Eq. 4: P/C^2 blocks of 2CBNH/P elements (a rank whose init source is itself skips one)
        want = cm.eq4_p2p(1, N, H, P, C) * 2
        assert ring == (want if recv != r else want - 2 * C * n * E * 2)
        # Eq. 3 in elements: Q/K/V gather (bf16) + O reduce-scatter (fp32 on our wire, c17)
        coll = (t[(0, "AG_Q")] + t[(0, "AG_KV")]) // 2 + t[(0, "RS_O")] // 4
        assert coll == cm.eq3_collective(1, N, H, P, C)


@pytest.mark.parametrize("P,C", [(2, 2), (4, 4), (8, 4)])
def test_library_bytes_extension_regime(P, C):
    h, d = 2, 64
    N = 256 * P
    n, E = N // P, h * d
    W = P // C
    by = cm.schedule_bytes(P, C, N, h, d)
    for r, t in by.items():
        a = r % C
        own = a * W <= r < (a + 1) * W
        assert t[(0, "SLICE_KV")] == (W - own) * 2 * n * E * 2
        assert t[(0, "AG_Q")] == (C - 1) * n * E * 2
        assert t[(0, "RING_KV")] == 0 and t[(0, "INIT_KV")] == 0


def test_workspace_scales_and_covers_team_buffers():
    for P, C in ((1, 1), (4, 2), (8, 2), (8, 4)):
        N, h, d = 16384 * P, 4, 128
        w1 = cm.memory(P, C, N, h, d, True)["workspace_bytes"]
        w2 = cm.memory(P, C, 2 * N, h, d, True)["workspace_bytes"]
        assert abs((w2 - 4096) - 2 * (w1 - 4096)) <= 64 * 1024  # linear in N up to 1 KB alignment
        m = cm.memory(P, C, N, h, d, True)
        if C > 1:
            assert m["workspace_bytes"] >= m["paper_team_3CA_bytes"] / 3  # at least the gathered Q


def test_predict_sanity():
    r = cm.predict(1, 1, 32768, 32, 128, True, 850, 1000)
    assert r["exposed_comm_frac"] == 0 and r["recv_bytes_max"] == 0
    ff, fb = cm.flops(32768, 32, 128, True)
    assert abs(r["total_ms"] - (ff / 850e12 + fb / 1000e12) * 1e3) < 1e-9
    slow = cm.predict(8, 1, 131072, 32, 128, True, 850, 1000, link_gbps=10)
    fast = cm.predict(8, 1, 131072, 32, 128, True, 850, 1000, link_gbps=1e6, latency_us=0)
    assert slow["total_ms"] > fast["total_ms"] and fast["exposed_comm_frac"] < 0.01


def test_predict_unit_pipelined_reductions():
    # extension regime (C^2 > P): of the C-1 member partials only the sender's last unit is
    # exposed after the pass; the rest travel during later units
    P, C, N, h, d = 4, 4, 65536, 32, 128
    r = cm.predict(P, C, N, h, d, True, 1000, 1000, link_gbps=100.0, latency_us=0)
    by = cm.schedule_bytes(P, C, N, h, d)
    for pas, name in ((0, "fwd"), (1, "bwd")):
        rs = max(sum(b for (p, k), b in dct.items() if p == pas and k in ("RS_O", "RS_LSE", "RS_DQ"))
                 for dct in by.values())
        rest = max(sum(b for (p, k), b in dct.items() if p == pas and k in ("RET_DQ", "REV_DKV"))
                   for dct in by.values())
        want = (rest + rs / (C - 1)) / 100e9 * 1e3
        assert abs(r[name]["post_ms"] - want) < 1e-9, (name, r[name]["post_ms"], want)
    # C = 2 at P = 2 has one partial per owner: all of it is exposed
    r2 = cm.predict(2, 2, 32768, h, d, True, 1000, 1000, link_gbps=100.0, latency_us=0)
    by2 = cm.schedule_bytes(2, 2, 32768, h, d)
    rs2 = max(sum(b for (p, k), b in dct.items() if p == 0 and k in ("RS_O", "RS_LSE")) for dct in by2.values())
    assert abs(r2["fwd"]["post_ms"] - rs2 / 100e9 * 1e3) < 1e-9
