"""Host-side tests of libwf.so (no GPU needed): the C ABI loads and exports every
symbol include/wf.h declares; the library's plan equals Alg. 2/3 as the oracle
transcribes it; its CommTrace (wf_plan_trace) equals the oracle's literal schedule
simulation record for record (bit-exact bookkeeping)."""
import os
import re
from collections import Counter

import pytest

from oracle.schedule import simulate_backward, simulate_forward
from oracle.sharding import unit_positions
from oracle.topology import ConfigError, build_plan, regime

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def wf():
    from paper_2407_00611_b200 import build
    build.build()
    import paper_2407_00611_b200 as m
    return m


def test_exports_every_declared_symbol(wf):
    from paper_2407_00611_b200._lib import EXPORTED, lib
    hdr = open(os.path.join(ROOT, "include", "wf.h")).read()
    declared = set(re.findall(r"^\s*(?:wf_status|int64_t|const char\*)\s+(wf_\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    L = lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(EXPORTED)


@pytest.mark.parametrize("P,C", [(P, C) for P in range(1, 17) for C in range(1, P + 1)])
def test_plan_matches_oracle(wf, P, C):
    try:
        o = build_plan(P, C)
    except ConfigError:
        with pytest.raises(wf.WFError):
            wf.plan(P, C, 0)
        return
    for r in range(P):
        p = wf.plan(P, C, r)
        assert (p["send"], p["recv"], p["next"], p["last"], p["R"], p["regime"]) == \
            (o["send"][r], o["recv"][r], o["next"][r], o["last"][r], o["R"], o["regime"])


def _oracle_trace(P, C, N, h, d, direct=False):
    _, _, ev_f, _ = simulate_forward(N, None, None, P, C, False, compute=False, heads=h, head_dim=d, direct=direct)
    _, _, _, ev_b = simulate_backward(N, None, None, None, None, None, P, C, False, compute=False, heads=h, head_dim=d,
                                      direct=direct)
    return Counter((e.pas, e.kind, e.step, e.src, e.dst, e.block, e.nbytes) for e in ev_f + ev_b)


CFGS = [(P, C) for P in (1, 2, 3, 4, 6, 8, 12, 16) for C in (1, 2, 3, 4, 8)
        if C <= P and P % C == 0 and (C * C > P or P % (C * C) == 0) and C <= 8 and P // C <= 8 or (P, C) == (16, 4)]


@pytest.mark.parametrize("P,C", CFGS)
def test_plan_trace_equals_oracle(wf, P, C):
    N, h, d = 256 * P, 2, 64
    lib_tr = Counter(wf.plan_trace(P, C, N, h, d))
    assert lib_tr == _oracle_trace(P, C, N, h, d)


@pytest.mark.parametrize("P,C", CFGS)
def test_plan_trace_direct_pull_equals_oracle(wf, P, C):
    # the DIRECT-PULL schedule variant (wf_set_schedule / wf_plan_trace_sched, reading c21)
    N, h, d = 256 * P, 2, 64
    lib_tr = Counter(wf.plan_trace(P, C, N, h, d, sched=wf.SCHED_DIRECT_PULL))
    assert lib_tr == _oracle_trace(P, C, N, h, d, direct=True)


def test_plan_trace_per_rank_partition(wf):
    P, C, N = 8, 2, 2048
    full = Counter(wf.plan_trace(P, C, N, 2, 64))
    parts = Counter()
    for r in range(P):
        tr = wf.plan_trace(P, C, N, 2, 64, rank=r)
        assert all(e[3] == r for e in tr)
        parts.update(tr)
    assert parts == full


def test_shard_ranges_match_dataloader(wf):
    for P in (1, 2, 4, 8):
        N = 1024 * P
        for causal in (False, True):
            for r in range(P):
                a0, a1, b0, b1 = wf.shard_ranges(P, r, N, causal)
                got = list(range(a0, a1)) + list(range(b0, b1))
                assert got == list(unit_positions(r, P, N, causal))


def test_bad_config_is_config_error(wf):
    from paper_2407_00611_b200._lib import lib
    import ctypes
    h = ctypes.c_void_p()
    assert lib().wf_init_emulated(8, 3, ctypes.byref(h)) == 2
    assert b"divide" in lib().wf_last_error(None)


def test_workspace_sized_by_regime():
    # one GPU keeps only the dQ accumulator and the statistics (bf16 O and dK/dV leave the
    # kernels directly); the C = 1 ring at P = 8 keeps two K/V slots, the fp32 state, two
    # dQ / Q-package slots, the home dQ and the dK/dV accumulators -- and no receive slots
    # for pulled partials (peer memory reads them in place).
    import paper_2407_00611_b200 as wf
    al = lambda b: (b + 1023) // 1024 * 1024  # noqa: E731
    E, h = 32 * 128, 32
    n = 32768
    # dQ accumulator, -D / sqrt(d), -LSE log2(e)
    assert wf.workspace_bytes(1, 1, 32768, 32, 128, True) == 4096 + al(n * E * 4) + 2 * al(h * n * 4)
    n = 131072 // 8
    ring = (4096 + 4 * al(n * E * 2) + al(n * E * 4) + al(h * n * 4) + 2 * al(h * n * 4)
            + 2 * (al(n * E * 4) + 2 * al(n * E * 2) + 2 * al(h * n * 4)) + al(n * E * 4) + 2 * al(n * E * 4))
    assert wf.workspace_bytes(8, 1, 131072, 32, 128, True) == ring
    # the paper regime (C^2 | P) needs no merge / dQ-sum receive slots; the extension does
    assert wf.workspace_bytes(8, 2, 131072, 32, 128, True) < wf.workspace_bytes(8, 4, 131072, 32, 128, True)
