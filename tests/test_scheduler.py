"""The Communication Topology Scheduler (§3.4, Eq. 8;
paper_2407_00611_b200/scheduler.py).

CPU: the candidate set is Eq. 8's C in [1, sqrt(P)] (C^2 | P) widened by reading
c2's extension (C | P, C^2 > P) and capped at BASELINE's C <= 4 -- checked against the
oracle's own validity rule (oracle/topology.py), independently of the scheduler's code;
the DIRECT-PULL variant is offered exactly for the paper-regime team sizes 1 < C <= sqrt P.
GPU: the search (all P ranks emulated on one GPU) profiles every candidate and returns the
argmin of its own table.
"""
import math

import pytest

from oracle.topology import ConfigError, regime
from paper_2407_00611_b200.scheduler import candidates, label, variants


def _valid(P, C):
    try:
        regime(P, C)
        return True
    except ConfigError:
        return False


@pytest.mark.parametrize("P", list(range(1, 65)))
def test_candidates_are_eq8_plus_extension(P):
    got = candidates(P)
    assert got == [C for C in range(1, min(P, 4) + 1) if _valid(P, C)]
    # Eq. 8's range: every C in [1, sqrt(P)] with C^2 | P ("from 1 to sqrt(P)")
    for C in range(1, min(4, math.isqrt(P)) + 1):
        if P % (C * C) == 0:
            assert C in got
    # the extension: C | P with C^2 > P (reading c2), e.g. P = 2, C = 2 and P = 8, C = 4
    for C in got:
        assert P % C == 0 and (C * C > P or P % (C * C) == 0)
    assert got[0] == 1  # Ring Attention (C = 1) is always a candidate


def test_candidates_baseline_configs():
    # BASELINE.json's metric grid: C in {1, 2, 4} where C | P
    assert candidates(1) == [1]
    assert candidates(2) == [1, 2]
    assert candidates(4) == [1, 2, 4]
    assert candidates(8) == [1, 2, 4]


@pytest.mark.parametrize("P", [1, 2, 4, 8, 16, 32])
def test_variants_direct_pull_only_in_paper_regime(P):
    v = variants(P)
    assert [c for c, s in v if s == 0] == candidates(P)
    assert sorted(c for c, s in v if s == 1) == [c for c in candidates(P) if 1 < c and c * c <= P]
    assert len({label(c, s) for c, s in v}) == len(v)


@pytest.mark.gpu
@pytest.mark.parametrize("P", [4, 8])
def test_search_emulated_returns_argmin(P):
    from paper_2407_00611_b200 import scheduler
    N = 2048 * P
    C, sched, table = scheduler.search(P, 0, N, 4, 128, True, steps=3, warmup=1, rounds=3, emulated=True)
    assert set(table) == {label(c, s) for c, s in variants(P)}
    best = min(table, key=lambda k: table[k]["ms"])
    assert label(C, sched) == best
    for row in table.values():
        assert row["ms"] > 0 and row["spread"] >= 0
