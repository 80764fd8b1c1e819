"""Sequence-Parallel Dataloader (§3.5) -- TEST INFRASTRUCTURE.

Full mask: "sequences are straightforwardly divided into sub-sequences of equal
lengths" -> unit u = [u n, (u+1) n), n = N/P.
Causal mask: the zigzag scheme of ring-flash-attention, "modified";
read as (reading c13): cut N into 2P chunks of c = N/(2P);
device u holds chunk u followed by chunk 2P-1-u.
"""
from __future__ import annotations

import numpy as np

__all__ = ["unit_positions", "team_positions", "causal_pairs"]


def unit_positions(u: int, P: int, N: int, causal: bool):
    """Global token positions of unit (= original device shard) u, in local order."""
    if causal:
        if N % (2 * P):
            raise ValueError("zigzag needs 2P | N")
        c = N // (2 * P)
        return np.concatenate([np.arange(u * c, (u + 1) * c), np.arange((2 * P - 1 - u) * c, (2 * P - u) * c)])
    if N % P:
        raise ValueError("naive split needs P | N")
    n = N // P
    return np.arange(u * n, (u + 1) * n)


def team_positions(units, P, N, causal):
    """Member-major concatenation of the given units (PAPER.md:193 team tensors)."""
    return np.concatenate([unit_positions(u, P, N, causal) for u in units])


def causal_pairs(P: int, N: int, zigzag: bool):
    """Per-device count of allowed (q, k) pairs, k <= q, by brute force."""
    out = []
    for u in range(P):
        if zigzag:
            qs = unit_positions(u, P, N, True)
        else:
            n = N // P
            qs = np.arange(u * n, (u + 1) * n)
        out.append(int(sum(int(q) + 1 for q in qs)))
    return out
