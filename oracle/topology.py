"""Communication Configuration Generator, literal (TEST INFRASTRUCTURE).

Alg. 2 get_init_send  -- PAPER.md:263-275 (§3.3)
get_init_recv         -- PAPER.md:261 "calculated similarly"; read as the inverse
                         permutation of get_init_send (reading c8).
Alg. 3 get_P2P_config -- PAPER.md:279-292 (§3.3); (r_t - 1) % g is the
                         mathematical modulo (reading c6), "/" is integer
                         division (reading c7).
Teams are contiguous in global rank, global = r_t * C + r_a (PAPER.md:167,
SPEC.md:112).  Valid C (reading c2): C | P and (C^2 <= P  =>  C^2 | P); the
C^2 > P "extension" regime has no ring (R = 1) and is flagged as ours.
"""
from __future__ import annotations

__all__ = ["ConfigError", "regime", "get_init_send", "get_init_recv", "get_p2p_config", "build_plan"]


class ConfigError(ValueError):
    pass


def regime(P: int, C: int) -> str:
    """'paper' (C^2 | P), 'ext' (C | P, C^2 > P) or raise ConfigError."""
    if P < 1 or C < 1:
        raise ConfigError(f"P={P}, C={C}: both must be >= 1")
    if C > P or P % C:
        raise ConfigError(f"C={C} must divide P={P}")
    if C * C <= P:
        if P % (C * C):
            raise ConfigError(f"C^2={C*C} must divide P={P} when C^2 <= P")
        return "paper"
    return "ext"


def get_init_send(r_t: int, r_a: int, d_t: int, d_a: int) -> int:
    """Alg. 2, line by line."""
    team_group_size = d_t // d_a                                   # l.1
    target_team_group_rank = r_a                                   # l.2
    target_team = target_team_group_rank * team_group_size + r_t // d_a  # l.3
    target_intra = r_t % d_a                                       # l.4
    return target_team * d_a + target_intra                        # l.5


def get_p2p_config(r_t: int, r_a: int, d_t: int, d_a: int):
    """Alg. 3, line by line.  Returns (next global rank, last global rank)."""
    g = d_t // d_a                                                 # l.1
    self_group = r_t // g                                          # l.2
    next_team = (r_t + 1) % g + g * self_group                     # l.3
    last_team = (r_t - 1) % g + g * self_group                     # l.4 (Python % is mathematical)
    return r_a + next_team * d_a, r_a + last_team * d_a            # l.5-6


def get_init_recv(r_t: int, r_a: int, d_t: int, d_a: int) -> int:
    """Inverse of Alg. 2: the unique rank whose init-send target is (r_t, r_a)."""
    me = r_t * d_a + r_a
    P = d_t * d_a
    hits = [x for x in range(P) if get_init_send(x // d_a, x % d_a, d_t, d_a) == me]
    if len(hits) != 1:
        raise ConfigError(f"init_send is not a permutation at rank {me}")
    return hits[0]


def build_plan(P: int, C: int) -> dict:
    """Per-rank init_send / init_recv / next / last and the ring length R."""
    reg = regime(P, C)
    T = P // C
    if reg == "ext":
        ident = list(range(P))
        return dict(P=P, C=C, T=T, R=1, regime=reg, send=ident, recv=list(ident), next=list(ident), last=list(ident))
    send, nxt, lst = [], [], []
    for r in range(P):
        r_t, r_a = divmod(r, C)
        send.append(get_init_send(r_t, r_a, T, C))
        n, l = get_p2p_config(r_t, r_a, T, C)
        nxt.append(n)
        lst.append(l)
    recv = [get_init_recv(r // C, r % C, T, C) for r in range(P)]
    return dict(P=P, C=C, T=T, R=P // (C * C), regime=reg, send=send, recv=recv, next=nxt, last=lst)
