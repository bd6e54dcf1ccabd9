"""Closed-form communication cost model of the paper (TEST INFRASTRUCTURE ONLY).

Only tests/ and bench.py's reporting may import this module.

PAPER.md:607 (§FE): "for R ranks participating in an all-reduce communication
for communication volume V, the cost is 2V(R-1)/R".
PAPER.md:609-611 (§FE): C_Emb = 2V(D-1)/D + 2V/2 = V(3D-2)/D.
PAPER.md:613-615 (§FE): C_Emb_fused = V(2D-1)/D (2D ranks).
SPEC.md:157-161 (compression_ratio): n*m / (r*(n+m)).
"""
from __future__ import annotations

from fractions import Fraction


def allreduce_cost(V, R):
    """Ring allreduce traffic per rank, 2V(R-1)/R."""
    if R < 1:
        raise ValueError("R >= 1")
    return Fraction(2) * V * (R - 1) / R


def c_emb(V, D):
    """Two-step embedding synchronisation: EMB-DP over D + EMB-sync over 2."""
    return allreduce_cost(V, D) + allreduce_cost(V, 2)


def c_emb_fused(V, D):
    """Fused embedding synchronisation: one allreduce over 2D ranks."""
    return allreduce_cost(V, 2 * D)


def compression_ratio(n, m, r):
    """Uncompressed / compressed element count for rank-r factors."""
    return Fraction(n * m, r * (n + m))
