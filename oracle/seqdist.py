"""Completion probabilities and batch relations (§6) --
test infrastructure only.

All sums run in ascending index order in plain Python floats (IEEE double) so
the C++ planner can reproduce them bit for bit.

Pins (tests/test_oracle_seqdist.py): SPEC.md:66-68 and :75-86 worked
examples; brute-force enumeration for S <= 64, N_D <= 16; per-S mass is 1 or
1/ceil(S/N_D).
"""
from __future__ import annotations

import math
from typing import Dict, List, Sequence


def completion_conditional(s: int, n_d: int) -> Dict[int, float]:
    """P_D(U | S=s), display equation PAPER.md:372-386:
    S <= N_D: all mass at U = S;  S > N_D: mass 1/ceil(S/N_D) at
    U = 1 + ((S-1) mod N_D), zero elsewhere."""
    if s <= n_d:
        return {s: 1.0}
    q = -(-s // n_d)
    return {1 + (s - 1) % n_d: 1.0 / q}


def completion_distribution(pmf_out: Sequence[float], n_d: int) -> List[float]:
    """P_D(U) = sum_S P_D(U|S) P_D(S), U = 1..N_D.
    pmf_out[k-1] = P_D(S=k)."""
    pu = [0.0] * n_d
    for k in range(1, len(pmf_out) + 1):
        p = float(pmf_out[k - 1])
        if k <= n_d:
            pu[k - 1] += p
        else:
            q = -(-k // n_d)
            pu[(k - 1) % n_d] += p * (1.0 / q)
    return pu


def completion_fraction(pu: Sequence[float]) -> float:
    """sum_U P_D(U): the expected fraction of the decode batch completing in
    one RRA phase."""
    f = 0.0
    for p in pu:
        f += p
    return f


def little_fraction(pmf_out: Sequence[float], n_d: int) -> float:
    """Steady-state (Little's law) alternative 1/E[ceil(S/N_D)] -- SURVEY.md
    §8(c) S3 flag; option `use_little_fraction`."""
    e = 0.0
    for k in range(1, len(pmf_out) + 1):
        e += float(pmf_out[k - 1]) * float(-(-k // n_d))
    return 1.0 / e


def rra_b_d(b_e: int, f: float) -> int:
    """B_E = B_D * f with B_E the control variable:
    B_D = max(B_E, floor(B_E/f + 1/2))."""
    return max(b_e, int(math.floor(b_e / f + 0.5)))


def waa_b_d(b_e: int, s_d_mean: float) -> int:
    """B_D = B_E * S_D, S_D rounded half-up to an integer."""
    return b_e * int(math.floor(s_d_mean + 0.5))


def rra_iteration_batches(b_d: int, pu: Sequence[float]) -> List[float]:
    """b_u = B_D * (1 - sum_{U<u} P_D(U)), u = 1..N_D: a row
    completing at U still runs iteration U."""
    out, acc = [], 0.0
    for u in range(len(pu)):
        out.append(b_d * (1.0 - acc))
        acc += pu[u]
    return out


def pmf_mean(pmf: Sequence[float]) -> float:
    m = 0.0
    for k in range(1, len(pmf) + 1):
        m += k * float(pmf[k - 1])
    return m
