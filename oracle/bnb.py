"""XScheduler: Algorithm 1 (§5.1) with the strategy and TP
outer loops -- test infrastructure only.

Rules the paper leaves open (listed in DESIGN.md):
 1 infeasible if perf(a1,a2).latency >= L_b;  2 return (b1,b2) if feasible;
 3 single-point blocks are terminal;  4 a degenerate axis forces the other;
 5 neither tl nor br feasible -> split the longer dimension (tie: x1);
 6 tl and br feasible with equal throughput -> vertical (cut x1);
 7 children whose upp is feasible are solved (candidates for T*, not queued);
 8 priority = lowr.thrput, ties -> earliest insertion;
 9 T* updated only from children's upp;  10 prune blocks with
   upp.thrput + eps_T < T*.
Perf evaluations are memoised; `evals` counts distinct points.

Outer loops: strategy x TP degree t x applied GPUs c, and
for WAA also the decoder micro-batch count M: like the TP degree, M is not a
monotone variable on its own (with weight-streaming-bound decode stages the
per-stage time hardly shrinks with B_m, so the fill F grows with M and
latency rises with M), so it is fixed per run of Algorithm 1, which then
searches B_E (reading S9').  RRA searches (B_E, N_D) in one run.

Pins: equals exhaustive argmax on strictly monotone grids; upper-corner
shortcut in <= 2 evaluations; infeasible lower corner
(tests/test_oracle_scheduler.py); schedule_find equals the exhaustive
optimum over strategy x t x c x (x1, x2) on 1/2/4-GPU problems with the
memory-limited B_E^max active (tests/test_oracle_pins.py).
"""
from __future__ import annotations

import heapq
import math
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Tuple

from . import simulator as sim

INF = float("inf")


@dataclass
class Perf:
    latency: float
    thrput: float


@dataclass
class BnBResult:
    x: Optional[Tuple[int, int]]
    perf: Optional[Perf]
    evals: int


class _Memo:
    def __init__(self, fn):
        self.fn, self.cache, self.order = fn, {}, []

    def __call__(self, x1, x2) -> Perf:
        k = (x1, x2)
        if k not in self.cache:
            self.cache[k] = self.fn(x1, x2)
            self.order.append(k)
        return self.cache[k]


def branch_and_bound(a1: int, b1: int, a2: int, b2: int, perf_fn: Callable[[int, int], Perf],
                     L_b: float, eps_t_frac: float = 0.02, eps_l_frac: float = 0.02) -> BnBResult:
    perf = _Memo(perf_fn)
    eps_l = eps_l_frac * L_b if L_b != INF else INF
    lowr = perf(a1, a2)
    if not lowr.latency < L_b:                                   # rule 1
        return BnBResult(None, None, len(perf.cache))
    upp = perf(b1, b2)
    if upp.latency < L_b:                                        # rule 2
        return BnBResult((b1, b2), upp, len(perf.cache))
    T_star, T_cfg = lowr.thrput, (a1, a2)                        # Alg.1 line 3
    heap: List = []
    seq = 0
    # block = (a1, a2, b1, b2, lowr, upp)
    heapq.heappush(heap, (-lowr.thrput, seq, (a1, a2, b1, b2, lowr, upp)))
    while heap:
        _, _, B = heapq.heappop(heap)
        ba1, ba2, bb1, bb2, blowr, bupp = B
        if ba1 == bb1 and ba2 == bb2:                            # rule 3
            continue
        if ba1 == bb1:                                           # rule 4
            axis = 2
        elif ba2 == bb2:
            axis = 1
        else:
            p_tl = perf(ba1, bb2)                                # topLeft (a1, b2)
            p_br = perf(bb1, ba2)                                # bottomRight (b1, a2)
            tl_ok, br_ok = p_tl.latency < L_b, p_br.latency < L_b
            if tl_ok and (not br_ok or p_tl.thrput >= p_br.thrput):
                axis = 1                                         # "vertically": cut x1 (rule 6 on ties)
            elif br_ok:
                axis = 2                                         # "horizontally": cut x2
            else:                                                # rule 5
                axis = 1 if (bb1 - ba1) >= (bb2 - ba2) else 2
        if axis == 1:
            m = (ba1 + bb1) // 2
            kids = [(ba1, ba2, m, bb2), (m + 1, ba2, bb1, bb2)]
        else:
            m = (ba2 + bb2) // 2
            kids = [(ba1, ba2, bb1, m), (ba1, m + 1, bb1, bb2)]
        best = None
        for (ka1, ka2, kb1, kb2) in kids:
            kupp = perf(kb1, kb2)                                # topRight
            klowr = perf(ka1, ka2)                               # bottomLeft
            if kupp.latency < L_b:                               # rule 7: solved
                if best is None or kupp.thrput > best[0].thrput:
                    best = (kupp, (kb1, kb2))
            elif klowr.latency < L_b + eps_l:                    # Alg.1 line 14
                seq += 1
                heapq.heappush(heap, (-klowr.thrput, seq, (ka1, ka2, kb1, kb2, klowr, kupp)))
        if best is not None and best[0].thrput > T_star:         # lines 16-19
            T_star, T_cfg = best[0].thrput, best[1]
            eps_t = eps_t_frac * T_star
            heap = [h for h in heap if not (h[2][5].thrput + eps_t < T_star)]
            heapq.heapify(heap)
    return BnBResult(T_cfg, perf(*T_cfg), len(perf.cache))


def exhaustive(a1: int, b1: int, a2: int, b2: int, perf_fn, L_b: float) -> BnBResult:
    """Plain definition: argmax throughput over the whole grid subject to
    latency < L_b; ties -> lower latency -> smallest (x1, x2)."""
    best, bx, n = None, None, 0
    for x1 in range(a1, b1 + 1):
        for x2 in range(a2, b2 + 1):
            p = perf_fn(x1, x2)
            n += 1
            if not p.latency < L_b:
                continue
            if best is None or p.thrput > best.thrput or (p.thrput == best.thrput and p.latency < best.latency):
                best, bx = p, (x1, x2)
    return BnBResult(bx, best, n)


def monotonicity_audit(grid: Dict[Tuple[int, int], Perf], axis: int, tol_t: float, tol_l: float):
    """Table 7 methodology: sweep one variable with the other
    fixed; count points whose throughput / latency decreases by more than the
    tolerance versus the previous point.  Returns (frac_latency, frac_thrput)."""
    xs1 = sorted({k[0] for k in grid})
    xs2 = sorted({k[1] for k in grid})
    n = bad_l = bad_t = 0
    outer, inner = (xs2, xs1) if axis == 1 else (xs1, xs2)
    for o in outer:
        prev = None
        for i in inner:
            k = (i, o) if axis == 1 else (o, i)
            p = grid[k]
            if prev is not None and math.isfinite(p.latency) and math.isfinite(prev.latency):
                n += 1
                if p.latency < prev.latency - tol_l:
                    bad_l += 1
                if p.thrput < prev.thrput - tol_t:
                    bad_t += 1
            prev = p
    return (bad_l / n if n else 0.0, bad_t / n if n else 0.0)


# ---------------------------------------------------------------------------
# outer loops (S12) over strategy x TP degree x applied GPUs
# ---------------------------------------------------------------------------
@dataclass
class SearchOpts:
    eps_t_frac: float = 0.02
    eps_l_frac: float = 0.02
    b_e_max: int = 256
    n_d_max: int = 0          # 0 -> max output length
    m_max: int = 8
    use_little_fraction: bool = False
    tp_degree_only: int = 0   # > 0: only this TP degree (a forced partial-TP plan)


@dataclass
class Found:
    schedule: sim.Schedule
    estimate: sim.Estimate
    evals: int


def _perf_of(est: sim.Estimate) -> Perf:
    # a point the simulator cannot evaluate (memory or profile hull) is
    # infeasible, and its throughput is unknown: +inf keeps it from acting as
    # a (wrong) upper bound in the pruning step (line 19)
    if not est.feasible:
        return Perf(INF, INF)
    return Perf(est.latency_s, est.thrput_seq_s)


def schedule_find(S: sim.Simulator, L_b: float, strategy_mask: int, opts: SearchOpts) -> Optional[Found]:
    N, H = S.cl.n_gpus, S.m.n_heads
    n_d_max = opts.n_d_max if opts.n_d_max > 0 else S.max_out
    best = None   # (key, Found)
    total_evals = 0
    for strat in (sim.RRA, sim.WAA_C, sim.WAA_M):
        if not (strategy_mask & strat):
            continue
        if strat != sim.RRA and N < 2:
            continue
        for t in (1, 2, 4, 8):
            if t > N or H % t != 0:
                continue
            if opts.tp_degree_only > 0 and t != opts.tp_degree_only:
                continue
            cs = [0] if t == 1 else list(range(t, N + 1, t))
            for c in cs:
                if strat == sim.RRA:
                    def mk(x1, x2, t=t, c=c):
                        return S.rra_schedule(x1, n_d_max + 1 - x2, t, c)
                    x2_ranges = [(1, n_d_max)]
                else:
                    def mk(x1, x2, t=t, c=c, strat=strat):
                        return S.waa_schedule(x1, opts.m_max + 1 - x2, t, c, strat)
                    # the micro-batch count is an outer variable like the TP
                    # degree: not monotone (DESIGN.md reading)
                    x2_ranges = [(x2, x2) for x2 in range(1, opts.m_max + 1)]

                def perf_fn(x1, x2, mk=mk):
                    s = mk(x1, x2)
                    if s is None:
                        return Perf(INF, INF)
                    return _perf_of(S.simulate(s))

                for a2, b2 in x2_ranges:
                    # B_E^max: largest B_E feasible at the least memory-hungry x2
                    b1 = 0
                    for be in range(1, opts.b_e_max + 1):
                        if math.isfinite(perf_fn(be, a2).latency):
                            b1 = be
                        else:
                            break
                    if b1 == 0:
                        continue
                    r = branch_and_bound(1, b1, a2, b2, perf_fn, L_b, opts.eps_t_frac, opts.eps_l_frac)
                    total_evals += r.evals + b1
                    if r.x is None:
                        continue
                    sch = mk(*r.x)
                    est = S.simulate(sch)
                    key = (-est.thrput_seq_s, est.latency_s, strat, t, c, r.x[0], r.x[1])
                    if best is None or key < best[0]:
                        best = (key, Found(sch, est, 0))
    if best is None:
        return None
    best[1].evals = total_evals
    return best[1]
