"""Pins for the oracle functions the round-1 review found unpinned
(VERDICT.md r1 "What's weak" #1): Simulator.simulate_waa, Simulator.waa_split,
interp2, and bnb.schedule_find's strategy x t x c outer loop.

Each pin is something other than the oracle itself: a printed value of the
paper, an independent discrete-event simulation, a closed form, or a brute
force over the same grid.
"""
import math
import random

import numpy as np
import pytest

from oracle import bnb, seqdist, simulator as sim
from workload import MODELS, task_dists, uniform_pmf


# =========================================================== WAA timeline ==
def waa_event_loop(te, h, td, M, b_m, B_E, S, n_batches, release=None, miss=0.0):
    """Independent event simulation of the WAA system of PAPER.md:198-225
    (Fig. 4b/c) under the S7 reading.

    Encoder: a FIFO flow shop over stage times te; batch j (B_E requests) is
    released at j*release (None: all at t=0, a saturated encoder).  Its output
    reaches the decoder after the handoff h, plus `miss` (the buffer of one
    missed handover).  Decoder: M micro-batches of b_m
    slots circulate through stage times td (every stage FIFO, one micro-batch
    at a time); when a micro-batch starts an iteration it drops its finished
    rows and absorbs arrived requests FIFO.  Every request emits S tokens (one
    per iteration of its micro-batch).  Returns [(completion time, latency from
    the start of its encode)]."""
    free = [0.0] * len(te)
    arrivals = []
    for j in range(n_batches):
        t = 0.0 if release is None else j * release
        start = None
        for k, v in enumerate(te):
            s = max(t, free[k])
            if k == 0:
                start = s
            t = s + v
            free[k] = t
        for _ in range(B_E):
            arrivals.append((t + h + miss, start))
    arrivals.sort()
    P = len(td)
    sfree = [0.0] * P
    rows = [[] for _ in range(M)]
    ready = [0.0] * M
    qi, total, done = 0, len(arrivals), []
    while len(done) < total:
        m = min(range(M), key=lambda i: (ready[i], i))
        t0 = max(ready[m], sfree[0])
        rows[m] = [r for r in rows[m] if r[0] > 0]
        if not rows[m] and qi < total and arrivals[qi][0] > t0 and all(not rows[i] for i in range(M)):
            t0 = arrivals[qi][0]
        while qi < total and arrivals[qi][0] <= t0 and len(rows[m]) < b_m:
            rows[m].append([S, arrivals[qi][1]])
            qi += 1
        if not rows[m]:
            ready[m] = max(t0, arrivals[qi][0]) if qi < total else math.inf
            continue
        t = t0
        for k in range(P):
            t = max(t, sfree[k]) + td[k]
            sfree[k] = t
        ready[m] = t
        for r in rows[m]:
            r[0] -= 1
            if r[0] == 0:
                done.append((t, t - r[1]))
    return done


def _steady(done):
    d = sorted(done)
    n = len(d)
    a, b = n // 4, 3 * n // 4
    return (b - a) / (d[b][0] - d[a][0]), max(x[1] for x in d[a:b])


def _simulate_waa_stage_times(te, td, M, B_E, S, h):
    """simulate_waa on a hand-built WAA layout whose stage times are te
    (encoder) and td (decoder): stage k holds round(1000 te[k]) (round(1000
    td[k])) layers of 1 ms each, pp_sync = 0 (the handoff term is pinned by
    test_simulate_waa_handoff_term), every output S tokens long."""
    assert h == 0.0
    scale = 1000
    lay_e = [int(round(v * scale)) for v in te]
    lay_d = [int(round(v * scale)) for v in td]
    L = max(sum(lay_e), sum(lay_d))
    prof = sim.Profile([1])
    prof.attn[("enc", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
    prof.attn[("dec", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
    prof.rest[("enc", 1)] = sim.Table1D([0, 1e12], [1.0 / scale, 1.0 / scale])
    prof.rest[("dec", 1)] = sim.Table1D([0, 1e12], [1.0 / scale, 1.0 / scale])
    prof.pp_sync = sim.Table1D([0, 1e18], [0.0, 0.0])
    m = sim.SimModel.from_spec(MODELS["opt-13b"])
    m.n_dec_layers = L
    pmf_out = [0.0] * S
    pmf_out[S - 1] = 1.0
    Sim = sim.Simulator(prof, m, sim.SimCluster(len(te) + len(td), 1e30),
                        uniform_pmf(1, 1), pmf_out, S)
    stages, g, l = [], 0, 0
    for n in lay_e:
        stages.append((g, 1, l, l + n))
        g += 1
        l += n
    l = 0
    for n in lay_d:
        stages.append((g, 1, l, l + n))
        g += 1
        l += n
    B_D = seqdist.waa_b_d(B_E, Sim.s_d)
    assert B_D == B_E * S
    b_m = -(-B_D // M)
    s = sim.Schedule(sim.WAA_C, B_E, B_D, b_m, 0, 1, 0, len(te), stages)
    return Sim.simulate_waa(s), b_m


_WAA_CASES = []
_rng = random.Random(7)
while len(_WAA_CASES) < 40:
    PE, PD = _rng.randint(1, 3), _rng.randint(1, 3)
    te = [_rng.choice([0.5, 1.0, 2.0, 3.0]) for _ in range(PE)]
    td = [_rng.choice([0.05, 0.1, 0.2]) for _ in range(PD)]
    S, B_E = _rng.randint(2, 8), _rng.randint(1, 4)
    M = _rng.choice([d for d in range(1, 5) if (B_E * S) % d == 0])   # M | B_D: no slack slots
    _WAA_CASES.append((te, td, M, B_E, S))


@pytest.mark.parametrize("te,td,M,B_E,S", _WAA_CASES)
def test_simulate_waa_throughput_equals_event_loop(te, td, M, B_E, S):
    """Long-run throughput of the event loop (saturated encoder, B_D = B_E S
    slots) equals simulate_waa's B_E / max(T_E, Pi(td, M)) -- encoder-bound
    and decoder-bound cases alike (a sum instead of the max, T_E = sum of the
    stages, or T_D = sum of td would all fail)."""
    est, b_m = _simulate_waa_stage_times(te, td, M, B_E, S, 0.0)
    thr, _ = _steady(waa_event_loop(te, 0.0, td, M, b_m, B_E, S, 400))
    assert est.thrput_seq_s == pytest.approx(thr, rel=4e-3)


@pytest.mark.parametrize("te,td,M,B_E,S", _WAA_CASES)
def test_simulate_waa_latency_vs_event_loop(te, td, M, B_E, S):
    """Worst steady-state latency of the event loop (encoder paced at the
    system period, one missed handover = one encoder period T_E of buffer):
    * never below T_trav + T_E + S * sum(td) (every iteration traverses every
      decoder stage) -- simulate_waa's latency is >= this bound too;
    * never above simulate_waa's latency + one decoder period (the wait for
      the running iteration to end, which the paper's buffer reading omits);
    * EQUAL to simulate_waa's latency when M = 1 and the decoder drains
      between encoder batches (T_E >= S * sum(td)): this fixes the T_trav,
      T_E, (S-1) Pi + F terms exactly."""
    est, b_m = _simulate_waa_stage_times(te, td, M, B_E, S, 0.0)
    T_E, T_trav, Pi = max(te), sum(te), sim.period(td, M)
    _, lat = _steady(waa_event_loop(te, 0.0, td, M, b_m, B_E, S, 400, release=max(T_E, Pi), miss=T_E))
    lower = T_trav + T_E + S * sum(td)
    assert lat >= lower - 1e-9
    assert est.latency_s >= lower - 1e-9
    assert lat <= est.latency_s + Pi + 1e-9
    if M == 1 and T_E >= S * sum(td):
        assert est.latency_s == pytest.approx(lat, abs=1e-9)


def test_simulate_waa_handoff_term():
    """The KV handoff is charged once per request on the
    latency, at pp_sync(B_E * S_E * L * KV bytes/token/layer), and not on the
    throughput."""
    d = task_dists("S")
    m = sim.SimModel.from_spec(MODELS["opt-13b"])
    m.n_dec_layers = 1

    def run(h_per_byte):
        prof = sim.Profile([1])
        prof.attn[("enc", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
        prof.attn[("dec", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
        prof.rest[("enc", 1)] = sim.Table1D([0, 1e12], [0.2, 0.2])
        prof.rest[("dec", 1)] = sim.Table1D([0, 1e12], [0.01, 0.01])
        prof.pp_sync = sim.Table1D([0, 1e15], [0.0, 1e15 * h_per_byte])
        S = sim.Simulator(prof, m, sim.SimCluster(2, 1e30), d.pmf_in, d.pmf_out, 63)
        s = sim.Schedule(sim.WAA_C, 4, 128, 128, 0, 1, 0, 1, [(0, 1, 0, 1), (1, 1, 0, 1)])
        return S, S.simulate_waa(s)

    S0, e0 = run(0.0)
    S1, e1 = run(1e-9)
    nbytes = 4 * S0.s_e * 1 * (2 * MODELS["opt-13b"].inner * 2)
    assert e1.thrput_seq_s == e0.thrput_seq_s
    assert e1.latency_s - e0.latency_s == pytest.approx(nbytes * 1e-9, rel=1e-12)


def test_simulate_waa_reproduces_table8_row1():
    """Table 8 row 1: WAA, B_E=4, 22.41 seq/s, latency 3.01 s
    for the p99 (63-token) query of task S; Table 9: WAA
    decoder single-stage time 0.041 +- 0.002 s.  An encoder-bound WAA timeline
    with T_E = 4/22.41 and the decoder stage at 0.041 -+ 0.002 s brackets the
    printed 3.01 s (2*0.1785 + 63*0.042 = 3.00); dropping the
    one-period buffer (2.76 s at 0.041), or charging T_E only once, misses it."""
    d = task_dists("S")
    assert d.target_len == 63
    m = sim.SimModel.from_spec(MODELS["opt-13b"])
    m.n_dec_layers = 1
    T_E = 4 / 22.41

    def est(t_dec):
        prof = sim.Profile([1])
        prof.attn[("enc", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
        prof.attn[("dec", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
        prof.rest[("enc", 1)] = sim.Table1D([0, 1e12], [T_E, T_E])
        prof.rest[("dec", 1)] = sim.Table1D([0, 1e12], [t_dec, t_dec])
        prof.pp_sync = sim.Table1D([0, 1e18], [0.0, 0.0])
        S = sim.Simulator(prof, m, sim.SimCluster(2, 1e30), d.pmf_in, d.pmf_out, 63)
        s = S.waa_schedule(4, 1, 1, 0)
        assert s.b_d == 128 and s.n_enc_gpus == 1
        return S.simulate_waa(s)

    lo, mid, hi = est(0.039), est(0.041), est(0.043)
    assert mid.thrput_seq_s == pytest.approx(22.41, rel=1e-12)
    assert lo.latency_s <= 3.01 <= hi.latency_s
    assert abs(mid.latency_s - 3.01) < 0.1
    # the printed value is NOT reproduced without the buffer term
    assert not (lo.latency_s - T_E <= 3.01 <= hi.latency_s - T_E)


# ============================================================ WAA split ==
def _split_sim(c_e, c_d, n):
    prof = sim.Profile([1])
    prof.attn[("enc", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
    prof.attn[("dec", 1)] = sim.Table2D([1, 1e9], [1, 1e9], [[0.0, 0.0], [0.0, 0.0]])
    prof.rest[("enc", 1)] = sim.Table1D([0, 1e12], [c_e, c_e])
    prof.rest[("dec", 1)] = sim.Table1D([0, 1e12], [c_d, c_d])
    prof.pp_sync = sim.Table1D([0, 1e18], [0.0, 0.0])
    m = sim.SimModel.from_spec(MODELS["opt-13b"])
    d = task_dists("S")
    return sim.Simulator(prof, m, sim.SimCluster(n, 1e30), d.pmf_in, d.pmf_out, 63)


@pytest.mark.parametrize("c_e,c_d,n,want", [(1.0, 3.0, 4, 1), (2.0, 2.0, 4, 2), (100.0, 1.0, 4, 3),
                                             (1.0, 100.0, 4, 1), (1.0, 1.0, 2, 1)])
def test_waa_split_spec_examples_through_the_oracle(c_e, c_d, n, want):
    """SPEC.md:235-237 through Simulator.waa_split on profiles whose per-layer
    encode / decode times are c_e / c_d: (1,3,4)->1 encoder GPU, (c,c,4)->2,
    (100,1,4)->3 (clamped: at least one decoder GPU); n=2 -> (1,1)
    (SPEC.md:246)."""
    S = _split_sim(c_e, c_d, n)
    assert S.waa_split(4, 128) == want
    s = S.waa_schedule(4, 1, 1, 0)
    assert s.n_enc_gpus == want and len(s.stages) == n


def test_waa_split_mirror_invariant_and_infeasible():
    """SPEC.md Invariants: n_enc(a, b) = n_dec(b, a) away from .5 rounding
    boundaries; WAA on one GPU is infeasible."""
    rng = random.Random(3)
    for _ in range(200):
        a, b, n = rng.uniform(0.01, 10), rng.uniform(0.01, 10), rng.randint(2, 8)
        if abs(n * a / (a + b) % 1 - 0.5) < 1e-6:
            continue
        assert _split_sim(a, b, n).waa_split(1, 1) == n - _split_sim(b, a, n).waa_split(1, 1)
    assert _split_sim(1.0, 1.0, 1).waa_schedule(4, 1, 1, 0) is None


# ============================================================== interp2 ==
def test_interp2_hand_values():
    """Hand-computed bilinear values on a non-constant, asymmetric table:
    b axis [1, 3], c axis [10, 20, 40]; t[b][c] below.  At (2, 15): ctx rows
    1.5 and 7.5, then 1.5 + (2-1)(7.5-1.5)/2 = 4.5.  At (3, 30): row b=3 at
    c=30 -> 10 + (30-20)(30-10)/20 = 20.  At (1, 40): 4.  Swapping the axes or
    bracketing the wrong row changes every one of these."""
    tb = sim.Table2D([1.0, 3.0], [10.0, 20.0, 40.0], [[1.0, 2.0, 4.0], [5.0, 10.0, 30.0]])
    assert sim.interp2(tb, 2.0, 15.0) == 4.5
    assert sim.interp2(tb, 3.0, 30.0) == 20.0
    assert sim.interp2(tb, 1.0, 40.0) == 4.0
    assert sim.interp2(tb, 0.5, 5.0) == 1.0                 # clamped below on both axes
    assert sim.interp2(tb, 2.5, 40.0) == 4.0 + 1.5 * 26.0 / 2.0
    with pytest.raises(sim.OutOfHull):
        sim.interp2(tb, 2.0, 41.0)
    with pytest.raises(sim.OutOfHull):
        sim.interp2(tb, 3.5, 20.0)


def test_interp2_exact_on_bilinear_functions():
    """Closed form: bilinear interpolation reproduces any function
    t = a + p b + q c + r b c exactly (up to rounding) inside each cell, on
    non-uniform grids."""
    rng = np.random.default_rng(9)
    for _ in range(50):
        bs = np.sort(rng.choice(np.arange(1, 200), size=rng.integers(2, 7), replace=False)).astype(float)
        cs = np.sort(rng.choice(np.arange(1, 3000), size=rng.integers(2, 7), replace=False)).astype(float)
        a, p, q, r = rng.uniform(-1, 1, 4)
        f = lambda b, c: a + p * b + q * c + r * b * c
        tb = sim.Table2D(list(bs), list(cs), [[f(b, c) for c in cs] for b in bs])
        for _ in range(20):
            b = rng.uniform(bs[0], bs[-1])
            c = rng.uniform(cs[0], cs[-1])
            assert sim.interp2(tb, b, c) == pytest.approx(f(b, c), abs=1e-9 * (1 + abs(r) * b * c))


# ===================================================== schedule_find ====
def _exhaustive_find(S, L_b, mask, opts):
    """Plain definition of PAPER.md:269-276 with the outer loops of
    PAPER.md:312, 348: argmax throughput over every strategy, TP degree t,
    applied-GPU count c and every (x1, x2) of the grid, latency < L_b
    strictly; ties -> lower latency -> smallest (strategy, t, c, x1, x2)."""
    N, H = S.cl.n_gpus, S.m.n_heads
    n_d_max = opts.n_d_max if opts.n_d_max > 0 else S.max_out
    best = None
    for strat in (sim.RRA, sim.WAA_C, sim.WAA_M):
        if not (mask & strat) or (strat != sim.RRA and N < 2):
            continue
        for t in (1, 2, 4, 8):
            if t > N or H % t:
                continue
            for c in ([0] if t == 1 else range(t, N + 1, t)):
                for x1 in range(1, opts.b_e_max + 1):
                    for x2 in range(1, (n_d_max if strat == sim.RRA else opts.m_max) + 1):
                        if strat == sim.RRA:
                            s = S.rra_schedule(x1, n_d_max + 1 - x2, t, c)
                        else:
                            s = S.waa_schedule(x1, opts.m_max + 1 - x2, t, c, strat)
                        if s is None:
                            continue
                        e = S.simulate(s)
                        if not (e.feasible and e.latency_s < L_b):
                            continue
                        key = (-e.thrput_seq_s, e.latency_s, strat, t, c, x1, x2)
                        if best is None or key < best[0]:
                            best = (key, s, e)
    return best


def _small_problem(n_gpus):
    from test_oracle_scheduler import _synthetic_profile
    spec = MODELS["opt-13b"]
    m = sim.SimModel.from_spec(spec)
    m.n_dec_layers = 8
    m.n_heads = 8
    out = uniform_pmf(1, 12)
    inp = uniform_pmf(32, 96)
    prof = _synthetic_profile(m)
    return sim.Simulator(prof, m, sim.SimCluster(n_gpus, 6.0e9, 0.2e9), inp, out, 12)


@pytest.mark.parametrize("n_gpus", [1, 2, 4])
def test_schedule_find_equals_exhaustive(n_gpus):
    """Algorithm 1 inside its strategy x t x c loops (bnb.schedule_find, eps
    = 0) returns the exhaustive optimum of the same grid, for every latency
    bound between the tightest and the loosest feasible point, with the
    memory-limited B_E^max rule active (6 GB per GPU)."""
    S = _small_problem(n_gpus)
    opts = bnb.SearchOpts(eps_t_frac=0.0, eps_l_frac=0.0, b_e_max=12, m_max=4)
    lats = []
    ex_inf = _exhaustive_find(S, math.inf, sim.RRA | sim.WAA_C | sim.WAA_M, opts)
    assert ex_inf is not None
    # latency bounds spread over the feasible range
    grid_lat = sorted({round(ex_inf[2].latency_s, 12)} | {
        S.simulate(S.rra_schedule(x1, nd, 1, 0)).latency_s for x1 in (1, 3, 6, 12) for nd in (1, 4, 12)})
    bounds = [v * 1.0001 for v in grid_lat if math.isfinite(v)] + [math.inf]
    n_match = 0
    for L_b in bounds:
        ex = _exhaustive_find(S, L_b, sim.RRA | sim.WAA_C | sim.WAA_M, opts)
        got = bnb.schedule_find(S, L_b, sim.RRA | sim.WAA_C | sim.WAA_M, opts)
        if ex is None:
            assert got is None
            continue
        assert got is not None
        assert got.estimate.latency_s < L_b
        assert got.estimate.thrput_seq_s == pytest.approx(ex[2].thrput_seq_s, rel=1e-12), (L_b, got.schedule, ex[1])
        n_match += 1
    assert n_match >= 3


# ======================================================== decode head term ==
def test_head_table_charged_once_per_iteration_on_the_last_stage():
    """The profile's `head` table (final norm + LM head + argmax per decode
    iteration) adds head(b) to the decode stage time of the last stage only:
    RRA P = 1 latency / cycle grow by exactly sum_u head(b_u) (closed form on a
    constant-cost profile), and profile-v1 round-trips it."""
    from test_oracle_scheduler import _const_profile, _one_layer_model
    d = task_dists("S")
    p0 = _const_profile(0.5, 0.01)
    p1 = sim.Profile.loads(p0.dumps())
    p1.head = sim.Table1D([1.0, 1000.0], [0.002, 0.002 + 999 * 1e-5])
    assert sim.Profile.loads(p1.dumps()).dumps() == p1.dumps()
    S0 = sim.Simulator(p0, _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out, 63)
    S1 = sim.Simulator(p1, _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out, 63)
    s = S0.rra_schedule(16, 8, 1, 0)
    e0, e1 = S0.simulate(s), S1.simulate(s)
    pu, f = S0.pu(8)
    bu = seqdist.rra_iteration_batches(s.b_d, pu)
    head = [0.002 + (b - 1) * 1e-5 for b in bu]
    T0, T1 = s.b_e / e0.thrput_seq_s, s.b_e / e1.thrput_seq_s
    assert T1 - T0 == pytest.approx(sum(head), rel=1e-9)
    # latency of the 63-token query: ceil(63/8) = 8 cycles, the last one to r = 7
    assert e1.latency_s - e0.latency_s == pytest.approx(7 * sum(head) + sum(head[:7]), rel=1e-9)
    # pipelines: only the last stage carries it
    st = sim.stage_layout(4, 1, 0, 8)
    t0 = S0.stage_times(st, "dec", 16.0)
    t1 = S1.stage_times(st, "dec", 16.0)
    assert t1[:3] == t0[:3] and t1[3] - t0[3] == pytest.approx(0.002 + 15 * 1e-5, rel=1e-12)
    assert S1.stage_times(st, "enc", 16.0) == S0.stage_times(st, "enc", 16.0)


def test_switch_table_and_rms_attention_length():
    """Encode -> decode switch (profile `switch`): the phase's first decode
    iteration carries switch(b_1) once per RRA cycle (closed form at P = 1);
    the static batch carries it once.  Encode attention is looked up at the
    RMS input length sqrt(E[n^2]) (closed form on a table linear in c^2)."""
    from test_oracle_scheduler import _const_profile, _one_layer_model
    d = task_dists("S")
    p0 = _const_profile(0.5, 0.01)
    p1 = sim.Profile.loads(p0.dumps())
    # cumulative extra time of the first k decode iterations: 0.003 + 2e-6 (b-1)
    # per iteration for k <= 8, flat beyond (the clock has recovered)
    ks = [1.0, 2.0, 4.0, 8.0, 16.0]
    p1.switch = sim.Table2D([1.0, 1000.0], ks, [[(0.003 + (b - 1) * 2e-6) * min(k, 8.0) for k in ks]
                                                for b in (1.0, 1000.0)])
    assert sim.Profile.loads(p1.dumps()).dumps() == p1.dumps()
    S0 = sim.Simulator(p0, _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out, 63)
    S1 = sim.Simulator(p1, _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out, 63)
    for n_d, k in ((8, 8.0), (4, 4.0), (30, 8.0)):
        s = S0.rra_schedule(16, n_d, 1, 0)
        e0, e1 = S0.simulate(s), S1.simulate(s)
        w = (0.003 + (s.b_d - 1) * 2e-6) * k                # b_1 = B_D, k = min(N_D, table)
        assert s.b_e / e1.thrput_seq_s - s.b_e / e0.thrput_seq_s == pytest.approx(w, rel=1e-9)
        assert e1.latency_s - e0.latency_s == pytest.approx(-(-63 // n_d) * w, rel=1e-9)   # one per cycle
    st0, st1 = S0.simulate_static(8), S1.simulate_static(8)
    assert st1.latency_s - st0.latency_s == pytest.approx((0.003 + 7 * 2e-6) * 8, rel=1e-9)
    # RMS length: an attention table t = c^2 (per request) makes the encode
    # attention term b * E[n^2]
    p2 = sim.Profile.loads(p0.dumps())
    cs = [float(c) for c in range(1, 600, 7)]
    p2.attn[("enc", 1)] = sim.Table2D([1.0, 4096.0], cs, [[c * c for c in cs], [4096 * c * c for c in cs]])
    S2 = sim.Simulator(p2, _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out, 63)
    e_n2 = sum(float(k * k) * float(d.pmf_in[k - 1]) for k in range(1, len(d.pmf_in) + 1))
    a = S2.layer_enc(1, 1.0) - S0.layer_enc(1, 1.0)
    assert a == pytest.approx(e_n2, rel=2e-3)           # piecewise-linear table of c^2
    assert e_n2 > 1.25 * S2.s_e ** 2                     # task S: RMS length ~1.14 x the mean


def test_rra_latency_buffer_closed_form():
    """RRA latency buffer (PAPER.md:397 reading): on a profile whose encode
    layer time is linear in tokens (slope a per token per layer) the latency
    grows by exactly L a z99 sqrt(q B_E) sigma_in -- the 99th-percentile excess
    of the encoder workload over the query's q phases -- and throughput is
    unchanged; sigma_in is the input PMF's standard deviation."""
    from test_oracle_scheduler import _one_layer_model
    d = task_dists("S")
    a = 2e-6

    def prof(slope):
        p = sim.Profile([1])
        p.attn[("enc", 1)] = sim.Table2D([1, 4096], [1, 4096], [[0.0, 0.0], [0.0, 0.0]])
        p.attn[("dec", 1)] = sim.Table2D([1, 4096], [1, 4096], [[0.0, 0.0], [0.0, 0.0]])
        p.rest[("enc", 1)] = sim.Table1D([0.0, 1e9], [0.01, 0.01 + slope * 1e9])
        p.rest[("dec", 1)] = sim.Table1D([1, 1e9], [0.01, 0.01])
        p.pp_sync = sim.Table1D([0, 1e15], [0.0, 0.0])
        return p
    S = sim.Simulator(prof(a), _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out, 63)
    mean = sum(k * d.pmf_in[k - 1] for k in range(1, len(d.pmf_in) + 1))
    sd = math.sqrt(sum((k - mean) ** 2 * d.pmf_in[k - 1] for k in range(1, len(d.pmf_in) + 1)))
    assert S.s_e_sd == pytest.approx(sd, rel=1e-9)
    for b_e, n_d in ((16, 8), (40, 32), (60, 63)):
        s = S.rra_schedule(b_e, n_d, 1, 0)
        e = S.simulate(s)
        q = -(-63 // n_d)
        T_enc = 0.01 + a * b_e * mean
        T_dec = 0.01
        r = 1 + (63 - 1) % n_d
        lat0 = (q - 1) * (T_enc + n_d * T_dec) + T_enc + r * T_dec
        assert e.latency_s - lat0 == pytest.approx(a * sim.Z99 * math.sqrt(q * b_e) * sd, rel=1e-6)
        assert e.thrput_seq_s == pytest.approx(b_e / (T_enc + n_d * T_dec), rel=1e-12)
