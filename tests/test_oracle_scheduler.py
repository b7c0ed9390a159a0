"""Pins for oracle/seqdist.py, oracle/simulator.py, oracle/bnb.py."""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import bnb, seqdist, simulator as sim
from workload import MODELS, task_dists, uniform_pmf


# ---------------------------------------------------------------- seqdist --
def test_completion_conditional_spec_examples():
    # SPEC.md:66-68
    assert seqdist.completion_conditional(3, 8) == {3: 1.0}
    assert seqdist.completion_conditional(10, 4) == {2: 1.0 / 3}
    assert seqdist.completion_conditional(8, 4) == {4: 0.5}


def test_completion_distribution_spec_examples():
    # SPEC.md:75-77, 84-86
    pd = np.zeros(4); pd[1] = 0.5; pd[3] = 0.5
    assert seqdist.completion_distribution(pd, 4) == [0.0, 0.5, 0.0, 0.5]
    pd = np.zeros(10); pd[9] = 1.0
    pu = seqdist.completion_distribution(pd, 4)
    assert pu[1] == pytest.approx(1 / 3) and seqdist.completion_fraction(pu) == pytest.approx(1 / 3)
    assert seqdist.completion_distribution([1.0], 1) == [1.0]
    pd = np.zeros(12); pd[[3, 7, 11]] = 1 / 3
    assert seqdist.completion_fraction(seqdist.completion_distribution(pd, 4)) == pytest.approx(11 / 18, abs=1e-15)


def _brute_conditional(s, n_d):
    """Enumerate the phases a length-s query occupies (uniform over its
    ceil(s/n_d) phases) and the iterations inside each."""
    q = 0
    while q * n_d < s:
        q += 1
    out = {}
    for phi in range(q):
        for u in range(1, n_d + 1):
            if phi * n_d + u == s:
                out[u] = out.get(u, Fraction(0)) + Fraction(1, q)
    return out


def test_completion_conditional_brute_force():
    for s in range(1, 65):
        for n_d in range(1, 17):
            got = seqdist.completion_conditional(s, n_d)
            ref = _brute_conditional(s, n_d)
            assert set(got) == set(ref)
            for u in ref:
                assert abs(got[u] - float(ref[u])) <= 1e-15
            mass = sum(got.values())
            assert mass == (1.0 if s <= n_d else 1.0 / math.ceil(s / n_d))


def test_completion_distribution_brute_force_mixture():
    rng = np.random.default_rng(3)
    for _ in range(50):
        L = int(rng.integers(1, 65))
        p = rng.random(L); p /= p.sum()
        n_d = int(rng.integers(1, 17))
        pu = seqdist.completion_distribution(p, n_d)
        ref = [0.0] * n_d
        for s in range(1, L + 1):
            for u, w in _brute_conditional(s, n_d).items():
                ref[u - 1] += p[s - 1] * float(w)
        assert np.allclose(pu, ref, atol=1e-12, rtol=0)


def test_full_phase_degenerates():
    d = task_dists("S")
    n_d = len(d.pmf_out)
    pu = seqdist.completion_distribution(d.pmf_out, n_d)
    assert seqdist.completion_fraction(pu) == pytest.approx(1.0, abs=1e-12)
    mean_u = sum((u + 1) * pu[u] for u in range(n_d))
    assert mean_u == pytest.approx(seqdist.pmf_mean(d.pmf_out), abs=1e-9)


def test_jensen_paper_fraction_exceeds_little():
    d = task_dists("S")
    for n_d in (1, 4, 7, 13, 32):
        f = seqdist.completion_fraction(seqdist.completion_distribution(d.pmf_out, n_d))
        assert f >= seqdist.little_fraction(d.pmf_out, n_d) - 1e-15
    # SURVEY.md S3 table, N_D = 13
    f13 = seqdist.completion_fraction(seqdist.completion_distribution(d.pmf_out, 13))
    assert f13 == pytest.approx(0.4037, abs=5e-4)


def test_batch_relations():
    # SPEC.md:253-261
    assert seqdist.rra_b_d(10, 1 / 3) == 30
    assert seqdist.waa_b_d(4, 32.0) == 128 and seqdist.waa_b_d(10, 3.0) == 30
    assert seqdist.rra_iteration_batches(16, [0.0, 0.5, 0.0, 0.5]) == [16, 16, 8, 8]
    assert seqdist.rra_iteration_batches(30, [0.0, 1 / 3, 0, 0]) == pytest.approx([30, 30, 20, 20])


def test_config1_schedule_relation():
    """Config 1: S ~ U{1..24}, B_D = 8 -> B_E = 4 at N_D = 6."""
    p = uniform_pmf(1, 24)
    f6 = seqdist.completion_fraction(seqdist.completion_distribution(p, 6))
    assert round(8 * f6) == 4 and f6 == pytest.approx(0.5208, abs=1e-4)
    assert seqdist.rra_b_d(4, f6) == 8


# -------------------------------------------------------------- simulator --
def _const_profile(t_enc_layer, t_dec_layer):
    p = sim.Profile([1])
    p.attn[("enc", 1)] = sim.Table2D([1, 4096], [1, 4096], [[0.0, 0.0], [0.0, 0.0]])
    p.attn[("dec", 1)] = sim.Table2D([1, 4096], [1, 4096], [[0.0, 0.0], [0.0, 0.0]])
    p.rest[("enc", 1)] = sim.Table1D([1, 1e9], [t_enc_layer, t_enc_layer])
    p.rest[("dec", 1)] = sim.Table1D([1, 1e9], [t_dec_layer, t_dec_layer])
    p.pp_sync = sim.Table1D([0, 1e15], [0.0, 0.0])
    return p


def _one_layer_model():
    m = sim.SimModel.from_spec(MODELS["opt-13b"])
    m.n_dec_layers = 1
    return m


@pytest.mark.parametrize("b_e,n_d,thr,lat", [(52, 13, 25.23, 10.23), (49, 7, 26.15, 16.87)])
def test_rra_timeline_reproduces_table8(b_e, n_d, thr, lat):
    """PAPER.md:722-724 (Table 8, RRA rows) with Table 9's decoder stage time
    0.038 s: T_cyc = B_E/thr, latency of the p99-length (63)
    query reproduces the printed latency."""
    T_cyc = b_e / thr
    t_dec = 0.038
    p = _const_profile(T_cyc - n_d * t_dec, t_dec)
    d = task_dists("S")
    S = sim.Simulator(p, _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out, 63)
    est = S.simulate(S.rra_schedule(b_e, n_d, 1, 0))
    assert est.thrput_seq_s == pytest.approx(thr, rel=1e-12)
    assert abs(est.latency_s - lat) < 0.01


def test_waa_pipeline_reproduces_fig4_counts():
    """with 1 encode stage + 3 decode stages, 2 tokens take
    7 stage-times unbatched and 3 2/3 with 3 micro-batches."""
    tau = 1.0
    K = 2
    M1 = (K - 1) * sim.period([tau] * 3, 1) + sim.fill([tau] * 3, 1)
    M3 = (K - 1) * sim.period([tau / 3] * 3, 3) + sim.fill([tau / 3] * 3, 3)
    assert tau + M1 == 7.0
    assert tau + M3 == pytest.approx(11 / 3, abs=1e-15)
    # hand-checked M > P_D case: M=4, P_D=2, K=2 -> 9 tau
    assert (K - 1) * sim.period([1.0, 1.0], 4) + sim.fill([1.0, 1.0], 4) == 9.0


def test_pipeline_algebra_equals_event_loop():
    rng = random.Random(11)
    for _ in range(2000):
        P, M, K = rng.randint(1, 6), rng.randint(1, 8), rng.randint(1, 6)
        if rng.random() < 0.5:
            ts = [rng.choice([0.5, 1.0, 2.0, 3.0]) for _ in range(P)]
        else:
            ts = [1.0] * P
        a = (K - 1) * sim.period(ts, M) + sim.fill(ts, M)
        assert a == pytest.approx(sim.pipeline_event_makespan(ts, M, K), abs=1e-9)
    assert sim.fill([1.0, 3.0], 2) == 7.0 and sim.fill([3.0, 1.0], 2) == 7.0


def test_rra_allocation_example():
    # PAPER.md:196 / SPEC.md:226: 8 layers on 4 GPUs -> 2 per GPU
    st = sim.stage_layout(4, 1, 0, 8)
    assert [(s[2], s[3]) for s in st] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    st = sim.stage_layout(4, 1, 0, 7)
    assert [s[3] - s[2] for s in st] == [2, 2, 2, 1]
    st = sim.stage_layout(8, 2, 4, 96)                     # 2 TP stages + 4 single
    assert [s[1] for s in st] == [2, 2, 1, 1, 1, 1] and sum(s[3] - s[2] for s in st) == 96


def test_waa_split_spec_examples():
    # SPEC.md:235-237 via the allocation rule
    def split(ce, cd, n):
        return min(max(int(math.floor(n * ce / (ce + cd) + 0.5)), 1), n - 1)
    assert split(1, 3, 4) == 1 and split(2, 2, 4) == 2 and split(100, 1, 4) == 3


def test_interp_exact_on_grid_and_hull():
    xs, ts = [1.0, 2.0, 4.0], [0.1, 0.3, 0.7]
    for x, t in zip(xs, ts):
        assert sim.interp1(xs, ts, x) == t
    assert sim.interp1(xs, ts, 3.0) == pytest.approx(0.5)
    assert sim.interp1(xs, ts, 0.5) == 0.1
    with pytest.raises(sim.OutOfHull):
        sim.interp1(xs, ts, 4.5)


def test_profile_roundtrip():
    p = _const_profile(0.1 / 3, 1e-3 / 7)
    p.tp_sync[2] = sim.Table1D([0.0, 1e6], [1e-5, 2.2e-5 / 3])
    q = sim.Profile.loads(p.dumps())
    assert q.dumps() == p.dumps()
    assert q.rest[("enc", 1)].t[0] == 0.1 / 3


# --------------------------------------------------------------------- B&B --
def _monotone_grid(rng, n1, n2):
    a = sorted(rng.random() for _ in range(n1))
    b = sorted(rng.random() for _ in range(n2))
    c = sorted(rng.random() for _ in range(n1))
    d = sorted(rng.random() for _ in range(n2))
    wt, wl = rng.uniform(0.2, 5), rng.uniform(0.2, 5)
    T = {(i + 1, j + 1): a[i] + wt * b[j] + 1e-9 * (i + j) for i in range(n1) for j in range(n2)}
    L = {(i + 1, j + 1): c[i] * wl + d[j] + 1e-9 * (i + j) for i in range(n1) for j in range(n2)}
    return T, L


def test_bnb_equals_exhaustive_on_strictly_monotone_grids():
    rng = random.Random(5)
    ev_frac = []
    for trial in range(300):
        n1, n2 = rng.randint(8, 32), rng.randint(8, 32)
        T, L = _monotone_grid(rng, n1, n2)
        Ls = sorted(L.values())
        L_b = Ls[rng.randint(0, len(Ls) - 1)] + 1e-12
        f = lambda x1, x2: bnb.Perf(L[(x1, x2)], T[(x1, x2)])
        r = bnb.branch_and_bound(1, n1, 1, n2, f, L_b, 0.0, 0.0)
        e = bnb.exhaustive(1, n1, 1, n2, f, L_b)
        if e.x is None:
            assert r.x is None
            continue
        assert r.perf.thrput == e.perf.thrput, trial
        assert r.perf.latency < L_b
        if n1 == 32 and n2 == 32 or n1 * n2 >= 600:
            ev_frac.append(r.evals / (n1 * n2))
    assert np.mean(ev_frac) <= 0.20


def test_bnb_upper_corner_shortcut_and_infeasible():
    f = lambda x1, x2: bnb.Perf(x1 + x2, x1 * x2)
    r = bnb.branch_and_bound(1, 10, 1, 10, f, 100.0)
    assert r.x == (10, 10) and r.evals <= 2
    r = bnb.branch_and_bound(1, 10, 1, 10, f, 1.5)
    assert r.x is None


def test_audit_counts_spike():
    g = {(i, j): bnb.Perf(float(i + j), float(i * j)) for i in range(1, 6) for j in range(1, 6)}
    assert bnb.monotonicity_audit(g, 1, 0.0, 0.0) == (0.0, 0.0)
    g[(3, 2)] = bnb.Perf(0.0, 0.0)
    fl, ft = bnb.monotonicity_audit(g, 1, 0.0, 0.0)
    assert fl == ft == pytest.approx(1 / 20)


def _synthetic_profile(model, tps=(1, 2, 4, 8)):
    """Roofline-shaped synthetic profile (test fixture only; the product
    profile is measured by exg_profile)."""
    p = sim.Profile(list(tps))
    d, ff, inner = model.d_model, model.d_ff, model.inner
    wbytes = (4 * d * inner + 2 * d * ff) * 2
    flops_tok = 2 * (4 * d * inner + 2 * d * ff)
    bs = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]
    cs = [1, 64, 128, 256, 512, 1024, 2048]
    toks = [1, 16, 64, 256, 1024, 4096, 16384, 65536, 262144, 1048576]
    for t in tps:
        for ph in ("enc", "dec"):
            p.attn[(ph, t)] = sim.Table2D(bs, cs, [[5e-6 + b * c * inner * 4 / t / 6e12 for c in cs] for b in bs])
            p.rest[(ph, t)] = sim.Table1D(toks, [8e-6 + max(wbytes / t / 6e12, x * flops_tok / t / 1.2e15) for x in toks])
        if t > 1:
            p.tp_sync[t] = sim.Table1D([0, 1e6, 1e9, 1e12], [1e-5, 1.2e-5, 1.5e-3, 1.5])
    p.pp_sync = sim.Table1D([0, 1e6, 1e9, 1e12, 1e15], [8e-6, 1e-5, 1.3e-3, 1.3, 1300.0])
    vbytes = model.vocab * d * 2
    p.head = sim.Table1D(bs, [4e-6 + max(vbytes / 6e12, b * 2 * model.vocab * d / 1.2e15) for b in bs])
    ks = [1, 2, 4, 8, 16, 32]
    p.switch = sim.Table2D(bs, ks, [[1e-4 * (1 + b / 512.0) * min(k, 8) / 3 for k in ks] for b in bs])
    return p


def test_schedule_find_bound_relaxation_trend():
    """SPEC.md:489 / Table 8 trend: relaxing L_B never lowers the optimum."""
    spec = MODELS["opt-13b"]
    m = sim.SimModel.from_spec(spec)
    d = task_dists("S")
    S = sim.Simulator(_synthetic_profile(m), m, sim.SimCluster(1, 180e9, 4e9), d.pmf_in, d.pmf_out, 63)
    prev = 0.0
    for L_b in (0.5, 1.0, 2.0, 4.0, float("inf")):
        f = bnb.schedule_find(S, L_b, sim.RRA, bnb.SearchOpts(b_e_max=64))
        if f is None:
            continue
        assert f.estimate.latency_s < L_b
        assert f.estimate.thrput_seq_s >= prev * (1 - 0.02)
        prev = f.estimate.thrput_seq_s
    assert prev > 0


def test_waa_m_split_balances_memory():
    """WAA-M (DESIGN.md reading): the encoder GPU count makes the
    per-GPU memory of the two sides as equal as any neighbouring split."""
    m = sim.SimModel.from_spec(MODELS["opt-66b"])
    d = task_dists("G")
    S = sim.Simulator(_synthetic_profile(m), m, sim.SimCluster(8, 180e9, 4e9), d.pmf_in, d.pmf_out, d.target_len)
    kv = S.kv_bytes_per_token_layer()
    W = S.n_layers * S.layer_bytes() + S.emb_bytes()
    for b_e in (1, 4, 16, 64):
        b_d = b_e * 192
        me = W + b_e * S.max_in * S.n_layers * kv
        md = W + b_d * (S.max_in + S.max_out) * S.n_layers * kv
        n = S.waa_split(b_e, b_d, sim.WAA_M)
        gap = lambda k: abs(me / k - md / (8 - k))
        for k in (n - 1, n + 1):
            if 1 <= k <= 7:
                assert gap(n) <= gap(k) * (1 + 1e-12), (b_e, n, k)
        s = S.waa_schedule(b_e, 2, 1, 0, sim.WAA_M)
        assert s.strategy == sim.WAA_M and s.n_enc_gpus == n
