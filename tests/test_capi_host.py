"""Host-side checks of libexegpt.so (no GPU needed):

* the library loads and exports every symbol include/*.h declares;
* the C++ planner (XSimulator + Algorithm 1) is bit-identical to the oracle
  on the same profile-v1 file (test tier T1);
* error statuses follow the header contract.
"""
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="session")
def L():
    from paper_2404_07947_b200 import _lib
    from paper_2404_07947_b200.build import build
    build()
    return _lib


def _declared_symbols():
    names = set()
    for h in ("exegpt.h", "exegpt_ops.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(exg_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol(L):
    import ctypes
    lib = ctypes.CDLL(L.LIB_PATH)
    names = _declared_symbols()
    assert len(names) >= 20
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert L.lib().exg_abi_version() == L.ABI_VERSION == 5


def _setup(task="S", model="opt-13b", n_gpus=1, mem=180e9, ws=4e9):
    from oracle import simulator as sim
    from workload import MODELS, task_dists
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_oracle_scheduler import _synthetic_profile
    spec = MODELS[model]
    m = sim.SimModel.from_spec(spec)
    prof = _synthetic_profile(m)
    d = task_dists(task)
    return spec, m, prof, d, sim.SimCluster(n_gpus, mem, ws)


def _c_objects(L, spec, prof, d, cl, tmp_path):
    path = str(tmp_path / "prof.txt")
    prof.save(path)
    P = L.Profile.load(path)
    mspec = L.model_spec(spec, 1)
    ccl = L.cluster_spec(cl.n_gpus, cl.mem_per_gpu_bytes, cl.workspace_bytes, cl.kv_page)
    return P, mspec, ccl, L.Pmf(d.pmf_in), L.Pmf(d.pmf_out)


def test_profile_roundtrip_through_library(L, tmp_path):
    spec, m, prof, d, cl = _setup()
    P, *_ = _c_objects(L, spec, prof, d, cl, tmp_path)
    out = str(tmp_path / "again.txt")
    P.save(out)
    assert open(out).read() == prof.dumps()


@pytest.mark.parametrize("b_e,n_d", [(1, 1), (4, 7), (16, 13), (52, 13), (49, 7), (64, 80), (200, 3)])
def test_simulate_rra_bit_identical(L, tmp_path, b_e, n_d):
    from oracle import simulator as sim
    spec, m, prof, d, cl = _setup()
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    S = sim.Simulator(prof, m, cl, d.pmf_in, d.pmf_out, d.target_len)
    s_o = S.rra_schedule(b_e, n_d, 1, 0)
    e_o = S.simulate(s_o)
    s_c = L.rra_schedule(b_e, 0, n_d)
    L.schedule_resolve(P, mspec, ccl, pin, pout, s_c)
    assert s_c.b_d == s_o.b_d and s_c.stages() == s_o.stages
    e_c = L.simulate(P, mspec, ccl, pin, pout, d.target_len, s_c)
    assert bool(e_c.feasible) == e_o.feasible
    if e_o.feasible:
        assert e_c.thrput_seq_s == e_o.thrput_seq_s and e_c.latency_s == e_o.latency_s


@pytest.mark.parametrize("n_gpus,t,c", [(4, 1, 0), (8, 2, 4), (8, 4, 8)])
def test_simulate_pipeline_bit_identical(L, tmp_path, n_gpus, t, c):
    from oracle import simulator as sim
    spec, m, prof, d, cl = _setup("G", "opt-66b", n_gpus)
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    S = sim.Simulator(prof, m, cl, d.pmf_in, d.pmf_out, d.target_len)
    for b_e, n_d in [(8, 10), (32, 50), (3, 480)]:
        s_o = S.rra_schedule(b_e, n_d, t, c)
        e_o = S.simulate(s_o)
        s_c = L.rra_schedule(b_e, 0, n_d)
        s_c.tp_degree, s_c.tp_gpus = t, c
        L.schedule_resolve(P, mspec, ccl, pin, pout, s_c)
        assert s_c.stages() == s_o.stages
        e_c = L.simulate(P, mspec, ccl, pin, pout, d.target_len, s_c)
        assert (e_c.thrput_seq_s, e_c.latency_s) == (e_o.thrput_seq_s, e_o.latency_s)
    # WAA with partial TP on the decoder side
    for b_e, M in [(2, 1), (4, 3), (8, 8)]:
        s_o = S.waa_schedule(b_e, M, t, c if c <= n_gpus - 1 else 0)
        if s_o is None:
            continue
        e_o = S.simulate(s_o)
        s_c = L.exg_schedule()
        s_c.strategy, s_c.b_e, s_c.tp_degree, s_c.tp_gpus = 2, b_e, s_o.tp_degree, s_o.tp_gpus
        L.schedule_resolve(P, mspec, ccl, pin, pout, s_c, M)
        assert (s_c.b_d, s_c.b_m, s_c.n_enc_gpus) == (s_o.b_d, s_o.b_m, s_o.n_enc_gpus)
        assert s_c.stages() == s_o.stages
        e_c = L.simulate(P, mspec, ccl, pin, pout, d.target_len, s_c)
        assert (e_c.thrput_seq_s, e_c.latency_s) == (e_o.thrput_seq_s, e_o.latency_s)


@pytest.mark.parametrize("task,model,n_gpus,mask", [("S", "opt-13b", 1, 1), ("S", "opt-13b", 4, 3),
                                                    ("G", "opt-66b", 8, 3), ("C1", "gpt3-175b", 8, 3),
                                                    ("G", "opt-66b", 4, 7), ("C1", "gpt3-175b", 8, 4)])
def test_schedule_find_bit_identical(L, tmp_path, task, model, n_gpus, mask):
    from oracle import bnb, simulator as sim
    spec, m, prof, d, cl = _setup(task, model, n_gpus)
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    S = sim.Simulator(prof, m, cl, d.pmf_in, d.pmf_out, d.target_len)
    opts = bnb.SearchOpts(b_e_max=48, m_max=6)
    copts = L.search_opts(b_e_max=48, m_max=6)
    for L_b in (0.3, 1.0, 3.0, math.inf):
        f = bnb.schedule_find(S, L_b, mask, opts)
        if f is None:
            with pytest.raises(L.ExgError) as ei:
                L.schedule_find(P, mspec, ccl, pin, pout, d.target_len, L_b, mask, copts)
            assert ei.value.status == L.EXG_E_INFEASIBLE
            continue
        s, est = L.schedule_find(P, mspec, ccl, pin, pout, d.target_len, L_b, mask, copts)
        assert (s.strategy, s.b_e, s.b_d, s.b_m, s.n_d, s.tp_degree, s.tp_gpus, s.n_enc_gpus) == (
            f.schedule.strategy, f.schedule.b_e, f.schedule.b_d, f.schedule.b_m, f.schedule.n_d,
            f.schedule.tp_degree, f.schedule.tp_gpus, f.schedule.n_enc_gpus)
        assert s.stages() == f.schedule.stages
        assert est.thrput_seq_s == f.estimate.thrput_seq_s and est.latency_s == f.estimate.latency_s
        assert est.perf_evals == f.evals
        assert est.latency_s < L_b


def test_static_batch_estimate_bit_identical(L, tmp_path):
    from oracle import simulator as sim
    spec, m, prof, d, cl = _setup()
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    S = sim.Simulator(prof, m, cl, d.pmf_in, d.pmf_out, d.target_len)
    for B in (1, 4, 8, 64, 256, 4000):
        e_o = S.simulate_static(B)
        s = L.exg_schedule()
        s.strategy, s.b_e = 8, B
        e_c = L.simulate(P, mspec, ccl, pin, pout, d.target_len, s)
        assert bool(e_c.feasible) == e_o.feasible
        if e_o.feasible:
            assert (e_c.thrput_seq_s, e_c.latency_s) == (e_o.thrput_seq_s, e_o.latency_s)


def test_static_latency_is_encode_plus_max_out_decodes():
    """Closed form of the FT-style static batch:
    latency = T_enc(B) + max_out * T_dec(B) on a constant-cost profile."""
    from oracle import simulator as sim
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_oracle_scheduler import _const_profile, _one_layer_model
    from workload import task_dists
    d = task_dists("S")
    S = sim.Simulator(_const_profile(0.5, 0.01), _one_layer_model(), sim.SimCluster(1, 1e30), d.pmf_in, d.pmf_out,
                      63)
    e = S.simulate_static(16)
    assert e.latency_s == pytest.approx(0.5 + 80 * 0.01, abs=1e-12)
    assert e.thrput_seq_s == pytest.approx(16 / 1.3, abs=1e-9)


def test_error_statuses(L, tmp_path):
    spec, m, prof, d, cl = _setup()
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    with pytest.raises(L.ExgError) as ei:
        L.schedule_find(P, mspec, ccl, pin, pout, d.target_len, 1e-9, 1, L.search_opts())
    assert ei.value.status == L.EXG_E_INFEASIBLE
    with pytest.raises(L.ExgError) as ei:
        L.schedule_find(P, mspec, ccl, pin, pout, 0, 1.0, 1, L.search_opts())
    assert ei.value.status == L.EXG_E_INPUT
    with pytest.raises(L.ExgError) as ei:
        L.Profile.load(str(tmp_path / "missing.txt"))
    assert ei.value.status == L.EXG_E_INPUT
    bad = str(tmp_path / "bad.txt")
    open(bad, "w").write("profile-v1\ntp 1 1\nbogus\n")
    with pytest.raises(L.ExgError):
        L.Profile.load(bad)


def test_profile_comm_model_tables(L, tmp_path):
    """exg_profile_comm_model: pp_sync = alpha + bytes/bw, tp_sync[t] = alpha +
    (t-1) bytes/bw for every t > 1 of the profile (DESIGN.md §3 reading)."""
    from oracle import simulator as sim
    spec, m, prof, d, cl = _setup("G", "opt-66b", 8)
    P, *_ = _c_objects(L, spec, prof, d, cl, tmp_path)
    alpha, bw = 12e-6, 450e9
    P.comm_model(alpha, bw)
    path = str(tmp_path / "cm.txt")
    P.save(path)
    Q = sim.Profile.loads(open(path).read())
    xs = Q.pp_sync.x
    assert xs[0] == 1024.0 and xs[-1] == 64.0 * 2 ** 30
    for x, t in zip(xs, Q.pp_sync.t):
        assert t == alpha + x / bw
    for tp in prof.tps:
        if tp > 1:
            for x, t in zip(Q.tp_sync[tp].x, Q.tp_sync[tp].t):
                assert t == alpha + (tp - 1) * x / bw
    with pytest.raises(L.ExgError):
        P.comm_model(alpha, 0.0)


def test_in_runner_baseline_picks(L, tmp_path):
    """bench.py's NEXT-4 legs: the FT static batch is the simulated
    max-throughput B within the bound (checked against a brute-force scan of
    the oracle simulator), and the ORCA-style schedule (Algorithm 1 with
    N_D^max = 1) admits every iteration."""
    import bench
    from oracle import simulator as sim
    spec, m, prof, d, cl = _setup()
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    S = sim.Simulator(prof, m, cl, d.pmf_in, d.pmf_out, d.target_len)
    lats = [S.simulate_static(B) for B in (1, 8, 64)]
    orca = 0
    for L_b in [e.latency_s * 1.01 for e in lats if e.feasible]:
        B, e = bench.static_pick(L, P, mspec, ccl, pin, pout, d.target_len, L_b)
        brute = [(S.simulate_static(b).thrput_tok_s, -b) for b in range(1, 1025)
                 if S.simulate_static(b).feasible and S.simulate_static(b).latency_s <= L_b]
        assert (e.thrput_tok_s, -B) == max(brute)
        assert e.latency_s <= L_b
        try:
            s, _ = L.schedule_find(P, mspec, ccl, pin, pout, d.target_len, L_b, L.EXG_RRA,
                                   L.search_opts(n_d_max=1, b_e_max=64))
        except L.ExgError:      # iteration-level admission can miss a tight bound
            continue
        assert s.n_d == 1
        orca += 1
    assert orca >= 1
    assert bench.static_pick(L, P, mspec, ccl, pin, pout, d.target_len, 1e-9) is None


@pytest.mark.parametrize("n_gpus,t,c", [(1, 1, 0), (4, 1, 0), (8, 2, 4), (8, 4, 8)])
def test_schedule_memory(L, tmp_path, n_gpus, t, c):
    """Memory-overhead accounting: C++ bit-identical to
    the oracle; pinned to closed forms -- summed over GPUs the model bytes
    are L x layer (x 2 for WAA's two sides) + the embeddings on every GPU of
    the first / last stage and the KV bytes are rows x ctx x L x (2 H dh 2 B); a
    schedule is memory-feasible exactly when every GPU's model + KV +
    workspace fits (mem_ok).  Embeddings are replicated on each GPU of a
    TP end stage."""
    from oracle import simulator as sim
    spec, m, prof, d, cl = _setup("G", "opt-66b", n_gpus)
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    S = sim.Simulator(prof, m, cl, d.pmf_in, d.pmf_out, d.target_len)
    kvb = 2 * spec.n_heads * spec.d_head * 2
    Lyr = S.n_layers
    cases = []
    for b_e, n_d in [(8, 10), (3, 480)]:
        s_o = S.rra_schedule(b_e, n_d, t, c)
        s_c = L.rra_schedule(b_e, 0, n_d)
        s_c.tp_degree, s_c.tp_gpus = t, c
        L.schedule_resolve(P, mspec, ccl, pin, pout, s_c)
        cases.append((s_o, s_c, s_o.b_d, S.max_in + S.max_out, None))
    if n_gpus > 1:
        for b_e, M in [(4, 3), (8, 8)]:
            s_o = S.waa_schedule(b_e, M, 1, 0)
            s_c = L.exg_schedule()
            s_c.strategy, s_c.b_e = 2, b_e
            L.schedule_resolve(P, mspec, ccl, pin, pout, s_c, M)
            cases.append((s_o, s_c, None, None, s_o))
    st_c = L.static_schedule(16)
    st_o = sim.Schedule(sim.STATIC, 16, 16, 0, 0, 1, 0, 0, [])
    cases.append((st_o, st_c, 16, S.max_in + S.max_out, None))
    for s_o, s_c, rows, ctx, waa in cases:
        w_o, kv_o = S.memory(s_o)
        w_c, kv_c = L.schedule_memory(P, mspec, ccl, pin, pout, s_c)
        assert (w_c, kv_c) == (w_o, kv_o)
        stages = s_o.stages if s_o.strategy != sim.STATIC else sim.stage_layout(n_gpus, 1, 0, Lyr)
        def end_gpus(side):   # the embeddings sit, replicated, on every GPU of a side's first / last stage
            return side[0][1] if len(side) == 1 else side[0][1] + side[-1][1]

        if waa is None:
            ends = end_gpus(stages)
            assert sum(w_o) == pytest.approx(Lyr * S.layer_bytes() + ends * S.emb_bytes(), rel=1e-12)
            assert sum(kv_o) == pytest.approx(rows * ctx * Lyr * kvb, rel=1e-12)
            ok = S.mem_ok(stages, rows, ctx)
        else:
            enc = [x for x in waa.stages if x[0] < waa.n_enc_gpus]
            dec = [x for x in waa.stages if x[0] >= waa.n_enc_gpus]
            ends = end_gpus(enc) + end_gpus(dec)
            assert sum(w_o) == pytest.approx(2 * Lyr * S.layer_bytes() + ends * S.emb_bytes(), rel=1e-12)
            assert sum(kv_o) == pytest.approx((waa.b_e * S.max_in + waa.b_d * (S.max_in + S.max_out)) * Lyr * kvb,
                                              rel=1e-12)
            ok = S.mem_ok(enc, waa.b_e, S.max_in) and S.mem_ok(dec, waa.b_d, S.max_in + S.max_out)
        fits = all(w + k + cl.workspace_bytes <= cl.mem_per_gpu_bytes for w, k in zip(w_o, kv_o) if w > 0)
        assert fits == ok


@pytest.mark.parametrize("n_gpus", [2, 4])
def test_schedule_find_bit_identical_on_exhaustive_pin_problems(L, tmp_path, n_gpus):
    """The small problems on which tests/test_oracle_pins.py pins the
    oracle's schedule_find to the exhaustive optimum: the C++ planner returns
    the same schedule, estimate and evaluation count (S15)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_oracle_pins import _small_problem
    from oracle import bnb
    from workload import MODELS
    S = _small_problem(n_gpus)
    path = str(tmp_path / "p.txt")
    S.p.save(path)
    P = L.Profile.load(path)
    spec = MODELS["opt-13b"]
    import dataclasses
    spec = dataclasses.replace(spec, n_dec_layers=S.m.n_dec_layers, n_heads=S.m.n_heads)
    mspec = L.model_spec(spec, 1)
    ccl = L.cluster_spec(S.cl.n_gpus, S.cl.mem_per_gpu_bytes, S.cl.workspace_bytes)
    pin, pout = L.Pmf(S.pmf_in), L.Pmf(S.pmf_out)
    opts = bnb.SearchOpts(eps_t_frac=0.0, eps_l_frac=0.0, b_e_max=12, m_max=4)
    copts = L.search_opts(eps_t=0.0, eps_l=0.0, b_e_max=12, m_max=4)
    for L_b in (0.005, 0.0103, 0.02, 0.05, math.inf):
        f = bnb.schedule_find(S, L_b, 7, opts)
        if f is None:
            with pytest.raises(L.ExgError):
                L.schedule_find(P, mspec, ccl, pin, pout, S.target_len, L_b, 7, copts)
            continue
        s, est = L.schedule_find(P, mspec, ccl, pin, pout, S.target_len, L_b, 7, copts)
        assert (s.strategy, s.b_e, s.b_d, s.b_m, s.n_d, s.tp_degree, s.tp_gpus, s.n_enc_gpus) == (
            f.schedule.strategy, f.schedule.b_e, f.schedule.b_d, f.schedule.b_m, f.schedule.n_d,
            f.schedule.tp_degree, f.schedule.tp_gpus, f.schedule.n_enc_gpus)
        assert est.thrput_seq_s == f.estimate.thrput_seq_s and est.latency_s == f.estimate.latency_s
        assert est.perf_evals == f.evals


def test_dtype_contract_without_gpu(L):
    """exg_create validates the dtype before touching a device: an unknown
    dtype, or EXG_FP32 outside the fp32 path's scope (encoder-decoder model,
    multi-GPU context), returns EXG_E_INPUT -- never a silent bf16 run
    (ADVICE r1)."""
    import ctypes as C
    from workload import MODELS
    for spec_name, dtype, ngpu in (("tiny", 7, 1), ("tiny-t5", 1, 1), ("tiny", 1, 2)):
        ms = L.model_spec(MODELS[spec_name], 1, dtype)
        h = C.c_void_p()
        st = L.lib().exg_create(C.byref(ms), C.byref(L.cluster_spec(ngpu)), 0, 0, 1, None, C.byref(h))
        assert st == L.EXG_E_INPUT, (spec_name, dtype, ngpu, st)


def test_profile_stage_time_matches_simulator_lookups(L, tmp_path):
    """exg_profile_stage_time = n_layers x (attention + rest) (+ head for a
    decode iteration), the XSimulator's per-layer lookups (oracle)."""
    from oracle import simulator as sim
    spec, m, prof, d, cl = _setup()
    P, *_ = _c_objects(L, spec, prof, d, cl, tmp_path)
    for rows, work in ((4.0, 1000.0), (37.0, 9000.5), (200.0, 51000.0)):
        enc = P.stage_time(0, rows, work, 40)
        ref = 40 * (sim.interp2(prof.attn[("enc", 1)], rows, work / rows) +
                    sim.interp1(prof.rest[("enc", 1)].x, prof.rest[("enc", 1)].t, work))
        assert enc == pytest.approx(ref, rel=1e-12)
        dec = P.stage_time(1, rows, work, 40)
        ref = 40 * (sim.interp2(prof.attn[("dec", 1)], rows, work / rows) +
                    sim.interp1(prof.rest[("dec", 1)].x, prof.rest[("dec", 1)].t, rows)) + \
            sim.interp1(prof.head.x, prof.head.t, rows)
        assert dec == pytest.approx(ref, rel=1e-12)
    with pytest.raises(L.ExgError):
        P.stage_time(2, 1.0, 1.0, 1)


# ------------------------------------------------------ paged KV (NEXT-2) --
def test_paged_kv_context_pins():
    """The paged memory model's per-row context (oracle kv_ctx_dec, DESIGN.md
    reading of PAPER.md:545) against (a) the row-iteration average of live
    keys evaluated from its definition by brute force over the two PMFs
    (sum_n sum_S p(n) p(S) sum_{u=1..S} (n - 1 + u) / E[S]) and (b) a
    discrete-event simulation of a full decode batch with refill (every
    finished row replaced at once), whose time-average of live keys per row
    converges to the same value (renewal-reward)."""
    from oracle import simulator as sim
    from workload import MODELS, task_dists
    d = task_dists("G")
    m = sim.SimModel.from_spec(MODELS["opt-66b"])
    P = 64
    S = sim.Simulator(None, m, sim.SimCluster(1, 180e9, 4e9, kv_page=P), d.pmf_in, d.pmf_out, d.target_len)
    pin, pout = np.asarray(d.pmf_in), np.asarray(d.pmf_out)
    num = den = 0.0
    for n in range(1, len(pin) + 1):
        if pin[n - 1] == 0:
            continue
        for So in range(1, len(pout) + 1):
            w = pin[n - 1] * pout[So - 1]
            num += w * sum(n - 1 + u for u in range(1, So + 1))
    for So in range(1, len(pout) + 1):
        den += pout[So - 1] * So
    live = num / den
    assert S.kv_ctx_dec == pytest.approx(live + 1.5 * P, rel=1e-12)
    # (b) event simulation: 64 rows, 4000 iterations, lengths drawn from the PMFs
    rng = np.random.default_rng(7)
    cin, cout = np.cumsum(pin), np.cumsum(pout)
    draw = lambda c: int(np.searchsorted(c, rng.random() * c[-1])) + 1
    rows = [[draw(cin), draw(cout), 1] for _ in range(64)]
    tot = cnt = 0
    for it in range(4000):
        for r in rows:
            if it >= 1000:
                tot += r[0] - 1 + r[2]
                cnt += 1
            r[2] += 1
            if r[2] > r[1]:
                r[:] = [draw(cin), draw(cout), 1]
    assert tot / cnt == pytest.approx(live, rel=0.02)
    # slots and T5 keep max_in + max_out
    S0 = sim.Simulator(None, m, sim.SimCluster(1, 180e9, 4e9), d.pmf_in, d.pmf_out, d.target_len)
    assert S0.kv_ctx_dec == len(pin) + len(pout)


@pytest.mark.parametrize("task,model,n_gpus,mask", [("G", "opt-66b", 1, 1), ("G", "opt-66b", 4, 7),
                                                    ("C2", "gpt3-175b", 8, 3)])
def test_paged_schedule_find_bit_identical(L, tmp_path, task, model, n_gpus, mask):
    """C++ planner == oracle with the paged memory model, and paging admits
    a larger decode batch where slots are memory-bound."""
    from oracle import bnb, simulator as sim
    spec, m, prof, d, cl = _setup(task, model, n_gpus)
    cl.kv_page = 64
    P, mspec, ccl, pin, pout = _c_objects(L, spec, prof, d, cl, tmp_path)
    S = sim.Simulator(prof, m, cl, d.pmf_in, d.pmf_out, d.target_len)
    opts = bnb.SearchOpts(b_e_max=48, m_max=6)
    copts = L.search_opts(b_e_max=48, m_max=6)
    for L_b in (1.0, 3.0, math.inf):
        f = bnb.schedule_find(S, L_b, mask, opts)
        if f is None:
            with pytest.raises(L.ExgError):
                L.schedule_find(P, mspec, ccl, pin, pout, d.target_len, L_b, mask, copts)
            continue
        s, est = L.schedule_find(P, mspec, ccl, pin, pout, d.target_len, L_b, mask, copts)
        assert (s.strategy, s.b_e, s.b_d, s.b_m, s.n_d, s.tp_degree, s.tp_gpus, s.n_enc_gpus) == (
            f.schedule.strategy, f.schedule.b_e, f.schedule.b_d, f.schedule.b_m, f.schedule.n_d,
            f.schedule.tp_degree, f.schedule.tp_gpus, f.schedule.n_enc_gpus)
        assert est.thrput_seq_s == f.estimate.thrput_seq_s and est.latency_s == f.estimate.latency_s
        w_c, kv_c = L.schedule_memory(P, mspec, ccl, pin, pout, s)
        assert (w_c, kv_c) == S.memory(f.schedule)
    if n_gpus == 1:
        # one 180 GB GPU under OPT-66B: slots cap the decode batch, pages do not
        S0 = sim.Simulator(prof, m, sim.SimCluster(1, cl.mem_per_gpu_bytes, cl.workspace_bytes), d.pmf_in,
                           d.pmf_out, d.target_len)
        b_slots = max(b for b in range(1, 400) if S0.mem_ok(S0.rra_schedule(1, 1, 1, 0).stages, b,
                                                               S0.kv_ctx_dec))
        b_paged = max(b for b in range(1, 400) if S.mem_ok(S.rra_schedule(1, 1, 1, 0).stages, b, S.kv_ctx_dec))
        assert b_paged > 2 * b_slots


@pytest.mark.parametrize("model,task", [("opt-13b", "S"), ("t5-11b", "T")])
def test_decode_context_pin(model, task):
    """The simulator's decode-attention context (ctx_mean, DESIGN.md reading):
    the keys a row holds, averaged over decode row-iterations -- brute force
    over the two PMFs from the definition (decoder-only: n - 1 + u keys at
    decode iteration u = 1..S; T5: n cross + u self keys), and a renewal
    check: a refilled batch's time-average converges to it."""
    from oracle import simulator as sim
    from workload import MODELS, task_dists
    d = task_dists(task)
    m = sim.SimModel.from_spec(MODELS[model])
    S = sim.Simulator(None, m, sim.SimCluster(1, 180e9, 4e9), d.pmf_in, d.pmf_out, d.target_len)
    pin, pout = np.asarray(d.pmf_in), np.asarray(d.pmf_out)
    off = 0 if model.startswith("t5") else -1
    num = den = 0.0
    for n in range(1, len(pin) + 1):
        for So in range(1, len(pout) + 1):
            w = pin[n - 1] * pout[So - 1]
            if w:
                num += w * sum(n + off + u for u in range(1, So + 1))
                den += w * So
    assert S.ctx_mean == pytest.approx(num / den, rel=1e-12)
    rng = np.random.default_rng(11)
    cin, cout = np.cumsum(pin), np.cumsum(pout)
    draw = lambda c: int(np.searchsorted(c, rng.random() * c[-1])) + 1
    rows = [[draw(cin), draw(cout), 1] for _ in range(64)]
    tot = cnt = 0
    for it in range(3000):
        for r in rows:
            if it >= 600:
                tot += r[0] + off + r[2]
                cnt += 1
            r[2] += 1
            if r[2] > r[1]:
                r[:] = [draw(cin), draw(cout), 1]
    assert tot / cnt == pytest.approx(S.ctx_mean, rel=0.02)
