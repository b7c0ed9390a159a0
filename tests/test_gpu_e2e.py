"""End-to-end parity of the CUDA runner (exg_run through the C-ABI) with the
oracle on config 1 (tiny model, RRA B_E=4, B_D=8, N_D=6; BASELINE.json
configs[0]) -- SURVEY.md §8(c) T4/T4a:

* greedy ids equal oracle mode (iii) (bf16-emulating KV loop), free-running;
  a mismatch at a step whose oracle top-2 margin exceeds 2*tol is a hard
  failure (tol = 2e-2);
* logits within max-abs 2e-2 of mode (iii) on every step;
* logits also compared with mode (ii) (fp64) teacher-forced on the run's own
  prefix;
* batch invariance (T13): every request run alone, and under another RRA
  schedule, gives bit-identical ids and logits.
"""
import numpy as np
import pytest

from parity import compare_free_running, decoder_only_tf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2404_07947_b200 as X
    from oracle import transformer as T
    from workload import MODELS, config1_requests, weight_seed
    spec = MODELS["tiny"]
    seed = weight_seed(1)
    reqs = config1_requests()
    ctx = X.Context(spec, seed)
    W = T.Weights(spec, seed)
    ora = T.greedy_kv(W, reqs, "bf16", record_logits=True)
    return X, T, spec, W, reqs, ctx, ora


def test_config1_ids_and_logits(setup):
    X, T, spec, W, reqs, ctx, ora = setup
    toks, lat, stats, logits = ctx.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
    # config 1's weight seed keeps every oracle margin >= 1e-3 (T4a fixture
    # choice), so no near tie is allowed here
    compare_free_running("config1", toks, logits, ora, TOL, decoder_only_tf(W, reqs), max_near_ties=0)
    assert stats["out_tokens"] == sum(q.output_len for q in reqs)
    assert stats["encode_phases"] >= 2 and stats["decode_iters"] >= max(q.output_len for q in reqs)
    assert np.all(lat > 0)


def test_config1_logits_vs_fp64_teacher_forced(setup):
    X, T, spec, W, reqs, ctx, ora = setup
    toks, _, _, logits = ctx.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
    worst = 0.0
    for r, q in enumerate(reqs):
        tf = T.teacher_forced_logits(W, q, toks[r], "fp64")
        for t in range(q.output_len):
            worst = max(worst, float(np.abs(logits[r][t] - tf[t]).max()))
    assert worst <= TOL, worst


def test_batch_invariance_across_schedules(setup):
    X, T, spec, W, reqs, ctx, ora = setup
    base_t, _, _, base_l = ctx.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
    for sched in (X.rra_schedule(1, 1, 1), X.rra_schedule(2, 3, 2), X.rra_schedule(8, 8, 24)):
        t2, _, _, l2 = ctx.run(sched, reqs, dump=range(len(reqs)))
        assert t2 == base_t
        for r in range(len(reqs)):
            assert np.array_equal(l2[r], base_l[r]), r
    for r in range(len(reqs)):
        t1, _, _, l1 = ctx.run(X.rra_schedule(1, 1, 3), [reqs[r]], dump=[0])
        assert t1[0] == base_t[r] and np.array_equal(l1[0], base_l[r])


def test_single_token_input_and_long_requests(setup):
    X, T, spec, W, reqs, ctx, ora = setup
    from workload import Request
    rng = np.random.default_rng(0)
    extra = [Request(np.array([5], np.int32), 1, 7),
             Request(rng.integers(0, 512, 40).astype(np.int32), 40, 24),
             Request(rng.integers(0, 512, 2).astype(np.int32), 2, 1)]
    o = T.greedy_kv(W, extra, "bf16", record_logits=True)
    toks, _, _, lg = ctx.run(X.rra_schedule(2, 3, 4), extra, dump=range(3))
    compare_free_running("edge-lengths", toks, lg, o, TOL, decoder_only_tf(W, extra), max_near_ties=1)


def test_input_errors(setup):
    X, T, spec, W, reqs, ctx, ora = setup
    from workload import Request
    with pytest.raises(X.ExgError) as ei:
        ctx.run(X.rra_schedule(1, 1, 1), [Request(np.array([600], np.int32), 1, 2)])
    assert ei.value.status == 1
    with pytest.raises(X.ExgError) as ei:
        ctx.run(X.rra_schedule(1, 1, 1), [Request(np.arange(60, dtype=np.int32), 60, 10)])
    assert ei.value.status == 1
    bad = X.rra_schedule(4, 2, 1)
    with pytest.raises(X.ExgError):
        ctx.run(bad, reqs)


def test_dynamic_workload_adjustment_keeps_results(setup):
    """the runtime B_E correction changes only which encode
    phase admits a request; per-request results are batch invariant (T13), so
    ids and logits are bit-identical to the plain schedule."""
    X, T, spec, W, reqs, ctx, ora = setup
    from workload import make_requests, uniform_pmf
    many = make_requests(40, uniform_pmf(4, 40), uniform_pmf(1, 20), spec.vocab, 77)
    a = ctx.run(X.rra_schedule(4, 10, 3), many, dump=range(len(many)))
    b = ctx.run(X.rra_schedule(4, 10, 3), many, dump=range(len(many)), dyn_threshold=0.1)
    assert a[0] == b[0]
    for r in range(len(many)):
        assert np.array_equal(a[3][r], b[3][r]), r
    st = b[2]
    assert st["mean_encode_batch"] > 0 and st["dec_stage_mean_s"] > 0 and st["dec_stage_p99dev_s"] >= 0
    assert a[2]["mean_encode_batch"] == pytest.approx(len(many) / a[2]["encode_phases"])


def test_profile_tp_shards(setup, tmp_path):
    """XProfiler over TP degrees: t > 1 times a one-layer shard
    of TP rank 0; every requested degree gets attention and rest tables."""
    X, T, spec, W, reqs, ctx, ora = setup
    from oracle import simulator as sim
    prof = ctx.profile([1, 4, 8], [16, 48], [16, 64, 256], reps=1, tps=[1, 2, 4])
    path = str(tmp_path / "p.txt")
    prof.comm_model(10e-6, 700e9)
    prof.save(path)
    P = sim.Profile.loads(open(path).read())
    assert P.tps == [1, 2, 4]
    for t in (1, 2, 4):
        for ph in ("enc", "dec"):
            assert np.all(np.array(P.attn[(ph, t)].t) > 0) and np.all(np.array(P.rest[(ph, t)].t) > 0)
    assert 2 in P.tp_sync and 4 in P.tp_sync and P.pp_sync is not None


def test_static_batch_baseline(setup):
    """FT-style static batch (EXG_STATIC; SURVEY.md §8(f)
    NEXT-4): finished rows keep being computed until the batch's longest
    output is done.  Per-request results are batch invariant (T13), so ids
    and logits are bit-identical to the RRA run; every request of a batch
    completes at the same iteration."""
    X, T, spec, W, reqs, ctx, ora = setup
    base_t, _, _, base_l = ctx.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
    for b in (1, 3, 8):
        toks, lat, st, lg = ctx.run(X.static_schedule(b), reqs, dump=range(len(reqs)))
        assert toks == base_t
        for r in range(len(reqs)):
            assert np.array_equal(lg[r], base_l[r]), (b, r)
        batches = [list(range(k, min(k + b, len(reqs)))) for k in range(0, len(reqs), b)]
        assert st["encode_phases"] == len(batches)
        assert st["decode_iters"] == sum(max(reqs[r].output_len for r in g) for g in batches)
        assert st["mean_decode_batch"] == pytest.approx(
            sum(len(g) * max(reqs[r].output_len for r in g) for g in batches) / st["decode_iters"])
        for g in batches:
            assert len({float(lat[r]) for r in g}) == 1, (b, g)
        assert np.all(lat > 0)
    # a finished row whose position runs past its slot / max_pos keeps being
    # computed (clamped inside its own slot) without touching its batch-mates
    from workload import Request
    rng = np.random.default_rng(1)
    two = [Request(rng.integers(0, 512, 60).astype(np.int32), 60, 4),
           Request(rng.integers(0, 512, 8).astype(np.int32), 8, 24)]
    ref_t, _, _, ref_l = ctx.run(X.rra_schedule(1, 1, 2), two, dump=range(2))
    toks, _, st, lg = ctx.run(X.static_schedule(2), two, dump=range(2))
    assert toks == ref_t and st["decode_iters"] == 24
    for r in range(2):
        assert np.array_equal(lg[r], ref_l[r]), r
    with pytest.raises(X.ExgError):
        ctx.run(X.static_schedule(0), reqs)


def test_long_context_split_merge():
    """Rows longer than one 512-key attention split: the
    decode attention's last split CTA merges the splits in-kernel; ids and
    logits are bit-identical to the separate combine kernel (diagnostics
    switch) and match the oracle's bf16-emulating KV loop."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2404_07947_b200 as X
    from oracle import transformer as T
    from workload import ModelSpec, Request
    spec = ModelSpec("long-ctx", "opt", 0, 2, 256, 2, 128, 1024, 512, 1100)
    seed = 0xE6E0_0077
    rng = np.random.default_rng(5)
    reqs = [Request(rng.integers(0, 512, n).astype(np.int32), n, s)
            for n, s in ((700, 6), (505, 12), (1030, 3), (40, 5))]
    ctx = X.Context(spec, seed)
    a = ctx.run(X.rra_schedule(2, 4, 4), reqs, dump=range(len(reqs)))
    X.lib().exg_diag_decode_merge(1)
    try:
        b = ctx.run(X.rra_schedule(2, 4, 4), reqs, dump=range(len(reqs)))
    finally:
        X.lib().exg_diag_decode_merge(0)
    assert a[0] == b[0]
    for r in range(len(reqs)):
        assert np.array_equal(a[3][r], b[3][r]), r
    Wl = T.Weights(spec, seed)
    ora = T.greedy_kv(Wl, reqs, "bf16", record_logits=True)
    compare_free_running("long-ctx", a[0], a[3], ora, TOL, decoder_only_tf(Wl, reqs), max_near_ties=1)
    ctx.close()


def test_dynamic_adjustment_narrow_inputs_stays_in_capacity(setup):
    """with every input the same length, the dynamic
    adjustment admits more than B_E rows (B_E' up to B_D); the encode tables
    and workspace are sized for that, the token sum never exceeds B_E x the
    longest input, and results stay bit-identical to the plain schedule."""
    X, T, spec, W, reqs, ctx, ora = setup
    from workload import make_requests, uniform_pmf
    same = make_requests(40, uniform_pmf(20, 20), uniform_pmf(1, 12), spec.vocab, 91)
    a = ctx.run(X.rra_schedule(4, 10, 3), same, dump=range(len(same)))
    b = ctx.run(X.rra_schedule(4, 10, 3), same, dump=range(len(same)), dyn_threshold=0.1)
    assert a[0] == b[0]
    for r in range(len(same)):
        assert np.array_equal(a[3][r], b[3][r]), r
    assert b[2]["encode_phases"] >= len(same) // 10


@pytest.mark.parametrize("n_req,b_d", [(24, 20), (160, 150)])
def test_deferred_stream_k_reduction_bit_identical(n_req, b_d):
    """Deferred stream-K reduction of the decode GEMMs (QKV segments summed
    in the attention kernel, O-projection / FFN2 segments in the following
    LayerNorm; gemm_tc.cuh) is the in-kernel fixup's arithmetic moved to the
    consumer: ids and logits bit-identical to the fixup path, on a model wide
    enough that every weight tile is split across CTAs (3-6 segments), at
    decode batches on the BN = 32 / 64 and BN = 256 token tiles."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2404_07947_b200 as X
    from workload import ModelSpec, make_requests, uniform_pmf
    spec = ModelSpec("defer-w2048", "opt", 0, 2, 2048, 16, 128, 8192, 4096, 512)
    reqs = make_requests(n_req, uniform_pmf(8, 64), uniform_pmf(2, 12), spec.vocab, 0xD3F)
    outs = []
    X.lib().exg_diag_chain(0)   # the per-kernel decode path carries the deferred reductions
    for mask in (0, 1, 2, 3):   # none / QKV / O-proj + FFN2 / all
        X.lib().exg_diag_deferred(mask)
        try:
            ctx = X.Context(spec, 0xE6E0_0D3F)
            outs.append(ctx.run(X.rra_schedule(min(n_req, b_d), b_d, 4), reqs, dump=range(len(reqs))))
            ctx.close()
        finally:
            X.lib().exg_diag_deferred(-1)
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        for r in range(len(reqs)):
            assert np.array_equal(o[3][r], outs[0][3][r]), r


@pytest.mark.parametrize("n_req,b_d,n_layers", [(24, 20, 3), (160, 150, 2), (9, 9, 1)])
def test_decode_chain_bit_identical(n_req, b_d, n_layers):
    """The decode GEMM chain (one persistent launch per layer for O-proj,
    LN2, FFN1, FFN2 and the next layer's LN1 + QKV; gemm_tc.cu) keeps every
    GEMM's stream-K cut, epilogue and fixup and the LayerNorm's arithmetic:
    ids and logits bit-identical to the separate launches, with split tiles
    (width 2048), every token tile class, 1-3 layers (chains with and
    without the next layer's QKV), repeated launches on the same counters."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2404_07947_b200 as X
    from workload import ModelSpec, make_requests, uniform_pmf
    spec = ModelSpec("chain-w2048", "gpt3", 0, n_layers, 2048, 16, 128, 8192, 4096, 512)
    reqs = make_requests(n_req, uniform_pmf(8, 64), uniform_pmf(2, 12), spec.vocab, 0xC4A1)
    outs = []
    for on in (0, 1):
        X.lib().exg_diag_chain(on)
        try:
            ctx = X.Context(spec, 0xE6E0_0C4A)
            outs.append(ctx.run(X.rra_schedule(min(n_req, b_d), b_d, 4), reqs, dump=range(len(reqs))))
            outs.append(ctx.run(X.rra_schedule(min(n_req, b_d), b_d, 4), reqs, dump=range(len(reqs))))
            ctx.close()
        finally:
            X.lib().exg_diag_chain(0)
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        for r in range(len(reqs)):
            assert np.array_equal(o[3][r], outs[0][3][r]), r
