"""Paged KV cache ("the addition of
vLLM's paging mechanism can further enhance WAA's performance") through
exg_run, on a decoder-only model with 128-wide heads (tcgen05 FMHA, 64-key
page halves) and 512 positions:

* paged without memory pressure is bit-identical to the slot cache (same
  arithmetic, pages shuffled by the allocator);
* under memory pressure rows are preempted and recomputed (re-encoded with
  their generated tokens appended): ids equal oracle mode (iii) free-running
  (near ties reported, parity.py), logits within 2e-2 -- the recomputed K/V
  come from the prefill GEMM instead of the decode GEMM, another valid
  evaluation of the same T4 rounding points;
* out-of-scope requests are rejected (EXG_E_INPUT).
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
    from workload import ModelSpec, make_requests, uniform_pmf
    spec = ModelSpec(name="paged-opt", arch="opt", n_enc_layers=0, n_dec_layers=2, d_model=256, n_heads=2,
                     d_head=128, d_ff=512, vocab=512, max_pos=512)
    seed = 0xE6E0_00A1
    reqs = make_requests(24, uniform_pmf(20, 200), uniform_pmf(10, 120), spec.vocab, 0xE6E1_00A1)
    ctx = X.Context(spec, seed)
    W = T.Weights(spec, seed)
    return X, T, spec, W, reqs, ctx


@pytest.fixture(scope="module")
def slots_run(setup):
    X, T, spec, W, reqs, ctx = setup
    return ctx.run(X.rra_schedule(4, 12, 4), reqs, dump=range(len(reqs)))


@pytest.mark.parametrize("P", [64, 128, 512])
def test_paged_without_pressure_is_bit_identical(setup, slots_run, P):
    X, T, spec, W, reqs, ctx = setup
    toks, _, st, lg = ctx.run(X.rra_schedule(4, 12, 4), reqs, dump=range(len(reqs)), kv_page=P)
    assert st["kv_preemptions"] == 0 and st["kv_pages_peak"] > 0
    assert toks == slots_run[0]
    for r in range(len(reqs)):
        assert np.array_equal(lg[r], slots_run[3][r]), r


def test_no_preemption_when_n_d_at_most_page(setup):
    """The admission reserve (one free page per active row) covers the
    growth of N_D <= P decode iterations: no preemption, even on a pool that
    throttles admission."""
    X, T, spec, W, reqs, ctx = setup
    _, _, st, _ = ctx.run(X.rra_schedule(4, 12, 4), reqs, kv_page=64, kv_pages=16)
    assert st["kv_preemptions"] == 0 and st["kv_pages_peak"] <= 16


@pytest.fixture(scope="module")
def long_reqs(setup):
    """Long outputs (100..300 tokens) on short inputs: rows outgrow a small
    pool between admissions."""
    X, T, spec, W, reqs, ctx = setup
    from workload import make_requests, uniform_pmf
    lr = make_requests(24, uniform_pmf(20, 100), uniform_pmf(100, 300), spec.vocab, 0xE6E1_00A2)
    ora = T.greedy_kv(W, lr, "bf16", record_logits=True)
    base = ctx.run(X.rra_schedule(8, 12, 200), lr, dump=range(len(lr)))
    return lr, ora, base


@pytest.mark.parametrize("P,pages", [(64, 16), (128, 8)])
def test_paged_preemption_matches_oracle(setup, long_reqs, P, pages):
    """N_D = 200 > P: rows cross several pages between admissions, the pool
    runs dry and the latest-admitted rows are preempted, re-encoded with their
    generated tokens and continued."""
    X, T, spec, W, reqs, ctx = setup
    lr, ora, base = long_reqs
    toks, lat, st, lg = ctx.run(X.rra_schedule(8, 12, 200), lr, dump=range(len(lr)), kv_page=P, kv_pages=pages)
    assert st["kv_preemptions"] > 0, st
    assert st["kv_pages_peak"] <= pages
    assert st["out_tokens"] == sum(q.output_len for q in lr) and np.all(lat > 0)
    compare_free_running("paged-P%d" % P, toks, lg, ora, TOL, decoder_only_tf(W, lr), max_near_ties=2)
    # requests never preempted are bitwise the slot run's (T13)
    same = sum(np.array_equal(lg[r], base[3][r]) for r in range(len(lr)))
    assert same >= 1


def test_paged_with_dynamic_adjustment(setup, slots_run):
    X, T, spec, W, reqs, ctx = setup
    toks, _, st, lg = ctx.run(X.rra_schedule(4, 12, 4), reqs, dump=range(len(reqs)), kv_page=64,
                              dyn_threshold=0.1)
    assert toks == slots_run[0]
    for r in range(len(reqs)):
        assert np.array_equal(lg[r], slots_run[3][r]), r


def test_paged_rejections(setup):
    X, T, spec, W, reqs, ctx = setup
    for kw in ({"kv_page": 96}, {"kv_page": 1024}, {"kv_page": 64, "kv_pages": 3}):
        with pytest.raises(X.ExgError) as ei:
            ctx.run(X.rra_schedule(4, 12, 4), reqs[:4], **kw)
        assert ei.value.status == 1, kw
    s = X.rra_schedule(4, 12, 4)
    s.strategy = 8   # EXG_STATIC: the FT baseline keeps slots
    with pytest.raises(X.ExgError) as ei:
        ctx.run(s, reqs[:4], kv_page=64)
    assert ei.value.status == 1


# ----------------------------------------------- paged KV under WAA (multi) --
# WAA's decoder GPUs page their KV; a row that finds no free page swaps the
# latest-admitted row's pages to pinned host memory and back (swap
# preemption), so paged WAA is bit-identical to slot WAA -- with or without
# memory pressure, across decoder pipeline stages, TP ranks and rank threads.
WAA_LAYOUTS = {
    "enc1_dec1": (4, 12, 0, 1, [(0, 1, 0, 2), (1, 1, 0, 2)], 1, 0),
    "dec_pp2_mb2": (4, 12, 6, 1, [(0, 1, 0, 2), (1, 1, 0, 1), (2, 1, 1, 2)], 1, 0),
    "dec_tp2": (4, 12, 6, 1, [(0, 1, 0, 2), (1, 2, 0, 2)], 2, 2),
}


@pytest.fixture(scope="module")
def multi(setup):
    X, T, spec, W, reqs, ctx = setup
    return X.Context(spec, 0xE6E0_00A1, cluster=X.cluster_spec(8))


@pytest.mark.parametrize("name", list(WAA_LAYOUTS))
def test_waa_paged_bit_identical(setup, long_reqs, multi, name):
    X, T, spec, W, reqs, ctx = setup
    from paper_2404_07947_b200 import _lib as L
    lr, ora, base = long_reqs
    b_e, b_d, b_m, n_enc, layout, t, c = WAA_LAYOUTS[name]
    s = L.make_schedule(X.EXG_WAA_C, b_e, b_d, layout, b_m=b_m, n_enc_gpus=n_enc, tp_degree=t, tp_gpus=c)
    ref_t, _, _, ref_l = multi.run(s, lr, dump=range(len(lr)))
    if t == 1:   # no TP: WAA is bit-identical to the one-GPU run too
        assert ref_t == base[0]
    else:
        compare_free_running("waa-" + name, ref_t, ref_l, ora, TOL, decoder_only_tf(W, lr), max_near_ties=2)
    for pages, swaps in ((0, False), (16, True)):
        toks, lat, st, lg = multi.run(s, lr, dump=range(len(lr)), kv_page=64, kv_pages=pages)
        assert (st["kv_preemptions"] > 0) == swaps, (pages, st["kv_preemptions"])
        if pages:
            assert st["kv_pages_peak"] <= pages
        assert toks == ref_t
        for r in range(len(lr)):
            assert np.array_equal(lg[r], ref_l[r]), (name, pages, r)


def test_waa_paged_rank_threads_bit_identical(setup, long_reqs):
    """Two rank threads (device-copy transport), paged decoder with swaps:
    the same decisions on every rank, results equal to the one-rank run."""
    X, T, spec, W, reqs, ctx = setup
    from paper_2404_07947_b200 import _lib as L
    lr, ora, base = long_reqs
    s = L.make_schedule(X.EXG_WAA_C, 4, 12, [(0, 1, 0, 2), (1, 1, 0, 1), (2, 1, 1, 2)], b_m=6, n_enc_gpus=1)
    group = X.local_group(spec, 0xE6E0_00A1, 2, X.cluster_spec(8))
    res = X.run_group(group, s, lr, dump=range(len(lr)), kv_page=64, kv_pages=16)
    toks, _, st, _ = res[0]
    assert st["kv_preemptions"] > 0
    assert toks == base[0]
    head_rank = max(range(2), key=lambda q: np.count_nonzero(res[q][3][0]))   # logits live on the LM head's rank
    for r in range(len(lr)):
        assert np.array_equal(res[head_rank][3][r], base[3][r]), r
    for g in group:
        g.close()


# ----------------------------------------- paged KV under multi-GPU RRA --
RRA_LAYOUTS = {
    "pp2": ([(0, 1, 0, 1), (1, 1, 1, 2)], 1, 0),
    "tp2": ([(0, 2, 0, 2)], 2, 2),
    "tp2_then_single": ([(0, 2, 0, 1), (2, 1, 1, 2)], 2, 2),
}


@pytest.mark.parametrize("name", list(RRA_LAYOUTS))
def test_rra_pipeline_paged_bit_identical(setup, long_reqs, multi, name):
    """RRA over pipeline stages / TP ranks with every stage paged (same page
    ids on every stage; swap preemption under pressure): bit-identical to the
    slot run of the same layout."""
    X, T, spec, W, reqs, ctx = setup
    from paper_2404_07947_b200 import _lib as L
    lr, ora, base = long_reqs
    layout, t, c = RRA_LAYOUTS[name]
    s = L.make_schedule(X.EXG_RRA, 8, 12, layout, n_d=200, tp_degree=t, tp_gpus=c)
    ref_t, _, _, ref_l = multi.run(s, lr, dump=range(len(lr)))
    if t == 1:
        assert ref_t == base[0]
    for pages, swaps in ((0, False), (16, True)):
        toks, _, st, lg = multi.run(s, lr, dump=range(len(lr)), kv_page=64, kv_pages=pages)
        assert (st["kv_preemptions"] > 0) == swaps, (pages, st["kv_preemptions"])
        assert toks == ref_t
        for r in range(len(lr)):
            assert np.array_equal(lg[r], ref_l[r]), (name, pages, r)


def test_rra_pipeline_paged_rank_threads(setup, long_reqs):
    X, T, spec, W, reqs, ctx = setup
    from paper_2404_07947_b200 import _lib as L
    lr, ora, base = long_reqs
    s = L.make_schedule(X.EXG_RRA, 8, 12, [(0, 1, 0, 1), (1, 1, 1, 2)], n_d=200)
    group = X.local_group(spec, 0xE6E0_00A1, 2, X.cluster_spec(8))
    res = X.run_group(group, s, lr, dump=range(len(lr)), kv_page=64, kv_pages=16)
    toks, _, st, _ = res[0]
    assert st["kv_preemptions"] > 0 and toks == base[0]
    head_rank = max(range(2), key=lambda q: np.count_nonzero(res[q][3][0]))
    for r in range(len(lr)):
        assert np.array_equal(res[head_rank][3][r], base[3][r]), r
    for g in group:
        g.close()
