"""Multi-GPU layouts of the method on one B200 (every GPU of a layout
emulated by its own Engine holding exactly that GPU's weight shard and KV):

* RRA over pipeline stages (PP) with P micro-batches;
* partial tensor parallelism (TP all-reduce of fp32
  partials in rank order, T4(i));
* WAA: encoder GPU(s) / decoder GPU(s), KV handoff layer by
  layer to the owning decoder stage and TP rank, rows merged at iteration
  boundaries, decoder micro-batches.

Parity bar: greedy ids equal to the oracle's
bf16-emulating decode (near-ties reported with their margin), logits within
2e-2; layouts without TP are bit-identical to the single-GPU run (same
per-row arithmetic, bit-exact transfers)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2404_07947_b200 as X
    from paper_2404_07947_b200 import _lib
    from oracle import transformer as T
    from workload import MODELS, config1_requests, weight_seed
    spec = MODELS["tiny"]
    seed = weight_seed(1)
    reqs = config1_requests()
    single = X.Context(spec, seed)
    multi = X.Context(spec, seed, cluster=X.cluster_spec(8))
    base_t, _, _, base_l = single.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
    ora = T.greedy_kv(T.Weights(spec, seed), reqs, "bf16", record_logits=True)
    return X, _lib, reqs, single, multi, base_t, base_l, ora


def _check_vs_oracle(reqs, toks, logits, ora):
    worst = 0.0
    for r, q in enumerate(reqs):
        for t in range(q.output_len):
            if toks[r][t] != ora.tokens[r][t]:
                assert ora.margins[r][t] <= 2 * TOL, "hard mismatch req %d step %d" % (r, t)
                pytest.fail("near-tie divergence req %d step %d (margin %.3g)" % (r, t, ora.margins[r][t]))
            worst = max(worst, float(np.abs(logits[r][t] - ora.logits[r][t]).max()))
    assert worst <= TOL, worst


PP_LAYOUTS = {
    "pp2": [(0, 1, 0, 1), (1, 1, 1, 2)],
}
TP_LAYOUTS = {
    "tp2_then_single": [(0, 2, 0, 1), (2, 1, 1, 2)],     # partial TP: c = 2 GPUs at the front, t = 2
    "tp4": [(0, 4, 0, 2)],
    "single_then_tp2": [(0, 1, 0, 1), (1, 2, 1, 2)],
}


@pytest.mark.parametrize("name", list(PP_LAYOUTS))
def test_rra_pipeline_bit_identical_to_single_gpu(env, name):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    s = L.make_schedule(X.EXG_RRA, 4, 8, PP_LAYOUTS[name], n_d=6)
    toks, lat, st, lg = multi.run(s, reqs, dump=range(len(reqs)))
    assert toks == base_t
    for r in range(len(reqs)):
        assert np.array_equal(lg[r], base_l[r]), r
    assert st["out_tokens"] == sum(q.output_len for q in reqs) and np.all(lat > 0)


@pytest.mark.parametrize("name", list(TP_LAYOUTS))
def test_rra_partial_tp_matches_oracle(env, name):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    s = L.make_schedule(X.EXG_RRA, 4, 8, TP_LAYOUTS[name], n_d=6, tp_degree=max(g[1] for g in TP_LAYOUTS[name]))
    toks, lat, st, lg = multi.run(s, reqs, dump=range(len(reqs)))
    _check_vs_oracle(reqs, toks, lg, ora)


@pytest.mark.parametrize("b_e,b_d,b_m,n_enc,layout", [
    (2, 8, 0, 1, [(0, 1, 0, 2), (1, 1, 0, 2)]),                     # 1 encoder GPU + 1 decoder GPU
    (3, 8, 4, 1, [(0, 1, 0, 2), (1, 1, 0, 1), (2, 1, 1, 2)]),      # decoder pipeline, 2 micro-batches
    (1, 5, 2, 2, [(0, 1, 0, 1), (1, 1, 1, 2), (2, 1, 0, 2)]),      # encoder pipeline of 2
])
def test_waa_bit_identical_to_single_gpu(env, b_e, b_d, b_m, n_enc, layout):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    s = L.make_schedule(X.EXG_WAA_C, b_e, b_d, layout, b_m=b_m, n_enc_gpus=n_enc)
    toks, lat, st, lg = multi.run(s, reqs, dump=range(len(reqs)))
    assert toks == base_t
    for r in range(len(reqs)):
        assert np.array_equal(lg[r], base_l[r]), r


def test_waa_with_decoder_tp_matches_oracle(env):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    layout = [(0, 1, 0, 2), (1, 2, 0, 1), (3, 1, 1, 2)]   # enc GPU 0; dec: TP-2 stage + single stage
    s = L.make_schedule(X.EXG_WAA_C, 2, 8, layout, b_m=4, n_enc_gpus=1, tp_degree=2, tp_gpus=2)
    toks, lat, st, lg = multi.run(s, reqs, dump=range(len(reqs)))
    _check_vs_oracle(reqs, toks, lg, ora)


def test_layout_validation(env):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    bad = L.make_schedule(X.EXG_RRA, 4, 8, [(0, 1, 0, 1)], n_d=6)          # misses layer 1
    with pytest.raises(X.ExgError) as ei:
        multi.run(bad, reqs)
    assert ei.value.status == 1
    too_many = L.make_schedule(X.EXG_RRA, 4, 8, [(0, 8, 0, 1), (8, 1, 1, 2)], n_d=6)
    with pytest.raises(X.ExgError):
        multi.run(too_many, reqs)


# ---------------------------------------------------------------------------
# multi-rank executor: `world` rank contexts (threads of this process on the
# one GPU, device-copy transport in place of NCCL), every GPU of the layout
# owned by rank g*world/G.  Same arithmetic in the same order as the
# single-rank run of the same layout => bit-identical ids and logits.
# ---------------------------------------------------------------------------
RANK_CASES = [
    # (name, strategy, b_e, b_d, b_m, n_enc, layout, tp_degree, world)
    ("pp2_w2", "rra", 4, 8, 0, 0, [(0, 1, 0, 1), (1, 1, 1, 2)], 1, 2),
    ("tp2_split_w2", "rra", 4, 8, 0, 0, [(0, 2, 0, 2)], 2, 2),
    ("tp2_then_single_w2", "rra", 4, 8, 0, 0, [(0, 2, 0, 1), (2, 1, 1, 2)], 2, 2),
    ("single_then_tp2_w3", "rra", 4, 8, 0, 0, [(0, 1, 0, 1), (1, 2, 1, 2)], 2, 3),
    ("waa_enc_dec_w2", "waa", 2, 8, 0, 1, [(0, 1, 0, 2), (1, 1, 0, 2)], 1, 2),
    ("waa_dec_pipeline_w2", "waa", 3, 8, 4, 1, [(0, 1, 0, 2), (1, 1, 0, 1), (2, 1, 1, 2)], 1, 2),
    ("waa_enc_pipeline_w3", "waa", 1, 5, 2, 2, [(0, 1, 0, 1), (1, 1, 1, 2), (2, 1, 0, 2)], 1, 3),
    ("waa_dec_tp_w4", "waa", 2, 8, 4, 1, [(0, 1, 0, 2), (1, 2, 0, 1), (3, 1, 1, 2)], 2, 4),
]


@pytest.mark.parametrize("case", RANK_CASES, ids=[c[0] for c in RANK_CASES])
def test_multi_rank_bit_identical_to_single_rank(env, case):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    name, strat, b_e, b_d, b_m, n_enc, layout, tp, world = case
    strategy = X.EXG_RRA if strat == "rra" else X.EXG_WAA_C
    tp_gpus = sum(g[1] for g in layout if g[1] > 1)
    s = L.make_schedule(strategy, b_e, b_d, layout, n_d=6, b_m=b_m, n_enc_gpus=n_enc, tp_degree=tp, tp_gpus=tp_gpus)
    ref_t, _, _, ref_l = multi.run(s, reqs, dump=range(len(reqs)))
    from workload import weight_seed
    group = X.local_group(multi.spec, weight_seed(1), world, X.cluster_spec(8))
    res = X.run_group(group, s, reqs, dump=range(len(reqs)))
    toks, lat, st, lg = res[0]
    assert toks == ref_t
    for r in range(len(reqs)):
        assert np.array_equal(lg[r], ref_l[r]) or not np.any(lg[r]), r   # logits live on the LM head's rank
    head_rank = max(range(world), key=lambda q: np.count_nonzero(res[q][3][0]))
    for r in range(len(reqs)):
        assert np.array_equal(res[head_rank][3][r], ref_l[r]), r
    assert st["out_tokens"] == sum(q.output_len for q in reqs)
    assert np.all(lat > 0) and st["wall_s"] >= lat.max()
    if tp == 1:
        assert toks == base_t
    for c in group:
        c.close()


def test_multi_rank_errors(env):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    from workload import weight_seed
    group = X.local_group(multi.spec, weight_seed(1), 3, X.cluster_spec(8))
    s = L.make_schedule(X.EXG_RRA, 4, 8, [(0, 1, 0, 1), (1, 1, 1, 2)], n_d=6)   # 2 GPUs < 3 ranks
    with pytest.raises(X.ExgError):
        X.run_group(group, s, reqs)
    for c in group:
        c.close()


# NCCL transport on one GPU: a one-rank communicator through which every
# exchange of the layout is sent to itself (ncclSend / ncclRecv in a group),
# bit-identical to the device-copy path
NCCL_CASES = [
    ("pp2", "rra", 4, 8, 0, 0, [(0, 1, 0, 1), (1, 1, 1, 2)], 1),
    ("tp2_then_single", "rra", 4, 8, 0, 0, [(0, 2, 0, 1), (2, 1, 1, 2)], 2),
    ("waa_dec_pipeline", "waa", 3, 8, 4, 1, [(0, 1, 0, 2), (1, 1, 0, 1), (2, 1, 1, 2)], 1),
    ("waa_dec_tp", "waa", 2, 8, 4, 1, [(0, 1, 0, 2), (1, 2, 0, 1), (3, 1, 1, 2)], 2),
]


@pytest.mark.parametrize("case", NCCL_CASES, ids=[c[0] for c in NCCL_CASES])
def test_nccl_loopback_bit_identical(env, case):
    X, L, reqs, single, multi, base_t, base_l, ora = env
    name, strat, b_e, b_d, b_m, n_enc, layout, tp = case
    strategy = X.EXG_RRA if strat == "rra" else X.EXG_WAA_C
    tp_gpus = sum(g[1] for g in layout if g[1] > 1)
    s = L.make_schedule(strategy, b_e, b_d, layout, n_d=6, b_m=b_m, n_enc_gpus=n_enc, tp_degree=tp, tp_gpus=tp_gpus)
    ref_t, _, _, ref_l = multi.run(s, reqs, dump=range(len(reqs)))
    from workload import weight_seed
    nc = X.nccl_loopback(multi.spec, weight_seed(1), X.cluster_spec(8))
    toks, lat, st, lg = nc.run(s, reqs, dump=range(len(reqs)))
    assert toks == ref_t
    for r in range(len(reqs)):
        assert np.array_equal(lg[r], ref_l[r]), r
    assert np.all(lat > 0)
    nc.close()


def test_profile_comm_tables_on_a_rank_group():
    """XProfiler's interconnect tables on a multi-rank context:
    every rank calls exg_profile_run (collective); tp_sync[t] for t <= world
    and pp_sync come back on the byte grid 1 KB .. 1 GB, positive and
    growing with the message; exg_profile_copy_comm merges them into a layer
    profile, which the simulator then reads (here over the thread-rank
    transport: device copies standing in for NVLink)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import threading
    import paper_2404_07947_b200 as X
    from oracle import simulator as sim
    from workload import MODELS, weight_seed
    spec = MODELS["tiny"]
    ctxs = X.local_group(spec, weight_seed(1), 4)
    res, err = [None] * 4, [None] * 4

    def go(r):
        try:
            res[r] = ctxs[r].profile([1], [1], [1], reps=2, tps=[1, 2, 4])
        except BaseException as e:  # noqa: BLE001
            err[r] = e
    th = [threading.Thread(target=go, args=(r,)) for r in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert all(e is None for e in err), err
    import tempfile, os
    with tempfile.TemporaryDirectory() as tmp:
        res[0].save(os.path.join(tmp, "c.txt"))
        P = sim.Profile.load(os.path.join(tmp, "c.txt"))
        assert set(P.tp_sync) == {2, 4}
        for t in (2, 4):
            ts = P.tp_sync[t].t
            assert P.tp_sync[t].x[0] == 1024.0 and P.tp_sync[t].x[-1] == float(1 << 30)
            assert all(v > 0 for v in ts) and ts[-1] > 10 * ts[0]
        # the thread-rank transport's hop has a ~40 us host-rendezvous floor, so
        # the table grows from it (1 KB) to the copy time of 1 GB
        assert all(v > 0 for v in P.pp_sync.t) and P.pp_sync.t[-1] > 3 * P.pp_sync.t[0]
        single = X.Context(spec, weight_seed(1))
        lay = single.profile([1, 4], [16, 48], [16, 64], reps=1, tps=[1, 2, 4])
        lay.copy_comm(res[0])
        lay.save(os.path.join(tmp, "m.txt"))
        M = sim.Profile.load(os.path.join(tmp, "m.txt"))
        assert M.tp_sync[2].t == P.tp_sync[2].t and M.pp_sync.t == P.pp_sync.t
        assert ("dec", 4) in M.rest
        single.close()
    for c in ctxs:
        c.close()


def test_waa_dynamic_adjustment_and_stage_variance(env):
    """NEXT-1 under WAA: the encoder batch follows the
    decode batch's drift and the token-sum window; results stay bit-identical
    (batch invariance, T13) and the run reports Table 9's single-stage
    statistics for the encoder and the decoder."""
    X, L, reqs, single, multi, base_t, base_l, ora = env
    from workload import make_requests, uniform_pmf
    many = make_requests(48, uniform_pmf(4, 40), uniform_pmf(1, 20), 512, 78)
    layout = [(0, 1, 0, 2), (1, 1, 0, 1), (2, 1, 1, 2)]
    s = L.make_schedule(X.EXG_WAA_C, 3, 12, layout, b_m=6, n_enc_gpus=1)
    a = multi.run(s, many, dump=range(len(many)))
    b = multi.run(s, many, dump=range(len(many)), dyn_threshold=0.1)
    assert a[0] == b[0]
    for r in range(len(many)):
        assert np.array_equal(a[3][r], b[3][r]), r
    for st in (a[2], b[2]):
        assert st["dec_stage_mean_s"] > 0 and st["enc_stage_mean_s"] > 0
        assert st["dec_stage_p99dev_s"] >= 0 and st["mean_encode_batch"] > 0 and st["tok_s_steady"] > 0
    assert a[2]["mean_encode_batch"] == pytest.approx(3.0, rel=0.05)
