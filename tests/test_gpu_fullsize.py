"""Parity at the bench's full sizes (config 2: OPT-13B, task S), in the launch
configuration bench.py times (tier rule ③):

* full width, sampled outputs: the first 2 of OPT-13B's 40 layers (identical
  weights: layer l is tensor slot 1001+l of the same seed) + embeddings + LM
  head run on the GPU with the bench's request recipe and its headline RRA
  control variables (B_E=31, B_D=77, N_D=16, 592-key slots); three sampled
  requests are recomputed one by one by the oracle (mode iii) over their
  first output steps (a step's logits depend only on the request's own
  prefix).  Tolerance at this width: two valid evaluations of
  the T4 rounding contract drift apart as the width grows (each fp32
  accumulation-order difference can flip a bf16 rounding), so the bar is
  calibrated per request by the oracle itself -- the distance between its
  fp64-accumulated and fp32-accumulated evaluations (measured ~0.02 max-abs,
  ~0.003 mean-abs at this width): GPU logits within max(2e-2, 2x that) max-abs
  and max(2e-3, 2x that) mean-abs; ids equal except at near ties (oracle
  top-2 margin within the bar, the GPU's token within it of the oracle's
  maximum), after which that request's prefixes differ;
* full depth, properties: all 40 layers, two schedules that put the same
  requests in different batches give bit-identical ids and logits (T13).
"""
import numpy as np
import pytest

from parity import compare_free_running, decoder_only_tf, t5_tf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 2e-2        # north_star's bf16 bar; widened per request by the calibration below
TOL_MEAN = 2e-3
STEPS = 6


@pytest.fixture(scope="module")
def X():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2404_07947_b200 as X
    return X


def _bench_requests(n):
    from workload import MODELS, make_requests, task_dists
    d = task_dists("S")
    return make_requests(n, d.pmf_in, d.pmf_out, MODELS["opt-13b"].vocab, 0xE6E1_0002)


@pytest.mark.parametrize("simt", [0])   # 1 routes dh=128 prefill to the fp32-P SIMT kernel (same result)
def test_opt13b_width_sampled_parity_in_bench_configuration(X, simt):
    from oracle import transformer as T
    from workload import MODELS, ModelSpec, Request, weight_seed
    full = MODELS["opt-13b"]
    spec = ModelSpec("opt-13b-first2", full.arch, 0, 2, full.d_model, full.n_heads, full.d_head, full.d_ff,
                     full.vocab, full.max_pos)
    reqs = _bench_requests(192)
    sample = [0, 95, 191]
    ctx = X.Context(spec, weight_seed(2))
    X.lib().exg_diag_prefill_simt(simt)
    toks, lat, st, lg = ctx.run(X.rra_schedule(31, 77, 16), reqs, dump=sample, slot_ctx=592)
    X.lib().exg_diag_prefill_simt(0)
    assert st["mean_decode_batch"] > 40          # steady decode batches in the bench's token-tile class (33..64)
    W = T.Weights(spec, weight_seed(2), cache_fp64=False)
    near_ties = []
    for r in sample:
        q = reqs[r]
        k = min(STEPS, q.output_len)
        rq = Request(q.ids, q.input_len, k)
        ora = T.greedy_kv(W, [rq], "bf16", record_logits=True)
        o32 = T.greedy_kv(W, [rq], "bf16", record_logits=True, accum="fp32")
        cal_max = cal_mean = 0.0
        for t in range(k):
            dd = np.abs(o32.logits[0][t] - ora.logits[0][t])
            cal_max, cal_mean = max(cal_max, float(dd.max())), max(cal_mean, float(dd.mean()))
            if o32.tokens[0][t] != ora.tokens[0][t]:
                break
        tol, tol_mean = max(TOL, 2 * cal_max), max(TOL_MEAN, 2 * cal_mean)
        worst, worst_mean, ev = compare_free_running(
            "opt13b-width req %d" % r, [toks[r][:k]], [lg[r][:k]], ora, tol,
            lambda _i, forced, rq=rq: T.teacher_forced_logits(W, rq, forced, "bf16"), max_near_ties=1,
            tol_mean=tol_mean)
        near_ties += ev
        print("req", r, "simt", simt, "gpu-vs-oracle max/mean %.4g/%.4g" % (worst, worst_mean),
              "oracle fp32-vs-fp64 %.4g/%.4g" % (cal_max, cal_mean), "bar %.4g" % tol)
    assert len(near_ties) <= 1, near_ties


@pytest.fixture(scope="module")
def full_depth(X):
    """All 40 layers of OPT-13B on 24 task-S requests under two schedules
    that put the requests in different batches."""
    from workload import MODELS, weight_seed
    reqs = _bench_requests(24)
    ctx = X.Context(MODELS["opt-13b"], weight_seed(2))
    dump = [0, 11, 23]
    a = ctx.run(X.rra_schedule(4, 8, 2), reqs, dump=dump, slot_ctx=592)
    b = ctx.run(X.rra_schedule(24, 24, 8), reqs, dump=dump, slot_ctx=592)
    ctx.close()
    return reqs, dump, a, b


def test_opt13b_full_depth_batch_invariance(full_depth):
    reqs, dump, a, b = full_depth
    assert a[0] == b[0]
    for r in dump:
        assert np.array_equal(a[3][r], b[3][r]), r
        assert np.all(np.isfinite(a[3][r]))


def _teacher_forced_layerwise(spec, seed, reqs, forced, accums=("fp64", "fp32")):
    """Oracle mode (iii) logits of every decode step of each request with the
    decode inputs forced to forced[r] (the GPU's own tokens), for each
    accumulation in `accums`.  One causal forward over each whole sequence
    x[0..n-1] + forced[0..S-2] -- the decode step t's logits are those of the
    row at position n-1+t (a row depends only on its own prefix) -- run layer
    by layer: each layer's weights are generated (T3), used for every
    sequence and both accumulations, then dropped, so a 40-layer OPT-13B
    never has to sit in host memory."""
    from oracle import transformer as T
    W = T.Weights(spec, seed, cache_fp64=False)
    toks, rows, out_rows = [], [], []
    for r, q in enumerate(reqs):
        seq = [int(v) for v in q.ids] + [int(v) for v in forced[r][:q.output_len - 1]]
        for p, v in enumerate(seq):
            if p >= q.input_len - 1:
                out_rows.append(len(toks))
            toks.append(v)
            rows.append((r, p))
    res = {}
    loops = {a: T.KVLoop(W, "bf16", a) for a in accums}
    H, dh, nL = spec.n_heads, spec.d_head, spec.n_dec_layers
    caches = {a: {r: ([None] * nL, [None] * nL) for r in range(len(reqs))} for a in accums}
    for a in accums:
        for r in range(len(reqs)):
            for l in range(nL):
                caches[a][r][0][l] = np.zeros((H, 0, dh))
                caches[a][r][1][l] = np.zeros((H, 0, dh))
    R = loops[accums[0]].R
    pos = np.array([p for _, p in rows])
    x0 = R.f32(W.emb_rows(np.array(toks)) + W.pos_emb[pos])
    xs = {a: x0.copy() for a in accums}
    for l in range(nL):
        for a in accums:
            xs[a] = loops[a]._layer(l, xs[a], rows, caches[a])
            for r in range(len(reqs)):      # keys of earlier layers are not needed again
                caches[a][r][0][l] = caches[a][r][1][l] = None
        W._layers.pop(l, None)
    for a in accums:
        lg = loops[a]._logits(xs[a][out_rows])
        k, res[a] = 0, []
        for q in reqs:
            res[a].append([lg[k + t] for t in range(q.output_len)])
            k += q.output_len
    return res


def test_opt13b_full_depth_vs_oracle(full_depth):
    """All 40 layers of OPT-13B (the bench's model, task-S requests) vs oracle
    mode (iii) on two sampled requests, weights regenerated per layer:
    the oracle is teacher-forced on the GPU's tokens (so a near tie early on
    does not end the comparison); every step's GPU id must be the oracle's
    argmax or a recorded near tie, and every step's logits lie within the
    calibrated bar max(2e-2, 2 x the oracle's own fp32-vs-fp64 accumulation
    spread at this depth) -- DESIGN.md §9."""
    from oracle import transformer as T
    from workload import MODELS, Request, weight_seed
    reqs, dump, a, _ = full_depth
    sample = dump[:2]
    steps = 8
    sreqs = [Request(reqs[r].ids, reqs[r].input_len, min(steps, reqs[r].output_len)) for r in sample]
    forced = [a[0][r][:sreqs[i].output_len] for i, r in enumerate(sample)]
    tf = _teacher_forced_layerwise(MODELS["opt-13b"], weight_seed(2), sreqs, forced)
    ev = []
    for i, r in enumerate(sample):
        ora, o32 = tf["fp64"][i], tf["fp32"][i]
        cal = max(float(np.abs(o32[t] - ora[t]).max()) for t in range(len(ora)))
        tol = max(TOL, 2 * cal)
        worst = 0.0
        for t in range(len(ora)):
            worst = max(worst, float(np.abs(a[3][r][t] - ora[t]).max()))
            y, yo = a[0][r][t], int(np.argmax(ora[t]))
            if y != yo:
                m = float(np.sort(ora[t])[-1] - np.sort(ora[t])[-2])
                assert m <= 2 * tol, "hard mismatch req %d step %d (margin %.4g)" % (r, t, m)
                assert ora[t][y] >= ora[t].max() - 2 * tol
                ev.append(("opt13b-40L req %d" % r, 0, t, m))
                print("NEAR-TIE opt13b 40 layers: request %d step %d margin %.3g" % (r, t, m))
        print("OPT-13B 40 layers req %d (n=%d): gpu-vs-oracle max %.4g, oracle fp32-vs-fp64 %.4g, bar %.4g"
              % (r, reqs[r].input_len, worst, cal, tol))
        assert worst <= tol, (r, worst, tol)
    from parity import NEAR_TIES
    NEAR_TIES.extend(ev)
    assert len(ev) <= 2


# ---------------------------------------------------------------------------
# configs 4 and 5 at their models' full width: one layer of OPT-66B under WAA
# with a TP-2 decoder group, one layer of GPT-3 175B under RRA with TP 8 --
# every GPU of the layout emulated on this device with exactly its shard --
# vs the oracle (calibrated bar as above) on short requests
# ---------------------------------------------------------------------------
def _width_case(X, model, layout, strategy, b_e, b_d, tp, n_enc, n_gpus):
    from oracle import transformer as T
    from workload import MODELS, ModelSpec, make_requests, uniform_pmf, weight_seed
    full = MODELS[model]
    spec = ModelSpec(model + "-1layer", full.arch, 0, 1, full.d_model, full.n_heads, full.d_head, full.d_ff,
                     full.vocab, full.max_pos)
    reqs = make_requests(4, uniform_pmf(24, 48), uniform_pmf(2, 3), full.vocab, 0xE6E10004)
    from paper_2404_07947_b200 import _lib
    ctx = X.Context(spec, weight_seed(4), cluster=X.cluster_spec(n_gpus))
    tp_gpus = sum(g[1] for g in layout if g[1] > 1)
    s = _lib.make_schedule(strategy, b_e, b_d, layout, n_d=2, b_m=0, n_enc_gpus=n_enc, tp_degree=tp, tp_gpus=tp_gpus)
    toks, lat, st, lg = ctx.run(s, reqs, dump=range(len(reqs)))
    W = T.Weights(spec, weight_seed(4), cache_fp64=False)
    ora = T.greedy_kv(W, reqs, "bf16", record_logits=True)
    o32 = T.greedy_kv(W, reqs, "bf16", record_logits=True, accum="fp32")
    cal = max(float(np.abs(o32.logits[r][t] - ora.logits[r][t]).max())
              for r, q in enumerate(reqs) for t in range(q.output_len))
    tol = max(TOL, 2 * cal)
    worst, _, _ = compare_free_running(model + "-width", toks, lg, ora, tol, decoder_only_tf(W, reqs), max_near_ties=1)
    print(model, "width: gpu-vs-oracle max %.4g, oracle fp32-vs-fp64 %.4g, bar %.4g" % (worst, cal, tol))


def test_config4_opt66b_width_waa_tp2(X):
    _width_case(X, "opt-66b", [(0, 1, 0, 1), (1, 2, 0, 1)], X.EXG_WAA_C, 2, 4, 2, 1, 3)


def test_config5_gpt3_width_rra_tp8(X):
    _width_case(X, "gpt3-175b", [(0, 8, 0, 1)], X.EXG_RRA, 2, 4, 8, 0, 8)


def test_config3_t5_11b_width_parity(X):
    """T5-11B width (d = 1024, 128 heads x 128, d_ff = 65536; one encoder and
    one decoder layer, identical weights) on task-T-shaped requests vs
    oracle/t5.py mode (iii), under RRA and under the 2-GPU WAA layout of config 3."""
    from oracle import t5 as T5
    from paper_2404_07947_b200 import _lib
    from workload import MODELS, ModelSpec, make_requests, uniform_pmf, weight_seed
    full = MODELS["t5-11b"]
    spec = ModelSpec("t5-11b-1+1", "t5", 1, 1, full.d_model, full.n_heads, full.d_head, full.d_ff, full.vocab,
                     full.max_pos)
    reqs = make_requests(4, uniform_pmf(40, 150), uniform_pmf(2, 4), full.vocab, 0xE6E10005)
    ora = T5.greedy_kv(T5.T5Weights(spec, weight_seed(3)), reqs, "bf16", record_logits=True)
    runs = [X.Context(spec, weight_seed(3)).run(X.rra_schedule(2, 4, 2), reqs, dump=range(len(reqs)))]
    s = _lib.make_schedule(X.EXG_WAA_C, 2, 4, [(0, 1, 0, 1), (1, 1, 0, 1)], n_enc_gpus=1)
    runs.append(X.Context(spec, weight_seed(3), cluster=X.cluster_spec(2)).run(s, reqs, dump=range(len(reqs))))
    W5 = T5.T5Weights(spec, weight_seed(3))
    for name, (toks, lat, st, lg) in zip(("rra", "waa"), runs):
        compare_free_running("t5-11b-width " + name, toks, lg, ora, TOL, t5_tf(W5, reqs), max_near_ties=1)
