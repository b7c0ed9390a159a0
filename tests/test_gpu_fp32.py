"""fp32 parity path (north_star: logits within 1e-4 of
the oracle on the fp32 path): exg_create with dtype EXG_FP32 runs every
intermediate in fp32 with FFMA contractions and precise expf / tanhf
(csrc/fp32_path.cu).  Compared with oracle mode (ii) -- the fp64 KV-cache
loop, itself pinned to the naive recompute loop (i) and to HuggingFace --
free-running: ids equal, logits within 1e-4 on every step.
"""
import numpy as np
import pytest

from parity import compare_free_running, decoder_only_tf

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL32 = 1e-4


@pytest.fixture(scope="module")
def X():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2404_07947_b200 as X
    return X


def test_config1_fp32_ids_and_logits(X):
    from oracle import transformer as T
    from workload import MODELS, config1_requests, weight_seed
    spec, seed = MODELS["tiny"], weight_seed(1)
    reqs = config1_requests()
    ctx = X.Context(spec, seed, dtype=X.EXG_FP32)
    toks, lat, st, lg = ctx.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
    W = T.Weights(spec, seed)
    ora = T.greedy_kv(W, reqs, "fp64", record_logits=True)
    worst, _, ev = compare_free_running("config1-fp32", toks, lg, ora, TOL32, decoder_only_tf(W, reqs, "fp64"),
                                        max_near_ties=0)
    print("config 1 fp32: max |logit - oracle(ii)| = %.3g" % worst)
    # the naive recompute loop (i) agrees too (it is the plain definition)
    for r in (0, 5):
        ids_i, lg_i = T.greedy_naive(W, reqs[r].ids, reqs[r].output_len, record_logits=True)
        assert ids_i == toks[r]
        assert max(float(np.abs(lg[r][t] - lg_i[t]).max()) for t in range(reqs[r].output_len)) <= TOL32
    assert st["out_tokens"] == sum(q.output_len for q in reqs)
    ctx.close()


def test_fp32_batch_invariance_and_static(X):
    from workload import MODELS, config1_requests, weight_seed
    spec, seed = MODELS["tiny"], weight_seed(1)
    reqs = config1_requests()
    ctx = X.Context(spec, seed, dtype=X.EXG_FP32)
    a = ctx.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
    for s in (X.rra_schedule(1, 1, 1), X.rra_schedule(3, 5, 2), X.static_schedule(3)):
        b = ctx.run(s, reqs, dump=range(len(reqs)))
        assert a[0] == b[0]
        for r in range(len(reqs)):
            assert np.array_equal(a[3][r], b[3][r]), r
    ctx.close()


@pytest.mark.parametrize("arch,dh,lens", [("opt", 128, ((700, 5), (1030, 3), (40, 6))), ("gpt3", 64, ((90, 9), (33, 4)))])
def test_fp32_wider_models_vs_oracle(X, arch, dh, lens):
    """dh = 64 / 128, OPT (ReLU) and GPT-3 (GELU-tanh) layers, rows of more
    than 1024 keys, ragged batches."""
    from oracle import transformer as T
    from workload import ModelSpec, Request
    spec = ModelSpec("fp32-" + arch, arch, 0, 2, 256, 256 // dh, dh, 1024, 512, 1100)
    seed = 0xE6E0_0F32
    rng = np.random.default_rng(11)
    reqs = [Request(rng.integers(0, 512, n).astype(np.int32), n, s) for n, s in lens]
    ctx = X.Context(spec, seed, dtype=X.EXG_FP32)
    toks, _, _, lg = ctx.run(X.rra_schedule(2, 3, 2), reqs, dump=range(len(reqs)))
    W = T.Weights(spec, seed)
    ora = T.greedy_kv(W, reqs, "fp64", record_logits=True)
    worst, _, _ = compare_free_running("fp32-" + arch, toks, lg, ora, TOL32, decoder_only_tf(W, reqs, "fp64"),
                                       max_near_ties=0)
    print(arch, "dh", dh, "fp32 max |logit diff| %.3g" % worst)
    ctx.close()


def test_fp32_scope_errors(X):
    from workload import MODELS, weight_seed
    with pytest.raises(X.ExgError) as ei:
        X.Context(MODELS["tiny-t5"], weight_seed(3), dtype=X.EXG_FP32)
    assert ei.value.status == 1
    with pytest.raises(X.ExgError) as ei:
        X.Context(MODELS["tiny"], weight_seed(1), dtype=X.EXG_FP32, cluster=X.cluster_spec(2))
    assert ei.value.status == 1
    ctx = X.Context(MODELS["tiny"], weight_seed(1), dtype=X.EXG_FP32)
    with pytest.raises(X.ExgError) as ei:
        ctx.profile([1, 4], [16], [16, 64], reps=1)
    assert ei.value.status == 1
    ctx.close()
