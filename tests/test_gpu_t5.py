"""T5 encoder-decoder on the CUDA path (SURVEY.md §8 rows a2, a3 and a5 for
T5), checked against oracle/t5.py:

* kernels: RMSNorm (with the folded head scale), bidirectional prefill
  attention with relative bias (SIMT dh=16 and tcgen05 FMHA dh=128, several
  128-key tiles and ragged tails), decode attention with the causal relative
  bias over one and several 512-key splits;
* end to end through exg_run: greedy ids equal oracle mode (iii) (near-ties
  reported with their margin), logits within 2e-2, for the dh=16 and the
  dh=128 parity models; batch invariance across RRA schedules (bit-identical);
* WAA layouts (config 3 shape): encoder GPU(s) project every decoder layer's
  cross K/V and hand it off to the decoder GPU(s) -- bit-identical to the
  single-GPU run, in one process and over 2 / 4 thread ranks.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gpu_util import bf16_round_np, bf16_tensor, dev, ptr, stream, to_np  # noqa: E402

TOL = 2e-2


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2404_07947_b200 import _lib
    return _lib


def _run(L, name, *args):
    L.check(getattr(L.lib(), name)(*args))


def _bias_table(rel, H, P, bidirectional):
    """fp32 [H][2P-1] table: tab[h][j] = rel[bucket(j - (P-1))][h] (oracle bucket rule)."""
    from oracle import t5 as T5
    idx = np.array([T5.bucket(j - (P - 1), bidirectional) for j in range(2 * P - 1)])
    return np.ascontiguousarray(rel[idx].T).astype(np.float32)


def test_rmsnorm(L):
    rng = np.random.default_rng(3)
    T, d = 37, 1024
    x = rng.standard_normal((T, d)).astype(np.float32) * 3
    g = bf16_round_np(1 + 0.1 * rng.standard_normal(d))
    y = torch.zeros((T, d), dtype=torch.bfloat16, device=dev())
    tx = torch.from_numpy(x).to(dev())
    tg = bf16_tensor(g)   # kept alive until the launch completes
    _run(L, "exg_op_rmsnorm", ptr(y), d, ptr(tx), d, ptr(tg), T, d, 1e-6, 1.0 / 32, stream())
    torch.cuda.synchronize()
    x64 = x.astype(np.float64)
    ref = x64 / np.sqrt((x64 ** 2).mean(axis=1, keepdims=True) + 1e-6) * g / 32
    assert np.all(np.abs(to_np(y) - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-6)


@pytest.mark.parametrize("dh", [16, 128])
def test_prefill_attention_bidirectional_bias(L, dh):
    rng = np.random.default_rng(dh + 7)
    H, max_ctx, P = 2, 400, 400
    lens = [1, 7, 100, 128, 129, 300]
    R = len(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    slot = np.array([3, 0, 5, 1, 4, 2], dtype=np.int32)
    n_slots = 6
    qkv = bf16_round_np(rng.standard_normal((T, 3 * H * dh)) * 0.5)
    K = np.zeros((n_slots, H, max_ctx, dh)); V = np.zeros((n_slots, H, max_ctx, dh))
    for r in range(R):
        for j in range(lens[r]):
            t = cu[r] + j
            K[slot[r], :, j] = qkv[t, H * dh:2 * H * dh].reshape(H, dh)
            V[slot[r], :, j] = qkv[t, 2 * H * dh:].reshape(H, dh)
    rel = bf16_round_np(rng.standard_normal((32, H)))
    tab = _bias_table(rel, H, P, True)
    out = torch.zeros((T, H * dh), dtype=torch.bfloat16, device=dev())
    tK, tV, tq, tb = bf16_tensor(K), bf16_tensor(V), bf16_tensor(qkv), torch.from_numpy(tab).to(dev())
    tcu, tsl = torch.from_numpy(cu).to(dev()), torch.from_numpy(slot).to(dev())
    tp0 = torch.zeros(R, dtype=torch.int32, device=dev())
    _run(L, "exg_op_prefill_attention", ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tcu), ptr(tsl), ptr(tp0), R,
         max(lens), ptr(out), H * dh, H, dh, max_ctx, n_slots, T, 1.0, 0, ptr(tb), 2 * P - 1, P - 1, stream())
    torch.cuda.synchronize()
    got = to_np(out)
    rtol, atol = (2.0 ** -8, 2e-3) if dh != 128 else (2.0 ** -7, 4e-3)
    for r in range(R):
        n = lens[r]
        pos = np.arange(n)
        for h in range(H):
            s = qkv[cu[r]:cu[r + 1], h * dh:(h + 1) * dh] @ K[slot[r], h, :n].T
            s = s + tab[h][(pos[None, :] - pos[:, None]) + P - 1]
            p = np.exp(s - s.max(axis=1, keepdims=True))
            ref = (p / p.sum(axis=1, keepdims=True)) @ V[slot[r], h, :n]
            g = got[cu[r]:cu[r + 1], h * dh:(h + 1) * dh]
            assert np.all(np.abs(g - ref) <= rtol * np.abs(ref) + atol), (r, h, np.abs(g - ref).max())


@pytest.mark.parametrize("dh", [16, 128])
def test_decode_attention_causal_bias(L, dh):
    rng = np.random.default_rng(dh + 11)
    H, max_ctx, P = 3, 1200, 1200
    nk = np.array([1, 2, 40, 511, 512, 513, 1100], dtype=np.int32)
    B = len(nk)
    slot = np.arange(B, dtype=np.int32)[::-1].copy()
    K = bf16_round_np(rng.standard_normal((B, H, max_ctx, dh)) * 0.5)
    V = bf16_round_np(rng.standard_normal((B, H, max_ctx, dh)))
    q = bf16_round_np(rng.standard_normal((B, H * dh)) * 0.5)
    rel = bf16_round_np(rng.standard_normal((32, H)))
    tab = _bias_table(rel, H, P, False)
    split, ms = 512, 3
    part = torch.zeros(B * H * ms * (dh + 2), dtype=torch.float32, device=dev())
    out = torch.zeros((B, H * dh), dtype=torch.bfloat16, device=dev())
    tK, tV, tq, tb = bf16_tensor(K), bf16_tensor(V), bf16_tensor(q), torch.from_numpy(tab).to(dev())
    ts, tn = torch.from_numpy(slot).to(dev()), torch.from_numpy(nk).to(dev())
    _run(L, "exg_op_decode_attention", ptr(tq), H * dh, ptr(tK), ptr(tV), ptr(ts), ptr(tn), ptr(out), H * dh, B, H,
         dh, max_ctx, 1.0, split, ms, ptr(part), ptr(tb), 2 * P - 1, P - 1, stream())
    torch.cuda.synchronize()
    got = to_np(out)
    for i in range(B):
        n = nk[i]
        for h in range(H):
            s = K[slot[i], h, :n] @ q[i, h * dh:(h + 1) * dh]
            s = s + tab[h][np.arange(n) - (n - 1) + P - 1]
            p = np.exp(s - s.max())
            ref = (p / p.sum()) @ V[slot[i], h, :n]
            g = got[i, h * dh:(h + 1) * dh]
            assert np.all(np.abs(g - ref) <= 2.0 ** -8 * np.abs(ref) + 2e-3), (i, h, np.abs(g - ref).max())


# ------------------------------------------------------------- end to end --
def _requests(name):
    from workload import MODELS, config1_requests, make_requests, uniform_pmf
    if name == "tiny-t5":
        return config1_requests()
    # dh = 128 model: inputs span one and two 128-key FMHA tiles
    return make_requests(6, uniform_pmf(60, 200), uniform_pmf(1, 12), MODELS[name].vocab, 0xE6E10003)


@pytest.fixture(scope="module", params=["tiny-t5", "small-t5"])
def t5env(request, L):
    import paper_2404_07947_b200 as X
    from oracle import t5 as T5
    from workload import MODELS, weight_seed
    spec = MODELS[request.param]
    seed = weight_seed(3)
    reqs = _requests(request.param)
    ctx = X.Context(spec, seed)
    ora = T5.greedy_kv(T5.T5Weights(spec, seed), reqs, "bf16", record_logits=True)
    return X, spec, reqs, ctx, ora


def test_t5_ids_and_logits_match_oracle(t5env):
    X, spec, reqs, ctx, ora = t5env
    toks, lat, st, lg = ctx.run(X.rra_schedule(3, 5, 4), reqs, dump=range(len(reqs)))
    worst = 0.0
    for r, q in enumerate(reqs):
        for t in range(q.output_len):
            if toks[r][t] != ora.tokens[r][t]:
                m = ora.margins[r][t]
                assert m <= 2 * TOL, "hard mismatch req %d step %d margin %.4g" % (r, t, m)
                pytest.fail("near-tie divergence req %d step %d (margin %.3g)" % (r, t, m))
            worst = max(worst, float(np.abs(lg[r][t] - ora.logits[r][t]).max()))
    assert worst <= TOL, worst
    assert st["out_tokens"] == sum(q.output_len for q in reqs) and np.all(lat > 0)


def test_t5_batch_invariance(t5env):
    X, spec, reqs, ctx, ora = t5env
    a = ctx.run(X.rra_schedule(3, 5, 4), reqs, dump=range(len(reqs)))
    b = ctx.run(X.rra_schedule(1, 8, 2), reqs, dump=range(len(reqs)))
    assert a[0] == b[0]
    for r in range(len(reqs)):
        assert np.array_equal(a[3][r], b[3][r]), r


def test_t5_static_batch_baseline(t5env):
    """FT-style static batch (EXG_STATIC) on the encoder-decoder: finished
    rows keep decoding at clamped decoder positions inside their own slots;
    ids and logits are bit-identical to the RRA run (T13), decode iterations
    = sum over batches of the batch's longest output."""
    X, spec, reqs, ctx, ora = t5env
    a = ctx.run(X.rra_schedule(3, 5, 4), reqs, dump=range(len(reqs)))
    b = 3
    toks, lat, st, lg = ctx.run(X.static_schedule(b), reqs, dump=range(len(reqs)))
    assert toks == a[0]
    for r in range(len(reqs)):
        assert np.array_equal(lg[r], a[3][r]), r
    groups = [range(k, min(k + b, len(reqs))) for k in range(0, len(reqs), b)]
    assert st["decode_iters"] == sum(max(reqs[r].output_len for r in g) for g in groups)
    for g in groups:
        assert len({float(lat[r]) for r in g}) == 1


@pytest.mark.parametrize("transport", ["one_rank", "two_ranks", "nccl_loopback"])
def test_t5_rra_pipeline_bit_identical(t5env, transport):
    """RRA over 2 pipeline stages, each holding encoder and decoder layers
    [l0, l1): the encoder output is broadcast from the last stage so every
    stage projects the cross K/V of its own decoder layers."""
    X, spec, reqs, ctx, ora = t5env
    from paper_2404_07947_b200 import _lib
    from workload import weight_seed
    base_t, _, _, base_l = ctx.run(X.rra_schedule(3, 5, 4), reqs, dump=range(len(reqs)))
    s = _lib.make_schedule(X.EXG_RRA, 3, 5, [(0, 1, 0, 1), (1, 1, 1, 2)], n_d=4)
    if transport == "one_rank":
        res = [X.Context(spec, weight_seed(3), cluster=X.cluster_spec(2)).run(s, reqs, dump=range(len(reqs)))]
    elif transport == "two_ranks":
        res = X.run_group(X.local_group(spec, weight_seed(3), 2, X.cluster_spec(2)), s, reqs, dump=range(len(reqs)))
    else:
        res = [X.nccl_loopback(spec, weight_seed(3), X.cluster_spec(2)).run(s, reqs, dump=range(len(reqs)))]
    assert res[0][0] == base_t
    head = [r[3] for r in res if np.any(r[3][0])]
    assert len(head) == 1
    for r in range(len(reqs)):
        assert np.array_equal(head[0][r], base_l[r]), r


# WAA for T5 (config 3: encoder GPU(s) + decoder GPU(s)): the last encoder
# stage projects the cross K/V of every decoder layer (K13) and hands each
# decoder stage its layers' n cross K/V rows per request (K12).  Same per-row
# arithmetic as the single-GPU run => bit-identical ids and logits, also with
# the GPUs split over thread ranks.
T5_WAA = [
    # (name, b_e, b_d, b_m, n_enc, layout, world)
    ("enc1_dec1", 2, 5, 0, 1, [(0, 1, 0, 2), (1, 1, 0, 2)], 1),
    ("enc1_dec1_w2", 2, 5, 0, 1, [(0, 1, 0, 2), (1, 1, 0, 2)], 2),
    ("enc2_dec2_mb", 3, 6, 3, 2, [(0, 1, 0, 1), (1, 1, 1, 2), (2, 1, 0, 1), (3, 1, 1, 2)], 1),
    ("enc2_dec2_mb_w4", 3, 6, 3, 2, [(0, 1, 0, 1), (1, 1, 1, 2), (2, 1, 0, 1), (3, 1, 1, 2)], 4),
]


@pytest.mark.parametrize("case", T5_WAA, ids=[c[0] for c in T5_WAA])
def test_t5_waa_bit_identical_to_single_gpu(t5env, case):
    X, spec, reqs, ctx, ora = t5env
    from paper_2404_07947_b200 import _lib
    from workload import weight_seed
    name, b_e, b_d, b_m, n_enc, layout, world = case
    base_t, _, _, base_l = ctx.run(X.rra_schedule(3, 5, 4), reqs, dump=range(len(reqs)))
    s = _lib.make_schedule(X.EXG_WAA_C, b_e, b_d, layout, b_m=b_m, n_enc_gpus=n_enc)
    if world == 1:
        multi = X.Context(spec, weight_seed(3), cluster=X.cluster_spec(4))
        toks, lat, st, lg = multi.run(s, reqs, dump=range(len(reqs)))
        heads = [lg]
    else:
        group = X.local_group(spec, weight_seed(3), world, X.cluster_spec(4))
        res = X.run_group(group, s, reqs, dump=range(len(reqs)))
        toks, lat, st, lg = res[0]
        heads = [r[3] for r in res if np.any(r[3][0])]
    assert toks == base_t
    assert len(heads) == 1
    for r in range(len(reqs)):
        assert np.array_equal(heads[0][r], base_l[r]), r
    assert st["out_tokens"] == sum(q.output_len for q in reqs) and np.all(lat > 0)
