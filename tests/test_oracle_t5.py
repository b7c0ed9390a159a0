"""Pins for oracle/t5.py (SURVEY.md §8(c) T1 T5 reading).

* relative position buckets == HuggingFace T5Attention._relative_position_bucket
  (an independent implementation of the published rule) for every distance in
  [-300, 300], both directions
* (i) naive recompute == HuggingFace T5ForConditionalGeneration in float64 with
  the same weights (its RMSNorm variance is taken in fp32; measured 5e-9, bar 1e-7)
* (i) naive == (ii) KV loop with projected cross K/V (two algorithms), 1e-10
* (iii) bf16 emulation within bf16-level error of (ii)
* closed form: with zero self/cross/FFN output projections the decoder is the
  identity and logits = RMS_f(E[y]) E^T d^-1/2 regardless of the input
"""
import numpy as np
import pytest
import torch

from oracle import t5 as T5
from workload import MODELS, ModelSpec, make_requests, uniform_pmf, weight_seed


def _spec():
    return ModelSpec("t", "t5", 2, 2, 32, 4, 8, 64, 97, 64)


def _reqs(n=3, V=97, seed=11):
    return make_requests(n, uniform_pmf(3, 9), uniform_pmf(1, 6), V, seed)


def test_bucket_matches_hf_rule():
    from transformers.models.t5.modeling_t5 import T5Attention
    rel = torch.arange(-300, 301)
    for bidir in (True, False):
        hf = T5Attention._relative_position_bucket(rel, bidirectional=bidir, num_buckets=32, max_distance=128)
        ours = [T5.bucket(int(r), bidir) for r in rel]
        assert ours == hf.tolist()


def _hf_model(W):
    from transformers import T5Config, T5ForConditionalGeneration
    s = W.spec
    cfg = T5Config(vocab_size=s.vocab, d_model=s.d_model, d_kv=s.d_head, d_ff=s.d_ff, num_layers=s.n_enc_layers,
                   num_decoder_layers=s.n_dec_layers, num_heads=s.n_heads, relative_attention_num_buckets=32,
                   relative_attention_max_distance=128, dropout_rate=0.0, layer_norm_epsilon=1e-6,
                   feed_forward_proj="relu", tie_word_embeddings=True, decoder_start_token_id=0)
    m = T5ForConditionalGeneration(cfg).double().eval()
    inner = s.inner
    t = lambda a: torch.tensor(a, dtype=torch.float64)
    sd = {"shared.weight": t(W.tok_emb), "encoder.final_layer_norm.weight": t(W.enc_lnf_g),
          "decoder.final_layer_norm.weight": t(W.lnf_g),
          "encoder.block.0.layer.0.SelfAttention.relative_attention_bias.weight": t(W.enc_rel),
          "decoder.block.0.layer.0.SelfAttention.relative_attention_bias.weight": t(W.dec_rel)}
    for side, layers in (("encoder", W.enc), ("decoder", W.dec)):
        for l, L in enumerate(layers):
            p = "%s.block.%d.layer." % (side, l)
            for i, n in enumerate("qkv"):
                sd[p + "0.SelfAttention.%s.weight" % n] = t(L["W_qkv"][:, i * inner:(i + 1) * inner].T)
            sd[p + "0.SelfAttention.o.weight"] = t(L["W_o"].T)
            sd[p + "0.layer_norm.weight"] = t(L["ln1_g"])
            f = 1 if side == "encoder" else 2
            if side == "decoder":
                sd[p + "1.EncDecAttention.q.weight"] = t(L["W_q_x"].T)
                sd[p + "1.EncDecAttention.k.weight"] = t(L["W_kv_x"][:, :inner].T)
                sd[p + "1.EncDecAttention.v.weight"] = t(L["W_kv_x"][:, inner:].T)
                sd[p + "1.EncDecAttention.o.weight"] = t(L["W_o_x"].T)
                sd[p + "1.layer_norm.weight"] = t(L["lnx_g"])
            sd[p + "%d.DenseReluDense.wi.weight" % f] = t(L["W_1"].T)
            sd[p + "%d.DenseReluDense.wo.weight" % f] = t(L["W_2"].T)
            sd[p + "%d.layer_norm.weight" % f] = t(L["ln2_g"])
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected
    assert all(k in ("lm_head.weight", "encoder.embed_tokens.weight", "decoder.embed_tokens.weight") for k in missing), missing
    m.lm_head.weight.data.copy_(t(W.tok_emb))
    return m


def test_naive_matches_huggingface_t5():
    W = T5.T5Weights(_spec(), 7)
    m = _hf_model(W)
    for q in _reqs():
        toks, lg = T5.greedy_naive(W, q.ids, q.output_len, record_logits=True)
        dec_in = torch.tensor([[0] + toks[:-1]])
        with torch.no_grad():
            out = m(input_ids=torch.from_numpy(q.ids.astype(np.int64))[None], decoder_input_ids=dec_in).logits[0].numpy()
        ref = np.stack(lg)
        assert np.abs(out - ref).max() <= 1e-7


def test_naive_equals_kv_fp64():
    W = T5.T5Weights(_spec(), 9)
    reqs = _reqs(4, seed=5)
    r2 = T5.greedy_kv(W, reqs, "fp64", record_logits=True)
    for i, q in enumerate(reqs):
        toks, lg = T5.greedy_naive(W, q.ids, q.output_len, True)
        assert toks == r2.tokens[i]
        for a, b in zip(lg, r2.logits[i]):
            assert np.abs(a - b).max() < 1e-10


def test_bf16_emulation_close_to_fp64():
    spec = MODELS["tiny-t5"]
    W = T5.T5Weights(spec, weight_seed(3))
    reqs = make_requests(3, uniform_pmf(16, 32), uniform_pmf(1, 12), spec.vocab, 3)
    a = T5.greedy_kv(W, reqs, "fp64", record_logits=True)
    b = T5.greedy_kv(W, reqs, "bf16", record_logits=True)
    for i in range(len(reqs)):
        # compare the first step (same inputs on both sides); later steps may diverge on near-ties
        assert np.abs(a.logits[i][0] - b.logits[i][0]).max() < 2e-2


def test_identity_decoder_closed_form():
    spec = _spec()
    W = T5.T5Weights(spec, 13)
    for L in W.dec:
        L["W_o"][:] = 0
        L["W_o_x"][:] = 0
        L["W_2"][:] = 0
    q = _reqs(1)[0]
    toks, lg = T5.greedy_naive(W, q.ids, 3, record_logits=True)
    prev = [0] + toks[:-1]
    for y_in, l in zip(prev, lg):
        e = W.tok_emb[y_in]
        h = e / np.sqrt((e * e).mean() + 1e-6) * W.lnf_g
        np.testing.assert_allclose(l, h @ W.tok_emb.T / np.sqrt(spec.d_model), atol=1e-12)
