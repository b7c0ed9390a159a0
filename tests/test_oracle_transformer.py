"""Pins for oracle/transformer.py (SURVEY.md §8(c) R1, c.3 'Transformer logits').

* (i) naive recompute == (ii) KV-cache loop (two independent algorithms), 1e-10
* (i) == HuggingFace GPT2LMHeadModel / OPTForCausalLM in float64 loaded with
  the same weights: an independent library implementation of the same
  architecture (T1: GPT-3-style = GPT-2 block with GELU-tanh; OPT = pre-LN,
  ReLU, q scaled by dh^-1/2; HF OPT's position offset of 2 is absorbed)
* closed forms: identity layers => logits = LN_f(emb+pos) E^T; constant keys
  => attention = causal running mean of V
* (iii) bf16 emulation stays within bf16-level error of (ii)
"""
import math

import numpy as np
import pytest
import torch

from oracle import transformer as T
from oracle import weights as wg
from workload import MODELS, ModelSpec, Request, config1_requests, make_requests, uniform_pmf, weight_seed


def _spec(arch, L=2, d=32, H=4, dh=8, ff=64, V=97, P=48):
    return ModelSpec("t", arch, 0, L, d, H, dh, ff, V, P)


def _weights(spec, seed=5):
    return T.Weights.from_dict(spec, wg.decoder_only_weights(spec, seed))


def test_naive_equals_kv_fp64_tiny_config1():
    spec = MODELS["tiny"]
    W = T.Weights(spec, weight_seed(1))
    reqs = config1_requests()
    r2 = T.greedy_kv(W, reqs, "fp64", record_logits=True)
    for i, q in enumerate(reqs):
        toks, lg = T.greedy_naive(W, q.ids, q.output_len, True)
        assert toks == r2.tokens[i]
        for a, b in zip(lg, r2.logits[i]):
            assert np.abs(a - b).max() < 1e-10


def _hf_gpt2(spec, W):
    from transformers import GPT2Config, GPT2LMHeadModel
    cfg = GPT2Config(vocab_size=spec.vocab, n_positions=spec.max_pos, n_embd=spec.d_model,
                     n_layer=spec.n_dec_layers, n_head=spec.n_heads, n_inner=spec.d_ff,
                     activation_function="gelu_new", layer_norm_epsilon=1e-5,
                     resid_pdrop=0.0, embd_pdrop=0.0, attn_pdrop=0.0, tie_word_embeddings=True)
    m = GPT2LMHeadModel(cfg).double().eval()
    t = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float64))
    with torch.no_grad():
        m.transformer.wte.weight.copy_(t(W.tok_emb))
        m.transformer.wpe.weight.copy_(t(W.pos_emb))
        m.transformer.ln_f.weight.copy_(t(W.lnf_g)); m.transformer.ln_f.bias.copy_(t(W.lnf_b))
        for l, blk in enumerate(m.transformer.h):
            L = W.layer(l)
            blk.ln_1.weight.copy_(t(L["ln1_g"])); blk.ln_1.bias.copy_(t(L["ln1_b"]))
            blk.attn.c_attn.weight.copy_(t(L["W_qkv"])); blk.attn.c_attn.bias.copy_(t(L["b_qkv"]))
            blk.attn.c_proj.weight.copy_(t(L["W_o"])); blk.attn.c_proj.bias.copy_(t(L["b_o"]))
            blk.ln_2.weight.copy_(t(L["ln2_g"])); blk.ln_2.bias.copy_(t(L["ln2_b"]))
            blk.mlp.c_fc.weight.copy_(t(L["W_1"])); blk.mlp.c_fc.bias.copy_(t(L["b_1"]))
            blk.mlp.c_proj.weight.copy_(t(L["W_2"])); blk.mlp.c_proj.bias.copy_(t(L["b_2"]))
    m.lm_head.weight = m.transformer.wte.weight
    return m


def _hf_opt(spec, W):
    from transformers import OPTConfig, OPTForCausalLM
    cfg = OPTConfig(vocab_size=spec.vocab, hidden_size=spec.d_model, num_hidden_layers=spec.n_dec_layers,
                    ffn_dim=spec.d_ff, num_attention_heads=spec.n_heads, max_position_embeddings=spec.max_pos,
                    do_layer_norm_before=True, word_embed_proj_dim=spec.d_model, dropout=0.0,
                    attention_dropout=0.0, activation_function="relu", enable_bias=True,
                    layer_norm_elementwise_affine=True, tie_word_embeddings=True, pad_token_id=None)
    m = OPTForCausalLM(cfg).double().eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)))
    inner = spec.inner
    with torch.no_grad():
        dec = m.model.decoder
        dec.embed_tokens.weight.copy_(t(W.tok_emb))
        dec.embed_positions.weight.zero_()
        dec.embed_positions.weight[2:2 + spec.max_pos].copy_(t(W.pos_emb))   # HF offset 2
        dec.final_layer_norm.weight.copy_(t(W.lnf_g)); dec.final_layer_norm.bias.copy_(t(W.lnf_b))
        for l, blk in enumerate(dec.layers):
            L = W.layer(l)
            Wq, Wk, Wv = np.split(L["W_qkv"], 3, axis=1)
            bq, bk, bv = np.split(L["b_qkv"], 3)
            a = blk.self_attn
            a.q_proj.weight.copy_(t(Wq.T)); a.q_proj.bias.copy_(t(bq))
            a.k_proj.weight.copy_(t(Wk.T)); a.k_proj.bias.copy_(t(bk))
            a.v_proj.weight.copy_(t(Wv.T)); a.v_proj.bias.copy_(t(bv))
            a.out_proj.weight.copy_(t(L["W_o"].T)); a.out_proj.bias.copy_(t(L["b_o"]))
            blk.self_attn_layer_norm.weight.copy_(t(L["ln1_g"])); blk.self_attn_layer_norm.bias.copy_(t(L["ln1_b"]))
            blk.final_layer_norm.weight.copy_(t(L["ln2_g"])); blk.final_layer_norm.bias.copy_(t(L["ln2_b"]))
            blk.fc1.weight.copy_(t(L["W_1"].T)); blk.fc1.bias.copy_(t(L["b_1"]))
            blk.fc2.weight.copy_(t(L["W_2"].T)); blk.fc2.bias.copy_(t(L["b_2"]))
    m.lm_head.weight = dec.embed_tokens.weight
    return m


@pytest.mark.parametrize("arch", ["gpt3", "opt"])
def test_forward_full_matches_huggingface(arch):
    spec = _spec(arch)
    W = _weights(spec)
    ids = np.random.default_rng(1).integers(0, spec.vocab, size=23)
    ours = T.forward_full(W, ids)
    m = _hf_gpt2(spec, W) if arch == "gpt3" else _hf_opt(spec, W)
    with torch.no_grad():
        ref = m(torch.from_numpy(ids[None].astype(np.int64))).logits[0].numpy()
    assert np.abs(ours - ref).max() < 1e-10


def test_tiny_model_matches_huggingface_gpt2():
    spec = MODELS["tiny"]
    W = T.Weights(spec, weight_seed(1))
    ids = config1_requests()[0].ids
    m = _hf_gpt2(spec, W)
    with torch.no_grad():
        ref = m(torch.from_numpy(ids[None].astype(np.int64))).logits[0].numpy()
    assert np.abs(T.forward_full(W, ids) - ref).max() < 1e-10


def test_identity_layers_closed_form():
    """W_o = W_2 = 0, b_o = b_2 = 0 => residual stream is emb + pos, so
    logits = LN_f(emb + pos) E^T exactly."""
    spec = _spec("opt")
    Wd = wg.decoder_only_weights(spec, 9)
    for L in Wd["layers"]:
        L["W_o"][:] = 0; L["b_o"][:] = 0; L["W_2"][:] = 0; L["b_2"][:] = 0
    W = T.Weights.from_dict(spec, Wd)
    ids = np.arange(11) * 7 % spec.vocab
    x = Wd["tok_emb"][ids] + Wd["pos_emb"][:11]
    mu = x.mean(1, keepdims=True)
    sd = np.sqrt(((x - mu) ** 2).mean(1, keepdims=True) + 1e-5)
    ref = ((x - mu) / sd * Wd["lnf_g"] + Wd["lnf_b"]) @ Wd["tok_emb"].T
    assert np.abs(T.forward_full(W, ids) - ref).max() < 1e-12


def test_constant_keys_give_causal_mean_of_values():
    """K projection = 0 with a constant key bias => every score in a row is
    equal, softmax is uniform over the visible prefix and the attention
    output is the running mean of V (1 layer, FFN zeroed)."""
    spec = _spec("gpt3", L=1)
    Wd = wg.decoder_only_weights(spec, 3)
    L = Wd["layers"][0]
    inner = spec.inner
    L["W_qkv"][:, inner:2 * inner] = 0.0
    L["b_qkv"][inner:2 * inner] = 0.37
    L["W_2"][:] = 0; L["b_2"][:] = 0
    W = T.Weights.from_dict(spec, Wd)
    ids = np.arange(9) * 5 % spec.vocab
    x = Wd["tok_emb"][ids] + Wd["pos_emb"][:9]
    mu = x.mean(1, keepdims=True)
    h = (x - mu) / np.sqrt(((x - mu) ** 2).mean(1, keepdims=True) + 1e-5) * L["ln1_g"] + L["ln1_b"]
    v = h @ L["W_qkv"][:, 2 * inner:] + L["b_qkv"][2 * inner:]
    cm = np.cumsum(v, axis=0) / np.arange(1, 10)[:, None]
    x2 = x + cm @ L["W_o"] + L["b_o"]
    mu = x2.mean(1, keepdims=True)
    hf = (x2 - mu) / np.sqrt(((x2 - mu) ** 2).mean(1, keepdims=True) + 1e-5) * Wd["lnf_g"] + Wd["lnf_b"]
    assert np.abs(T.forward_full(W, ids) - hf @ Wd["tok_emb"].T).max() < 1e-12


def test_bf16_mode_close_to_fp64_and_same_ids_on_config1():
    spec = MODELS["tiny"]
    W = T.Weights(spec, weight_seed(1))
    reqs = config1_requests()
    r2 = T.greedy_kv(W, reqs, "fp64", record_logits=True)
    r3 = T.greedy_kv(W, reqs, "bf16", record_logits=True)
    assert r2.tokens == r3.tokens
    err = max(np.abs(a - b).max() for i in range(len(reqs)) for a, b in zip(r2.logits[i], r3.logits[i]))
    assert 0 < err < 2e-2
    # config-1 fixture choice (T4a): oracle min top-2 margin >= 1e-3
    assert min(min(m) for m in r3.margins) >= 1e-3


def test_teacher_forced_logits_equal_free_running_on_own_prefix():
    spec = _spec("opt")
    W = _weights(spec)
    req = Request(np.array([3, 14, 15, 92, 65], np.int32), 5, 6)
    r = T.greedy_kv(W, [req], "fp64", record_logits=True)
    tf = T.teacher_forced_logits(W, req, r.tokens[0], "fp64")
    for a, b in zip(tf, r.logits[0]):
        assert np.abs(a - b).max() < 1e-12


def test_single_token_input_has_empty_encode():
    spec = _spec("gpt3")
    W = _weights(spec)
    req = Request(np.array([4], np.int32), 1, 3)
    assert T.greedy_kv(W, [req], "fp64").tokens[0] == T.greedy_naive(W, req.ids, 3)


def test_fp32_accumulation_variant_agrees_at_small_width():
    """The accum="fp32" evaluation (used only to calibrate the full-width
    tolerance) follows the same rounding points: at config-1 width it agrees
    with the fp64-accumulated reference to well inside the parity bar."""
    spec = MODELS["tiny"]
    W = T.Weights(spec, weight_seed(1))
    reqs = config1_requests()[:3]
    a = T.greedy_kv(W, reqs, "bf16", record_logits=True)
    b = T.greedy_kv(W, reqs, "bf16", record_logits=True, accum="fp32")
    for i in range(len(reqs)):
        for t in range(len(a.logits[i])):
            if a.tokens[i][t] != b.tokens[i][t]:
                break
            assert np.abs(a.logits[i][t] - b.logits[i][t]).max() < 2e-3
