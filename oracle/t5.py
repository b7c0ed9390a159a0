"""T5 encoder-decoder greedy decoding oracle (SURVEY.md §8(c) T1 T5 reading,
PAPER.md:97-98 self-/cross-attention, PAPER.md:415 T5 11B) -- test
infrastructure only.

Architecture (standard T5 v1.0; PAPER.md gives only sizes):
  encoder layer:  x += SelfAttn(RMS(x), bidirectional relative bias)
                  x += W_2 relu(W_1 RMS(x))
  encoder out:    RMS_enc(x)
  decoder layer:  x += SelfAttn(RMS(x), causal relative bias)
                  x += CrossAttn(RMS_x(x), encoder out)      (no bias)
                  x += W_2 relu(W_1 RMS(x))
  logits:         (RMS_f(x) E^T) * d^-1/2   (tied embedding)
No biases, no 1/sqrt(dh) score scaling, RMSNorm eps 1e-6, relative bias
(32 buckets, max distance 128) computed from layer 0's table and shared by all
layers, decoder start token 0.  Token accounting T6: the encode phase runs the
encoder over all n input tokens (and projects the cross K/V of every decoder
layer, K13); decode iteration u consumes the start token (u = 1) or y[u-1].

Weight tensors (T3 generator, canonical W[in][out]): encoder layer l at slot
1+l, decoder layer l at slot 1001+l, kinds ln1_g (self-attn norm), W_qkv,
W_o, ln2_g (FFN norm), W_1, W_2, rel_bias [buckets][H] (layer 0 only),
decoder adds lnx_g (cross norm), W_q_x [d][inner], W_kv_x [d][2 inner],
W_o_x [inner][d]; slot 0: tok_emb, lnf_g (decoder final norm), lnx_g
(encoder final norm; a reading: T3 lists no separate kind for it).

Modes as in transformer.py: (i) fp64 naive recompute, (ii) fp64 KV loop,
(iii) bf16-emulating KV loop (T4 rounding points; RMS output bf16, q/k/v and
cross K/V bf16, scores fp32(q.k) + fp32 bias, ctx bf16, FFN1 relu fp32 -> bf16,
residual fp32, logits fp32(bf16(RMS_f(x) d^-1/2) E^T): the head scale is
applied to the normed state before its bf16 rounding -- a reading; equal to
scaling the logits whenever d^-1/2 is a power of two, as for every T5 shape
here (d = 64, 256, 1024)).

Pins: (i) vs HuggingFace T5ForConditionalGeneration (fp64, same weights);
(i) == (ii); bucket table vs the published bucket rule on hand cases.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import weights as wgen
from .transformer import Rounding, argmax_first, top2_margin

NUM_BUCKETS = 32
MAX_DISTANCE = 128
EPS = 1e-6


def bucket(rel: int, bidirectional: bool, num_buckets: int = NUM_BUCKETS, max_distance: int = MAX_DISTANCE) -> int:
    """T5 relative position bucket of rel = key_pos - query_pos (double
    precision log, floor; T9)."""
    ret = 0
    n = num_buckets
    if bidirectional:
        n //= 2
        if rel > 0:
            ret += n
        rel = abs(rel)
    else:
        rel = -min(rel, 0)
    max_exact = n // 2
    if rel < max_exact:
        return ret + rel
    large = max_exact + int(math.log(rel / max_exact) / math.log(max_distance / max_exact) * (n - max_exact))
    return ret + min(large, n - 1)


def rms(x, g):
    return x / np.sqrt((x * x).mean(axis=-1, keepdims=True) + EPS) * g


class T5Weights:
    def __init__(self, spec, seed: int):
        self.spec, self.seed = spec, seed
        d, inner, ff, V = spec.d_model, spec.inner, spec.d_ff, spec.vocab
        g = lambda slot, kind, shape: wgen.gen_tensor(seed, slot, kind, shape).astype(np.float64)
        self.tok_emb = g(0, "tok_emb", (V, d))
        self.lnf_g = g(0, "lnf_g", (d,))
        self.enc_lnf_g = g(0, "lnx_g", (d,))
        H = spec.n_heads
        self.enc_rel = g(1, "rel_bias", (NUM_BUCKETS, H))
        self.dec_rel = g(1001, "rel_bias", (NUM_BUCKETS, H))
        self.enc = []
        for l in range(spec.n_enc_layers):
            s = wgen.enc_slot(l)
            self.enc.append({"ln1_g": g(s, "ln1_g", (d,)), "W_qkv": g(s, "W_qkv", (d, 3 * inner)),
                             "W_o": g(s, "W_o", (inner, d)), "ln2_g": g(s, "ln2_g", (d,)),
                             "W_1": g(s, "W_1", (d, ff)), "W_2": g(s, "W_2", (ff, d))})
        self.dec = []
        for l in range(spec.n_dec_layers):
            s = wgen.dec_slot(l)
            self.dec.append({"ln1_g": g(s, "ln1_g", (d,)), "W_qkv": g(s, "W_qkv", (d, 3 * inner)),
                             "W_o": g(s, "W_o", (inner, d)), "lnx_g": g(s, "lnx_g", (d,)),
                             "W_q_x": g(s, "W_q_x", (d, inner)), "W_kv_x": g(s, "W_kv_x", (d, 2 * inner)),
                             "W_o_x": g(s, "W_o_x", (inner, d)), "ln2_g": g(s, "ln2_g", (d,)),
                             "W_1": g(s, "W_1", (d, ff)), "W_2": g(s, "W_2", (ff, d))})


def _bias(table, qpos, kpos, bidirectional):
    """[H, len(qpos), len(kpos)] relative bias."""
    b = np.array([[bucket(int(k) - int(q), bidirectional) for k in kpos] for q in qpos], dtype=np.int64)
    return table[b].transpose(2, 0, 1)


def _mha(q, k, v, bias, causal, R):
    """q [Tq,H,dh], k/v [Tk,H,dh], bias [H,Tq,Tk] or None -> ctx [Tq,H*dh]."""
    Tq, H, dh = q.shape
    s = R.f32(np.einsum("qhd,khd->hqk", q, k))
    if bias is not None:
        s = R.f32(s + bias)
    if causal is not None:
        s = np.where(causal[None], s, -np.inf)
    m = s.max(axis=-1, keepdims=True)
    e = np.exp(s - m)
    p = e / e.sum(axis=-1, keepdims=True)
    return np.einsum("hqk,khd->qhd", p, v).reshape(Tq, H * dh)


def encoder_forward(W: T5Weights, ids, R: Optional[Rounding] = None):
    """Encoder over one request's tokens -> final RMS-normed states."""
    R = R or Rounding("fp64")
    spec = W.spec
    H, dh, inner = spec.n_heads, spec.d_head, spec.inner
    n = len(ids)
    pos = np.arange(n)
    bias = R.f32(_bias(W.enc_rel, pos, pos, True))
    x = R.f32(W.tok_emb[np.asarray(ids)])
    for L in W.enc:
        h = R.bf16(rms(x, L["ln1_g"]))
        qkv = R.bf16(h @ L["W_qkv"])
        q, k, v = (qkv[:, i * inner:(i + 1) * inner].reshape(n, H, dh) for i in range(3))
        ctx = R.bf16(_mha(q, k, v, bias, None, R))
        x = R.f32(x + R.f32(ctx @ L["W_o"]))
        h = R.bf16(rms(x, L["ln2_g"]))
        f = R.bf16(np.maximum(R.f32(h @ L["W_1"]), 0.0))
        x = R.f32(x + R.f32(f @ L["W_2"]))
    return R.bf16(rms(x, W.enc_lnf_g))


def decoder_full(W: T5Weights, enc_out, dec_ids):
    """(i) naive: decoder over the whole decoder input prefix, fp64 -> logits [T, V]."""
    R = Rounding("fp64")
    spec = W.spec
    H, dh, inner, d = spec.n_heads, spec.d_head, spec.inner, spec.d_model
    T = len(dec_ids)
    pos = np.arange(T)
    bias = _bias(W.dec_rel, pos, pos, False)
    causal = pos[None, :] <= pos[:, None]
    x = W.tok_emb[np.asarray(dec_ids)]
    n = enc_out.shape[0]
    for L in W.dec:
        h = rms(x, L["ln1_g"])
        qkv = h @ L["W_qkv"]
        q, k, v = (qkv[:, i * inner:(i + 1) * inner].reshape(T, H, dh) for i in range(3))
        x = x + _mha(q, k, v, bias, causal, R) @ L["W_o"]
        h = rms(x, L["lnx_g"])
        qx = (h @ L["W_q_x"]).reshape(T, H, dh)
        kvx = enc_out @ L["W_kv_x"]
        kx, vx = kvx[:, :inner].reshape(n, H, dh), kvx[:, inner:].reshape(n, H, dh)
        x = x + _mha(qx, kx, vx, None, None, R) @ L["W_o_x"]
        h = rms(x, L["ln2_g"])
        x = x + np.maximum(h @ L["W_1"], 0.0) @ L["W_2"]
    hf = rms(x, W.lnf_g)
    return (hf @ W.tok_emb.T) * d ** -0.5


def greedy_naive(W: T5Weights, ids, S: int, record_logits=False):
    enc = encoder_forward(W, ids)
    seq = [0]
    out, logs = [], []
    for _ in range(S):
        lg = decoder_full(W, enc, seq)[-1]
        y = argmax_first(lg)
        out.append(y)
        logs.append(lg)
        seq.append(y)
    return (out, logs) if record_logits else out


@dataclass
class Result:
    tokens: List[List[int]]
    logits: List[List[np.ndarray]] = field(default_factory=list)
    margins: List[List[float]] = field(default_factory=list)


def greedy_kv(W: T5Weights, requests, mode: str = "bf16", record_logits: bool = False,
              forced: Optional[List[List[int]]] = None) -> Result:
    """(ii)/(iii): encoder once per request, cross K/V projected once (K13),
    decoder self-attention KV cache, one token per decode iteration.
    forced[r]: decode inputs forced to these tokens (teacher forcing on
    another run's output) instead of the greedy ids."""
    R = Rounding(mode)
    spec = W.spec
    H, dh, inner, d = spec.n_heads, spec.d_head, spec.inner, spec.d_model
    head_scale = d ** -0.5
    toks, logs, margins = [], [], []
    for qi, q in enumerate(requests):
        enc = encoder_forward(W, q.ids, R)
        n = enc.shape[0]
        cross = []
        for L in W.dec:
            kvx = R.bf16(enc @ L["W_kv_x"])
            cross.append((kvx[:, :inner].reshape(n, H, dh), kvx[:, inner:].reshape(n, H, dh)))
        Kc = [np.zeros((0, H, dh)) for _ in W.dec]
        Vc = [np.zeros((0, H, dh)) for _ in W.dec]
        cur, out, lg_r, mg_r = 0, [], [], []
        for t in range(q.output_len):
            x = R.f32(W.tok_emb[[cur]])
            for li, L in enumerate(W.dec):
                h = R.bf16(rms(x, L["ln1_g"]))
                qkv = R.bf16(h @ L["W_qkv"])
                qs = qkv[:, :inner].reshape(1, H, dh)
                Kc[li] = np.concatenate([Kc[li], qkv[:, inner:2 * inner].reshape(1, H, dh)])
                Vc[li] = np.concatenate([Vc[li], qkv[:, 2 * inner:].reshape(1, H, dh)])
                bias = R.f32(_bias(W.dec_rel, [t], np.arange(t + 1), False))
                ctx = R.bf16(_mha(qs, Kc[li], Vc[li], bias, None, R))
                x = R.f32(x + R.f32(ctx @ L["W_o"]))
                h = R.bf16(rms(x, L["lnx_g"]))
                qx = R.bf16(h @ L["W_q_x"]).reshape(1, H, dh)
                ctx = R.bf16(_mha(qx, cross[li][0], cross[li][1], None, None, R))
                x = R.f32(x + R.f32(ctx @ L["W_o_x"]))
                h = R.bf16(rms(x, L["ln2_g"]))
                f = R.bf16(np.maximum(R.f32(h @ L["W_1"]), 0.0))
                x = R.f32(x + R.f32(f @ L["W_2"]))
            hf = R.bf16(rms(x, W.lnf_g) * head_scale)
            lg = R.f32(hf @ W.tok_emb.T)[0]
            y = argmax_first(lg)
            out.append(y)
            mg_r.append(top2_margin(lg))
            if record_logits:
                lg_r.append(lg)
            cur = y if forced is None else forced[qi][t]
        toks.append(out)
        logs.append(lg_r)
        margins.append(mg_r)
    return Result(toks, logs, margins)
