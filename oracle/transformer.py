"""Greedy decoding oracle for decoder-only models
(OPT: ReLU; GPT-3 / tiny: GELU-tanh), test infrastructure only.

Definition (§2; forced output lengths PAPER.md:486):

    y_r[t] = argmax_v logits(x_r || y_r[1..t-1])[v],  t = 1..S_r

for each request in isolation; lowest index wins ties (T7).  Architecture
readings T1/T10 (pre-LN, biases, learned absolute positions 0-based, final
LN, tied LM head, q scaled by dh^-1/2, LN eps 1e-5, biased variance).

Three implementations:
  (i)   `greedy_naive`      fp64, full causal forward over the whole prefix at
                            every step, no cache (the "independent naive loop").
  (ii)  `greedy_kv(...,"fp64")`  fp64 KV-cache loop, token accounting T6
                            (encode writes positions 0..n-2, decode iteration u
                            consumes x[n-1] (u=1) or y[u-1]).
  (iii) `greedy_kv(...,"bf16")`  same loop with the rounding points of T4:
                            residual fp32, norm out bf16, QKV bf16, K/V bf16,
                            scores fp32(q.k)*fp32(scale), ctx bf16, FFN1
                            bias+act on fp32 then bf16, O/FFN2 fp32, logits
                            fp32.  Accumulation in fp64.

Pins: (i) == (ii) to 1e-10; (i) vs HuggingFace GPT2/OPT in fp64 with the same
weights (library implementation of the same architecture); closed-form special
cases (tests/test_oracle_transformer.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import weights as wgen


# ---------------------------------------------------------------------------
# rounding policy (T4)
# ---------------------------------------------------------------------------
class Rounding:
    def __init__(self, mode: str):
        assert mode in ("fp64", "bf16")
        self.emulate = mode == "bf16"

    def f32(self, x):
        return np.asarray(x, dtype=np.float32).astype(np.float64) if self.emulate else x

    def bf16(self, x):
        if not self.emulate:
            return x
        return wgen.bf16_round(np.asarray(x, dtype=np.float32)).astype(np.float64)

    def scale(self, dh: int) -> float:
        s = 1.0 / math.sqrt(dh)
        return float(np.float32(s)) if self.emulate else s


def layer_norm(x: np.ndarray, g: np.ndarray, b: np.ndarray, eps: float = 1e-5) -> np.ndarray:
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def gelu_tanh(x: np.ndarray) -> np.ndarray:
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def relu(x: np.ndarray) -> np.ndarray:
    return np.maximum(x, 0.0)


def act_fn(arch: str):
    return relu if arch == "opt" else gelu_tanh


# ---------------------------------------------------------------------------
# weights
# ---------------------------------------------------------------------------
class Weights:
    """Parameter provider.  Small models are materialised in fp64; large ones
    keep bf16-exact values in float32 and upcast one layer at a time."""

    def __init__(self, spec, seed: int, cache_fp64: Optional[bool] = None):
        self.spec, self.seed = spec, seed
        params = spec.n_dec_layers * (4 * spec.d_model * spec.inner + 2 * spec.d_model * spec.d_ff)
        self.cache_fp64 = params < 50_000_000 if cache_fp64 is None else cache_fp64
        d = spec.d_model
        self.tok_emb = wgen.gen_tensor(seed, 0, "tok_emb", (spec.vocab, d))
        self.pos_emb = wgen.gen_tensor(seed, 0, "pos_emb", (spec.max_pos, d)).astype(np.float64)
        self.lnf_g = wgen.gen_tensor(seed, 0, "lnf_g", (d,)).astype(np.float64)
        self.lnf_b = wgen.gen_tensor(seed, 0, "lnf_b", (d,)).astype(np.float64)
        self._layers: Dict[int, Dict] = {}
        if self.cache_fp64:
            self.tok_emb = self.tok_emb.astype(np.float64)

    @classmethod
    def from_dict(cls, spec, W: Dict):
        """Explicit weights (fp64 dict as produced by weights.decoder_only_weights)."""
        self = cls.__new__(cls)
        self.spec, self.seed, self.cache_fp64 = spec, None, True
        self.tok_emb, self.pos_emb = W["tok_emb"], W["pos_emb"]
        self.lnf_g, self.lnf_b = W["lnf_g"], W["lnf_b"]
        self._layers = {l: L for l, L in enumerate(W["layers"])}
        return self

    def layer(self, l: int) -> Dict:
        if l in self._layers:
            L = self._layers[l]
            return L if self.cache_fp64 else {k: v.astype(np.float64) for k, v in L.items()}
        L = wgen.decoder_layer_weights(self.spec, self.seed, wgen.dec_slot(l),
                                       np.float64 if self.cache_fp64 else np.float32)
        self._layers[l] = L
        return L if self.cache_fp64 else {k: v.astype(np.float64) for k, v in L.items()}

    def emb_rows(self, ids) -> np.ndarray:
        return np.asarray(self.tok_emb[np.asarray(ids)], dtype=np.float64)

    def head(self) -> np.ndarray:
        return np.asarray(self.tok_emb, dtype=np.float64)


# ---------------------------------------------------------------------------
# (i) naive recompute, fp64
# ---------------------------------------------------------------------------
def forward_full(W: Weights, ids: np.ndarray) -> np.ndarray:
    """Textbook causal forward over a whole sequence; returns fp64 logits
    [T, V].  No cache, no rounding."""
    spec = W.spec
    T = len(ids)
    H, dh = spec.n_heads, spec.d_head
    act = act_fn(spec.arch)
    x = W.emb_rows(ids) + W.pos_emb[:T]
    mask = np.triu(np.full((T, T), -np.inf), k=1)
    for l in range(spec.n_dec_layers):
        L = W.layer(l)
        h = layer_norm(x, L["ln1_g"], L["ln1_b"])
        qkv = h @ L["W_qkv"] + L["b_qkv"]
        q, k, v = np.split(qkv, 3, axis=1)
        q = q.reshape(T, H, dh).transpose(1, 0, 2)
        k = k.reshape(T, H, dh).transpose(1, 0, 2)
        v = v.reshape(T, H, dh).transpose(1, 0, 2)
        s = q @ k.transpose(0, 2, 1) / math.sqrt(dh) + mask
        s = s - s.max(axis=-1, keepdims=True)
        p = np.exp(s)
        p = p / p.sum(axis=-1, keepdims=True)
        ctx = (p @ v).transpose(1, 0, 2).reshape(T, H * dh)
        x = x + ctx @ L["W_o"] + L["b_o"]
        h2 = layer_norm(x, L["ln2_g"], L["ln2_b"])
        x = x + act(h2 @ L["W_1"] + L["b_1"]) @ L["W_2"] + L["b_2"]
    hf = layer_norm(x, W.lnf_g, W.lnf_b)
    return hf @ W.head().T


def argmax_first(v: np.ndarray) -> int:
    """Lowest index among the maxima (T7); NaN is an error."""
    if np.isnan(v).any():
        raise FloatingPointError("NaN logit")
    return int(np.argmax(v))


def top2_margin(v: np.ndarray) -> float:
    if len(v) < 2:
        return float("inf")
    part = np.partition(v, -2)[-2:]
    return float(part[1] - part[0])


def greedy_naive(W: Weights, ids: np.ndarray, S: int, record_logits: bool = False):
    seq = list(int(t) for t in ids)
    out, logits = [], []
    for _ in range(S):
        lg = forward_full(W, np.array(seq))[-1]
        y = argmax_first(lg)
        out.append(y)
        if record_logits:
            logits.append(lg)
        seq.append(y)
    return (out, logits) if record_logits else out


# ---------------------------------------------------------------------------
# (ii)/(iii) KV-cache loop, batched over requests (results are per-request
# isolated: attention never crosses requests, T9)
# ---------------------------------------------------------------------------
@dataclass
class Result:
    tokens: List[List[int]]
    logits: List[List[np.ndarray]] = field(default_factory=list)   # per request, per step
    margins: List[List[float]] = field(default_factory=list)


class KVLoop:
    """accum = "fp64" (default): every product accumulated in fp64 and rounded
    once at the T4 rounding point -- the reference.  accum = "fp32": the same
    rounding points with fp32 accumulation (numpy float32 matmuls), a second
    valid evaluation of the contract used only to measure how far two valid
    evaluations can drift apart at a given model width (calibrates the
    full-width parity tolerance)."""

    def __init__(self, W: Weights, mode: str, accum: str = "fp64"):
        self.W, self.spec, self.R = W, W.spec, Rounding(mode)
        self.act = act_fn(self.spec.arch)
        assert accum in ("fp64", "fp32")
        self.f32acc = accum == "fp32"

    def mm(self, a, b):
        if self.f32acc:
            return (np.asarray(a, dtype=np.float32) @ np.asarray(b, dtype=np.float32)).astype(np.float64)
        return a @ b

    def _layer(self, l, x, rows, caches):
        """x: [T, d] residual (fp32-valued in bf16 mode) for tokens `rows`
        = list of (request r, position p); caches[r] = (K, V) lists per layer
        with arrays [H, len, dh].  Each request's new tokens are consecutive
        positions and are appended before attention."""
        spec, R = self.spec, self.R
        H, dh = spec.n_heads, spec.d_head
        L = self.W.layer(l)
        h = R.bf16(layer_norm(x, L["ln1_g"], L["ln1_b"]))
        qkv = R.bf16(self.mm(h, L["W_qkv"]) + L["b_qkv"])
        T = x.shape[0]
        q = qkv[:, :H * dh].reshape(T, H, dh)
        k = qkv[:, H * dh:2 * H * dh].reshape(T, H, dh)
        v = qkv[:, 2 * H * dh:].reshape(T, H, dh)
        ctx = np.empty((T, H, dh))
        scale = R.scale(dh)
        # group consecutive tokens per request
        i = 0
        while i < T:
            r, p0 = rows[i]
            j = i
            while j < T and rows[j][0] == r:
                j += 1
            K, Vc = caches[r]
            K[l] = np.concatenate([K[l], k[i:j].transpose(1, 0, 2)], axis=1)
            Vc[l] = np.concatenate([Vc[l], v[i:j].transpose(1, 0, 2)], axis=1)
            n_new = j - i
            klen = K[l].shape[1]
            assert klen == p0 + n_new
            qs = q[i:j].transpose(1, 0, 2)                         # [H, n_new, dh]
            s = R.f32(self.mm(qs, K[l].transpose(0, 2, 1)))        # [H, n_new, klen]
            s = R.f32(s * scale)
            qpos = p0 + np.arange(n_new)[:, None]
            s = np.where(np.arange(klen)[None, :] <= qpos, s, -np.inf)
            m = s.max(axis=-1, keepdims=True)
            e = np.exp(s - m)
            pr = e / e.sum(axis=-1, keepdims=True)
            ctx[i:j] = self.mm(pr, Vc[l]).transpose(1, 0, 2)
            i = j
        ctx = R.bf16(ctx.reshape(T, H * dh))
        x = R.f32(x + R.f32(self.mm(ctx, L["W_o"]) + L["b_o"]))
        h2 = R.bf16(layer_norm(x, L["ln2_g"], L["ln2_b"]))
        f = R.bf16(self.act(R.f32(self.mm(h2, L["W_1"]) + L["b_1"])))
        x = R.f32(x + R.f32(self.mm(f, L["W_2"]) + L["b_2"]))
        return x

    def _forward(self, tokens, rows, caches):
        R = self.R
        pos = np.array([p for _, p in rows])
        x = R.f32(self.W.emb_rows(tokens) + self.W.pos_emb[pos])
        for l in range(self.spec.n_dec_layers):
            x = self._layer(l, x, rows, caches)
        return x

    def _logits(self, x):
        R = self.R
        hf = R.bf16(layer_norm(x, self.W.lnf_g, self.W.lnf_b))
        return R.f32(self.mm(hf, self.W.head().T))

    def run(self, requests, record_logits: bool = False, record: Optional[set] = None) -> Result:
        """Greedy decode every request; token accounting T6."""
        nL = self.spec.n_dec_layers
        H, dh = self.spec.n_heads, self.spec.d_head
        caches = {r: ([np.zeros((H, 0, dh)) for _ in range(nL)],
                      [np.zeros((H, 0, dh)) for _ in range(nL)]) for r in range(len(requests))}
        # encode: positions 0..n-2 of every request, packed
        toks, rows = [], []
        for r, q in enumerate(requests):
            for p in range(q.input_len - 1):
                toks.append(int(q.ids[p]))
                rows.append((r, p))
        if toks:
            self._forward(np.array(toks), rows, caches)
        out = [[] for _ in requests]
        logs = [[] for _ in requests]
        margins = [[] for _ in requests]
        cur = {r: (int(q.ids[-1]), q.input_len - 1) for r, q in enumerate(requests)}
        active = [r for r, q in enumerate(requests) if q.output_len > 0]
        while active:
            toks = np.array([cur[r][0] for r in active])
            rows = [(r, cur[r][1]) for r in active]
            x = self._forward(toks, rows, caches)
            lg = self._logits(x)
            nxt = []
            for i, r in enumerate(active):
                y = argmax_first(lg[i])
                out[r].append(y)
                margins[r].append(top2_margin(lg[i]))
                if record_logits and (record is None or r in record):
                    logs[r].append(lg[i].copy())
                cur[r] = (y, cur[r][1] + 1)
                if len(out[r]) < requests[r].output_len:
                    nxt.append(r)
            active = nxt
        return Result(out, logs, margins)


def greedy_kv(W: Weights, requests, mode: str = "bf16", record_logits: bool = False,
              record: Optional[set] = None, accum: str = "fp64") -> Result:
    return KVLoop(W, mode, accum).run(requests, record_logits, record)


def teacher_forced_logits(W: Weights, request, forced: List[int], mode: str = "fp64",
                          accum: str = "fp64") -> List[np.ndarray]:
    """Logits of every decode step when the decode inputs are forced to
    `forced` (the tokens some other run emitted): used to compare a run's
    logits with mode (ii) on that run's own prefix, and to keep checking a
    run past a near-tie divergence (tests/parity.py)."""
    loop = KVLoop(W, mode, accum)
    nL, H, dh = W.spec.n_dec_layers, W.spec.n_heads, W.spec.d_head
    caches = {0: ([np.zeros((H, 0, dh)) for _ in range(nL)], [np.zeros((H, 0, dh)) for _ in range(nL)])}
    n = request.input_len
    if n > 1:
        loop._forward(np.array(request.ids[:n - 1]), [(0, p) for p in range(n - 1)], caches)
    cur, pos, out = int(request.ids[-1]), n - 1, []
    for t in range(len(forced)):
        x = loop._forward(np.array([cur]), [(0, pos)], caches)
        out.append(loop._logits(x)[0])
        cur, pos = forced[t], pos + 1
    return out
