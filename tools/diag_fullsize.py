"""Diagnose GPU-vs-oracle logit differences at OPT-13B width.

GPU box:  python tools/diag_fullsize.py gpu   -> gpurun_out/diag_fullsize.npz
here:     python tools/diag_fullsize.py cpu   -> oracle rounding-point variants vs the GPU logits
"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from workload import MODELS, ModelSpec, Request, make_requests, task_dists, weight_seed

full = MODELS["opt-13b"]
NL = 1
spec = ModelSpec("w", full.arch, 0, NL, full.d_model, full.n_heads, full.d_head, full.d_ff, full.vocab, full.max_pos)
d = task_dists("S")
q = make_requests(4, d.pmf_in, d.pmf_out, full.vocab, 0xE6E1_0002)[1]
r1 = Request(q.ids[:40], 40, 2)
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "diag_fullsize.npz")

if sys.argv[1] == "gpu":
    import paper_2404_07947_b200 as X
    ctx = X.Context(spec, weight_seed(2))
    toks, lat, st, lg = ctx.run(X.rra_schedule(1, 1, 1), [r1], dump=[0], slot_ctx=64)
    np.savez(OUT, logits=lg[0], toks=np.array(toks[0]))
    sys.exit(0)

from oracle import transformer as T
g = np.load(OUT)
W = T.Weights(spec, weight_seed(2), cache_fp64=False)
base = T.KVLoop(W, "bf16")
orig_bf16 = base.R.bf16
sites = ["h", "qkv", "ctx", "h2", "f", "hf"]


def run(skip):
    R = T.Rounding("bf16")
    loop = T.KVLoop(W, "bf16")
    counter = {"i": 0}
    names = []

    def bf16(x):
        # call order inside _layer: h, qkv, ctx, h2, f ; _logits: hf
        i = counter["i"]
        counter["i"] += 1
        name = names[i] if i < len(names) else "?"
        return x if name in skip else orig_bf16(x)
    per_layer = ["h", "qkv", "ctx", "h2", "f"]
    # prefill (n-1 tokens), then decode steps with logits
    names[:] = per_layer * NL + (per_layer * NL + ["hf"]) * 2
    loop.R.bf16 = bf16
    res = loop.run([r1], record_logits=True)
    return res.logits[0]


for skip in []:
    lg = run(skip)
    print("skip %-8s step0 max|gpu-ora| %.4g mean %.4g   step1 %.4g" % (",".join(sorted(skip)) or "-",
          np.abs(g["logits"][0] - lg[0]).max(), np.abs(g["logits"][0] - lg[0]).mean(),
          np.abs(g["logits"][1] - lg[1]).max()))

# variant: the same rounding points with fp32 matmuls (the GPU's accumulation precision)
class F32Loop(T.KVLoop):
    pass

_mm = np.matmul


def f32_matmul_run():
    import builtins
    loop = T.KVLoop(W, "bf16")
    orig_layer = loop.W.layer

    def layer32(l):
        return {k: v.astype(np.float32) for k, v in orig_layer(l).items()}
    loop.W.layer = layer32
    orig_head = loop.W.head
    loop.W.head = lambda: orig_head().astype(np.float32)
    res = loop.run([r1], record_logits=True)
    loop.W.layer, loop.W.head = orig_layer, orig_head
    return res.logits[0]


lg64 = run(set())
lg32 = f32_matmul_run()
print("oracle fp32-matmul vs fp64-matmul: step0 max %.4g mean %.4g" % (np.abs(lg32[0] - lg64[0]).max(),
                                                                       np.abs(lg32[0] - lg64[0]).mean()))
print("gpu vs oracle fp32-matmul: step0 max %.4g mean %.4g" % (np.abs(g["logits"][0] - lg32[0]).max(),
                                                                 np.abs(g["logits"][0] - lg32[0]).mean()))


def manual(dt):
    """(iii) rounding points, matmuls accumulated in dtype (fp32 = the GPU's)."""
    R = T.Rounding("bf16")
    L = {k: v.astype(dt) for k, v in W.layer(0).items()}
    H, dh = spec.n_heads, spec.d_head
    inner = H * dh
    ids = np.asarray(r1.ids)
    x = R.f32(W.emb_rows(ids) + W.pos_emb[:len(ids)])
    h = R.bf16(T.layer_norm(x, L["ln1_g"], L["ln1_b"])).astype(dt)
    qkv = R.bf16((h @ L["W_qkv"]).astype(np.float64) + L["b_qkv"])
    K = qkv[:, inner:2 * inner].reshape(-1, H, dh)
    V = qkv[:, 2 * inner:].reshape(-1, H, dh)
    t = len(ids) - 1
    q = qkv[t, :inner].reshape(H, dh)
    s = R.f32(np.einsum("hd,khd->hk", q.astype(dt), K.astype(dt)).astype(np.float64)) * np.float32(1 / np.sqrt(dh))
    s = R.f32(s)
    p = np.exp(s - s.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    ctx = R.bf16(np.einsum("hk,khd->hd", p.astype(dt), V.astype(dt)).reshape(1, inner).astype(np.float64))
    xt = x[t:t + 1]
    xt = R.f32(xt + R.f32((ctx.astype(dt) @ L["W_o"]).astype(np.float64) + L["b_o"]))
    h2 = R.bf16(T.layer_norm(xt, L["ln2_g"], L["ln2_b"]))
    f = R.bf16(np.maximum(R.f32((h2.astype(dt) @ L["W_1"]).astype(np.float64) + L["b_1"]), 0))
    xt = R.f32(xt + R.f32((f.astype(dt) @ L["W_2"]).astype(np.float64) + L["b_2"]))
    hf = R.bf16(T.layer_norm(xt, W.lnf_g, W.lnf_b))
    return R.f32((hf.astype(dt) @ W.head().astype(dt).T).astype(np.float64))[0]


m64, m32 = manual(np.float64), manual(np.float32)
print("manual64 vs oracle(iii): %.4g" % np.abs(m64 - lg64[0]).max())
print("manual32 vs manual64: max %.4g mean %.4g" % (np.abs(m32 - m64).max(), np.abs(m32 - m64).mean()))
print("gpu vs manual32: max %.4g mean %.4g" % (np.abs(g["logits"][0] - m32).max(), np.abs(g["logits"][0] - m32).mean()))
