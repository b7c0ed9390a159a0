"""FMHA P-in-TMEM diagnosis: the T5 bidirectional + relative-bias case of
tests/test_gpu_t5.py and a 4-tile causal / bidirectional case, run repeatedly
with P in shared memory (0) and in TMEM (1); prints the max error vs fp64 and
whether the outputs are finite and repeatable.

    python tools/fmha_pt_check.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2404_07947_b200 import _lib as L  # noqa: E402
from gpu_util import bf16_round_np, bf16_tensor, ptr  # noqa: E402
from test_gpu_t5 import _bias_table  # noqa: E402

dev = torch.device("cuda:0")
st = lambda: torch.cuda.current_stream().cuda_stream


def case(bias, causal, lens, H=2, dh=128, max_ctx=512, seed=7):
    rng = np.random.default_rng(seed)
    R = len(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    qkv = bf16_round_np(rng.standard_normal((T, 3 * H * dh)) * 0.5)
    K = np.zeros((R, H, max_ctx, dh)); V = np.zeros((R, H, max_ctx, dh))
    for r in range(R):
        for j in range(lens[r]):
            t = cu[r] + j
            K[r, :, j] = qkv[t, H * dh:2 * H * dh].reshape(H, dh)
            V[r, :, j] = qkv[t, 2 * H * dh:].reshape(H, dh)
    P = 400
    tab = _bias_table(bf16_round_np(rng.standard_normal((32, H))), H, P, True) if bias else None
    tK, tV, tq = bf16_tensor(K), bf16_tensor(V), bf16_tensor(qkv)
    tb = torch.from_numpy(tab).to(dev) if bias else None
    tcu = torch.from_numpy(cu).to(dev)
    tsl = torch.arange(R, dtype=torch.int32, device=dev)
    tp0 = torch.zeros(R, dtype=torch.int32, device=dev)
    scale = 1.0 if bias else float(np.float32(1 / np.sqrt(dh)))

    def run():
        out = torch.zeros((T, H * dh), dtype=torch.bfloat16, device=dev)
        L.check(L.lib().exg_op_prefill_attention(ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tcu), ptr(tsl), ptr(tp0),
                                                 R, max(lens), ptr(out), H * dh, H, dh, max_ctx, R, T, scale, causal,
                                                 ptr(tb) if bias else None, 2 * P - 1 if bias else 0,
                                                 P - 1 if bias else 0, st()))
        torch.cuda.synchronize()
        return out.float().cpu().numpy()

    worst = 0.0
    outs = [run() for _ in range(8)]
    for r in range(R):
        n = lens[r]
        pos = np.arange(n)
        for h in range(H):
            s = (qkv[cu[r]:cu[r + 1], h * dh:(h + 1) * dh] @ K[r, h, :n].T) * scale
            if bias:
                s = s + tab[h][(pos[None, :] - pos[:, None]) + P - 1]
            if causal:
                s = np.where(np.tril(np.ones_like(s)) > 0, s, -np.inf)
            p = np.exp(s - s.max(axis=1, keepdims=True))
            ref = (p / p.sum(axis=1, keepdims=True)) @ V[r, h, :n]
            worst = max(worst, float(np.nanmax(np.abs(outs[0][cu[r]:cu[r + 1], h * dh:(h + 1) * dh] - ref))))
    finite = all(np.isfinite(o).all() for o in outs)
    same = all(np.array_equal(o, outs[0]) for o in outs)
    return worst, finite, same


for on in (0, 1):
    L.lib().exg_diag_fmha_p_tmem(on)
    for name, bias, causal, lens in (("t5-bias", True, 0, [1, 7, 100, 128, 129, 300]),
                                     ("bidir", False, 0, [512, 300, 257, 129, 511, 384]),
                                     ("causal", False, 1, [512, 300, 257, 129, 511, 384])):
        w, f, same = case(bias, causal, lens)
        print("P in %-4s %-8s max err %.3g finite %s repeatable %s" % ("TMEM" if on else "smem", name, w, f, same))
L.lib().exg_diag_fmha_p_tmem(1)
