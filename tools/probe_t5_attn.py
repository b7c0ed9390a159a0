"""T5-11B decode attention per-key cost, self (relative bias) vs cross (no
bias), at batch 64: the XProfiler times the T5 decode attention at an even
self / cross split of the keys; task T rows hold ~40 % self / 60 % cross.

    python tools/probe_t5_attn.py
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_07947_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda:0")
st = lambda: torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)


def timeit(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def dattn(B, keys, bias, H=128, dh=128, max_ctx=512, ragged=None):
    kc = torch.randn(B, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    vc = torch.randn(B, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    q = torch.randn(B, 3 * H * dh, device=dev).to(torch.bfloat16)
    slot = torch.arange(B, dtype=torch.int32, device=dev)
    if ragged is None:
        nk = torch.full((B,), keys, dtype=torch.int32, device=dev)
    else:   # per-row key counts, longest first (the runner's row order)
        nk = torch.tensor(sorted(ragged, reverse=True), dtype=torch.int32, device=dev)
        keys = int(max(ragged))
    out = torch.empty(B, H * dh, device=dev, dtype=torch.bfloat16)
    ms = max(1, math.ceil(keys / 512))
    part = torch.empty(B * H * ms * (dh + 2), device=dev, dtype=torch.float32)
    tab = torch.randn(H, 2 * max_ctx - 1, device=dev) if bias else None

    def fn():
        L.check(L.lib().exg_op_decode_attention(q.data_ptr(), 3 * H * dh, kc.data_ptr(), vc.data_ptr(),
                                                slot.data_ptr(), nk.data_ptr(), out.data_ptr(), H * dh, B, H, dh,
                                                max_ctx, 1.0, 512, ms, part.data_ptr(),
                                                tab.data_ptr() if bias else None, 2 * max_ctx - 1 if bias else 0,
                                                max_ctx - 1 if bias else 0, st()))
    return timeit(fn)


B = 64
for keys in (64, 86, 107, 128, 160, 214):
    ts, tc = dattn(B, keys, True), dattn(B, keys, False)
    print("B=%d keys %4d: self (bias) %7.1f us  cross %7.1f us  ratio %.3f" % (B, keys, ts * 1e6, tc * 1e6, ts / tc))
even = dattn(B, 107, True) + dattn(B, 107, False)
real = dattn(B, 86, True) + dattn(B, 128, False)
print("even split 107+107: %.1f us   task-T split 86 self + 128 cross: %.1f us   real/even %.3f" % (
    even * 1e6, real * 1e6, real / even))
# raggedness: the same total keys as uniform rows vs spread rows (task T's self
# keys ~ U(1..2*86), cross keys ~ the input PMF)
rng = np.random.default_rng(0)
for mean in (86, 128, 214):
    rag = list(np.clip(rng.integers(1, 2 * mean, size=B), 1, 511))
    rag = [int(x) for x in rag]
    tu = dattn(B, int(round(np.mean(rag))), False)
    tr = dattn(B, 0, False, ragged=rag)
    print("B=%d mean keys %.0f: uniform %7.1f us  ragged (1..%d) %7.1f us  ragged/uniform %.3f" % (
        B, np.mean(rag), tu * 1e6, 2 * mean, tr * 1e6, tr / tu))
