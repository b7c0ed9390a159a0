"""In-situ decode GEMM launch spans (earliest CTA entry -> latest CTA exit,
%globaltimer) with PDL active, OPT-13B RRA: per position of the decode
iteration (QKV, O, FFN1, FFN2 of each layer, LM head) the median duration, the
achieved weight bandwidth, and the gap to the previous GEMM (which contains the
LayerNorm / KV scatter / attention kernels in between).
    python tools/probe_spans.py [n_requests]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_07947_b200 as X  # noqa: E402
from workload import MODELS, make_requests, task_dists, weight_seed  # noqa: E402

spec = MODELS["opt-13b"]
d = task_dists("S")
ctx = X.Context(spec, weight_seed(2))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reqs = make_requests(n, d.pmf_in, d.pmf_out, spec.vocab, 0xE6E10002)
ctx.run(X.rra_schedule(24, 79, 9), reqs, slot_ctx=592)   # warm
lib = X.lib()
lib.exg_diag_gemm_spans.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
lib.exg_diag_gemm_spans_reset()
lib.exg_diag_gemm_flags(16)
toks, lat, st, _ = ctx.run(X.rra_schedule(24, 79, 9), reqs, slot_ctx=592)
lib.exg_diag_gemm_flags(0)
lo = np.zeros(4096, dtype=np.uint64)
hi = np.zeros(4096, dtype=np.uint64)
dep = np.zeros(4096, dtype=np.uint64)
cnt = lib.exg_diag_gemm_spans(lo.ctypes.data, hi.ctypes.data, dep.ctypes.data)
cnt = min(cnt, 4096)
lo, hi, dep = lo[:cnt].astype(np.float64), hi[:cnt].astype(np.float64), dep[:cnt].astype(np.float64)
dur = (hi - dep) / 1e3          # dependency resolved -> last CTA exit
pre = (dep - lo) / 1e3          # first CTA resident -> dependency resolved (overlapped with the predecessor)
per_it = 4 * spec.n_dec_layers + 1
d_, K, ff, V = spec.d_model, spec.d_model, spec.d_ff, spec.vocab
wbytes = [2 * 3 * d_ * K, 2 * d_ * d_, 2 * ff * d_, 2 * d_ * ff]
names = ["QKV", "O", "FFN1", "FFN2"]
iters = cnt // per_it
print("decode GEMM launches recorded %d (%d iterations), run decode_s %.4f iters %d mean batch %.1f" %
      (cnt, iters, st["decode_s"], st["decode_iters"], st["mean_decode_batch"]))
tot_gemm = tot_gap = 0.0
for k in range(4):
    idx = np.array([it * per_it + l * 4 + k for it in range(iters) for l in range(spec.n_dec_layers)])
    dd = dur[idx]
    j = idx[idx > 0]
    gap = (dep[j] - hi[j - 1]) / 1e3    # previous GEMM's exit -> this one's dependency resolved
    tot_gemm += dd.sum()
    tot_gap += gap.sum()
    print("%-5s dep->exit median %6.1f us p90 %6.1f -> %5.2f TB/s | resident early by %5.1f us | prev GEMM exit -> dep %6.1f us" %
          (names[k], np.median(dd), np.percentile(dd, 90), wbytes[k] / np.median(dd) / 1e6, np.median(pre[idx]),
           np.median(gap)))
hidx = np.array([it * per_it + per_it - 1 for it in range(iters)])
print("head  median %6.1f us  -> %5.2f TB/s" % (np.median(dur[hidx]), 2 * V * d_ / np.median(dur[hidx]) / 1e6))
span = (hi[iters * per_it - 1] - lo[0]) / 1e3
print("window %.1f us: GEMM time %.1f us (%.0f%%), gaps %.1f us" % (span, tot_gemm, 100 * tot_gemm / span, tot_gap))
