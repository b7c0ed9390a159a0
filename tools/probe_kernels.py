"""Kernel timing probe at the workload's shapes (OPT-13B, task S): prefill
GEMMs, decode GEMMs, decode attention, prefill attention.  Prints achieved
TFLOP/s or GB/s per kernel (CUDA events, L2 flushed between reps)."""
import math
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_07947_b200 import _lib as L  # noqa: E402
L.LIB_PATH = os.environ.get("EXG_PROBE_LIB", L.LIB_PATH)   # A/B against another build

dev = torch.device("cuda:0")
st = lambda: torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 * 1024 * 1024, dtype=torch.int8, device=dev)


def timeit(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        flush.sum()          # read-only L2 flush: leaves no dirty lines to write back
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return float(np.median(ts))


def gemm(tokens, features, K, decode, mode=0):
    X = torch.randn(tokens, K, device=dev).to(torch.bfloat16)
    W0 = (torch.randn(features, K, device=dev) * 0.02).to(torch.bfloat16)
    W = torch.empty(int(L.lib().exg_op_blocked_elems(features, K)), dtype=torch.bfloat16, device=dev)
    L.check(L.lib().exg_op_pack_weight(W.data_ptr(), W0.data_ptr(), features, K, K, st()))
    out = torch.zeros(tokens, features, device=dev, dtype=torch.float32 if mode in (2, 3) else torch.bfloat16)
    nws = int(L.lib().exg_op_decode_workspace(features, K, tokens)) if decode else 0
    ws = torch.zeros(max(nws, 1), device=dev, dtype=torch.float32)   # fixup counters start at 0
    resid = out.data_ptr() if mode == 2 else None
    split = nws

    def fn():
        L.check(L.lib().exg_op_linear(X.data_ptr(), K, W.data_ptr(), tokens, features, K, mode, 0, None,
                                      out.data_ptr(), features, resid, features, int(decode), ws.data_ptr(), nws,
                                      st()))
    t = timeit(fn)
    flops = 2.0 * tokens * features * K
    byts = 2.0 * (features * K + tokens * K + tokens * features)
    print("gemm %s T=%5d N=%5d K=%5d split=%d: %8.1f us  %7.1f TFLOP/s  %7.1f GB/s" %
          ("dec" if decode else "pre", tokens, features, K, split, t * 1e6, flops / t / 1e12, byts / t / 1e9))


def pgemm_ab(tokens, features, K, mode=0, reps_sus=0):
    """Prefill GEMM: CTA-pair kernel vs the 1-CTA kernel (diagnostics flag
    bit 6): time both, and compare their outputs bit for bit."""
    X = torch.randn(tokens, K, device=dev).to(torch.bfloat16)
    W0 = (torch.randn(features, K, device=dev) * 0.02).to(torch.bfloat16)
    W = torch.empty(int(L.lib().exg_op_blocked_elems(features, K)), dtype=torch.bfloat16, device=dev)
    L.check(L.lib().exg_op_pack_weight(W.data_ptr(), W0.data_ptr(), features, K, K, st()))
    bias = (torch.randn(features, device=dev) * 0.1).to(torch.bfloat16)
    outs = {}
    for flag in (64, 0):
        L.lib().exg_diag_gemm_flags(flag)
        out = torch.zeros(tokens, features, device=dev, dtype=torch.float32 if mode in (2, 3) else torch.bfloat16)
        resid = out.data_ptr() if mode == 2 else None

        def fn():
            L.check(L.lib().exg_op_linear(X.data_ptr(), K, W.data_ptr(), tokens, features, K, mode, 1,
                                          bias.data_ptr(), out.data_ptr(), features, resid, features, 0, None, 0,
                                          st()))
        if mode == 2:
            out.zero_()
        fn()
        torch.cuda.synchronize()
        outs[flag] = out.clone()
        t = timeit(fn)
        flops = 2.0 * tokens * features * K
        line = "pgemm %s T=%5d N=%5d K=%5d mode %d: %8.1f us %7.1f TFLOP/s" % (
            "1cta" if flag else "pair", tokens, features, K, mode, t * 1e6, flops / t / 1e12)
        if reps_sus:
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps_sus):
                fn()
            b.record()
            torch.cuda.synchronize()
            ts = a.elapsed_time(b) * 1e-3 / reps_sus
            line += "  sustained x%d: %8.1f us %7.1f TFLOP/s" % (reps_sus, ts * 1e6, flops / ts / 1e12)
        print(line, flush=True)
    L.lib().exg_diag_gemm_flags(0)
    if mode == 2:
        print("   (resid mode: accumulated over different rep counts, not compared)")
    else:
        same = torch.equal(outs[0], outs[64])
        print("   pair == 1cta bitwise:", same, " max |diff|", float((outs[0].float() - outs[64].float()).abs().max()))


def dattn(B, c, H=40, dh=128, split_len=512):
    max_ctx = ((c + 63) // 64) * 64
    kc = torch.randn(B, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    vc = torch.randn(B, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    q = torch.randn(B, 3 * H * dh, device=dev).to(torch.bfloat16)
    slot = torch.arange(B, dtype=torch.int32, device=dev)
    nk = torch.full((B,), c, dtype=torch.int32, device=dev)
    ms = (c + split_len - 1) // split_len
    part = torch.empty(B * H * ms * (dh + 2), device=dev)
    out = torch.empty(B, H * dh, device=dev, dtype=torch.bfloat16)

    def fn():
        L.check(L.lib().exg_op_decode_attention(q.data_ptr(), 3 * H * dh, kc.data_ptr(), vc.data_ptr(),
                                                slot.data_ptr(), nk.data_ptr(), out.data_ptr(), H * dh, B, H, dh,
                                                max_ctx, 0.0883883, split_len, ms, part.data_ptr(), None, 0, 0, st()))
    t = timeit(fn)
    byts = B * H * (2.0 * c * dh * 2 + 2 * dh * 2)
    print("decode-attn B=%4d c=%5d H=%d: %8.1f us  %7.1f GB/s" % (B, c, H, t * 1e6, byts / t / 1e9))


def dattn_mix(B, split_len=512, H=40, dh=128, seed=0):
    """Decode attention at the bench's context mix: row contexts n + u with n
    from task S's input PMF and u uniform in the output range."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from workload import task_dists
    d = task_dists("S")
    rng = np.random.default_rng(seed)
    n = rng.choice(np.arange(1, len(d.pmf_in) + 1), size=B, p=np.asarray(d.pmf_in) / np.sum(d.pmf_in))
    u = rng.integers(1, 40, size=B)
    ctxs = (n + u).astype(np.int32)
    max_ctx = 592
    kc = torch.randn(B, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    vc = torch.randn(B, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    q = torch.randn(B, 3 * H * dh, device=dev).to(torch.bfloat16)
    slot = torch.arange(B, dtype=torch.int32, device=dev)
    nk = torch.from_numpy(ctxs).to(dev)
    ms = (int(ctxs.max()) + split_len - 1) // split_len
    part = torch.empty(B * H * ms * (dh + 2), device=dev)
    out = torch.empty(B, H * dh, device=dev, dtype=torch.bfloat16)

    def fn():
        L.check(L.lib().exg_op_decode_attention(q.data_ptr(), 3 * H * dh, kc.data_ptr(), vc.data_ptr(),
                                                slot.data_ptr(), nk.data_ptr(), out.data_ptr(), H * dh, B, H, dh,
                                                max_ctx, 0.0883883, split_len, ms, part.data_ptr(), None, 0, 0, st()))
    t = timeit(fn)
    byts = H * (2.0 * ctxs.sum() * dh * 2 + B * 2 * dh * 2)
    print("decode-attn mix B=%4d mean ctx %5.0f split %4d: %8.1f us  %7.1f GB/s" % (B, ctxs.mean(), split_len,
                                                                                    t * 1e6, byts / t / 1e9))


def pattn(R, n, H=40, dh=128):
    T = R * n
    max_ctx = n
    kc = torch.randn(R, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    vc = torch.randn(R, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    q = torch.randn(T, 3 * H * dh, device=dev).to(torch.bfloat16)
    cu = torch.arange(0, T + 1, n, dtype=torch.int32, device=dev)
    slot = torch.arange(R, dtype=torch.int32, device=dev)
    p0 = torch.zeros(R, dtype=torch.int32, device=dev)
    out = torch.empty(T, H * dh, device=dev, dtype=torch.bfloat16)

    def fn():
        L.check(L.lib().exg_op_prefill_attention(q.data_ptr(), 3 * H * dh, kc.data_ptr(), vc.data_ptr(),
                                                 cu.data_ptr(), slot.data_ptr(), p0.data_ptr(), R, n, out.data_ptr(),
                                                 H * dh, H, dh, max_ctx, R, T, 0.0883883, 1, None, 0, 0, st()))
    t = timeit(fn)
    flops = 4.0 * H * dh * R * n * (n + 1) / 2
    print("prefill-attn R=%d n=%d: %8.1f us  %7.1f TFLOP/s" % (R, n, t * 1e6, flops / t / 1e12))


def pattn_mix(R, H=40, dh=128, seed=0):
    """Prefill attention at the task-S input-length mix (R requests)."""
    from workload import make_requests, task_dists
    d = task_dists("S")
    lens = [max(1, r.input_len - 1) for r in make_requests(R, d.pmf_in, d.pmf_out, 50272, 0xE6E10002 + seed)]
    T, max_ctx = sum(lens), max(lens)
    kc = torch.randn(R, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    vc = torch.randn(R, H, max_ctx, dh, device=dev).to(torch.bfloat16)
    q = torch.randn(T, 3 * H * dh, device=dev).to(torch.bfloat16)
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32, device=dev)
    slot = torch.arange(R, dtype=torch.int32, device=dev)
    p0 = torch.zeros(R, dtype=torch.int32, device=dev)
    out = torch.empty(T, H * dh, device=dev, dtype=torch.bfloat16)

    def fn():
        L.check(L.lib().exg_op_prefill_attention(q.data_ptr(), 3 * H * dh, kc.data_ptr(), vc.data_ptr(),
                                                 cu.data_ptr(), slot.data_ptr(), p0.data_ptr(), R, max_ctx,
                                                 out.data_ptr(), H * dh, H, dh, max_ctx, R, T, 0.0883883, 1, None, 0,
                                                 0, st()))
    t = timeit(fn)
    flops = sum(4.0 * H * dh * n * (n + 1) / 2 for n in lens)
    print("prefill-attn mix R=%d mean n %.0f: %8.1f us  %7.1f TFLOP/s  %7.1f GB/s (q,k,v,o)" % (
        R, T / R, t * 1e6, flops / t / 1e12, 4.0 * T * H * dh * 2 / t / 1e9))


def stream_probe():
    """HBM ceiling of the bulk-copy ring (no MMA): 148..592 CTAs x chunk x stages."""
    import ctypes
    f = L.lib().exg_diag_stream_probe
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                  ctypes.c_void_p]
    buf = torch.zeros(1 << 30, dtype=torch.uint8, device=dev)
    sink = torch.zeros(1, dtype=torch.int32, device=dev)
    for total in (1 << 30, 157286400, 52428800):
        for ctas, chunk, stages in ((148, 16384, 8), (148, 32768, 6), (296, 16384, 6), (444, 16384, 4)):
            per = (total // ctas) // chunk * chunk
            t = timeit(lambda: f(buf.data_ptr(), per, ctas, chunk, stages, sink.data_ptr(), st()))
            print("stream %4d MB ctas=%d chunk=%d stages=%d: %6.1f us %.1f GB/s" %
                  (total >> 20, ctas, chunk, stages, t * 1e6, per * ctas / t / 1e9))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "gemm":
        T, N, K = map(int, sys.argv[2:5])
        gemm(T, N, K, sys.argv[5] == "dec", int(sys.argv[6]) if len(sys.argv) > 6 else 0)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "nomma":
        for flags in (0, 1):
            L.lib().exg_diag_gemm_flags(flags)
            print("flags", flags)
            for B in (16, 64):
                gemm(B, 15360, 5120, True)
                gemm(B, 5120, 5120, True, 2)
                gemm(B, 5120, 20480, True, 2)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "stream":
        stream_probe()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "dattn":
        dattn(int(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "slab":
        for mb in (16, 32, 48, 64, 96):
            L.lib().exg_diag_gemm_slab_mb(mb)
            print("A slab MB", mb)
            for T in (4096, 8192, 16384):
                gemm(T, 15360, 5120, False)
                gemm(T, 20480, 5120, False)
                gemm(T, 5120, 20480, False, 2)
        L.lib().exg_diag_gemm_slab_mb(32)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "skctas":
        for cap in (148, 120, 100, 74):
            L.lib().exg_diag_gemm_sk_ctas(cap)
            print("stream-K CTAs", cap)
            for T in (16, 64):
                gemm(T, 15360, 5120, True)
                gemm(T, 5120, 5120, True, 2)
                gemm(T, 20480, 5120, True)
                gemm(T, 5120, 20480, True, 2)
        L.lib().exg_diag_gemm_sk_ctas(0)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "dmix":
        for stages in (int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,27,1,16,4").split(",")):
            L.lib().exg_diag_decode_stages(stages)
            print("stages", stages)
            for B in (16, 56, 79, 256):
                dattn_mix(B, 512)
        L.lib().exg_diag_decode_stages(0)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pgemm":
        d, ff = 5120, 20480
        for T in (12544, 8192, 300):
            pgemm_ab(T, 3 * d, d, 0, 200 if T == 12544 else 0)
            pgemm_ab(T, d, d, 0)
            pgemm_ab(T, ff, d, 1 if False else 0, 100 if T == 12544 else 0)
            pgemm_ab(T, d, ff, 0)
        pgemm_ab(1000, 300, 512, 0)
        pgemm_ab(777, 1024, 5120, 2)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pmix":
        for R in (8, 32, 52, 64):
            pattn_mix(R)
        for R, n in ((16, 256), (16, 512), (8, 1024), (64, 128)):
            pattn(R, n)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pmix_pf":
        # A/B of the FMHA's L2 prefetch distance (exg_diag_fmha_prefetch)
        for ahead in (0, 1, 2, 4):
            L.lib().exg_diag_fmha_prefetch(ahead)
            print("-- FMHA L2 prefetch ahead = %d" % ahead)
            for R in (32, 52):
                pattn_mix(R)
            pattn(32, 256)
        L.lib().exg_diag_fmha_prefetch(2)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pmix_pt":
        # A/B of the FMHA's P buffer: shared memory (0) vs TMEM (1) (exg_diag_fmha_p_tmem)
        for rep in range(2):
            for on in (0, 1):
                L.lib().exg_diag_fmha_p_tmem(on)
                print("-- FMHA P in %s" % ("TMEM" if on else "shared memory"))
                for R in (32, 52):
                    pattn_mix(R)
                pattn(32, 256)
        L.lib().exg_diag_fmha_p_tmem(1)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "pattn":
        pattn(int(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    d, ff = 5120, 20480
    for T in (2048, 8192):
        gemm(T, 3 * d, d, False)
        gemm(T, d, d, False, 2)
        gemm(T, ff, d, False)
        gemm(T, d, ff, False, 2)
    for B in (16, 64, 256):
        gemm(B, 3 * d, d, True)
        gemm(B, d, d, True, 2)
        gemm(B, ff, d, True)
        gemm(B, d, ff, True, 2)
        gemm(B, 50272, d, True, 3)
    for B, c in ((64, 300), (256, 300), (256, 592), (16, 1600)):
        dattn(B, c)
    pattn(16, 256)
    pattn(8, 512)

