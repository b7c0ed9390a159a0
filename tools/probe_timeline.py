"""Per-CTA timeline of one decode GEMM launch (globaltimer marks, exg_diag_gemm
flag bit 2): where the time of a launch goes -- ramp, first data, mainloop,
epilogue / stream-K fixup, exit.

    python tools/probe_timeline.py T N K [mode]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_07947_b200 import _lib as L  # noqa: E402
L.LIB_PATH = os.environ.get("EXG_PROBE_LIB", L.LIB_PATH)   # A/B against another build

dev = torch.device("cuda:0")
st = lambda: torch.cuda.current_stream().cuda_stream
MARKS = ["entry", "setup", "griddep", "first_full", "last_commit", "epi_done", "exit"]


def run(T, N, K, mode=0):
    X = torch.randn(T, K, device=dev).to(torch.bfloat16)
    W0 = (torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16)
    W = torch.empty(int(L.lib().exg_op_blocked_elems(N, K)), dtype=torch.bfloat16, device=dev)
    L.check(L.lib().exg_op_pack_weight(W.data_ptr(), W0.data_ptr(), N, K, K, st()))
    out = torch.zeros(T, N, device=dev, dtype=torch.float32 if mode in (2, 3) else torch.bfloat16)
    nws = int(L.lib().exg_op_decode_workspace(N, K, T))
    ws = torch.zeros(max(nws, 1), device=dev, dtype=torch.float32)
    resid = out.data_ptr() if mode == 2 else None
    flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
    lib = L.lib()
    lib.exg_diag_gemm_timeline.argtypes = [C.c_void_p]

    def fn():
        L.check(lib.exg_op_linear(X.data_ptr(), K, W.data_ptr(), T, N, K, mode, 0, None, out.data_ptr(), N, resid, N,
                                  1, ws.data_ptr(), nws, st()))
    fn()
    lib.exg_diag_gemm_flags(4 | int(os.environ.get("EXG_EXTRA_FLAGS", "0")))   # e.g. 128: no early fixup
    for rep in range(3):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        tl = np.zeros(256 * 8, dtype=np.uint64)
        lib.exg_diag_gemm_timeline(tl.ctypes.data)
        tl = tl.reshape(256, 8)
        rows = tl[:, 0] > 0
        t = tl[rows, :7].astype(np.float64)
        t0 = t[:, 0].min()
        t = (t - t0) / 1e3
        print("T=%d N=%d K=%d mode=%d rep %d: event %.1f us, CTAs %d" % (T, N, K, mode, rep, a.elapsed_time(b) * 1e3,
                                                                          rows.sum()))
        for k, m in enumerate(MARKS):
            v = t[:, k]
            print("   %-12s min %7.2f  med %7.2f  max %7.2f us" % (m, v.min(), np.median(v), v.max()))
    lib.exg_diag_gemm_flags(0)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    if a:
        run(*a)
    else:
        for T, N, K, mode in ((64, 20480, 5120, 0), (64, 5120, 5120, 2), (64, 5120, 20480, 2), (16, 15360, 5120, 0)):
            run(T, N, K, mode)
