"""A/B: a decode GEMM as a one-phase (or n-phase) chain launch vs exg_op_linear."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_07947_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda:0")
st = lambda: torch.cuda.current_stream().cuda_stream
flush = torch.empty(256 << 20, dtype=torch.int8, device=dev)
lib = L.lib()
lib.exg_diag_chain_gemm.restype = C.c_int
lib.exg_diag_chain_gemm.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                    C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_uint, C.c_int, C.c_void_p]


def timeit(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        flush.sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


for T, N, K in ((56, 20480, 5120), (56, 5120, 5120), (56, 5120, 20480)):
    X = torch.randn(T, K, device=dev).to(torch.bfloat16)
    W0 = (torch.randn(N, K, device=dev) * 0.02).to(torch.bfloat16)
    W = torch.empty(int(lib.exg_op_blocked_elems(N, K)), dtype=torch.bfloat16, device=dev)
    L.check(lib.exg_op_pack_weight(W.data_ptr(), W0.data_ptr(), N, K, K, st()))
    out = torch.zeros(T, N, device=dev, dtype=torch.bfloat16)
    nws = int(lib.exg_op_decode_workspace(N, K, T))
    ws = torch.zeros(max(nws, 1), device=dev, dtype=torch.float32)
    t_lin = timeit(lambda: L.check(lib.exg_op_linear(X.data_ptr(), K, W.data_ptr(), T, N, K, 0, 0, None, out.data_ptr(),
                                                     N, None, N, 1, ws.data_ptr(), nws, st())))
    ref = out.clone()
    for n_rep in (1, 2):
        cws_n = lib.exg_diag_chain_gemm(X.data_ptr(), K, W.data_ptr(), T, N, K, out.data_ptr(), N, None, 0, None, 0,
                                        n_rep, st())
        cws = torch.zeros(max(cws_n, 1), device=dev, dtype=torch.float32)
        sync = torch.zeros(16, device=dev, dtype=torch.int32)
        ep = [0]

        def ch():
            ep[0] += 1
            rc = lib.exg_diag_chain_gemm(X.data_ptr(), K, W.data_ptr(), T, N, K, out.data_ptr(), N, cws.data_ptr(),
                                         cws_n, sync.data_ptr(), ep[0], n_rep, st())
            assert rc == 0
        t_ch = timeit(ch)
        same = torch.equal(out, ref)
        print("T=%d N=%d K=%d: linear %.1f us | chain x%d %.1f us (%.1f us per GEMM) identical %s" %
              (T, N, K, t_lin, n_rep, t_ch, t_ch / n_rep, same), flush=True)
