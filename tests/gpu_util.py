"""Helpers for the -m gpu tests: torch CUDA tensors as device memory, and
bf16 <-> numpy conversions.  Test infrastructure only."""
import numpy as np
import torch


def dev():
    return torch.device("cuda:0")


def ptr(t):
    return t.data_ptr() if t is not None else None


def stream():
    return torch.cuda.current_stream().cuda_stream


def bf16_tensor(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).to(dev())


def to_np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def blocked(L, W):
    """Pack a row-major bf16 CUDA matrix [rows][K] into the GEMM blocked
    layout (exg_op_pack_weight); returns the new tensor (keep it alive)."""
    rows, K = W.shape
    out = torch.empty(int(L.lib().exg_op_blocked_elems(rows, K)), dtype=torch.bfloat16, device=W.device)
    L.check(L.lib().exg_op_pack_weight(out.data_ptr(), W.data_ptr(), rows, K, W.stride(0), stream()))
    return out


def bf16_round_np(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy().astype(np.float64)
