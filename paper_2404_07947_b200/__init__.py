"""B200-native (sm_100a) runner for the decoupled-inference computation that
ExeGPT (arXiv 2404.07947) schedules: encode (prefill) and decode phases run
under an RRA / WAA schedule, behind the C-ABI of libexegpt.so
(include/exegpt.h).  This package is the thin Python binding (ctypes); every
step of the hot path runs in the library's CUDA kernels.
"""
from ._lib import (EXG_BF16, EXG_FP32, EXG_RRA, EXG_STATIC, EXG_WAA_C, EXG_WAA_M, Context, ExgError, Pmf, Profile, cluster_spec, lib,
                   local_group, model_spec, nccl_loopback, rra_schedule, run_group, schedule_find,
                   schedule_memory, schedule_resolve, search_opts, simulate, static_schedule, unique_id)

__all__ = ["EXG_BF16", "EXG_FP32", "EXG_RRA", "EXG_STATIC", "EXG_WAA_C", "EXG_WAA_M", "Context", "ExgError", "Pmf", "Profile", "cluster_spec", "lib",
           "local_group", "model_spec", "nccl_loopback", "rra_schedule", "run_group", "schedule_find", "schedule_memory", "schedule_resolve",
           "search_opts", "simulate", "static_schedule", "unique_id"]
