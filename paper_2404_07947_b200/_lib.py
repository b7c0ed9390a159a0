"""ctypes binding of libexegpt.so (include/exegpt.h, include/exegpt_ops.h).

Argument marshalling only: every step of the hot path runs inside the
library's sm_100a kernels.  Loading fails loudly if the library is missing;
there is no fallback implementation.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libexegpt.so")

EXG_OK, EXG_E_INPUT, EXG_E_INFEASIBLE, EXG_E_CUDA, EXG_E_NCCL, EXG_E_OOM, EXG_E_INTERNAL = range(7)
EXG_ARCH_OPT, EXG_ARCH_GPT3, EXG_ARCH_T5 = 0, 1, 2
EXG_RRA, EXG_WAA_C, EXG_WAA_M, EXG_STATIC = 1, 2, 4, 8
MAX_STAGES = 8

STATUS_NAMES = {0: "EXG_OK", 1: "EXG_E_INPUT", 2: "EXG_E_INFEASIBLE", 3: "EXG_E_CUDA", 4: "EXG_E_NCCL",
                5: "EXG_E_OOM", 6: "EXG_E_INTERNAL"}


class ExgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status


class exg_model_spec(C.Structure):
    _fields_ = [("arch", C.c_int), ("n_enc_layers", C.c_int32), ("n_dec_layers", C.c_int32),
                ("d_model", C.c_int32), ("n_heads", C.c_int32), ("d_head", C.c_int32), ("d_ff", C.c_int32),
                ("vocab", C.c_int32), ("max_pos", C.c_int32), ("dtype", C.c_int), ("weight_seed", C.c_uint64)]


class exg_cluster_spec(C.Structure):
    _fields_ = [("n_gpus", C.c_int32), ("mem_per_gpu_bytes", C.c_int64), ("workspace_bytes", C.c_int64),
                ("kv_page", C.c_int32)]


class exg_pmf(C.Structure):
    _fields_ = [("max_len", C.c_int32), ("prob", C.POINTER(C.c_double))]


class exg_schedule(C.Structure):
    _fields_ = [("strategy", C.c_int), ("b_e", C.c_int32), ("b_d", C.c_int32), ("b_m", C.c_int32),
                ("n_d", C.c_int32), ("tp_degree", C.c_int32), ("tp_gpus", C.c_int32), ("n_enc_gpus", C.c_int32),
                ("n_stages", C.c_int32), ("stage_first_gpu", C.c_int32 * MAX_STAGES),
                ("stage_n_gpus", C.c_int32 * MAX_STAGES), ("stage_layer_begin", C.c_int32 * MAX_STAGES),
                ("stage_layer_end", C.c_int32 * MAX_STAGES)]

    def stages(self):
        return [(self.stage_first_gpu[k], self.stage_n_gpus[k], self.stage_layer_begin[k], self.stage_layer_end[k])
                for k in range(self.n_stages)]

    def as_dict(self):
        return {"strategy": {1: "RRA", 2: "WAA-C", 4: "WAA-M"}.get(self.strategy, self.strategy),
                "b_e": self.b_e, "b_d": self.b_d, "b_m": self.b_m, "n_d": self.n_d,
                "tp_degree": self.tp_degree, "tp_gpus": self.tp_gpus, "n_enc_gpus": self.n_enc_gpus,
                "stages": self.stages()}


class exg_estimate(C.Structure):
    _fields_ = [("thrput_seq_s", C.c_double), ("thrput_tok_s", C.c_double), ("latency_s", C.c_double),
                ("perf_evals", C.c_int64), ("feasible", C.c_int32)]


class exg_search_opts(C.Structure):
    _fields_ = [("eps_t_frac", C.c_double), ("eps_l_frac", C.c_double), ("b_e_max", C.c_int32),
                ("n_d_max", C.c_int32), ("m_max", C.c_int32), ("use_little_fraction", C.c_int32),
                ("tp_degree_only", C.c_int32)]


class exg_profile_grid(C.Structure):
    _fields_ = [("n_batch", C.c_int32), ("batch", C.POINTER(C.c_int32)), ("n_ctx", C.c_int32),
                ("ctx", C.POINTER(C.c_int32)), ("n_tokens", C.c_int32), ("tokens", C.POINTER(C.c_int32)),
                ("n_tp", C.c_int32), ("tp", C.POINTER(C.c_int32)), ("reps", C.c_int32)]


class exg_request(C.Structure):
    _fields_ = [("input_ids", C.POINTER(C.c_int32)), ("input_len", C.c_int32), ("output_len", C.c_int32)]


class exg_run_opts(C.Structure):
    _fields_ = [("logits_out", C.POINTER(C.c_float)), ("dump_mask", C.POINTER(C.c_uint8)),
                ("slot_ctx", C.c_int32), ("pin_nccl_algo", C.c_int32), ("kernel_timing", C.c_int32),
                ("dyn_threshold", C.c_double), ("trace_out", C.POINTER(C.c_double)), ("trace_cap", C.c_int32),
                ("kv_page", C.c_int32), ("kv_pages", C.c_int32)]


K_CLASSES = ["prefill_gemm", "decode_gemm", "decode_attn", "prefill_attn"]


class exg_run_stats(C.Structure):
    _fields_ = [("tok_s", C.c_double), ("tok_s_steady", C.c_double), ("seq_s", C.c_double),
                ("lat_p50_s", C.c_double), ("lat_p99_s", C.c_double), ("lat_max_s", C.c_double),
                ("wall_s", C.c_double), ("out_tokens", C.c_int64), ("decode_iters", C.c_int64),
                ("encode_phases", C.c_int64), ("mean_decode_batch", C.c_double), ("encode_s", C.c_double),
                ("decode_s", C.c_double), ("kernel_launches", C.c_int64), ("k_time_s", C.c_double * 4),
                ("k_work", C.c_double * 4), ("k_launches", C.c_int64 * 4),
                ("enc_stage_mean_s", C.c_double), ("enc_stage_p99dev_s", C.c_double),
                ("dec_stage_mean_s", C.c_double), ("dec_stage_p99dev_s", C.c_double),
                ("mean_encode_batch", C.c_double), ("trace_records", C.c_int64),
                ("kv_preemptions", C.c_int64), ("kv_pages_peak", C.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if not k.startswith("k_")}
        d["kernels"] = {K_CLASSES[c]: {"time_s": self.k_time_s[c], "work": self.k_work[c],
                                       "launches": self.k_launches[c]} for c in range(4)}
        return d


_P = C.c_void_p
_SIGS = {
    "exg_abi_version": (C.c_int32, []),
    "exg_last_error": (C.c_char_p, []),
    "exg_get_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "exg_create": (C.c_int, [C.POINTER(exg_model_spec), C.POINTER(exg_cluster_spec), C.c_int32, C.c_int32,
                             C.c_int32, C.POINTER(C.c_uint8), C.POINTER(_P)]),
    "exg_destroy": (None, [_P]),
    "exg_create_local_group": (C.c_int, [C.POINTER(exg_model_spec), C.POINTER(exg_cluster_spec), C.c_int32,
                                         C.c_int32, C.POINTER(_P)]),
    "exg_create_nccl_loopback": (C.c_int, [C.POINTER(exg_model_spec), C.POINTER(exg_cluster_spec), C.c_int32,
                                           C.POINTER(_P)]),
    "exg_profile_run": (C.c_int, [_P, C.POINTER(exg_profile_grid), C.POINTER(_P)]),
    "exg_profile_save": (C.c_int, [_P, C.c_char_p]),
    "exg_profile_load": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "exg_profile_free": (None, [_P]),
    "exg_profile_comm_model": (C.c_int, [_P, C.c_double, C.c_double]),
    "exg_profile_copy_comm": (C.c_int, [_P, _P]),
    "exg_profile_stage_time": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                         C.POINTER(C.c_double)]),
    "exg_simulate": (C.c_int, [_P, C.POINTER(exg_model_spec), C.POINTER(exg_cluster_spec), C.POINTER(exg_pmf),
                               C.POINTER(exg_pmf), C.c_int32, C.POINTER(exg_schedule), C.POINTER(exg_estimate)]),
    "exg_schedule_memory": (C.c_int, [_P, C.POINTER(exg_model_spec), C.POINTER(exg_cluster_spec), C.POINTER(exg_pmf),
                                      C.POINTER(exg_pmf), C.POINTER(exg_schedule), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]),
    "exg_schedule_resolve": (C.c_int, [_P, C.POINTER(exg_model_spec), C.POINTER(exg_cluster_spec),
                                       C.POINTER(exg_pmf), C.POINTER(exg_pmf), C.c_int32, C.POINTER(exg_schedule)]),
    "exg_schedule_find": (C.c_int, [_P, C.POINTER(exg_model_spec), C.POINTER(exg_cluster_spec), C.POINTER(exg_pmf),
                                    C.POINTER(exg_pmf), C.c_int32, C.c_double, C.c_uint32,
                                    C.POINTER(exg_search_opts), C.POINTER(exg_schedule), C.POINTER(exg_estimate)]),
    "exg_run": (C.c_int, [_P, C.POINTER(exg_schedule), C.POINTER(exg_request), C.c_int32, C.POINTER(C.c_int32),
                          C.POINTER(C.c_double), C.POINTER(exg_run_stats), C.POINTER(exg_run_opts)]),
    # ops (device pointers as void*)
    "exg_op_weightgen": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_int32,
                                   C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _P]),
    "exg_op_pack_weight": (C.c_int, [_P, _P, C.c_int64, C.c_int64, C.c_int64, _P]),
    "exg_op_blocked_elems": (C.c_int64, [C.c_int64, C.c_int64]),
    "exg_op_linear": (C.c_int, [_P, C.c_int64, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_int32, _P, _P, C.c_int64, _P, C.c_int64, C.c_int32, _P, C.c_int64, _P]),
    "exg_op_layernorm": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _P, _P, C.c_int32, C.c_int32, C.c_float, _P]),
"exg_op_rmsnorm": (C.c_int, [_P, C.c_int64, _P, C.c_int64, _P, C.c_int32, C.c_int32, C.c_float, C.c_float, _P]),
    "exg_op_embed": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int32, _P]),
    "exg_op_kv_scatter": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    "exg_op_decode_attention": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, C.c_int64, C.c_int32, C.c_int32,
                                          C.c_int32, C.c_int32, C.c_float, C.c_int32, C.c_int32, _P,
                                          _P, C.c_int32, C.c_int32, _P]),
    "exg_op_prefill_attention": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, C.c_int32, C.c_int32, _P,
                                           C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_float, C.c_int32, _P, C.c_int32, C.c_int32, _P]),
    "exg_op_decode_attention_paged": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, C.c_int64, C.c_int32,
                                                C.c_int32, C.c_int32, C.c_int32, C.c_float, C.c_int32,
                                                C.c_int32, _P, _P, C.c_int32, C.c_int32, _P, C.c_int32, _P]),
    "exg_op_prefill_attention_paged": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P, _P, C.c_int32, C.c_int32, _P,
                                                 C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                 C.c_int32, C.c_float, C.c_int32, _P, C.c_int32, C.c_int32, _P,
                                                 C.c_int32, _P]),
    "exg_op_argmax": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, _P, _P]),
    "exg_op_decode_workspace": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
}

_lib = None
ABI_VERSION = 5   # include/exegpt.h EXG_ABI_VERSION


def lib():
    """Load libexegpt.so (raises if it is missing: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libexegpt.so not built (%s); run `python -m paper_2404_07947_b200.build`" % LIB_PATH)
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.exg_abi_version() != ABI_VERSION:
            raise ImportError("libexegpt.so ABI %d != binding ABI %d: rebuild" % (L.exg_abi_version(), ABI_VERSION))
        _lib = L
    return _lib


def check(status: int):
    if status != EXG_OK:
        raise ExgError(status, lib().exg_last_error().decode(errors="replace"))


# ---------------------------------------------------------------- helpers --
ARCH_OF = {"opt": EXG_ARCH_OPT, "gpt3": EXG_ARCH_GPT3, "t5": EXG_ARCH_T5}


EXG_BF16, EXG_FP32 = 0, 1


def model_spec(spec, seed: int, dtype: int = EXG_BF16) -> exg_model_spec:
    return exg_model_spec(ARCH_OF[spec.arch], spec.n_enc_layers, spec.n_dec_layers, spec.d_model, spec.n_heads,
                          spec.d_head, spec.d_ff, spec.vocab, spec.max_pos, dtype, seed)


def cluster_spec(n_gpus: int = 1, mem_per_gpu: float = 180e9, workspace: float = 6e9,
                 kv_page: int = 0) -> exg_cluster_spec:
    return exg_cluster_spec(n_gpus, int(mem_per_gpu), int(workspace), int(kv_page))


class Pmf:
    """Keeps the probability array alive while the struct is in use."""

    def __init__(self, prob: Sequence[float]):
        self.arr = np.ascontiguousarray(np.asarray(prob, dtype=np.float64))
        self.c = exg_pmf(len(self.arr), self.arr.ctypes.data_as(C.POINTER(C.c_double)))


def search_opts(eps_t=0.02, eps_l=0.02, b_e_max=256, n_d_max=0, m_max=8, little=False,
                tp_only=0) -> exg_search_opts:
    return exg_search_opts(eps_t, eps_l, b_e_max, n_d_max, m_max, int(little), int(tp_only))


def unique_id() -> bytes:
    """NCCL unique id of a multi-rank group (rank 0; broadcast the bytes)."""
    buf = (C.c_uint8 * 128)()
    check(lib().exg_get_unique_id(buf))
    return bytes(buf)


class Context:
    """One rank's context.  world > 1: one process per GPU, NCCL (uid from
    unique_id() on rank 0); every rank calls run() with identical arguments and
    rank 0 receives the outputs."""

    def __init__(self, spec, seed: int, device: int = 0, cluster: Optional[exg_cluster_spec] = None,
                 rank: int = 0, world: int = 1, uid: Optional[bytes] = None, _handle=None, dtype: int = EXG_BF16):
        self.spec = spec
        self.mspec = model_spec(spec, seed, dtype)
        self.cluster = cluster or cluster_spec()
        self.rank, self.world = rank, world
        if _handle is not None:
            self.h = _handle
            return
        h = _P()
        ubuf = (C.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
        check(lib().exg_create(C.byref(self.mspec), C.byref(self.cluster), device, rank, world, ubuf, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().exg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def profile(self, batch, ctx, tokens, reps: int = 3, tps=(1,)) -> "Profile":
        arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.int32)) for a in (batch, ctx, tokens, tps)]
        ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
        g = exg_profile_grid(len(arrs[0]), ptr(arrs[0]), len(arrs[1]), ptr(arrs[1]), len(arrs[2]), ptr(arrs[2]),
                             len(arrs[3]), ptr(arrs[3]), reps)
        h = _P()
        check(lib().exg_profile_run(self.h, C.byref(g), C.byref(h)))
        return Profile(h)

    def run(self, sched: exg_schedule, requests, dump: Optional[Sequence[int]] = None, slot_ctx: int = 0,
            kernel_timing: bool = False, dyn_threshold: float = 0.0, trace: Optional[list] = None,
            pin_nccl_algo: bool = False, kv_page: int = 0, kv_pages: int = 0):
        """Returns (tokens per request, latencies [s], stats dict, logits per
        dumped request [S_r][V] or None).  trace: a list that receives the
        per-stage records [kind, start, duration, rows, work] (exegpt.h)."""
        n = len(requests)
        keep = []
        reqs = (exg_request * n)()
        for i, r in enumerate(requests):
            ids = np.ascontiguousarray(np.asarray(r.ids, dtype=np.int32))
            keep.append(ids)
            reqs[i] = exg_request(ids.ctypes.data_as(C.POINTER(C.c_int32)), int(r.input_len), int(r.output_len))
        total = sum(int(r.output_len) for r in requests)
        out = np.zeros(total, dtype=np.int32)
        lat = np.zeros(n, dtype=np.float64)
        stats = exg_run_stats()
        opts = exg_run_opts(None, None, slot_ctx, int(pin_nccl_algo), int(kernel_timing), float(dyn_threshold))
        opts.kv_page = int(kv_page)
        opts.kv_pages = int(kv_pages)
        tbuf = None
        if trace is not None:
            cap = 8 * (n + 16) + 4 * total
            tbuf = np.zeros((cap, 5), dtype=np.float64)
            opts.trace_out = tbuf.ctypes.data_as(C.POINTER(C.c_double))
            opts.trace_cap = cap
        logits = None
        if dump is not None:
            mask = np.zeros(n, dtype=np.uint8)
            mask[list(dump)] = 1
            nd = sum(int(requests[i].output_len) for i in dump)
            logits = np.zeros((max(nd, 1), self.spec.vocab), dtype=np.float32)
            keep += [mask, logits]
            opts.logits_out = logits.ctypes.data_as(C.POINTER(C.c_float))
            opts.dump_mask = mask.ctypes.data_as(C.POINTER(C.c_uint8))
        check(lib().exg_run(self.h, C.byref(sched), reqs, n, out.ctypes.data_as(C.POINTER(C.c_int32)),
                            lat.ctypes.data_as(C.POINTER(C.c_double)), C.byref(stats), C.byref(opts)))
        if trace is not None:
            trace.extend(tbuf[:int(stats.trace_records)].tolist())
        toks, off = [], 0
        for r in requests:
            toks.append(out[off:off + r.output_len].tolist())
            off += r.output_len
        dumped = None
        if dump is not None:
            dumped, off = {}, 0
            for i in sorted(dump):
                S = int(requests[i].output_len)
                dumped[i] = logits[off:off + S]
                off += S
        return toks, lat, stats.as_dict(), dumped


def local_group(spec, seed: int, world: int, cluster: Optional[exg_cluster_spec] = None, device: int = 0):
    """`world` rank contexts in this process on one device, joined by the
    device-copy transport (exg_create_local_group); drive them with run_group."""
    cluster = cluster or cluster_spec(world)
    mspec = model_spec(spec, seed)
    hs = (_P * world)()
    check(lib().exg_create_local_group(C.byref(mspec), C.byref(cluster), device, world, hs))
    return [Context(spec, seed, device, cluster, rank=r, world=world, _handle=_P(hs[r])) for r in range(world)]


def nccl_loopback(spec, seed: int, cluster: Optional[exg_cluster_spec] = None, device: int = 0) -> Context:
    """One-rank context whose layout exchanges all go through NCCL (send /
    recv to self): the NCCL transport on a single GPU."""
    cluster = cluster or cluster_spec(8)
    h = _P()
    check(lib().exg_create_nccl_loopback(C.byref(model_spec(spec, seed)), C.byref(cluster), device, C.byref(h)))
    return Context(spec, seed, device, cluster, _handle=h)


def run_group(ctxs, sched: exg_schedule, requests, **kw):
    """Call run() on every rank context from its own thread (the calls are
    collective); returns the per-rank results, rank 0's being authoritative.
    The first rank error is re-raised."""
    import threading
    res = [None] * len(ctxs)
    err = [None] * len(ctxs)

    def go(r):
        try:
            res[r] = ctxs[r].run(sched, requests, **kw)
        except BaseException as e:  # noqa: BLE001 -- reported below
            err[r] = e

    th = [threading.Thread(target=go, args=(r,), daemon=True) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return res


class Profile:
    def __init__(self, h):
        self.h = h

    @classmethod
    def load(cls, path: str) -> "Profile":
        h = _P()
        check(lib().exg_profile_load(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str):
        check(lib().exg_profile_save(self.h, path.encode()))

    def comm_model(self, alpha_s: float, bw_bytes_per_s: float):
        """Fill tp_sync / pp_sync from an alpha-beta interconnect model."""
        check(lib().exg_profile_comm_model(self.h, alpha_s, bw_bytes_per_s))

    def stage_time(self, phase: int, rows: float, work: float, n_layers: int, tp: int = 1) -> float:
        """exg_profile_stage_time: the profile's time of one encode phase (0) /
        decode iteration (1) of a single-GPU stage."""
        out = C.c_double()
        check(lib().exg_profile_stage_time(self.h, phase, tp, n_layers, float(rows), float(work), C.byref(out)))
        return out.value

    def copy_comm(self, other: "Profile"):
        """tp_sync / pp_sync tables from a multi-rank profile (exg_profile_copy_comm)."""
        check(lib().exg_profile_copy_comm(self.h, other.h))

    def __del__(self):
        try:
            if self.h:
                lib().exg_profile_free(self.h)
        except Exception:
            pass


def rra_schedule(b_e: int, b_d: int, n_d: int) -> exg_schedule:
    """A caller-filled single-GPU RRA schedule (config 1 style)."""
    s = exg_schedule()
    s.strategy, s.b_e, s.b_d, s.n_d, s.tp_degree, s.tp_gpus = EXG_RRA, b_e, b_d, n_d, 1, 0
    s.n_stages = 1
    s.stage_first_gpu[0], s.stage_n_gpus[0], s.stage_layer_begin[0], s.stage_layer_end[0] = 0, 1, 0, 0
    return s


def static_schedule(b: int) -> exg_schedule:
    """FasterTransformer-style static batch of b requests on one GPU
    (the in-runner baseline)."""
    s = exg_schedule()
    s.strategy, s.b_e, s.b_d, s.n_d, s.tp_degree, s.tp_gpus = EXG_STATIC, b, b, 0, 1, 0
    s.n_stages = 1
    s.stage_first_gpu[0], s.stage_n_gpus[0], s.stage_layer_begin[0], s.stage_layer_end[0] = 0, 1, 0, 0
    return s


def make_schedule(strategy: int, b_e: int, b_d: int, stages, n_d: int = 0, b_m: int = 0, n_enc_gpus: int = 0,
                  tp_degree: int = 1, tp_gpus: int = 0) -> exg_schedule:
    """A caller-filled multi-stage schedule; stages = [(first_gpu, n_gpus,
    layer_begin, layer_end), ...] (WAA: encoder stages first)."""
    s = exg_schedule()
    s.strategy, s.b_e, s.b_d, s.b_m, s.n_d = strategy, b_e, b_d, b_m, n_d
    s.tp_degree, s.tp_gpus, s.n_enc_gpus, s.n_stages = tp_degree, tp_gpus, n_enc_gpus, len(stages)
    for k, (g, ng, l0, l1) in enumerate(stages):
        s.stage_first_gpu[k], s.stage_n_gpus[k], s.stage_layer_begin[k], s.stage_layer_end[k] = g, ng, l0, l1
    return s


def simulate(prof: Profile, mspec: exg_model_spec, cl: exg_cluster_spec, pin: Pmf, pout: Pmf, target_len: int,
             sched: exg_schedule) -> exg_estimate:
    est = exg_estimate()
    check(lib().exg_simulate(prof.h, C.byref(mspec), C.byref(cl), C.byref(pin.c), C.byref(pout.c), target_len,
                             C.byref(sched), C.byref(est)))
    return est


def schedule_memory(prof: Profile, mspec, cl, pin: Pmf, pout: Pmf, sched: exg_schedule):
    """Per-GPU (model bytes, KV-cache bytes) lists of a schedule
    (exg_schedule_memory)."""
    n = int(cl.n_gpus)
    w, kv = (C.c_double * n)(), (C.c_double * n)()
    check(lib().exg_schedule_memory(prof.h, C.byref(mspec), C.byref(cl), C.byref(pin.c), C.byref(pout.c),
                                    C.byref(sched), w, kv))
    return list(w), list(kv)


def schedule_resolve(prof: Profile, mspec, cl, pin: Pmf, pout: Pmf, sched: exg_schedule, m_count: int = 1):
    check(lib().exg_schedule_resolve(prof.h, C.byref(mspec), C.byref(cl), C.byref(pin.c), C.byref(pout.c),
                                     m_count, C.byref(sched)))
    return sched


def schedule_find(prof: Profile, mspec, cl, pin: Pmf, pout: Pmf, target_len: int, L_b: float, mask: int,
                  opts: Optional[exg_search_opts] = None):
    s, est = exg_schedule(), exg_estimate()
    o = opts or search_opts()
    check(lib().exg_schedule_find(prof.h, C.byref(mspec), C.byref(cl), C.byref(pin.c), C.byref(pout.c), target_len,
                                  L_b, mask, C.byref(o), C.byref(s), C.byref(est)))
    return s, est
