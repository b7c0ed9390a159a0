"""Seeded synthetic inputs shared by the oracle and the product path.

This module holds NO arithmetic of the method (no attention, no GEMM, no
scheduling math).  It only describes the workload the paper evaluates on:

* model shapes (Table 1; SURVEY.md §8 model table),
* the task length distributions of Table 3 as discrete PMFs
  -- the paper's "given distributions P_E and P_D" are INPUTS to
  the scheduler, so building them is input modelling, not the method,
* seeded request generation.

Both `oracle/` and the CUDA path consume what this module returns; neither
side's arithmetic lives here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def splitmix64_np(z: np.ndarray) -> np.ndarray:
    """Vigna's splitmix64 finaliser on the state after one golden-ratio step.

    z is uint64; arithmetic wraps mod 2**64 (numpy uint64 semantics)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


# ----------------------------------------------------------------------------
# Model shapes (Table 1; OPT-66B public shape; tiny per config 1)
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class ModelSpec:
    name: str
    arch: str            # "gpt3" (GELU-tanh), "opt" (ReLU), "t5"
    n_enc_layers: int
    n_dec_layers: int
    d_model: int
    n_heads: int
    d_head: int
    d_ff: int
    vocab: int
    max_pos: int

    @property
    def inner(self) -> int:
        return self.n_heads * self.d_head


MODELS = {
    # config 1 (BASELINE.json configs[0]); SURVEY.md §8(c) T1 "tiny"
    "tiny": ModelSpec("tiny", "gpt3", 0, 2, 64, 4, 16, 256, 512, 64),
    # PAPER.md:417 (OPT 13B: 40 layers, hidden 5120, 40 heads); FFN=4d, V=50272
    "opt-13b": ModelSpec("opt-13b", "opt", 0, 40, 5120, 40, 128, 20480, 50272, 2048),
    # not in the paper; public OPT-66B shape
    "opt-66b": ModelSpec("opt-66b", "opt", 0, 64, 9216, 72, 128, 36864, 50272, 2048),
    # PAPER.md:421 (GPT-3 175B: 96 layers, 12288 hidden, 96 heads)
    "gpt3-175b": ModelSpec("gpt3-175b", "gpt3", 0, 96, 12288, 96, 128, 49152, 50257, 2048),
    # PAPER.md:415 (T5 11B: 48 layers = 24 enc + 24 dec, hidden 1024, 128 heads)
    "t5-11b": ModelSpec("t5-11b", "t5", 24, 24, 1024, 128, 128, 65536, 32128, 2048),
    # encoder-decoder parity cases (T5 architecture at config-1 scale; the
    # dh=128 one exercises the tensor-core attention paths)
    "tiny-t5": ModelSpec("tiny-t5", "t5", 2, 2, 64, 4, 16, 256, 512, 64),
    "small-t5": ModelSpec("small-t5", "t5", 2, 2, 256, 2, 128, 512, 512, 256),
}


# ----------------------------------------------------------------------------
# Table 3 task distributions
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class Task:
    name: str
    in_avg: float
    in_std: float
    in_max: int
    out_avg: float
    out_std: float
    out_p99: int       # printed 99th percentile, used as the latency target length
    out_max: int


TASKS = {
    "S": Task("S", 256, 252, 512, 32, 13, 63, 80),
    "T": Task("T", 128, 81, 256, 128, 68, 292, 320),
    "G": Task("G", 64, 23, 128, 192, 93, 417, 480),
    "C1": Task("C1", 256, 115, 512, 64, 30, 137, 160),
    "C2": Task("C2", 512, 252, 1024, 256, 134, 579, 640),
}


def _phi(z: float) -> float:
    """Standard normal CDF via glibc erfc (deterministic)."""
    return 0.5 * math.erfc(-z / math.sqrt(2.0))


def truncnorm_pmf(mu: float, sigma: float, max_len: int) -> np.ndarray:
    """Discretised truncated normal on [1, max_len].

    Cell k receives the normal mass of (k-1/2, k+1/2]; truncation at 1/2 and
    max_len+1/2; renormalised.  Returns prob[k-1] = P(len = k), float64."""
    if sigma <= 0 or max_len < 1:
        raise ValueError("sigma must be > 0 and max_len >= 1")
    edges = [_phi((k - 0.5 - mu) / sigma) for k in range(1, max_len + 2)]
    cells = np.array([edges[i + 1] - edges[i] for i in range(max_len)], dtype=np.float64)
    total = 0.0
    for c in cells:
        total += c
    if not total > 0.0:
        # mass far outside the support: degenerate to the nearest end
        cells = np.zeros(max_len)
        cells[min(max(int(round(mu)), 1), max_len) - 1] = 1.0
        return cells
    return cells / total


def uniform_pmf(lo: int, hi: int, max_len: Optional[int] = None) -> np.ndarray:
    max_len = hi if max_len is None else max_len
    p = np.zeros(max_len, dtype=np.float64)
    p[lo - 1:hi] = 1.0 / (hi - lo + 1)
    return p


def pmf_mean(p: np.ndarray) -> float:
    k = np.arange(1, len(p) + 1, dtype=np.float64)
    return float(np.dot(k, p))


def pmf_std(p: np.ndarray) -> float:
    k = np.arange(1, len(p) + 1, dtype=np.float64)
    m = float(np.dot(k, p))
    return math.sqrt(max(float(np.dot((k - m) ** 2, p)), 0.0))


def _trunc_moments(mu0: float, s0: float, max_len: int) -> Tuple[float, float]:
    p = truncnorm_pmf(mu0, s0, max_len)
    return pmf_mean(p), pmf_std(p)


def fit_reading_b(mean: float, std: float, max_len: int) -> Tuple[float, float]:
    """Underlying (mu0, sigma0) whose *truncated, discretised* PMF has the
    table's mean and std (SURVEY.md §8(c) S1 'Reading B').  Damped Newton on
    the two moment equations, deterministic start at the table values."""
    mu0, s0 = float(mean), float(std)
    for _ in range(100):
        m, s = _trunc_moments(mu0, s0, max_len)
        f = np.array([m - mean, s - std])
        if abs(f[0]) < 1e-10 and abs(f[1]) < 1e-10:
            break
        h = 1e-4
        m1, s1 = _trunc_moments(mu0 + h, s0, max_len)
        m2, s2 = _trunc_moments(mu0, s0 + h, max_len)
        J = np.array([[(m1 - m) / h, (m2 - m) / h], [(s1 - s) / h, (s2 - s) / h]])
        step = np.linalg.solve(J, f)
        lam = 1.0
        while lam > 1e-4:
            nm, ns = mu0 - lam * step[0], s0 - lam * step[1]
            if ns > 0:
                mm, ss = _trunc_moments(nm, ns, max_len)
                if abs(mm - mean) + abs(ss - std) < abs(f[0]) + abs(f[1]):
                    mu0, s0 = nm, ns
                    break
            lam *= 0.5
        else:
            break
    return mu0, s0


def truncnorm_quantile(mu0: float, s0: float, max_len: int, q: float) -> float:
    """Continuous quantile of N(mu0, s0^2) truncated to [0.5, max_len+0.5]."""
    lo_c, hi_c = _phi((0.5 - mu0) / s0), _phi((max_len + 0.5 - mu0) / s0)
    target = lo_c + q * (hi_c - lo_c)
    a, b = 0.5, max_len + 0.5
    for _ in range(200):
        m = 0.5 * (a + b)
        if _phi((m - mu0) / s0) < target:
            a = m
        else:
            b = m
    return 0.5 * (a + b)


@dataclass
class TaskDists:
    task: str
    pmf_in: np.ndarray      # Reading A
    pmf_out: np.ndarray     # Reading B
    mu0: float
    sigma0: float
    target_len: int         # Table 3's 99th column


_TASK_CACHE = {}


def task_dists(task: str) -> TaskDists:
    """Input PMF: Reading A (table values as the underlying normal).
    Output PMF: Reading B (fitted so the truncated PMF has the table's
    mean/std).  SURVEY.md §8(c) S1."""
    if task in _TASK_CACHE:
        return _TASK_CACHE[task]
    t = TASKS[task]
    pin = truncnorm_pmf(t.in_avg, t.in_std, t.in_max)
    mu0, s0 = fit_reading_b(t.out_avg, t.out_std, t.out_max)
    pout = truncnorm_pmf(mu0, s0, t.out_max)
    d = TaskDists(task, pin, pout, mu0, s0, t.out_p99)
    _TASK_CACHE[task] = d
    return d


# ----------------------------------------------------------------------------
# Requests
# ----------------------------------------------------------------------------
@dataclass
class Request:
    ids: np.ndarray     # int32 [input_len]
    input_len: int
    output_len: int


def _inv_cdf(pmf: np.ndarray, u: float) -> int:
    c = 0.0
    for k, p in enumerate(pmf):
        c += p
        if c >= u:
            return k + 1
    return len(pmf)


def make_requests(n: int, pmf_in: np.ndarray, pmf_out: np.ndarray, vocab: int,
                  seed: int, max_pos: Optional[int] = None) -> List[Request]:
    """n requests; lengths by inverse CDF on a 53-bit hash uniform, ids by
    multiply-shift of a hash stream.  Input and output lengths independent
    (PAPER.md:363)."""
    reqs = []
    idx = np.arange(n, dtype=np.uint64)
    seed = np.uint64(seed & MASK64)
    h_in = splitmix64_np(seed ^ (np.uint64(1) << np.uint64(40)) ^ idx)
    h_out = splitmix64_np(seed ^ (np.uint64(2) << np.uint64(40)) ^ idx)
    for r in range(n):
        u_in = float(int(h_in[r]) >> 11) * 2.0 ** -53
        u_out = float(int(h_out[r]) >> 11) * 2.0 ** -53
        nin = _inv_cdf(pmf_in, u_in)
        nout = _inv_cdf(pmf_out, u_out)
        if max_pos is not None and nin + nout > max_pos:
            nin = max(1, max_pos - nout)
        j = (np.uint64(r) << np.uint64(20)) + np.arange(nin, dtype=np.uint64)
        h = splitmix64_np(seed ^ (np.uint64(3) << np.uint64(40)) ^ j)
        ids = (((h >> np.uint64(32)) * np.uint64(vocab)) >> np.uint64(32)).astype(np.int32)
        reqs.append(Request(ids, nin, nout))
    return reqs


def config1_requests(seed: int = 0xE6E10001) -> List[Request]:
    """Config 1: 8 requests, n ~ U{16..32}, S ~ U{1..24}, ids U[0,512)."""
    return make_requests(8, uniform_pmf(16, 32), uniform_pmf(1, 24), 512, seed)


# weight seeds (0xE6E0_0000 + config#)
def weight_seed(config: int) -> int:
    return 0xE6E00000 + config


def request_seed(config: int) -> int:
    return 0xE6E10000 + config
