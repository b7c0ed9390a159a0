"""XSimulator (§6) -- test infrastructure
only.  Plain double-precision arithmetic in a fixed operation order so the C++
planner can match it bit for bit.

Readings (listed in DESIGN.md):
* profile lookups: linear / bilinear interpolation t0+(x-x0)*(t1-t0)/(x1-x0),
  exact on grid points, clamped below the first grid point, out-of-hull above
  the last (=> infeasible);
* layer time = attn + rest + k * tp_sync, k = 2 all-reduces per layer
  (3 for a T5 decoder layer), messages in fp32 (T4(i));
* decode stage time of the last stage + head(b): final norm, LM head and
  argmax once per iteration (profile table `head`, when present);
* RRA timeline via the pipeline algebra F/Pi (S6), P micro-batches;
* WAA timeline (S7): throughput = B_E / max(T_E, T_D); latency =
  T_E^trav + T_handoff + T_E + (S-1) Pi + F;
* partial TP (S8): c GPUs at the pipeline front form c/t TP stages; layers per
  stage proportional to GPUs per stage, remainder one per stage from the front.

Pins: Table 8 rows 3-4 identities (RRA P=1), Fig. 4 "7" and "3 2/3" (WAA
pipeline), pipeline algebra == FIFO event loop (tests/test_oracle_scheduler.py);
simulate_waa vs Table 8 row 1 + Table 9's WAA decoder stage, vs an independent
WAA event loop (throughput equal; latency bracketed, equal for M = 1 with a
draining decoder), the handoff term; waa_split through SPEC.md:235-237 and the
mirror invariant; interp2 on hand values and bilinear closed forms
(tests/test_oracle_pins.py).  The RRA P > 1 timeline is pinned only by the
pipeline algebra identities (Fig. 4a is missing from PAPER.md).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import seqdist

INF = float("inf")


class OutOfHull(Exception):
    pass


# ---------------------------------------------------------------------------
# profile-v1 (D3): attn(phase,tp,batch,ctx), rest(phase,tp,tokens),
# tp_sync(tp,bytes), pp_sync(bytes).  Plain whitespace text, %.17g numbers.
# ---------------------------------------------------------------------------
@dataclass
class Table1D:
    x: List[float]
    t: List[float]


@dataclass
class Table2D:
    b: List[float]
    c: List[float]
    t: List[List[float]]   # t[ib][ic]


@dataclass
class Profile:
    tps: List[int]
    attn: Dict[Tuple[str, int], Table2D] = field(default_factory=dict)
    rest: Dict[Tuple[str, int], Table1D] = field(default_factory=dict)
    tp_sync: Dict[int, Table1D] = field(default_factory=dict)
    pp_sync: Optional[Table1D] = None
    head: Optional[Table1D] = None     # decode head (final norm + LM head + argmax) vs batch
    switch: Optional[Table2D] = None   # cumulative extra time of the first k decode iterations after an encode phase [b][k]

    def save(self, path: str):
        with open(path, "w") as f:
            f.write(self.dumps())

    def dumps(self) -> str:
        g = lambda v: "%.17g" % v
        out = ["profile-v1", "tp %d %s" % (len(self.tps), " ".join(str(t) for t in self.tps))]
        for (ph, tp), tb in sorted(self.attn.items()):
            out.append("attn %s %d %d %d" % (ph, tp, len(tb.b), len(tb.c)))
            out.append(" ".join(g(v) for v in tb.b))
            out.append(" ".join(g(v) for v in tb.c))
            out.append(" ".join(g(v) for row in tb.t for v in row))
        for (ph, tp), tb in sorted(self.rest.items()):
            out.append("rest %s %d %d" % (ph, tp, len(tb.x)))
            out.append(" ".join(g(v) for v in tb.x))
            out.append(" ".join(g(v) for v in tb.t))
        for tp, tb in sorted(self.tp_sync.items()):
            out.append("tp_sync %d %d" % (tp, len(tb.x)))
            out.append(" ".join(g(v) for v in tb.x))
            out.append(" ".join(g(v) for v in tb.t))
        if self.pp_sync is not None:
            out.append("pp_sync %d" % len(self.pp_sync.x))
            out.append(" ".join(g(v) for v in self.pp_sync.x))
            out.append(" ".join(g(v) for v in self.pp_sync.t))
        if self.head is not None:
            out.append("head %d" % len(self.head.x))
            out.append(" ".join(g(v) for v in self.head.x))
            out.append(" ".join(g(v) for v in self.head.t))
        if self.switch is not None:
            out.append("switch %d %d" % (len(self.switch.b), len(self.switch.c)))
            out.append(" ".join(g(v) for v in self.switch.b))
            out.append(" ".join(g(v) for v in self.switch.c))
            out.append(" ".join(g(v) for row in self.switch.t for v in row))
        out.append("end")
        return "\n".join(out) + "\n"

    @classmethod
    def loads(cls, text: str) -> "Profile":
        tok = text.split()
        pos = 0

        def nxt():
            nonlocal pos
            pos += 1
            return tok[pos - 1]

        if nxt() != "profile-v1":
            raise ValueError("not a profile-v1 file")
        assert nxt() == "tp"
        n = int(nxt())
        p = cls([int(nxt()) for _ in range(n)])
        while True:
            kw = nxt()
            if kw == "end":
                return p
            if kw == "attn":
                ph, tp, nb, nc = nxt(), int(nxt()), int(nxt()), int(nxt())
                b = [float(nxt()) for _ in range(nb)]
                c = [float(nxt()) for _ in range(nc)]
                t = [[float(nxt()) for _ in range(nc)] for _ in range(nb)]
                p.attn[(ph, tp)] = Table2D(b, c, t)
            elif kw == "rest":
                ph, tp, n = nxt(), int(nxt()), int(nxt())
                x = [float(nxt()) for _ in range(n)]
                p.rest[(ph, tp)] = Table1D(x, [float(nxt()) for _ in range(n)])
            elif kw == "tp_sync":
                tp, n = int(nxt()), int(nxt())
                x = [float(nxt()) for _ in range(n)]
                p.tp_sync[tp] = Table1D(x, [float(nxt()) for _ in range(n)])
            elif kw == "pp_sync":
                n = int(nxt())
                x = [float(nxt()) for _ in range(n)]
                p.pp_sync = Table1D(x, [float(nxt()) for _ in range(n)])
            elif kw == "head":
                n = int(nxt())
                x = [float(nxt()) for _ in range(n)]
                p.head = Table1D(x, [float(nxt()) for _ in range(n)])
            elif kw == "switch":
                nb, nc = int(nxt()), int(nxt())
                b = [float(nxt()) for _ in range(nb)]
                c = [float(nxt()) for _ in range(nc)]
                p.switch = Table2D(b, c, [[float(nxt()) for _ in range(nc)] for _ in range(nb)])
            else:
                raise ValueError("bad keyword %r" % kw)

    @classmethod
    def load(cls, path: str) -> "Profile":
        with open(path) as f:
            return cls.loads(f.read())


def interp1(xs: Sequence[float], ts: Sequence[float], x: float) -> float:
    """Linear interpolation: exact on grid points, clamp below
    the first point, out of hull above the last (no extrapolation)."""
    n = len(xs)
    if x <= xs[0]:
        return ts[0]
    for i in range(1, n):
        if x == xs[i]:
            return ts[i]
        if x < xs[i]:
            x0, x1, t0, t1 = xs[i - 1], xs[i], ts[i - 1], ts[i]
            return t0 + (x - x0) * (t1 - t0) / (x1 - x0)
    raise OutOfHull(x)


def interp2(tb: Table2D, b: float, c: float) -> float:
    """Bilinear: interpolate along ctx within the bracketing batch rows, then
    along batch."""
    bs = tb.b
    if b <= bs[0]:
        return interp1(tb.c, tb.t[0], c)
    for i in range(1, len(bs)):
        if b == bs[i]:
            return interp1(tb.c, tb.t[i], c)
        if b < bs[i]:
            f0 = interp1(tb.c, tb.t[i - 1], c)
            f1 = interp1(tb.c, tb.t[i], c)
            return f0 + (b - bs[i - 1]) * (f1 - f0) / (bs[i] - bs[i - 1])
    raise OutOfHull(b)


# ---------------------------------------------------------------------------
# model / cluster / schedule
# ---------------------------------------------------------------------------
@dataclass
class SimModel:
    arch: str          # "opt" | "gpt3" | "t5"
    n_enc_layers: int  # 0 for decoder-only
    n_dec_layers: int
    d_model: int
    n_heads: int
    d_head: int
    d_ff: int
    vocab: int
    max_pos: int

    @classmethod
    def from_spec(cls, s):
        return cls(s.arch, s.n_enc_layers, s.n_dec_layers, s.d_model, s.n_heads, s.d_head,
                   s.d_ff, s.vocab, s.max_pos)

    @property
    def inner(self):
        return self.n_heads * self.d_head


@dataclass
class SimCluster:
    n_gpus: int
    mem_per_gpu_bytes: float
    workspace_bytes: float = 0.0
    kv_page: int = 0     # > 0: paged KV of this page length (decoder-only; NEXT-2)


RRA, WAA_C, WAA_M, STATIC = 1, 2, 4, 8
Z99 = 2.3263478740408408   # standard normal 0.99 quantile (RRA latency buffer)


@dataclass
class Schedule:
    strategy: int
    b_e: int
    b_d: int = 0
    b_m: int = 0
    n_d: int = 0
    tp_degree: int = 1
    tp_gpus: int = 0
    n_enc_gpus: int = 0
    stages: List[Tuple[int, int, int, int]] = field(default_factory=list)  # (first_gpu, n_gpus, layer_begin, layer_end)


@dataclass
class Estimate:
    thrput_seq_s: float
    thrput_tok_s: float
    latency_s: float
    feasible: bool = True


def stage_layout(n_gpus: int, t: int, c: int, n_layers: int, first_gpu: int = 0):
    """S8: c GPUs (a multiple of t) at the front form c/t TP stages of t GPUs;
    the rest are 1-GPU stages.  Layers proportional to GPUs per stage,
    remainder one per stage from the front."""
    g = []
    if t > 1:
        g += [t] * (c // t)
        rest = n_gpus - c
    else:
        rest = n_gpus
    g += [1] * rest
    base = [n_layers * gk // n_gpus for gk in g]
    rem = n_layers - sum(base)
    for k in range(rem):
        base[k] += 1
    stages, gpu, layer = [], first_gpu, 0
    for gk, lk in zip(g, base):
        stages.append((gpu, gk, layer, layer + lk))
        gpu += gk
        layer += lk
    return stages


def fill(ts: Sequence[float], M: int) -> float:
    """F(t, M) = sum_k t_k + (M-1) max_k t_k: flow-shop makespan of M
    identical micro-batches."""
    s, m = 0.0, 0.0
    for v in ts:
        s += v
        m = max(m, v)
    return s + (M - 1) * m


def period(ts: Sequence[float], M: int) -> float:
    """Pi(t, M) = max(sum_k t_k, M max_k t_k): closed-pipeline period."""
    s, m = 0.0, 0.0
    for v in ts:
        s += v
        m = max(m, v)
    return max(s, M * m)


def pipeline_event_makespan(ts: Sequence[float], M: int, K: int) -> float:
    """FIFO discrete-event reference for the pipeline algebra: M micro-batches
    each run K iterations through stages ts; micro-batch m may start
    iteration j+1 only after finishing iteration j at the last stage; each
    stage serves one micro-batch at a time, in arrival order.  Returns the
    completion time of the last micro-batch's K-th iteration."""
    P = len(ts)
    free = [0.0] * P
    ready = [0.0] * M          # when micro-batch m may enter stage 0
    done = 0.0
    for j in range(K):
        for m in range(M):
            t = ready[m]
            for k in range(P):
                start = max(t, free[k])
                t = start + ts[k]
                free[k] = t
            ready[m] = t
            done = max(done, t)
    return done


class Simulator:
    def __init__(self, prof: Profile, model: SimModel, cluster: SimCluster,
                 pmf_in: Sequence[float], pmf_out: Sequence[float], target_len: int,
                 use_little_fraction: bool = False):
        self.p, self.m, self.cl = prof, model, cluster
        self.pmf_in, self.pmf_out = list(pmf_in), list(pmf_out)
        self.target_len = target_len
        self.s_e = seqdist.pmf_mean(self.pmf_in)
        self.s_d = seqdist.pmf_mean(self.pmf_out)
        self.max_in, self.max_out = len(self.pmf_in), len(self.pmf_out)
        # decode-attention context of a row at a decode iteration (DESIGN.md
        # reading, round 2; S5 used S_E + S_D/2): rows stay in the batch for
        # S iterations, so an iteration sees a request with probability
        # proportional to S and at a uniform age u = 1..S (renewal-reward) --
        # the row-iteration mean of u is E[S(S+1)] / (2 E[S]); keys = n - 1 + u
        # (decoder-only: n - 1 encoded positions + u decoded) or n cross + u
        # self keys (T5, the profile's total at c = self + cross)
        m2o_ = 0.0
        for k in range(1, len(self.pmf_out) + 1):
            m2o_ += float(k) * float(k) * float(self.pmf_out[k - 1])
        self.age_mean = (m2o_ + self.s_d) / (2.0 * self.s_d)
        self.ctx_mean = self.s_e + self.age_mean - (0.0 if model.arch == "t5" else 1.0)
        # encode-attention lookup length: the RMS input length (a request's
        # attention cost grows as n^2; DESIGN.md reading)
        m2 = 0.0
        for k in range(1, len(self.pmf_in) + 1):
            m2 += float(k) * float(k) * float(self.pmf_in[k - 1])
        self.s_e_rms = math.sqrt(m2)
        var = m2 - self.s_e * self.s_e                       # input-length variance
        self.s_e_sd = math.sqrt(var if var > 0.0 else 0.0)
        self.use_little = use_little_fraction
        self.n_layers = model.n_dec_layers                   # decoder-only: every layer runs both phases
        # decoder KV context per row: slots hold Max_in + Max_out positions
        # (S13); with paged KV (SimCluster.kv_page = P, decoder-only) a row
        # holds only its live positions, and the memory model charges the
        # row-iteration average of those (DESIGN.md reading):
        # a request with input n and output S holds n - 1 + u keys at its
        # decode iteration u = 1..S, so over its S iterations the mean is
        # n - 1 + (S + 1)/2; weighting requests by their S iterations
        # (renewal-reward) gives S_E - 1 + E[S(S+1)] / (2 E[S]), plus 3P/2:
        # half a page of rounding on average and the one-page-per-row reserve
        # the runner keeps at admission.  Fluctuations above the mean are
        # absorbed by the runner's preemption.
        self.kv_ctx_dec = float(self.max_in + self.max_out)
        if cluster.kv_page > 0 and model.arch != "t5":
            live = self.s_e - 1.0 + self.age_mean
            self.kv_ctx_dec = min(live + 1.5 * float(cluster.kv_page), float(self.max_in + self.max_out))
        self.k_dec = 3 if model.arch == "t5" else 2
        self._pu_cache: Dict[int, Tuple[List[float], float]] = {}

    # -- profile lookups ---------------------------------------------------
    def _tp_sync(self, t: int, nbytes: float) -> float:
        if t <= 1:
            return 0.0
        tb = self.p.tp_sync[t]
        return interp1(tb.x, tb.t, nbytes)

    def _pp_sync(self, nbytes: float) -> float:
        tb = self.p.pp_sync
        return interp1(tb.x, tb.t, nbytes)

    def layer_enc(self, t: int, b: float) -> float:
        toks = b * self.s_e
        a = interp2(self.p.attn[("enc", t)], b, self.s_e_rms)
        tb = self.p.rest[("enc", t)]
        r = interp1(tb.x, tb.t, toks)
        return a + r + 2 * self._tp_sync(t, toks * self.m.d_model * 4.0)

    def layer_dec(self, t: int, b: float) -> float:
        a = interp2(self.p.attn[("dec", t)], b, self.ctx_mean)
        tb = self.p.rest[("dec", t)]
        r = interp1(tb.x, tb.t, b)
        return a + r + self.k_dec * self._tp_sync(t, b * self.m.d_model * 4.0)

    def stage_times(self, stages, phase: str, b: float) -> List[float]:
        out = []
        P = len(stages)
        for k, (g0, ng, l0, l1) in enumerate(stages):
            per = self.layer_enc(ng, b) if phase == "enc" else self.layer_dec(ng, b)
            v = (l1 - l0) * per
            if k < P - 1:
                toks = b * self.s_e if phase == "enc" else b
                v += self._pp_sync(toks * self.m.d_model * 2.0)
            if phase == "dec" and k == P - 1 and self.p.head is not None:
                # the decode head (final norm + LM head + argmax) runs once per
                # iteration on the last stage (DESIGN.md reading)
                v += interp1(self.p.head.x, self.p.head.t, b)
            out.append(v)
        return out

    # -- completion statistics -------------------------------------------
    def pu(self, n_d: int) -> Tuple[List[float], float]:
        if n_d not in self._pu_cache:
            pu = seqdist.completion_distribution(self.pmf_out, n_d)
            f = seqdist.little_fraction(self.pmf_out, n_d) if self.use_little else seqdist.completion_fraction(pu)
            self._pu_cache[n_d] = (pu, f)
        return self._pu_cache[n_d]

    # -- memory (S13) -------------------------------------------------------
    def layer_bytes(self) -> float:
        d, inner, ff = self.m.d_model, self.m.inner, self.m.d_ff
        params = d * 3 * inner + 3 * inner + inner * d + d + d * ff + ff + ff * d + d + 4 * d
        return params * 2.0

    def emb_bytes(self) -> float:
        return (self.m.vocab * self.m.d_model + self.m.max_pos * self.m.d_model + 2 * self.m.d_model) * 2.0

    def kv_bytes_per_token_layer(self) -> float:
        return 2.0 * self.m.inner * 2.0

    def memory(self, s: Schedule):
        """Per-GPU (model bytes, KV-cache bytes) of a schedule under the
        memory model of mem_ok (weight shard, embeddings on the first / last
        stage of each side, KV slots at kv_rows x ctx for the stage's layers):
        the memory-overhead accounting of PAPER.md:548-560 (WAA holds more
        model copies and less KV than RRA / FT).  Lists of length n_gpus."""
        w = [0.0] * self.cl.n_gpus
        kv = [0.0] * self.cl.n_gpus

        def account(stages, rows, ctx):
            P = len(stages)
            for k, (g0, ng, l0, l1) in enumerate(stages):
                b = (l1 - l0) * self.layer_bytes() / ng
                if k == 0 or k == P - 1:
                    b += self.emb_bytes()
                c = rows * ctx * (l1 - l0) * self.kv_bytes_per_token_layer() / ng
                for g in range(g0, min(g0 + ng, self.cl.n_gpus)):
                    w[g] += b
                    kv[g] += c

        if s.strategy == STATIC:
            account(stage_layout(self.cl.n_gpus, 1, 0, self.n_layers), s.b_e, self.max_in + self.max_out)
        elif s.strategy == RRA:
            account(s.stages, s.b_d, self.kv_ctx_dec)
        else:
            account([st for st in s.stages if st[0] < s.n_enc_gpus], s.b_e, self.max_in)
            account([st for st in s.stages if st[0] >= s.n_enc_gpus], s.b_d, self.kv_ctx_dec)
        return w, kv

    def mem_ok(self, stages, kv_rows: int, ctx: int) -> bool:
        P = len(stages)
        for k, (g0, ng, l0, l1) in enumerate(stages):
            b = (l1 - l0) * self.layer_bytes() / ng
            if k == 0 or k == P - 1:
                b += self.emb_bytes()
            b += kv_rows * ctx * (l1 - l0) * self.kv_bytes_per_token_layer() / ng
            b += self.cl.workspace_bytes
            if b > self.cl.mem_per_gpu_bytes:
                return False
        return True

    # -- RRA (S6) -----------------------------------------------------------
    def rra_schedule(self, b_e: int, n_d: int, t: int, c: int) -> Schedule:
        pu, f = self.pu(n_d)
        b_d = seqdist.rra_b_d(b_e, f)
        st = stage_layout(self.cl.n_gpus, t, c, self.n_layers)
        return Schedule(RRA, b_e, b_d, 0, n_d, t, c, 0, st)

    def simulate_rra(self, s: Schedule) -> Estimate:
        if not self.mem_ok(s.stages, s.b_d, self.kv_ctx_dec):
            return Estimate(0.0, 0.0, INF, False)
        pu, f = self.pu(s.n_d)
        P = len(s.stages)
        try:
            t_enc = self.stage_times(s.stages, "enc", s.b_e / P)
            T_encph = fill(t_enc, P)
            bu = seqdist.rra_iteration_batches(s.b_d, pu)
            Pi, Fu = [], []
            for u in range(s.n_d):
                tu = self.stage_times(s.stages, "dec", bu[u] / P)
                if u == 0 and self.p.switch is not None:
                    # the phase's decode iterations follow an encode phase: the
                    # clock recovers from the power cap over the first few; their
                    # cumulative extra time (profile `switch` at k = min(N_D,
                    # k_max)) is charged to the first iteration, each stage its
                    # layer share (DESIGN.md reading)
                    w = interp2(self.p.switch, bu[0] / P, min(float(s.n_d), self.p.switch.c[-1]))
                    for k in range(P):
                        tu[k] = tu[k] + w * float(s.stages[k][3] - s.stages[k][2]) / self.n_layers
                Pi.append(period(tu, P))
                Fu.append(fill(tu, P))
        except OutOfHull:
            return Estimate(0.0, 0.0, INF, False)
        T_decph = 0.0
        for u in range(s.n_d - 1):
            T_decph += Pi[u]
        T_decph += Fu[s.n_d - 1]
        T_cyc = T_encph + T_decph
        thr = s.b_e / T_cyc
        S = self.target_len
        q = -(-S // s.n_d)
        r = 1 + (S - 1) % s.n_d
        lat = (q - 1) * T_cyc + T_encph
        for u in range(r - 1):
            lat += Pi[u]
        lat += Fu[r - 1]
        # buffer time: the encoder workload of the query's q
        # encode phases varies with the input lengths (Table 9);
        # its 99th-percentile excess, z99 sqrt(q B_E) sigma_in tokens spread
        # over the q phases, at the profile's encode cost (DESIGN.md reading)
        if self.s_e_sd > 0.0:
            db = Z99 * self.s_e_sd * math.sqrt(q * s.b_e) / (q * self.s_e)
            try:
                T_buf = fill(self.stage_times(s.stages, "enc", (s.b_e + db) / P), P)
            except OutOfHull:
                return Estimate(0.0, 0.0, INF, False)
            lat += q * (T_buf - T_encph)
        return Estimate(thr, thr * self.s_d, lat)

    # -- WAA (S7) -----------------------------------------------------------
    def waa_split(self, b_e: int, b_d: int, strat: int = WAA_C) -> int:
        """Encoder GPUs out of N.  WAA-C (S7): proportional to the encoder /
        decoder compute per iteration.  WAA-M (reading): so the
        per-GPU memory of the two sides is equal -- M_E = weights + B_E max_in
        KV rows, M_D = weights + B_D kv_ctx_dec KV rows (max_in + max_out;
        paged: the live average), n_enc =
        round(N M_E / (M_E + M_D))."""
        N = self.cl.n_gpus
        if strat == WAA_M:
            kv = self.kv_bytes_per_token_layer()
            W = self.n_layers * self.layer_bytes() + self.emb_bytes()
            M_E = W + (b_e * self.max_in * self.n_layers) * kv
            M_D = W + (b_d * self.kv_ctx_dec * self.n_layers) * kv
            n_enc = int(math.floor(N * M_E / (M_E + M_D) + 0.5))
        else:
            C_E = self.n_layers * self.layer_enc(1, b_e)
            C_D = self.n_layers * self.layer_dec(1, b_d)
            n_enc = int(math.floor(N * C_E / (C_E + C_D) + 0.5))
        return min(max(n_enc, 1), N - 1)

    def waa_schedule(self, b_e: int, M: int, t: int, c: int, strat: int = WAA_C) -> Optional[Schedule]:
        if self.cl.n_gpus < 2:
            return None
        b_d = seqdist.waa_b_d(b_e, self.s_d)
        M = min(M, b_d)
        b_m = -(-b_d // M)
        try:
            n_enc = self.waa_split(b_e, b_d, strat)
        except OutOfHull:
            return None
        n_dec = self.cl.n_gpus - n_enc
        if c > n_dec:
            return None
        enc = stage_layout(n_enc, 1, 0, self.n_layers, 0)
        dec = stage_layout(n_dec, t, c, self.n_layers, n_enc)
        return Schedule(strat, b_e, b_d, b_m, 0, t, c, n_enc, enc + dec)

    def simulate_waa(self, s: Schedule) -> Estimate:
        enc = [st for st in s.stages if st[0] < s.n_enc_gpus]
        dec = [st for st in s.stages if st[0] >= s.n_enc_gpus]
        if not (self.mem_ok(enc, s.b_e, self.max_in) and self.mem_ok(dec, s.b_d, self.kv_ctx_dec)):
            return Estimate(0.0, 0.0, INF, False)
        M = -(-s.b_d // s.b_m)
        try:
            te = self.stage_times(enc, "enc", float(s.b_e))
            td = self.stage_times(dec, "dec", float(s.b_m))
            handoff = self._pp_sync(s.b_e * self.s_e * self.n_layers * self.kv_bytes_per_token_layer())
        except OutOfHull:
            return Estimate(0.0, 0.0, INF, False)
        T_E, T_trav = 0.0, 0.0
        for v in te:
            T_E = max(T_E, v)
            T_trav += v
        T_D = period(td, M)
        thr = s.b_e / max(T_E, T_D)
        lat = T_trav + handoff + T_E + (self.target_len - 1) * T_D + fill(td, M)
        return Estimate(thr, thr * self.s_d, lat)

    # -- FT-style static batch ----------
    def simulate_static(self, B: int) -> Estimate:
        """Encode B requests, then decode all B rows for max_out iterations
        with no early termination (dead rows still computed): the baseline
        the paper derives its latency bounds from.  Latency applies to a
        max-length output; throughput = B / latency.  P = 1 (TP maxed within
        the box is the paper's FT setting; single-GPU here)."""
        st = stage_layout(self.cl.n_gpus, 1, 0, self.n_layers)
        if not self.mem_ok(st, B, self.max_in + self.max_out):
            return Estimate(0.0, 0.0, INF, False)
        try:
            t_enc = self.stage_times(st, "enc", float(B))
            t_dec = self.stage_times(st, "dec", float(B))
            lat = fill(t_enc, 1) + self.max_out * fill(t_dec, 1)
            if self.p.switch is not None:
                # the decode iterations follow the encode phase (clock recovery)
                lat += interp2(self.p.switch, float(B), min(float(self.max_out), self.p.switch.c[-1]))
        except OutOfHull:
            return Estimate(0.0, 0.0, INF, False)
        thr = B / lat
        return Estimate(thr, thr * self.s_d, lat)

    def simulate(self, s: Schedule) -> Estimate:
        return self.simulate_rra(s) if s.strategy == RRA else self.simulate_waa(s)
