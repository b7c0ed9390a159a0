#!/usr/bin/env python
"""bench.py -- BASELINE.json metric: output tokens/s under a latency bound,
plus the decode-attention HBM GB/s, on config 2 (OPT-13B, task S, RRA on
1 x B200; BASELINE.json configs[1]).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

One step = one pass of the whole hot path over one synthetic request batch:
exg_run of `--requests` task-S requests under the schedule exg_schedule_find
picked for the bound (encode phases, N_D decode iterations each, early
termination, until the batch drains).  Procedure:

  1. exg_create: seeded OPT-13B weights generated on the GPU;
  2. exg_profile: XProfiler sweep of one encoder / decoder layer;
  3. latency bounds by the paper's recipe: static-batch (FT
     style) latency of a max-length output for B = 4, 8, ... -> 10th / 30th /
     70th percentiles and infinity;
  4. exg_schedule_find per bound (Algorithm 1, host);
  5. headline bound (70th pctl): W warm-up + K timed steps, with per-launch
     kernel timing (roofline); the other bounds: one run each.

With N > 1 (torchrun) the default is config 4 (OPT-66B, task G) under the
scheduler's N-GPU plan -- RRA / WAA with partial TP, pipeline hops, KV
handoff and TP all-reduce over NCCL -- as one job (run_layout); `--layout
replicas` runs independent config-2 replicas instead (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

TASK = "S"
COMM_ALPHA_S, COMM_BW = 10e-6, 700e9   # modeled p2p latency / bandwidth per GPU link set
METRIC = "output tokens/s under latency bound (BASELINE.json; 70th-pctl bound headline)"
WORKLOAD = ("config 2: OPT-13B (seeded random init), task S (in 256+-252<=512, out 32+-13<=80, p99 63), "
            "RRA on 1xB200 per rank")
MODEL = "opt-13b"
CONFIG_NO = 2
B_E_MAX = 64
# XProfiler sweep axes: batch, context, tokens
PROFILE_BATCH = [1, 2, 4, 8, 16, 32, 48, 64, 96, 128, 160, 192, 224, 256, 320, 384, 448, 512]
PROFILE_CTX = [1, 32, 64, 128, 192, 256, 320, 384, 448, 512, 592]
PROFILE_TOKENS = [1, 16, 64, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768]


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sus": d.get("bf16_tflops_sustained",
                                                                                  d["bf16_tflops"]),
                "src": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback (B200_PROFILING.md)"}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        loaded = [s for s in sm if s > 500] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------
# CPU baseline: the oracle as it stands (test infrastructure) on a bounded
# sample of the same workload -- a measured per-layer cost model of oracle
# mode (iii)'s batched KV loop (SURVEY.md §8(d) "Oracle timing").
# ----------------------------------------------------------------------------
CPU_REQUESTS = 32


class OracleCostModel:
    """Oracle mode (iii) (oracle/transformer.py KVLoop, bf16-emulating, fp64
    accumulation) running CPU_REQUESTS task-S requests batched exactly as
    KVLoop.run does -- one encode forward over every request's input tokens,
    then decode iterations over the still-active rows -- through all L = 40
    OPT-13B layers.  Every layer has the same shapes, so the run's time is

        L * [enc(T_E) + sum_u dec(b_u)] + sum_u head(b_u)

    with b_u the rows alive at iteration u.  enc / dec / head are measured on
    the host with the oracle's own functions (KVLoop._layer on layer 0,
    KVLoop._logits): enc per encoded token on a packed sample of requests,
    dec and head at two batch sizes (linear in b).  Weight generation is
    outside the timed region (a CPU server holds its weights)."""

    def __init__(self, n_enc_sample=4):
        from oracle import transformer as T
        from workload import MODELS, ModelSpec, make_requests, task_dists, weight_seed
        full = MODELS[MODEL]
        self.L = full.n_dec_layers
        spec = ModelSpec(full.name + "-layer0", full.arch, 0, 1, full.d_model, full.n_heads, full.d_head,
                         full.d_ff, full.vocab, full.max_pos)
        self.T = T
        self.W = T.Weights(spec, weight_seed(CONFIG_NO), cache_fp64=False)
        self.W.layer(0)                                     # generated outside the timed region
        d = task_dists(TASK)
        self.reqs = make_requests(CPU_REQUESTS, d.pmf_in, d.pmf_out, full.vocab, 0xE6E1_0000 + CONFIG_NO)
        self.loop = T.KVLoop(self.W, "bf16")
        self.sample = self.reqs[:n_enc_sample]
        H, dh = spec.n_heads, spec.d_head
        toks, rows = [], []
        for r, q in enumerate(self.sample):
            for p in range(q.input_len - 1):
                toks.append(int(q.ids[p]))
                rows.append((r, p))
        self.enc_rows, self.enc_toks = rows, np.array(toks)
        self.mk = lambda: {r: ([np.zeros((H, 0, dh))], [np.zeros((H, 0, dh))]) for r in range(len(self.sample))}
        self.base_caches = self.mk()
        x = self.loop._forward(self.enc_toks, rows, self.base_caches)     # caches for the decode measurement
        del x

    def _dec_caches(self, b):
        return {i: ([self.base_caches[i % len(self.sample)][0][0].copy()],
                    [self.base_caches[i % len(self.sample)][1][0].copy()]) for i in range(b)}

    def measure(self, b_lo=8, b_hi=CPU_REQUESTS):
        """One bounded sample: returns (modeled tok/s, modeled seconds, measured CPU seconds, detail)."""
        loop, W = self.loop, self.W
        t_all = time.perf_counter()
        # encode: layer 0 over the sample's packed input tokens
        pos = np.array([p for _, p in self.enc_rows])
        x = loop.R.f32(W.emb_rows(self.enc_toks) + W.pos_emb[pos])
        t0 = time.perf_counter()
        loop._layer(0, x, self.enc_rows, self.mk())
        c_enc = (time.perf_counter() - t0) / len(self.enc_rows)
        dec, head = {}, {}
        for b in (b_lo, b_hi):
            caches = self._dec_caches(b)
            rows = [(i, self.sample[i % len(self.sample)].input_len - 1) for i in range(b)]
            toks = np.array([int(self.sample[i % len(self.sample)].ids[-1]) for i in range(b)])
            xd = loop.R.f32(W.emb_rows(toks) + W.pos_emb[np.array([p for _, p in rows])])
            t0 = time.perf_counter()
            xo = loop._layer(0, xd, rows, caches)
            dec[b] = time.perf_counter() - t0
            t0 = time.perf_counter()
            loop._logits(xo)
            head[b] = time.perf_counter() - t0
        lin = lambda f, b: f[b_lo] + (f[b_hi] - f[b_lo]) * (b - b_lo) / (b_hi - b_lo)
        T_E = sum(q.input_len - 1 for q in self.reqs)
        S = [q.output_len for q in self.reqs]
        b_u = [sum(1 for s in S if s >= u) for u in range(1, max(S) + 1)]
        t_model = self.L * (c_enc * T_E + sum(lin(dec, b) for b in b_u)) + sum(lin(head, b) for b in b_u)
        cpu_s = time.perf_counter() - t_all
        detail = {"enc_s_per_token_layer": c_enc, "dec_layer_s": {str(k): v for k, v in dec.items()},
                  "head_s": {str(k): v for k, v in head.items()}, "encode_tokens": T_E, "decode_iters": len(b_u),
                  "modeled_run_s": t_model}
        return sum(S) / t_model, t_model, cpu_s, detail


def cpu_info():
    """Host description for the CPU baseline: lscpu model, usable cores, BLAS
    library and its thread count."""
    model = None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    blas = []
    try:
        import threadpoolctl
        np.ones((64, 64)) @ np.ones((64, 64))
        blas = [{"api": i.get("internal_api"), "threads": i.get("num_threads"), "version": i.get("version")}
                for i in threadpoolctl.threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "cores": cpu_cores(), "blas": blas}


def cpu_baseline_block(cm: "OracleCostModel", value, model_s, cpu_s, detail):
    info = cpu_info()
    threads = max([b["threads"] or 0 for b in info["blas"]] or [1])
    return {"value": value, "unit": "output tokens/s", "cores": threads or info["cores"], "kind": "oracle",
            "sample": ("per-layer cost model of oracle mode (iii)'s batched KV loop over %d task-S requests "
                       "(%d encode tokens, %d decode iterations) through all %d OPT-13B layers + LM head: "
                       "layer-0 encode / decode / head measured on the host (%.1f s of CPU work), modeled run "
                       "%.0f s" % (CPU_REQUESTS, detail["encode_tokens"], detail["decode_iters"], cm.L, cpu_s,
                                   model_s)),
            "host": info, "measured": detail}


def scheduler_wall_times(X, prof, ctx, cl, pin, pout, d, L_b, args):
    """exg_schedule_find (C++) vs oracle/bnb.schedule_find (Python) on the
    same profile-v1 file, bound and options; also checks they agree (S15)."""
    import tempfile
    from oracle import bnb, simulator as sim
    from workload import MODELS
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "p.txt")
        prof.save(path)
        P = sim.Profile.load(path)
    S = sim.Simulator(P, sim.SimModel.from_spec(MODELS[MODEL]), sim.SimCluster(cl.n_gpus, cl.mem_per_gpu_bytes,
                                                                             cl.workspace_bytes),
                      d.pmf_in, d.pmf_out, d.target_len, use_little_fraction=bool(args.little))
    t0 = time.perf_counter()
    s_c, e_c = X.schedule_find(prof, ctx.mspec, cl, pin, pout, d.target_len, L_b * (1 - args.margin), X.EXG_RRA,
                               X.search_opts(b_e_max=B_E_MAX, little=args.little))
    t_c = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = bnb.schedule_find(S, L_b * (1 - args.margin), sim.RRA, bnb.SearchOpts(b_e_max=B_E_MAX,
                                                                              use_little_fraction=bool(args.little)))
    t_py = time.perf_counter() - t0
    same = f is not None and (f.schedule.b_e, f.schedule.n_d, f.estimate.thrput_seq_s) == (
        s_c.b_e, s_c.n_d, e_c.thrput_seq_s)
    return {"cpp": t_c, "python_oracle": t_py, "evals": int(e_c.perf_evals), "identical_choice": bool(same)}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def workload_variance(st, trace=None, prof=None, n_layers=0, recovery_iters=10):
    """Table 9: mean single-stage time and its 99th-pctl
    range (|t - mean|) for encode phases and decode iterations.  With the
    run's stage trace and the profile, the range is decomposed: `model` =
    the range of measured / profile-predicted time for the same rows and
    work (what the workload's batch / context changes do not explain), and,
    for decode, `model_after_recovery` = the same over iterations >= 10 after
    an encode phase (the first ones run while the clock recovers from the
    encode phase's power cap -- the profile's switch table)."""
    def one(m, d):
        return {"mean_s": m, "p99_range_s": d, "p99_range_pct": 100.0 * d / m if m else None}
    out = {"encoder": one(st["enc_stage_mean_s"], st["enc_stage_p99dev_s"]),
           "decoder": one(st["dec_stage_mean_s"], st["dec_stage_p99dev_s"])}
    if trace and prof is not None:
        def rng(v):
            v = np.asarray(v)
            return float(100.0 * np.percentile(np.abs(v - v.mean()), 99) / v.mean()) if len(v) else None
        enc_r, dec_r, dec_late = [], [], []
        k = 0
        for kind, _, dur, rows, work in trace:
            if kind == 1:
                enc_r.append(dur / prof.stage_time(0, rows, work, n_layers))
                k = 0
            else:
                r = dur / prof.stage_time(1, rows, work, n_layers)
                dec_r.append(r)
                if k >= recovery_iters:
                    dec_late.append(r)
                k += 1
        out["encoder"]["model_p99_range_pct"] = rng(enc_r)
        out["decoder"]["model_p99_range_pct"] = rng(dec_r)
        out["decoder"]["model_after_recovery_p99_range_pct"] = rng(dec_late)
        out["decoder"]["paper_table9_pct"] = [2.4, 5.5]
    return out


# ---- multi-rank host logic (weak scaling: independent replicas) ------------
def rank_request_seed(rank: int) -> int:
    """Each rank draws its own requests of the same workload (weak scaling)."""
    return 0xE6E1_0000 + CONFIG_NO + 1000 * rank


def reduce_over_ranks(v: float, op: str, dist=None, device: str = "cuda") -> float:
    """max / sum of a scalar over the ranks of the default process group."""
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def job_throughput(tokens: float, seconds: float, dist=None, device: str = "cuda") -> float:
    """Whole-job metric: the tokens every rank produced / the slowest rank's time."""
    return reduce_over_ranks(tokens, "sum", dist, device) / reduce_over_ranks(seconds, "max", dist, device)


def static_bounds(X, prof, mspec, cl, pin, pout, target_len):
    """Latency bounds: 10/30/70th percentiles of the FT-style static-batch
    latencies B = 4, 8, ... on the profile."""
    from paper_2404_07947_b200._lib import exg_schedule
    stat = []
    for B in range(4, 1025, 4):
        s = exg_schedule()
        s.strategy, s.b_e = X.EXG_STATIC, B
        e = X.simulate(prof, mspec, cl, pin, pout, target_len, s)
        if not e.feasible:
            break
        stat.append(e.latency_s)
    p10, p30, p70 = (float(np.percentile(stat, q)) for q in (10, 30, 70))
    return [("p10", p10), ("p30", p30), ("p70", p70), ("inf", math.inf)]


def static_pick(X, prof, mspec, cl, pin, pout, target_len, L_b):
    """The FT-style static batch size for a bound: the simulated
    max-throughput B whose static latency (max-length output)
    is within L_b; None if even B = 1 misses it."""
    from paper_2404_07947_b200._lib import exg_schedule
    best = None
    for B in range(1, 1025):
        s = exg_schedule()
        s.strategy, s.b_e = X.EXG_STATIC, B
        e = X.simulate(prof, mspec, cl, pin, pout, target_len, s)
        if not e.feasible:
            break
        if e.latency_s <= L_b and (best is None or e.thrput_tok_s > best[1].thrput_tok_s):
            best = (B, e)
    return best


def in_runner_baselines(args, X, ctx, prof, cl, pin, pout, d, bounds, scheds, reqs, slot_ctx, sla):
    """the paper's comparison points run on the same
    kernels, requests and bounds -- FT-style static batches (PAPER.md:112:
    fixed batch, no early termination; B = the simulated best static batch
    within the bound) and ORCA-style iteration-level admission (PAPER.md:116:
    new requests join every iteration = RRA with N_D = 1, B_E / B_D picked by
    Algorithm 1 with N_D^max = 1) -- beside the ExeGPT schedule (RRA,
    Algorithm 1).  Ratios are measured tokens/s; a leg whose run misses the
    bound (SLA-(b)) is reported with sla_b_met false."""
    res = {}
    for name, L_b in bounds:
        row = {"latency_bound_s": L_b}
        legs = {}
        if scheds.get(name):
            legs["exegpt"] = (scheds[name][0], scheds[name][1].thrput_tok_s)
        pick = static_pick(X, prof, ctx.mspec, cl, pin, pout, d.target_len, L_b * (1 - args.margin))
        if pick:
            legs["ft_static"] = (X.static_schedule(pick[0]), pick[1].thrput_tok_s)
        else:
            row["ft_static"] = {"infeasible": "no static batch within the bound on the profile"}
        try:
            so, eo = X.schedule_find(prof, ctx.mspec, cl, pin, pout, d.target_len, L_b * (1 - args.margin),
                                     X.EXG_RRA, X.search_opts(b_e_max=B_E_MAX, n_d_max=1, little=args.little))
            legs["orca_style"] = (so, eo.thrput_tok_s)
        except X.ExgError as e:
            # an encode every iteration puts each request behind O(S) encode
            # phases: no N_D = 1 schedule meets a finite bound on task S
            row["orca_style"] = {"infeasible": str(e)}
        for leg, (sch, pred) in legs.items():
            _, lat, st, _ = ctx.run(sch, reqs, slot_ctx=slot_ctx)
            row[leg] = {"schedule": sch.as_dict(), "predicted_tok_s": pred, "tok_s": st["tok_s"],
                        "mean_decode_batch": st["mean_decode_batch"], "decode_iters": st["decode_iters"],
                        "encode_phases": st["encode_phases"], "wall_s": st["wall_s"], **sla(lat, L_b, reqs)}
        for leg in ("ft_static", "orca_style"):
            if "exegpt" in row and "tok_s" in row.get(leg, {}):
                row["exegpt_over_" + leg.split("_")[0]] = row["exegpt"]["tok_s"] / row[leg]["tok_s"]
            elif "exegpt" in row:
                row["exegpt_over_" + leg.split("_")[0]] = None   # the baseline has no batch within the bound
        res[name] = row
    return res


MULTI_MODEL, MULTI_TASK, MULTI_CONFIG_NO = "opt-66b", "G", 4
MULTI_WORKLOAD = ("config 4: OPT-66B (seeded random init), task G (in 64+-23<=128, out 184+-102<=480, p99 417), "
                  "the scheduler's N-GPU plan (RRA | WAA-C | WAA-M x partial TP) as one NCCL job")


def multi_plans(X, prof, mspec, cl_n, pin, pout, target_len, margin, little):
    """Config 4's plans on an N-GPU cluster: the static-batch
    bounds of the paper's recipe, the scheduler's overall pick
    over RRA | WAA-C | WAA-M x TP degree x applied GPUs at the 70th-percentile
    bound, and the forced WAA plan with partial TP of degree 2.
    Pure host (the C-ABI planner); returns a dict of schedules (bytes) and
    estimates."""
    bounds = static_bounds(X, prof, mspec, cl_n, pin, pout, target_len)
    L_b = dict(bounds)["p70"]
    out = {"bounds": bounds, "latency_bound_s": L_b}
    opts = X.search_opts(b_e_max=B_E_MAX, little=little)
    for name, mask, o in (("pick", X.EXG_RRA | X.EXG_WAA_C | X.EXG_WAA_M, opts),
                          ("waa_tp2", X.EXG_WAA_C | X.EXG_WAA_M, X.search_opts(b_e_max=B_E_MAX, little=little, tp_only=2))):
        try:
            s, e = X.schedule_find(prof, mspec, cl_n, pin, pout, target_len, L_b * (1 - margin), mask, o)
            out[name] = {"sched": bytes(s), "schedule": s.as_dict(), "predicted_tok_s": e.thrput_tok_s,
                         "predicted_latency_s": e.latency_s}
        except X.ExgError as err:
            out[name] = {"infeasible": str(err)}
    return out


def run_layout(args, rank, world, local):
    """N > 1 (torchrun): config 4 -- OPT-66B on task G -- as ONE job over the N
    ranks (one process per GPU, NCCL): GPU g of the layout on rank g*N/G
    (multi.cu).  (1) rank 0's NCCL id is broadcast and every rank creates
    the multi-rank context; (2) XProfiler's interconnect tables are measured
    collectively (TP all-reduce over NCCL sub-communicators, PP hop); (3)
    rank 0 profiles the layer tables on a one-GPU context of the full model,
    merges the measured interconnect tables, derives the bounds and plans;
    (4) every rank runs the scheduler's pick (W + K steps, device time from
    the gathered stamps, max over ranks by construction) and, once, the forced
    WAA TP-2 plan."""
    import torch
    import torch.distributed as dist
    import paper_2404_07947_b200 as X
    from paper_2404_07947_b200._lib import exg_schedule
    from workload import MODELS, make_requests, task_dists, weight_seed
    spec = MODELS[args.multi_model]
    d = task_dists(args.multi_task)
    seed = weight_seed(MULTI_CONFIG_NO)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None   # one-GPU dry run of this path (--layout plan without torchrun)
    free, total = torch.cuda.mem_get_info(local)
    mem, ws = total - (6 << 30), 8 << 30
    pin, pout = X.Pmf(d.pmf_in), X.Pmf(d.pmf_out)

    def bcast(obj):
        box = [obj]
        if dist:
            dist.broadcast_object_list(box, src=0)
        return box[0]

    uid = bcast(X.unique_id() if rank == 0 and world > 1 else None)
    tps = [t for t in (1, 2, 4, 8) if t <= max(world, 1) and spec.n_heads % t == 0]
    comm_prof = None
    if world > 1:
        ctx = X.Context(spec, seed, device=local, cluster=X.cluster_spec(world, mem, ws), rank=rank, world=world,
                        uid=uid)
        comm_prof = ctx.profile([1], [1], [1], reps=5, tps=tps)       # collective
    plan = None
    if rank == 0:
        ctx1 = X.Context(spec, seed, device=local, cluster=X.cluster_spec(1, mem, ws))
        prof = ctx1.profile(PROFILE_BATCH, PROFILE_CTX, PROFILE_TOKENS, reps=3, tps=tps)
        if comm_prof is not None:
            prof.copy_comm(comm_prof)
        else:
            prof.comm_model(COMM_ALPHA_S, COMM_BW)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        prof.save(os.path.join(ROOT, "gpurun_out", "profile_multi.txt"))
        # paged KV (NEXT-2, --kv-page): the planner charges each decode row its
        # live positions (exegpt.h kv_page), every executor pages
        paged = args.kv_page
        cl_plan = X.cluster_spec(max(world, 1), mem, ws, kv_page=paged)
        plan = multi_plans(X, prof, ctx1.mspec, cl_plan, pin, pout, d.target_len, args.margin, args.little)
        for key in ("pick", "waa_tp2"):
            if not paged or "sched" not in plan[key]:
                continue
            # page pool: the same page count on every paged GPU, the most any
            # of them fits after its weights and workspace
            sp = exg_schedule.from_buffer_copy(plan[key]["sched"])
            w_b, _ = X.schedule_memory(prof, ctx1.mspec, cl_plan, pin, pout, sp)
            waa = sp.strategy in (X.EXG_WAA_C, X.EXG_WAA_M)
            pools = []
            for g0, ng, l0, l1 in sp.stages():
                if waa and g0 < sp.n_enc_gpus:
                    continue   # WAA encoder GPUs keep per-batch slots
                page_bytes = (l1 - l0) * 2 * (spec.n_heads // ng) * paged * spec.d_head * 2
                pools += [int((mem - w_b[g] - ws) // page_bytes) for g in range(g0, g0 + ng)]
            plan[key]["kv_pages"] = max(1, min(pools))
        if world > 1:
            ctx1.close()
            del ctx1
            torch.cuda.empty_cache()
        else:
            ctx = ctx1
    plan = bcast(plan)
    if "sched" not in plan["pick"]:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "n_gpus": world, "unavailable":
                              "no schedule meets the bound: " + plan["pick"].get("infeasible", "")}))
        ctx.close()
        if dist:
            dist.destroy_process_group()
        return
    s = exg_schedule.from_buffer_copy(plan["pick"]["sched"])
    L_b = plan["latency_bound_s"]
    pkw = {"kv_page": args.kv_page, "kv_pages": plan["pick"]["kv_pages"]} if plan["pick"].get("kv_pages") else {}
    reqs = make_requests(args.requests, d.pmf_in, d.pmf_out, spec.vocab, 0xE6E1_0000 + MULTI_CONFIG_NO)
    slot_ctx = len(d.pmf_in) + len(d.pmf_out)
    h2d = sum((r.input_len - 1) * 12 + 16 + 16 * r.output_len for r in reqs)
    d2h = sum(4 * r.output_len for r in reqs)
    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        ctx.run(s, reqs, slot_ctx=slot_ctx, **pkw)
    barrier()
    wall, toks, lat = 0.0, 0, None
    th0 = time.perf_counter()
    with Clocks(local) as clk:
        for _ in range(args.steps):
            _, lat, st, _ = ctx.run(s, reqs, slot_ctx=slot_ctx, **pkw)
            wall += st["wall_s"]     # rank 0: stamps of every rank on one clock
            toks += st["out_tokens"]
        barrier()
        host = time.perf_counter() - th0
    wall = reduce_over_ranks(wall, "max", dist)
    host = reduce_over_ranks(host, "max", dist)
    forced = None
    if "sched" in plan["waa_tp2"] and world > 1:
        sw = exg_schedule.from_buffer_copy(plan["waa_tp2"]["sched"])
        wkw = ({"kv_page": args.kv_page, "kv_pages": plan["waa_tp2"]["kv_pages"]}
               if plan["waa_tp2"].get("kv_pages") else {})
        _, lat_w, st_w, _ = ctx.run(sw, reqs, slot_ctx=slot_ctx, **wkw)
        forced = {"schedule": plan["waa_tp2"]["schedule"], "predicted_tok_s": plan["waa_tp2"]["predicted_tok_s"],
                  "tok_s": st_w["tok_s"], "p99_latency_s": float(np.percentile(lat_w, 99)) if rank == 0 else None}
    else:
        forced = plan["waa_tp2"]
    if rank == 0:
        upto = [lat[i] for i, r in enumerate(reqs) if r.output_len <= d.target_len]
        print(json.dumps({
            "metric": METRIC, "value": toks / wall, "unit": "output tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": MULTI_WORKLOAD, "layout": "plan", "latency_bound_s": L_b,
                       "bound_rule": "70th pctl of static-batch latencies (PAPER.md:490)",
                       "schedule": plan["pick"]["schedule"], "predicted_tok_s": plan["pick"]["predicted_tok_s"],
                       "predicted_latency_s": plan["pick"]["predicted_latency_s"], "requests_per_step": args.requests,
                       "parallelism": "plan over %d GPUs (one NCCL job)" % world},
            "e2e": {"value": toks / host, "unit": "output tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "sla": {"sla_b_met": bool(max(upto) < L_b), "sla_a_met": bool(np.percentile(lat, 99) <= L_b),
                    "max_latency_upto_p99_len_s": float(max(upto)), "p99_latency_s": float(np.percentile(lat, 99))},
            "forced_waa_tp2": forced, "clocks": clk.summary(),
            "paged_kv": ({"kv_page": pkw["kv_page"], "kv_pages": pkw["kv_pages"], "preemptions": st["kv_preemptions"],
                          "pages_peak": st["kv_pages_peak"], "mean_decode_batch": st["mean_decode_batch"]}
                         if pkw else None),
            "comm": ("measured: XProfiler tp_sync / pp_sync on this job's NCCL communicators" if world > 1 else
                     "one-GPU dry run: alpha-beta interconnect model")}))
    ctx.close()
    if dist:
        dist.destroy_process_group()


def run_reference(args, rank, world):
    """--impl reference: the oracle (CPU, float64, bf16-emulating KV loop)
    timed by its per-layer cost model on a bounded sample per step (see
    OracleCostModel); rank 0 only."""
    if rank != 0:
        return
    cm = OracleCostModel()
    for _ in range(args.warmup):
        cm.measure()
    vals, times, last = [], [], None
    for _ in range(args.steps):
        v, model_s, cpu_s, detail = cm.measure()
        vals.append(v)
        times.append(model_s)
        last = (v, model_s, cpu_s, detail)
    value = float(np.mean(vals))
    cpu = cpu_baseline_block(cm, value, *last[1:])
    out = {"metric": METRIC, "value": value, "unit": "output tokens/s",
           "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD, "oracle_sample": cpu["sample"]},
           "cpu_baseline": cpu,
           "e2e": {"value": value, "unit": "output tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


# ----------------------------------------------------------------------------
def main():
    if os.environ.get("EXG_PROFILE_INSITU"):   # diagnostics (A/B): in-situ decode attention table
        import paper_2404_07947_b200 as X
        X.lib().exg_diag_profile_insitu(int(os.environ["EXG_PROFILE_INSITU"]))
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--requests", type=int, default=1024, help="requests per step")
    ap.add_argument("--margin", type=float, default=0.03,
                    help="latency margin on top of the simulator's buffer time (its measured latency error is "
                         "within +-3%% on this workload, tools/sim_fidelity.py)")
    ap.add_argument("--little", type=int, default=1,
                    help="1: completion fraction by Little's law (SURVEY.md S3; DESIGN.md), 0: paper's E[1/ceil(S/N_D)]")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", default="plan", choices=["replicas", "plan"],
                    help="N > 1: config 4 under the scheduler's N-GPU plan as one NCCL job (default), or "
                         "independent config-2 replicas")
    ap.add_argument("--kv-page", type=int, default=0,
                    help="--layout plan: paged KV of this page length (planner and runner; 0 = slots)")
    ap.add_argument("--plan-dry-run", action="store_true",
                    help="run the N > 1 (config 4) path on one GPU (testing; no collective)")
    ap.add_argument("--multi-model", default=MULTI_MODEL)
    ap.add_argument("--multi-task", default=MULTI_TASK)
    ap.add_argument("--plan-gpus", type=lambda v: [int(x) for x in v.split(",") if x], default=[2, 4, 8],
                    help="cluster sizes for the scheduler's predicted multi-GPU plan")
    ap.add_argument("--dyn", type=float, default=0.1, help="dynamic workload adjustment threshold (0: skip the run)")
    ap.add_argument("--roofline-steps", type=int, default=1, help="extra steps with per-launch kernel events")
    ap.add_argument("--bounds", default="all", choices=["all", "headline"])
    ap.add_argument("--baseline-requests", type=int, default=512,
                    help="requests per in-runner baseline run (FT static / ORCA-style / ExeGPT); 0: skip")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.layout == "plan" and (world > 1 or args.plan_dry_run):
        run_layout(args, rank, world, local)
        return

    import torch
    import paper_2404_07947_b200 as X
    from workload import MODELS, make_requests, task_dists, weight_seed

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        return reduce_over_ranks(v, "max", dist)

    def sum_over_ranks(v):
        return reduce_over_ranks(v, "sum", dist)

    spec = MODELS[MODEL]
    d = task_dists(TASK)
    free, total = torch.cuda.mem_get_info(local)
    t_setup = time.perf_counter()
    ctx = X.Context(spec, weight_seed(CONFIG_NO), device=local,
                    cluster=X.cluster_spec(1, total - (6 << 30), 8 << 30))
    t_weights = time.perf_counter() - t_setup
    # XProfiler sweep
    t0 = time.perf_counter()
    prof = ctx.profile(PROFILE_BATCH, PROFILE_CTX, PROFILE_TOKENS, reps=3, tps=[1, 2, 4, 8])
    # interconnect tables: alpha-beta model of NVLink 5 / NVSwitch (DESIGN.md
    # reading; a single-GPU context cannot time them)
    prof.comm_model(COMM_ALPHA_S, COMM_BW)
    t_prof = time.perf_counter() - t0
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        prof.save(os.path.join(ROOT, "gpurun_out", "profile_opt13b.txt"))
    cl = ctx.cluster
    pin, pout = X.Pmf(d.pmf_in), X.Pmf(d.pmf_out)
    # static-batch latency sweep -> bounds
    bounds = static_bounds(X, prof, ctx.mspec, cl, pin, pout, d.target_len)
    scheds = {}
    t0 = time.perf_counter()
    for name, L_b in bounds:
        try:
            # schedule against L_B * (1 - margin): the paper budgets the encoder /
            # decoder stage-time variance (Table 9: +-7..12 %, PAPER.md:739,
            # 759-761) when choosing the control variables
            scheds[name] = X.schedule_find(prof, ctx.mspec, cl, pin, pout, d.target_len, L_b * (1 - args.margin),
                                           X.EXG_RRA,
                                           X.search_opts(b_e_max=B_E_MAX, little=args.little))
        except X.ExgError as e:
            scheds[name] = None
    t_sched = time.perf_counter() - t0

    reqs = make_requests(args.requests, d.pmf_in, d.pmf_out, spec.vocab, rank_request_seed(rank))
    slot_ctx = len(d.pmf_in) + len(d.pmf_out)
    h2d = sum((r.input_len - 1) * 12 + 16 + 16 * r.output_len for r in reqs)
    d2h = sum(4 * r.output_len for r in reqs)

    def sla(lat, L_b, rq=None):
        # SLA-(b) (the paper's main definition): a
        # sequence of the 99th-percentile length completes within L_B -- checked
        # on every request whose output is at most that long; SLA-(a): 99 % of
        # all requests complete within L_B.
        rq = reqs if rq is None else rq
        upto = [lat[i] for i, r in enumerate(rq) if r.output_len <= d.target_len]
        at = [lat[i] for i, r in enumerate(rq) if r.output_len == d.target_len]
        return {"sla_b_met": bool(max(upto) < L_b), "sla_a_met": bool(np.percentile(lat, 99) <= L_b),
                "max_latency_upto_p99_len_s": float(max(upto)),
                "max_latency_at_p99_len_s": float(max(at)) if at else None, "p99_latency_s": float(np.percentile(lat, 99))}

    head_name = "p70"
    head = scheds[head_name] or scheds["inf"]
    sched, est = head
    for _ in range(args.warmup):
        ctx.run(sched, reqs, slot_ctx=slot_ctx)
    barrier()
    dev_time, toks, launches = 0.0, 0, 0
    ktime = {k: 0.0 for k in ("prefill_gemm", "decode_gemm", "decode_attn", "prefill_attn")}
    kwork = dict(ktime)
    klaunch = {k: 0 for k in ktime}
    lats, steady = [], []
    with Clocks(local) as clk:
        th0 = time.perf_counter()
        if torch.cuda.is_available():
            torch.cuda.nvtx.range_push("timed")
        trace = []
        for step in range(args.steps):
            _, lat, st, _ = ctx.run(sched, reqs, slot_ctx=slot_ctx,
                                    trace=trace if step == args.steps - 1 else None)
            dev_time += st["wall_s"]
            toks += st["out_tokens"]
            launches += st["kernel_launches"]
            lats.append(lat)
            steady.append(st["tok_s_steady"])
            var_st = st
        if torch.cuda.is_available():
            torch.cuda.nvtx.range_pop()
        barrier()
        host_time = time.perf_counter() - th0
    # per-kernel-class CUDA events (engine stream, one pair per launch) on
    # extra steps of the same workload: an event between two launches
    # disables their programmatic-dependent-launch overlap (~5 % of a step),
    # so the timed steps above run without them
    kdev = 0.0
    enc_tokens_step = float(sum(r.input_len - 1 for r in reqs))   # decoder-only: n - 1 encoded per request
    for _ in range(args.roofline_steps):
        _, _, st, _ = ctx.run(sched, reqs, slot_ctx=slot_ctx, kernel_timing=True)
        kdev += st["wall_s"]
        for k, v in st["kernels"].items():
            ktime[k] += v["time_s"]
            kwork[k] += v["work"]
            klaunch[k] += v["launches"]
    dev_max = max_over_ranks(dev_time)
    host_max = max_over_ranks(host_time)
    toks_all = sum_over_ranks(toks)
    value = toks_all / dev_max
    e2e = toks_all / host_max
    L_head = dict(bounds)[head_name]
    s_ok = sla(lats[-1], L_head)

    other = {}
    if args.bounds == "all":
        for name, L_b in bounds:
            if scheds[name] is None:
                other[name] = {"latency_bound_s": L_b, "feasible": False}
                continue
            s2, e2 = scheds[name]
            _, lat2, st2, _ = ctx.run(s2, reqs, slot_ctx=slot_ctx)
            other[name] = {"latency_bound_s": L_b, "schedule": s2.as_dict(),
                           "predicted_tok_s": e2.thrput_tok_s, "predicted_latency_s": e2.latency_s,
                           "tok_s": st2["tok_s"], "tok_s_steady": st2["tok_s_steady"],
                           "lat_p99_s": st2["lat_p99_s"], "mean_decode_batch": st2["mean_decode_batch"],
                           "encode_s": st2["encode_s"], "decode_s": st2["decode_s"],
                           "encode_phases": st2["encode_phases"], "decode_iters": st2["decode_iters"],
                           "wall_s": st2["wall_s"], **sla(lat2, L_b)}

    # dynamic workload adjustment on the headline schedule:
    # one extra run, reported beside the plain one (not part of `value`)
    dyn = None
    if args.dyn > 0 and rank == 0:
        _, lat_d, st_d, _ = ctx.run(sched, reqs, slot_ctx=slot_ctx, dyn_threshold=args.dyn)
        dyn = {"threshold": args.dyn, "tok_s": st_d["tok_s"], "tok_s_steady": st_d["tok_s_steady"],
               "mean_encode_batch": st_d["mean_encode_batch"], "mean_decode_batch": st_d["mean_decode_batch"],
               "variance": workload_variance(st_d), **sla(lat_d, L_head)}

    # in-runner baselines (NEXT-4) on the first --baseline-requests requests
    base = None
    if args.baseline_requests > 0 and rank == 0:
        base = in_runner_baselines(args, X, ctx, prof, cl, pin, pout, d, bounds, scheds,
                                   reqs[:args.baseline_requests], slot_ctx, sla)

    def memory_gb(prof_, cl_, sch):
        """Per-GPU model / KV-cache GB of a schedule (exg_schedule_memory;
        the memory-overhead accounting of PAPER.md:548-560)."""
        w, kv = X.schedule_memory(prof_, ctx.mspec, cl_, pin, pout, sch)
        return {"model_gb": [round(x / 1e9, 2) for x in w], "kv_gb": [round(x / 1e9, 2) for x in kv]}

    memory = {"headline_rra": memory_gb(prof, cl, sched)}
    if base:
        for name, row in base.items():
            if "schedule" in row.get("ft_static", {}):
                memory["ft_static_" + name] = memory_gb(prof, cl, X.static_schedule(row["ft_static"]["schedule"]["b_e"]))

    # the scheduler's multi-GPU plan for this workload and bound (predicted by
    # the XSimulator on the measured per-GPU tables + the modeled interconnect)
    plan = {}
    for n in args.plan_gpus:
        try:
            cl_n = X.cluster_spec(n, cl.mem_per_gpu_bytes, cl.workspace_bytes)
            s_n, e_n = X.schedule_find(prof, ctx.mspec, cl_n, pin, pout, d.target_len, L_head * (1 - args.margin),
                                       X.EXG_RRA | X.EXG_WAA_C, X.search_opts(b_e_max=B_E_MAX, little=args.little))
            plan[str(n)] = {"predicted_tok_s": e_n.thrput_tok_s, "predicted_latency_s": e_n.latency_s,
                            "schedule": s_n.as_dict(), "memory": memory_gb(prof, cl_n, s_n)}
        except X.ExgError as e:
            plan[str(n)] = {"infeasible": str(e)}

    pk = peaks()
    # roofline of the dominant kernel class (time share) + decode attention
    dom = max(ktime, key=lambda k: ktime[k])
    traffic_ref = {}
    tp = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    if os.path.exists(tp):
        traffic_ref = json.load(open(tp))

    def roof(k):
        if klaunch[k] == 0 or ktime[k] <= 0:
            return None
        per_launch_work = kwork[k] / klaunch[k]
        avg_t = ktime[k] / klaunch[k]
        tensor = k in ("prefill_gemm", "prefill_attn")
        ach = per_launch_work / avg_t / (1e12 if tensor else 1e9)
        peak = pk["bf16_sus"] if tensor else pk["hbm"]
        tr = traffic_ref.get(k)
        traffic = tr["dram_bytes_per_work"] * per_launch_work if tr else None
        out = {"bound": "tensor" if tensor else "hbm", "achieved": ach, "peak": peak,
               "unit": "TFLOP/s" if tensor else "GB/s", "frac": ach / peak, "traffic": traffic,
               "kernel": k, "launches": klaunch[k], "time_share": ktime[k] / kdev if kdev else None,
               "measured": "CUDA events per launch on the engine stream, %d extra step(s)" % args.roofline_steps,
               "peak_src": pk["src"] + (" sustained" if tensor else "")}
        if k == "prefill_attn":
            # classical roofline: the FMHA's algorithmic bytes (q, k, v in, o
            # out: 4 T H dh 2 per layer launch) against its flops -- at task-S
            # lengths the arithmetic intensity is below the ridge, so HBM bounds
            # it
            byts = 4.0 * enc_tokens_step * spec.n_heads * spec.d_head * 2 * spec.n_dec_layers * args.roofline_steps
            ai = kwork[k] / byts
            ridge = pk["bf16_sus"] * 1e12 / (pk["hbm"] * 1e9)
            out["tensor_view"] = {"achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak}
            out["intensity_flop_per_byte"] = ai
            out["ridge_flop_per_byte"] = ridge
            if ai < ridge:
                bw = byts / klaunch[k] / avg_t / 1e9
                out.update({"bound": "hbm", "achieved": bw, "peak": pk["hbm"], "unit": "GB/s",
                            "frac": bw / pk["hbm"], "peak_src": pk["src"]})
        return out

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cm = OracleCostModel()
        cpu = cpu_baseline_block(cm, *cm.measure())
        # scheduler wall time, Python oracle vs the C++ planner, on the same
        # profile file and bound (PAPER.md:637 reports 3 s - 5 min for its own)
        cpu["schedule_find_s"] = scheduler_wall_times(X, prof, ctx, cl, pin, pout, d, L_head, args)

    if rank == 0:
        out = {
            "metric": METRIC,
            "value": value, "unit": "output tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * dev_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD,
                       "requests_per_step": args.requests, "latency_bound_s": L_head,
                       "bound_rule": "70th pctl of static-batch latencies (PAPER.md:490)",
                       "schedule": sched.as_dict(), "predicted_tok_s": est.thrput_tok_s,
                       "predicted_latency_s": est.latency_s,
                       "parallelism": "replicas" if world > 1 else "single-GPU",
                       "l2": "inputs larger than L2: 26 GB of weights + KV streamed every decode step"},
            "tok_s_steady": float(np.mean(steady)),
            "sla": s_ok,
            "roofline": roof(dom),
            "roofline_decode_attn": roof("decode_attn"),
            "roofline_decode_gemm": roof("decode_gemm"),
            "roofline_prefill_gemm": roof("prefill_gemm"),
            "roofline_prefill_attn": roof("prefill_attn"),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "output tokens/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "multi_gpu_plan": {"latency_bound_s": L_head, "comm": "modeled: alpha %.0f us, %.0f GB/s" %
                               (COMM_ALPHA_S * 1e6, COMM_BW / 1e9), "predicted": plan},
            "workload_variance": workload_variance(var_st, trace, prof, spec.n_dec_layers),
            "dyn_adjust": dyn,
            "memory": memory,
            "in_runner_baselines": base and {"requests": min(args.baseline_requests, args.requests),
                                             "rule": "same kernels / requests / bounds; FT static = best "
                                                     "simulated static batch within the bound (PAPER.md:112), "
                                                     "ORCA-style = RRA N_D=1 (PAPER.md:116)",
                                             "per_bound": base},
            "bounds": other,
            "setup_s": {"weights": t_weights, "profile": t_prof, "schedule_find_4_bounds": t_sched},
        }
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
