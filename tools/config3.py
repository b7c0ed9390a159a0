"""Config 3 end to end on one B200: T5-11B (seeded random init), task T
(translation-shaped lengths) -- XProfiler on the full model,
static-batch bounds, the scheduler's 1-GPU RRA schedule (measured) and its
2-GPU plan (predicted; run in single-device emulation to check it reproduces
the 1-GPU tokens bit for bit).

    python tools/config3.py [n_requests] > profiles/r1_config3.json
"""
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2404_07947_b200 as X  # noqa: E402
from workload import MODELS, TASKS, make_requests, task_dists, weight_seed  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    import torch
    spec = MODELS["t5-11b"]
    t = TASKS["T"]
    d = task_dists("T")
    free, total = torch.cuda.mem_get_info(0)
    if os.environ.get("EXG_PROFILE_INSITU"):   # diagnostics: in-situ decode attention table
        X.lib().exg_diag_profile_insitu(int(os.environ["EXG_PROFILE_INSITU"]))
    t0 = time.perf_counter()
    ctx = X.Context(spec, weight_seed(3), cluster=X.cluster_spec(1, total - (40 << 30), 8 << 30))
    prof = ctx.profile([1, 2, 4, 8, 16, 32, 64, 96, 128, 192, 256], [1, 32, 64, 128, 192, 256, 384, 512, 576],
                       [1, 16, 64, 256, 512, 1024, 2048, 4096, 8192, 16384], reps=3)
    prof.comm_model(bench.COMM_ALPHA_S, bench.COMM_BW)
    t_prof = time.perf_counter() - t0
    cl = ctx.cluster
    pin, pout = X.Pmf(d.pmf_in), X.Pmf(d.pmf_out)
    bounds = bench.static_bounds(X, prof, ctx.mspec, cl, pin, pout, d.target_len)
    L_b = dict(bounds)["p70"]
    opts = X.search_opts(b_e_max=64, little=1)
    s1, e1 = X.schedule_find(prof, ctx.mspec, cl, pin, pout, d.target_len, L_b * 0.85, X.EXG_RRA, opts)
    cl2 = X.cluster_spec(2, cl.mem_per_gpu_bytes, cl.workspace_bytes)
    try:
        s2, e2 = X.schedule_find(prof, ctx.mspec, cl2, pin, pout, d.target_len, L_b * 0.85,
                                 X.EXG_RRA | X.EXG_WAA_C | X.EXG_WAA_M, opts)
    except X.ExgError as e:
        s2, e2 = None, str(e)
    reqs = make_requests(n, d.pmf_in, d.pmf_out, spec.vocab, 0xE6E1_0003)
    slot_ctx = t.out_max
    ctx.run(s1, reqs, slot_ctx=slot_ctx)
    trace = []
    toks1, lat, st, _ = ctx.run(s1, reqs, slot_ctx=slot_ctx, trace=trace)
    # simulator fidelity per stage: measured encode phases / decode iterations
    # against the profile's time for the same rows and work
    # (exg_profile_stage_time), and the batch trajectory
    fid = {}
    # decode iterations >= 16 after the last encode phase (outside the clock
    # recovery the simulator charges separately through its switch table)
    since, late = 10 ** 9, []
    for r in trace:
        if int(r[0]) == 1 and r[3] > 0:
            since = 0
        elif int(r[0]) == 2:
            since += 1
            late.append(since > 16)
    # mean decode batch between the third and the last encode phase (the
    # steady state: after the ramp-up, before the drain) vs the model's mean b_u
    enc_idx = [i for i, r in enumerate(trace) if int(r[0]) == 1 and r[3] > 0]
    if len(enc_idx) >= 4:
        mid = [r[3] for r in trace[enc_idx[2]:enc_idx[-1]] if int(r[0]) == 2]
        fid["steady_mean_decode_batch"] = float(np.mean(mid)) if mid else None
    for kind, name, ph in ((1, "encode", 0), (2, "decode", 1), (3, "decode_after_recovery", 1)):
        if kind == 3:
            recs = [r for r, ok in zip([r for r in trace if int(r[0]) == 2], late) if ok and r[3] > 0]
        else:
            recs = [r for r in trace if int(r[0]) == kind and r[3] > 0]
        meas = sum(r[2] for r in recs)
        pred = sum(prof.stage_time(ph, r[3], r[4], spec.n_dec_layers) for r in recs)
        fid[name] = {"stages": len(recs), "measured_s": meas, "profile_s": pred,
                     "measured_over_profile": meas / pred if pred > 0 else None,
                     "mean_rows": float(np.mean([r[3] for r in recs])) if recs else 0.0}
    out = {"workload": "config 3: T5-11B (seeded random init), task T, %d requests" % n,
           "profile_s": t_prof, "latency_bound_s": L_b, "bounds": bounds,
           "one_gpu": {"schedule": s1.as_dict(), "predicted_tok_s": e1.thrput_tok_s,
                       "predicted_latency_s": e1.latency_s, "tok_s": st["tok_s"], "tok_s_steady": st["tok_s_steady"],
                       "p99_latency_s": float(np.percentile(lat, 99)), "mean_decode_batch": st["mean_decode_batch"],
                       "encode_s": st["encode_s"], "decode_s": st["decode_s"],
                       "sla_a_met": bool(np.percentile(lat, 99) <= L_b), "stage_fidelity": fid}}
    if s2 is not None:
        ctx.close()
        del ctx
        out["two_gpu_plan"] = {"schedule": s2.as_dict(), "predicted_tok_s": e2.thrput_tok_s,
                               "predicted_latency_s": e2.latency_s}
        try:
            # both GPUs of the plan emulated on this device (their weights and KV
            # share its memory): per-request results must equal the 1-GPU run's
            m = X.Context(spec, weight_seed(3), cluster=cl2)
            k = min(n, 32)
            toks2, _, _, _ = m.run(s2, reqs[:k], slot_ctx=slot_ctx)
            out["two_gpu_plan"]["emulated_tokens_equal_one_gpu"] = toks2 == toks1[:k]
            m.close()
        except X.ExgError as e:
            out["two_gpu_plan"]["emulation"] = "skipped: %s" % e
    else:
        out["two_gpu_plan"] = {"infeasible": e2}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
