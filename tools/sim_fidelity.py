"""Simulator fidelity on one B200 (VERDICT r1 "next" #7): run the bench's
config-2 schedules with the per-stage trace (exg_run_opts.trace_out) and
compare every measured encode phase / decode iteration with the XSimulator's
stage time for the same rows and work, and the run's throughput / latency
with the simulator's estimate.  Writes gpurun_out/sim_fidelity.json.

    python tools/sim_fidelity.py [--requests 1024] [--margin 0.15]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=1024)
    ap.add_argument("--margins", default="0.15", help="comma-separated latency margins to run")
    ap.add_argument("--little", type=int, default=1)
    ap.add_argument("--bounds", default="p10,p30,p70,inf")
    args = ap.parse_args()
    import torch
    import paper_2404_07947_b200 as X
    from oracle import simulator as sim
    from workload import MODELS, make_requests, task_dists, weight_seed
    spec = MODELS[bench.MODEL]
    d = task_dists(bench.TASK)
    free, total = torch.cuda.mem_get_info(0)
    ctx = X.Context(spec, weight_seed(bench.CONFIG_NO), cluster=X.cluster_spec(1, total - (6 << 30), 8 << 30))
    prof = ctx.profile(bench.PROFILE_BATCH, bench.PROFILE_CTX, bench.PROFILE_TOKENS, reps=3, tps=[1])
    prof.comm_model(bench.COMM_ALPHA_S, bench.COMM_BW)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out", "profile_fidelity.txt")
    prof.save(path)
    P = sim.Profile.load(path)
    m = sim.SimModel.from_spec(spec)
    cl = ctx.cluster
    S = sim.Simulator(P, m, sim.SimCluster(1, cl.mem_per_gpu_bytes, cl.workspace_bytes), d.pmf_in, d.pmf_out,
                      d.target_len, use_little_fraction=bool(args.little))
    pin, pout = X.Pmf(d.pmf_in), X.Pmf(d.pmf_out)
    bounds = dict(bench.static_bounds(X, prof, ctx.mspec, cl, pin, pout, d.target_len))
    reqs = make_requests(args.requests, d.pmf_in, d.pmf_out, spec.vocab, bench.rank_request_seed(0))
    slot_ctx = len(d.pmf_in) + len(d.pmf_out)
    L = m.n_dec_layers
    out = {"bounds": {}}
    ctx.run(X.rra_schedule(8, 16, 8), reqs[:64], slot_ctx=slot_ctx)   # warm-up
    for name, margin in [(b, float(m)) for b in args.bounds.split(",") for m in args.margins.split(",")]:
        L_b = bounds[name]
        s, e = X.schedule_find(prof, ctx.mspec, cl, pin, pout, d.target_len, L_b * (1 - margin), X.EXG_RRA,
                               X.search_opts(b_e_max=bench.B_E_MAX, little=args.little))
        tr = []
        _, lat, st, _ = ctx.run(s, reqs, slot_ctx=slot_ctx, trace=tr)
        tr = np.array(tr)
        np.save(os.path.join(ROOT, "gpurun_out", "sim_trace_%s_m%g.npy" % (name, margin)), tr)
        enc, dec = tr[tr[:, 0] == 1], tr[tr[:, 0] == 2]

        def pred_enc(rows, toks):
            a = sim.interp2(P.attn[("enc", 1)], rows, toks / rows)
            r = sim.interp1(P.rest[("enc", 1)].x, P.rest[("enc", 1)].t, toks)
            return L * (a + r)

        def pred_dec(rows, keys):
            a = sim.interp2(P.attn[("dec", 1)], rows, keys / rows)
            r = sim.interp1(P.rest[("dec", 1)].x, P.rest[("dec", 1)].t, rows)
            h = sim.interp1(P.head.x, P.head.t, rows) if P.head is not None else 0.0
            return L * (a + r) + h

        pe = np.array([pred_enc(r[3], r[4]) for r in enc])
        pd = np.array([pred_dec(r[3], r[4]) for r in dec])
        re, rd = enc[:, 2] / pe, dec[:, 2] / pd
        # residual of decode iteration time after the batch / context
        # dependence the profile explains: the noise part of Table 9's spread
        dev = np.abs(dec[:, 2] - dec[:, 2].mean())
        resid = np.abs(dec[:, 2] - pd * rd.mean())
        sched = s.as_dict()
        sim_s = S.rra_schedule(s.b_e, s.n_d, 1, 0)
        pu, f = S.pu(s.n_d)
        import oracle.seqdist as sq
        bu = sq.rra_iteration_batches(sim_s.b_d, pu)
        upto = [lat[i] for i, r in enumerate(reqs) if r.output_len <= d.target_len]
        row = {
            "latency_bound_s": L_b, "margin": margin, "schedule": sched,
            "predicted": {"tok_s": e.thrput_tok_s, "latency_s": e.latency_s, "b_d": sim_s.b_d,
                          "mean_b_u": float(np.mean(bu)), "T_enc_s": pred_enc(s.b_e, s.b_e * S.s_e),
                          "T_dec_mean_s": float(np.mean([pred_dec(b, b * S.ctx_mean) for b in bu]))},
            "measured": {"tok_s": st["tok_s"], "tok_s_steady": st["tok_s_steady"],
                         "max_latency_upto_p99_len_s": float(max(upto)), "lat_p99_s": st["lat_p99_s"],
                         "mean_decode_batch": st["mean_decode_batch"], "mean_encode_batch": st["mean_encode_batch"],
                         "encode_phases": int(len(enc)), "decode_iters": int(len(dec)),
                         "T_enc_mean_s": float(enc[:, 2].mean()), "T_dec_mean_s": float(dec[:, 2].mean())},
            "stage_ratio_measured_over_profile": {
                "encode_mean": float(re.mean()), "encode_p10_p90": [float(np.percentile(re, 10)), float(np.percentile(re, 90))],
                "decode_mean": float(rd.mean()), "decode_p10_p90": [float(np.percentile(rd, 10)), float(np.percentile(rd, 90))]},
            "decode_variance": {"p99_range_pct": float(100 * np.percentile(dev, 99) / dec[:, 2].mean()),
                                "p99_residual_pct_after_profile_model": float(100 * np.percentile(resid, 99) / dec[:, 2].mean())},
            "decode_gap_s_mean": float(np.mean(np.diff(dec[:, 1]) - dec[:-1, 2])) if len(dec) > 1 else None,
        }
        row["sla_b_met"] = bool(max(upto) < L_b)
        out["bounds"]["%s_m%g" % (name, margin)] = row
        print(name, margin, json.dumps(row))
        sys.stdout.flush()
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sim_fidelity.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
