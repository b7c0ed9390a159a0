"""NEXT-3: distribution-shift robustness on config 2.

The p70-bound schedule chosen for task S is run on requests
drawn from shifted length distributions (mean / std of the input or output
length scaled; PAPER.md:593-632 studies the same question with shifted
statistics), next to a schedule re-optimised for the shifted distribution under
the same bound.  Reports throughput, p99 latency and the SLA readings.

    python tools/shift_experiment.py [n_requests] > profiles/r1_shift.json
"""
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2404_07947_b200 as X  # noqa: E402
from workload import (MODELS, TASKS, make_requests, task_dists, truncnorm_pmf, truncnorm_quantile,  # noqa: E402
                      weight_seed)

MARGIN = 0.15
SHIFTS = [  # (name, in_mu x, in_sigma x, out_mu x, out_sigma x)
    ("nominal", 1.0, 1.0, 1.0, 1.0),
    ("out_mean_x0.7", 1.0, 1.0, 0.7, 1.0),
    ("out_mean_x1.3", 1.0, 1.0, 1.3, 1.0),
    ("out_std_x1.3", 1.0, 1.0, 1.0, 1.3),
    ("in_mean_x0.7", 0.7, 1.0, 1.0, 1.0),
    ("in_mean_x1.3", 1.3, 1.0, 1.0, 1.0),
    ("in_std_x0.7", 1.0, 0.7, 1.0, 1.0),
]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    import torch
    spec = MODELS["opt-13b"]
    t = TASKS["S"]
    d = task_dists("S")
    free, total = torch.cuda.mem_get_info(0)
    ctx = X.Context(spec, weight_seed(2), cluster=X.cluster_spec(1, total - (6 << 30), 8 << 30))
    prof = ctx.profile([1, 2, 4, 8, 16, 32, 48, 64, 96, 128, 160, 192, 224, 256, 320, 384, 448, 512],
                       [1, 32, 64, 128, 192, 256, 320, 384, 448, 512, 592],
                       [1, 16, 64, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768], reps=3)
    cl = ctx.cluster
    pin0, pout0 = X.Pmf(d.pmf_in), X.Pmf(d.pmf_out)
    L_b = dict(bench.static_bounds(X, prof, ctx.mspec, cl, pin0, pout0, d.target_len))["p70"]
    opts = X.search_opts(b_e_max=bench.B_E_MAX, little=1)
    s_nom, e_nom = X.schedule_find(prof, ctx.mspec, cl, pin0, pout0, d.target_len, L_b * (1 - MARGIN), X.EXG_RRA,
                                   opts)
    slot_ctx = t.in_max + t.out_max
    for name, fi_m, fi_s, fo_m, fo_s in SHIFTS:
        pin = truncnorm_pmf(t.in_avg * fi_m, t.in_std * fi_s, t.in_max)
        pout = truncnorm_pmf(d.mu0 * fo_m, d.sigma0 * fo_s, t.out_max)
        target = int(math.ceil(truncnorm_quantile(d.mu0 * fo_m, d.sigma0 * fo_s, t.out_max, 0.99)))
        reqs = make_requests(n, pin, pout, spec.vocab, 0xE6E1_3000)
        row = {"shift": name, "latency_bound_s": L_b, "p99_output_len": target,
               "mean_in": float(np.mean([r.input_len for r in reqs])),
               "mean_out": float(np.mean([r.output_len for r in reqs]))}
        try:
            s_re, e_re = X.schedule_find(prof, ctx.mspec, cl, X.Pmf(pin), X.Pmf(pout), target, L_b * (1 - MARGIN),
                                         X.EXG_RRA, opts)
        except X.ExgError:
            s_re = None
        for tag, s in (("nominal_schedule", s_nom), ("reoptimised", s_re)):
            if s is None:
                row[tag] = {"feasible": False}
                continue
            _, lat, st, _ = ctx.run(s, reqs, slot_ctx=slot_ctx)
            upto = [lat[i] for i, r in enumerate(reqs) if r.output_len <= target]
            row[tag] = {"schedule": {k: s.as_dict()[k] for k in ("b_e", "b_d", "n_d")}, "tok_s": st["tok_s"],
                        "p99_latency_s": float(np.percentile(lat, 99)),
                        "sla_a_met": bool(np.percentile(lat, 99) <= L_b),
                        "sla_b_met": bool(max(upto) < L_b) if upto else None}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
