"""The scheduler's plans for configs 4 and 5 (BASELINE.json), which do not fit
one B200 as whole models: per-layer tables are profiled on a ONE-layer context
of the model's exact shape (and its TP-rank-0 shards for t = 2, 4, 8), the
interconnect from the alpha-beta model; Algorithm 1 then plans the full model on
N GPUs.  Predictions only (the layouts' arithmetic is checked at full width in
tests/test_gpu_fullsize.py).

    python tools/plan_configs.py > profiles/r2_plans.json

Each config is planned with KV slots and with paged KV (kv_page = 64).
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2404_07947_b200 as X  # noqa: E402
from workload import MODELS, ModelSpec, task_dists, weight_seed  # noqa: E402

CONFIGS = [  # (config, model, task, GPU counts, strategies)
    ("config 4", "opt-66b", "G", (4, 8), X.EXG_RRA | X.EXG_WAA_C | X.EXG_WAA_M),
    ("config 5 (C1)", "gpt3-175b", "C1", (8,), X.EXG_RRA | X.EXG_WAA_C | X.EXG_WAA_M),
    ("config 5 (C2)", "gpt3-175b", "C2", (8,), X.EXG_RRA | X.EXG_WAA_C | X.EXG_WAA_M),
]


bench_margin = 0.03   # the bench's scheduler margin on top of the simulator's buffer time


def main():
    import torch
    free, total = torch.cuda.mem_get_info(0)
    profs = {}
    for name, model, task, gpus, mask in CONFIGS:
        full = MODELS[model]
        d = task_dists(task)
        if model not in profs:
            one = ModelSpec(model + "-1layer", full.arch, 0, 1, full.d_model, full.n_heads, full.d_head, full.d_ff,
                            full.vocab, full.max_pos)
            ctx1 = X.Context(one, weight_seed(4))
            tps = [t for t in (1, 2, 4, 8) if full.n_heads % t == 0]
            prof = ctx1.profile([1, 2, 4, 8, 16, 32, 64, 128, 256, 512], [1, 64, 128, 256, 512, 1024, 1664],
                                [1, 64, 256, 1024, 4096, 8192, 16384, 32768], reps=3, tps=tps)
            prof.comm_model(bench.COMM_ALPHA_S, bench.COMM_BW)
            profs[model] = (prof, ctx1)
        prof, ctx1 = profs[model]
        mspec = X.model_spec(full, weight_seed(4))   # the full model for the planner
        pin, pout = X.Pmf(d.pmf_in), X.Pmf(d.pmf_out)
        row = {"config": name, "model": model, "task": task, "plans": {}}
        for n in gpus:
            for kv_page, key in ((0, "plans"), (64, "plans_paged_kv")):
                # paged KV (NEXT-2): the planner charges a decode row its live
                # positions; the static-batch bounds keep slots (FT does not page)
                cl = X.cluster_spec(n, total - (6 << 30), 8 << 30, kv_page=kv_page)
                try:
                    bounds = bench.static_bounds(X, prof, mspec, cl, pin, pout, d.target_len)
                except Exception as e:  # noqa: BLE001
                    row.setdefault(key, {})[str(n)] = {"bounds": "static baseline infeasible: %s" % e}
                    continue
                per = {}
                for bname, L_b in bounds:
                    try:
                        s, e = X.schedule_find(prof, mspec, cl, pin, pout, d.target_len,
                                               L_b * (1 - bench_margin) if math.isfinite(L_b) else L_b, mask,
                                               X.search_opts(b_e_max=64, little=1))
                        mem_w, mem_kv = X.schedule_memory(prof, mspec, cl, pin, pout, s)
                        per[bname] = {"bound_s": L_b, "schedule": s.as_dict(), "predicted_tok_s": e.thrput_tok_s,
                                      "predicted_latency_s": e.latency_s,
                                      "max_gpu_gb": round(max(a + b for a, b in zip(mem_w, mem_kv)) / 1e9, 2)}
                    except X.ExgError as ex:
                        per[bname] = {"bound_s": L_b, "infeasible": str(ex)}
                row.setdefault(key, {})[str(n)] = per
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
