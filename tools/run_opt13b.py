"""Run config 2 (OPT-13B, task S) under a fixed RRA schedule and print the
run statistics -- a small driver for ncu launch lists and timing checks.

    python tools/run_opt13b.py [n_requests] [b_e b_d n_d] [--timing] [--repeat R]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_07947_b200 as X  # noqa: E402
from workload import MODELS, make_requests, task_dists, weight_seed  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 64
b_e, b_d, n_d = (int(x) for x in args[1:4]) if len(args) >= 4 else (24, 79, 9)
rep = int(sys.argv[sys.argv.index("--repeat") + 1]) if "--repeat" in sys.argv else 2
spec = MODELS["opt-13b"]
d = task_dists("S")
ctx = X.Context(spec, weight_seed(2))
reqs = make_requests(n, d.pmf_in, d.pmf_out, spec.vocab, 0xE6E10002)
for r in range(rep):
    toks, lat, st, _ = ctx.run(X.rra_schedule(b_e, b_d, n_d), reqs, slot_ctx=592, kernel_timing="--timing" in sys.argv)
    k = st.pop("kernels")
    print(json.dumps({"rep": r, **{x: st[x] for x in ("tok_s", "wall_s", "encode_s", "decode_s", "decode_iters",
                                                     "mean_decode_batch", "kernel_launches")},
                      "kernels": {c: {"t": v["time_s"], "n": v["launches"],
                                      "rate": (v["work"] / v["time_s"] if v["time_s"] else 0)} for c, v in k.items()}}))
