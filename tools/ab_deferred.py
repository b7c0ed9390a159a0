"""A/B of the deferred stream-K reduction (gemm_tc.cuh) on the OPT-13B RRA
run: two contexts built with the reduction off / on (exg_diag_deferred),
runs interleaved on the same box; decode / encode phase times, tokens (must
be identical) and per-class kernel times.

    python tools/ab_deferred.py [requests] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_07947_b200 as X  # noqa: E402
from workload import MODELS, make_requests, task_dists, weight_seed  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = MODELS["opt-13b"]
d = task_dists("S")
reqs = make_requests(n, d.pmf_in, d.pmf_out, spec.vocab, 0xE6E10002)
# modes: 0..3 = deferred mask with the per-kernel decode path; 10 = decode GEMM chain
MODES = [int(x) for x in os.environ.get("EXG_DEFER_MODES", "2,10").split(",")]
ctxs = {}
for on in MODES:
    X.lib().exg_diag_chain(1 if on == 10 else 0)
    X.lib().exg_diag_deferred(on if on < 10 else -1)
    ctxs[on] = X.Context(spec, weight_seed(2))
X.lib().exg_diag_deferred(-1)
X.lib().exg_diag_chain(0)
sched = X.rra_schedule(56, 83, 32)
toks = {}
for r in range(reps):
    for on in MODES:
        t, lat, st, _ = ctxs[on].run(sched, reqs, slot_ctx=592)
        toks[on] = t
        print("deferred %d rep %d tok_s %.1f decode_s %.4f encode_s %.4f iters %d" % (
            on, r, st["tok_s"], st["decode_s"], st["encode_s"], st["decode_iters"]))
        sys.stdout.flush()
print("tokens identical:", all(toks[m] == toks[MODES[0]] for m in MODES))
for on in MODES:
    _, _, st, _ = ctxs[on].run(sched, reqs, slot_ctx=592, kernel_timing=True)
    print("deferred %d kernels: %s" % (on, {k: (round(v["time_s"], 4), v["launches"]) for k, v in st["kernels"].items()}))
