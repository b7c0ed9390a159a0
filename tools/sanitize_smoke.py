"""compute-sanitizer target (SURVEY.md §4 tier T5): small runs through every
kernel family -- config 1 bf16 (RRA, static batch, dynamic adjustment) and
fp32, a T5 model with tensor-core attention (dh = 128), a width-2048 model
with split stream-K tiles (deferred and in-kernel reductions), an emulated
WAA layout with a TP-2 decoder stage, a small profile, and paged KV (one-GPU
RRA with recompute preemption, WAA with swap preemption; dh = 128 pages of 64).

    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_07947_b200 as X  # noqa: E402
from paper_2404_07947_b200 import _lib as L  # noqa: E402
from workload import MODELS, ModelSpec, config1_requests, make_requests, uniform_pmf, weight_seed  # noqa: E402

reqs = config1_requests()
tiny = MODELS["tiny"]
c = X.Context(tiny, weight_seed(1))
c.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
c.run(X.static_schedule(3), reqs)
c.run(X.rra_schedule(4, 8, 3), reqs, dyn_threshold=0.1)
c.profile([1, 4], [16, 48], [16, 64], reps=1, tps=[1, 2])
c.close()
c = X.Context(tiny, weight_seed(1), dtype=X.EXG_FP32)
c.run(X.rra_schedule(4, 8, 6), reqs, dump=range(len(reqs)))
c.close()
t5 = MODELS["small-t5"]
r5 = make_requests(3, uniform_pmf(100, 160), uniform_pmf(2, 4), t5.vocab, 0xE6E10003)
c = X.Context(t5, weight_seed(3))
c.run(X.rra_schedule(2, 3, 2), r5, dump=range(3))
c.close()
w = ModelSpec("san-w2048", "opt", 0, 1, 2048, 16, 128, 8192, 4096, 256)
rw = make_requests(20, uniform_pmf(8, 64), uniform_pmf(2, 6), w.vocab, 5)
for mask in (0, 3):
    X.lib().exg_diag_deferred(mask)
    c = X.Context(w, 77)
    c.run(X.rra_schedule(10, 20, 3), rw)
    c.close()
X.lib().exg_diag_deferred(-1)
m = X.Context(tiny, weight_seed(1), cluster=X.cluster_spec(4))
s = L.make_schedule(X.EXG_WAA_C, 2, 8, [(0, 1, 0, 2), (1, 2, 0, 1), (3, 1, 1, 2)], b_m=4, n_enc_gpus=1, tp_degree=2,
                    tp_gpus=2)
m.run(s, reqs, dump=range(len(reqs)))
m.close()
pg = ModelSpec("san-paged", "opt", 0, 2, 256, 2, 128, 512, 512, 512)
rp = make_requests(12, uniform_pmf(20, 100), uniform_pmf(100, 300), pg.vocab, 0xE6E1_00A2)
c = X.Context(pg, 0xE6E0_00A1)
c.run(X.rra_schedule(8, 12, 200), rp, kv_page=64, kv_pages=12)
c.close()
m = X.Context(pg, 0xE6E0_00A1, cluster=X.cluster_spec(4))
s = L.make_schedule(X.EXG_WAA_C, 4, 12, [(0, 1, 0, 2), (1, 1, 0, 1), (2, 1, 1, 2)], b_m=6, n_enc_gpus=1)
m.run(s, rp, kv_page=64, kv_pages=12)
m.close()
print("sanitize smoke done")
