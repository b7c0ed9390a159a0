"""Per-CTA timeline of one decode-chain launch (OPT-13B layer shapes) from
the chain's %globaltimer marks (exg_diag_chain_timeline)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_07947_b200 as X  # noqa: E402
from workload import MODELS, make_requests, task_dists, uniform_pmf  # noqa: E402

spec = MODELS["opt-13b"]
from workload import ModelSpec  # noqa: E402
sp = ModelSpec("opt13b-2l", "opt", 0, 2, spec.d_model, spec.n_heads, spec.d_head, spec.d_ff, spec.vocab, spec.max_pos)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 56
reqs = make_requests(B, uniform_pmf(200, 300), uniform_pmf(6, 6), sp.vocab, 3)
ctx = X.Context(sp, 11)
lib = X.lib()
lib.exg_diag_chain_timeline.argtypes = [C.c_int, C.c_void_p]
ctx.run(X.rra_schedule(B, B, 8), reqs)
lib.exg_diag_chain_timeline(1, None)
ctx.run(X.rra_schedule(B, B, 8), reqs)
tl = np.zeros(256 * 32, dtype=np.uint64)
lib.exg_diag_chain_timeline(0, tl.ctypes.data)
tl = tl.reshape(256, 32)[:148].astype(np.float64)
t0 = tl[:, 0].min()
names = {0: "entry", 1: "in0", 2: "in1", 3: "in2", 4: "in3", 5: "fin0", 6: "fin1", 7: "fin2", 8: "fin3",
         9: "ln0", 10: "ln1", 11: "ln2", 12: "ln3", 13: "prod_end", 14: "epi_exit",
         16: "mma0_first", 17: "mma1_first", 18: "mma2_first", 19: "mma3_first",
         20: "mma0_last", 21: "mma1_last", 22: "mma2_last", 23: "mma3_last"}
for k, nm in names.items():
    v = tl[:, k]
    v = v[v > 0]
    if len(v) == 0:
        continue
    v = (v - t0) / 1e3
    print("%-9s n=%3d min %7.2f med %7.2f max %7.2f us" % (nm, len(v), v.min(), np.median(v), v.max()))
