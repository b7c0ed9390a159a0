"""Chain vs separate decode launches: where do results differ?"""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_2404_07947_b200 as X
from workload import ModelSpec, make_requests, uniform_pmf
spec = ModelSpec("chain-w2048", "gpt3", 0, 2, 2048, 16, 128, 8192, 4096, 512)
reqs = make_requests(160, uniform_pmf(8, 64), uniform_pmf(2, 12), spec.vocab, 0xC4A1)
outs = {}
for on in (0, 1):
    X.lib().exg_diag_chain(on)
    ctx = X.Context(spec, 0xE6E0_0C4A)
    for rep in range(3):
        outs[(on, rep)] = ctx.run(X.rra_schedule(150, 150, 4), reqs, dump=range(len(reqs)))
    ctx.close()
X.lib().exg_diag_chain(1)
ref = outs[(0, 0)]
for k, o in outs.items():
    bad = [r for r in range(len(reqs)) if not np.array_equal(o[3][r], ref[3][r])]
    first = None
    for r in bad:
        t = next(t for t in range(reqs[r].output_len) if not np.array_equal(o[3][r][t], ref[3][r][t]))
        first = (r, t) if first is None or t < first[1] else first
    print(k, "tokens equal", o[0] == ref[0], "bad rows", len(bad), "earliest (row, step)", first, flush=True)
