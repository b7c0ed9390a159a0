"""A/B a GEMM diagnostics flag on the OPT-13B RRA run (decode / encode phase times).
    python tools/ab_decode.py FLAG [FLAG ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_07947_b200 as X  # noqa: E402
from paper_2404_07947_b200 import _lib as _L  # noqa: E402
_L.LIB_PATH = os.environ.get("EXG_PROBE_LIB", _L.LIB_PATH)   # A/B against another build
from workload import MODELS, make_requests, task_dists, weight_seed  # noqa: E402

spec = MODELS["opt-13b"]
d = task_dists("S")
ctx = X.Context(spec, weight_seed(2))
reqs = make_requests(256, d.pmf_in, d.pmf_out, spec.vocab, 0xE6E10002)
if os.environ.get("EXG_DECODE_MERGE"):   # 1: separate combine kernel for attention splits
    X.lib().exg_diag_decode_merge(int(os.environ["EXG_DECODE_MERGE"]))
if os.environ.get("EXG_DECODE_STAGES"):   # decode-attention ring depth / CTAs per SM variant
    X.lib().exg_diag_decode_stages(int(os.environ["EXG_DECODE_STAGES"]))
if os.environ.get("EXG_LN_PRELOAD"):    # 0: deferred LayerNorm preloads only the first segment
    X.lib().exg_diag_ln_preload(int(os.environ["EXG_LN_PRELOAD"]))
if os.environ.get("EXG_DECODE_SPLIT"):
    X.lib().exg_diag_decode_split(int(os.environ["EXG_DECODE_SPLIT"]))
for f in [int(x) for x in sys.argv[1:]] or [0]:
    X.lib().exg_diag_gemm_flags(f)
    for r in range(3):
        toks, lat, st, _ = ctx.run(X.rra_schedule(24, 79, 9), reqs, slot_ctx=592)
        print("flag %d rep %d tok_s %.1f decode_s %.4f encode_s %.4f tokens_hash %d" % (
            f, r, st["tok_s"], st["decode_s"], st["encode_s"], hash(tuple(map(tuple, toks))) & 0xffffffff))
X.lib().exg_diag_gemm_flags(0)
