"""Does the XProfiler's encode table depend on the GPU's power state?  Profile
cold, then after a sustained OPT-13B run, then again; print rest(enc, T)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_07947_b200 as X  # noqa: E402
from oracle import simulator as sim  # noqa: E402
from workload import MODELS, make_requests, task_dists, weight_seed  # noqa: E402

spec = MODELS["opt-13b"]
d = task_dists("S")
ctx = X.Context(spec, weight_seed(2))
reqs = make_requests(256, d.pmf_in, d.pmf_out, spec.vocab, 0xE6E10002)


def prof(tag):
    p = ctx.profile([1, 16, 64], [64, 256], [1024, 4096, 8192], reps=3)
    path = "/tmp/p_%s.txt" % tag
    p.save(path)
    P = sim.Profile.loads(open(path).read())
    tb = P.rest[("enc", 1)]
    print(tag, "enc rest", " ".join("%d:%.0f" % (x, y * 1e6) for x, y in zip(tb.x, tb.t)),
          "| dec rest", " ".join("%d:%.0f" % (x, y * 1e6) for x, y in zip(P.rest[("dec", 1)].x, P.rest[("dec", 1)].t)))


prof("cold")
t0 = time.time()
_, _, st, _ = ctx.run(X.rra_schedule(30, 74, 16), reqs, slot_ctx=592)
print("run: encode_s %.3f phases %d -> %.1f ms/phase" % (st["encode_s"], st["encode_phases"],
                                                         1e3 * st["encode_s"] / st["encode_phases"]))
prof("after_run")
ctx.run(X.rra_schedule(30, 74, 16), reqs, slot_ctx=592)
prof("after_run2")
