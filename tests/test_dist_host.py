"""Multi-rank host logic on CPU (world_size 2, gloo, 127.0.0.1): the bench's
weak-scaling reductions (whole-job tokens / slowest rank's time) and the
per-rank request streams.  The device-side multi-rank executor is covered by
tests/test_gpu_multi.py (thread ranks on one GPU)."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from workload import make_requests, task_dists
    try:
        toks = 100.0 * (rank + 1)
        secs = 2.0 + rank
        value = bench.job_throughput(toks, secs, dist, "cpu")
        mx = bench.reduce_over_ranks(float(rank), "max", dist, "cpu")
        d = task_dists("S")
        reqs = make_requests(4, d.pmf_in, d.pmf_out, 50272, bench.rank_request_seed(rank))
        q.put((rank, value, mx, [r.ids[:4].tolist() for r in reqs]))
    finally:
        dist.destroy_process_group()


def test_weak_scaling_reductions_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, value, mx, ids in out:
        assert value == pytest.approx((100.0 + 200.0) / 3.0)   # sum of tokens / max of times
        assert mx == 1.0
    assert out[0][3] != out[1][3]                               # independent request streams per rank


def _plan_inputs():
    """config 4's planner inputs on a synthetic roofline profile (test
    fixture; the bench measures the real one)."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import tempfile
    import bench
    from oracle import simulator as sim
    from paper_2404_07947_b200 import _lib as L
    from test_oracle_scheduler import _synthetic_profile
    from workload import MODELS, task_dists
    spec = MODELS[bench.MULTI_MODEL]
    d = task_dists(bench.MULTI_TASK)
    prof = _synthetic_profile(sim.SimModel.from_spec(spec))
    with tempfile.TemporaryDirectory() as tmp:
        prof.save(os.path.join(tmp, "p.txt"))
        P = L.Profile.load(os.path.join(tmp, "p.txt"))
    return bench, L, spec, d, prof, P


def _plan_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bench, L, spec, d, prof, P = _plan_inputs()
        from paper_2404_07947_b200._lib import exg_schedule
        box = [None]
        if rank == 0:   # the bench's rank-0 planning step, broadcast to every rank
            box[0] = bench.multi_plans(L, P, L.model_spec(spec, 1), L.cluster_spec(4, 180e9, 8e9), L.Pmf(d.pmf_in),
                                       L.Pmf(d.pmf_out), d.target_len, 0.03, 1)
        dist.broadcast_object_list(box, src=0)
        plan = box[0]
        s = exg_schedule.from_buffer_copy(plan["pick"]["sched"])
        w = exg_schedule.from_buffer_copy(plan["waa_tp2"]["sched"])
        q.put((rank, s.as_dict(), w.as_dict(), plan["latency_bound_s"]))
    finally:
        dist.destroy_process_group()


def test_config4_plan_broadcast_gloo_world2():
    """bench.py's N > 1 host path (config 4): rank 0 plans -- overall pick
    over RRA | WAA x TP and the forced WAA TP-2 plan -- and every rank
    reconstructs the same schedules from the broadcast bytes."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda x: x[0])
    assert out[0][1:] == out[1][1:]
    pick, waa = out[0][1], out[0][2]
    assert waa["strategy"] in ("WAA-C", "WAA-M") and waa["tp_degree"] == 2 and waa["tp_gpus"] >= 2
    assert sum(st[1] for st in pick["stages"]) <= 4


def test_forced_tp_plan_cpp_equals_oracle():
    """exg_search_opts.tp_degree_only (the forced partial-TP plan): C++
    planner bit-identical to oracle/bnb.py with SearchOpts(tp_degree_only)."""
    bench, L, spec, d, prof, P = _plan_inputs()
    from oracle import bnb, simulator as sim
    S = sim.Simulator(prof, sim.SimModel.from_spec(spec), sim.SimCluster(4, 180e9, 8e9), d.pmf_in, d.pmf_out,
                      d.target_len)
    for L_b in (2.0, 6.0, float("inf")):
        f = bnb.schedule_find(S, L_b, sim.WAA_C | sim.WAA_M, bnb.SearchOpts(b_e_max=32, m_max=4, tp_degree_only=2))
        args = (P, L.model_spec(spec, 1), L.cluster_spec(4, 180e9, 8e9), L.Pmf(d.pmf_in), L.Pmf(d.pmf_out),
                d.target_len, L_b, sim.WAA_C | sim.WAA_M, L.search_opts(b_e_max=32, m_max=4, tp_only=2))
        if f is None:
            with pytest.raises(L.ExgError):
                L.schedule_find(*args)
            continue
        n_found = locals().get("n_found", 0) + 1
        s, e = L.schedule_find(*args)
        assert f.schedule.tp_degree == 2 == s.tp_degree
        assert (s.b_e, s.b_d, s.b_m, s.n_enc_gpus, s.tp_gpus) == (f.schedule.b_e, f.schedule.b_d, f.schedule.b_m,
                                                                 f.schedule.n_enc_gpus, f.schedule.tp_gpus)
        assert e.thrput_seq_s == f.estimate.thrput_seq_s and e.latency_s == f.estimate.latency_s
    assert n_found >= 1
