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
