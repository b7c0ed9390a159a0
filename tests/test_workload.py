"""Workload generator pins: Table 3."""
import math

import numpy as np
import pytest

from workload import (TASKS, MODELS, config1_requests, make_requests, pmf_mean, pmf_std,
                      task_dists, truncnorm_pmf, truncnorm_quantile, uniform_pmf, splitmix64_np)


@pytest.mark.parametrize("task", list(TASKS))
def test_reading_b_reproduces_table3_p99(task):
    """Reading B: the fitted truncated PMF has the table's
    mean/std and its continuous 0.99-quantile rounds up to the printed 99th
    column for all five tasks."""
    t = TASKS[task]
    d = task_dists(task)
    assert abs(pmf_mean(d.pmf_out) - t.out_avg) < 1e-6
    assert abs(pmf_std(d.pmf_out) - t.out_std) < 1e-6
    q = truncnorm_quantile(d.mu0, d.sigma0, t.out_max, 0.99)
    assert math.ceil(q) == t.out_p99


@pytest.mark.parametrize("task,mean", [("S", 256), ("T", 128), ("G", 64), ("C1", 256), ("C2", 512)])
def test_reading_a_input_means(task, mean):
    d = task_dists(task)
    assert abs(pmf_mean(d.pmf_in) - mean) < 0.4
    assert abs(d.pmf_in.sum() - 1) < 1e-12


def test_truncnorm_spec_examples():
    # SPEC.md:48 mean within 1 token of 32.1; SPEC.md:49 point mass; SPEC.md:50 half-normal
    assert abs(pmf_mean(truncnorm_pmf(32, 13, 80)) - 32.1) < 1
    p = truncnorm_pmf(5, 1e-6, 10)
    assert p[4] == pytest.approx(1.0)
    assert abs(pmf_mean(truncnorm_pmf(0, 10, 100)) - 8.0) < 1.0


def test_splitmix64_reference_vector():
    # first outputs of Vigna's splitmix64 with state 0 (published reference sequence)
    z = np.array([0, 0x9E3779B97F4A7C15], dtype=np.uint64)
    h = splitmix64_np(z)
    assert int(h[0]) == 0xE220A8397B1DCDAF
    assert int(h[1]) == 0x6E789E6AA1B965F4


def test_requests_deterministic_and_in_range():
    a, b = config1_requests(), config1_requests()
    assert len(a) == 8
    for x, y in zip(a, b):
        assert np.array_equal(x.ids, y.ids) and x.output_len == y.output_len
        assert 16 <= x.input_len <= 32 and 1 <= x.output_len <= 24
        assert x.ids.min() >= 0 and x.ids.max() < 512 and len(x.ids) == x.input_len


def test_request_lengths_follow_pmf():
    d = task_dists("S")
    reqs = make_requests(4000, d.pmf_in, d.pmf_out, 50272, 7)
    outs = np.array([r.output_len for r in reqs])
    assert abs(outs.mean() - 32) < 1.0
    assert abs(outs.std() - 13) < 1.0
    assert outs.max() <= 80 and outs.min() >= 1
