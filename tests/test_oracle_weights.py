"""Pins for oracle/weights.py."""
import numpy as np
import torch

from oracle import weights as wg


def test_splitmix64_reference_vector():
    assert int(wg.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF


def test_bf16_round_matches_torch_rne():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100000).astype(np.float32) * 0.05,
                        # halfway cases: low 16 bits == 0x8000 with both parities
                        (np.arange(2000, dtype=np.uint32) << 16 | 0x8000).view(np.float32),
                        np.array([0.0, -0.0, 1.0, 65504.0, 1e-30], np.float32)])
    x = x[np.isfinite(x)]
    ours = wg.bf16_round(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(ours.view(np.uint32), ref.view(np.uint32))


def test_uniform_moments_and_range():
    v = wg.gen_values(123, wg.tensor_id(1001, "W_qkv"), 200000, "W_qkv").astype(np.float64)
    half = np.sqrt(3) * 0.02
    assert np.abs(v).max() <= half * 1.01
    assert abs(v.mean()) < 2e-4
    assert abs(v.std() - 0.02) < 2e-4
    g = wg.gen_values(123, wg.tensor_id(1001, "ln1_g"), 100000, "ln1_g").astype(np.float64)
    assert g.min() >= 0.9 - 4e-3 and g.max() <= 1.1 + 8e-3 and abs(g.mean() - 1) < 1e-3


def test_values_are_bf16_exact_and_index_addressable():
    tid = wg.tensor_id(1002, "W_1")
    full = wg.gen_values(7, tid, 5000, "W_1")
    part = wg.gen_values(7, tid, 1000, "W_1", start=3000)
    assert np.array_equal(full[3000:4000], part)
    assert np.array_equal(wg.bf16_round(full), full)


def test_distinct_tensors_decorrelated():
    a = wg.gen_values(7, wg.tensor_id(1001, "W_o"), 50000, "W_o").astype(np.float64)
    b = wg.gen_values(7, wg.tensor_id(1002, "W_o"), 50000, "W_o").astype(np.float64)
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.02


def test_chunked_generation_is_the_same_array(monkeypatch):
    """gen_values splits large tensors into index chunks on a thread pool;
    every value depends on its own index only, so the array is unchanged."""
    import numpy as np
    from oracle import weights as wgen
    ref = wgen._gen_values(7, 12345, 100_003, "W_1", 17)
    monkeypatch.setattr(wgen, "_CHUNK", 1000)
    assert np.array_equal(wgen.gen_values(7, 12345, 100_003, "W_1", 17), ref)
    ref_g = wgen._gen_values(7, 99, 50_001, "ln1_g", 0)
    assert np.array_equal(wgen.gen_values(7, 99, 50_001, "ln1_g"), ref_g)
