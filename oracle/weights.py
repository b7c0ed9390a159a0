"""Seeded random-init weights, SURVEY.md §8(c) T3 (the north star asks for
"seeded random-init weights"; PAPER.md is silent on the distribution).

    w = bf16_rne( fp32( fp32(u - 1/2) * c ) ),  c = fp32(2*sqrt(3)*sigma)
    u = (splitmix64(seed ^ tensor_id<<40 ^ i) >> 40) * 2^-24

* sigma = 0.02 for embeddings, matrices, biases, relative-bias table;
* norm gains: 1 + U(+-0.1) computed as fp32(1 + fp32((u-1/2)*fp32(0.2)));
* norm biases: sigma = 0.02 like matrices;
* i is the row-major index in the canonical unsharded layout W[in][out]
  (y = x @ W); vectors are indexed 0..n-1.

Pins (tests/test_oracle_weights.py): splitmix64(0) = 0xE220A8397B1DCDAF (the
first output of Vigna's reference splitmix64 seeded with 0); bf16 rounding vs
torch's float32->bfloat16 conversion (library RNE); uniform moments.
"""
from __future__ import annotations

import math
from typing import Dict

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

KINDS = ["tok_emb", "pos_emb", "ln1_g", "ln1_b", "W_qkv", "b_qkv", "W_o", "b_o",
         "ln2_g", "ln2_b", "W_1", "b_1", "W_2", "b_2", "lnf_g", "lnf_b",
         "rel_bias", "W_q_x", "W_kv_x", "W_o_x", "lnx_g"]
KIND = {k: i for i, k in enumerate(KINDS)}
GAIN_KINDS = {"ln1_g", "ln2_g", "lnf_g", "lnx_g"}

SIGMA = 0.02
C_MAT = np.float32(2.0 * math.sqrt(3.0) * SIGMA)   # fp32(2*sqrt(3)*sigma)
C_GAIN = np.float32(0.2)                           # U(+-0.1)


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def bf16_round(x32: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 round-to-nearest-even, returned as float32 values."""
    x32 = np.ascontiguousarray(x32, dtype=np.float32)
    b = x32.view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
    return (r & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)


def tensor_id(layer_slot: int, kind: str) -> int:
    return layer_slot * 64 + KIND[kind]


def enc_slot(l: int) -> int:
    return 1 + l


def dec_slot(l: int) -> int:
    return 1001 + l


_CHUNK = 1 << 22


def gen_values(seed: int, tid: int, n: int, kind: str, start: int = 0) -> np.ndarray:
    """n consecutive values (indices start..start+n-1) of tensor `tid`, as
    float32 arrays holding bf16-exact values.  Large tensors are generated in
    index chunks on a thread pool (every value depends on its own index only,
    so the result is the same array)."""
    if n > 2 * _CHUNK:
        import concurrent.futures as cf
        import os
        out = np.empty(n, np.float32)

        def job(s):
            e = min(n, s + _CHUNK)
            out[s:e] = _gen_values(seed, tid, e - s, kind, start + s)

        with cf.ThreadPoolExecutor(max(1, min(32, os.cpu_count() or 1))) as ex:
            list(ex.map(job, range(0, n, _CHUNK)))
        return out
    return _gen_values(seed, tid, n, kind, start)


def _gen_values(seed: int, tid: int, n: int, kind: str, start: int) -> np.ndarray:
    i = np.arange(start, start + n, dtype=np.uint64)
    key = np.uint64(seed) ^ (np.uint64(tid) << np.uint64(40))
    h = splitmix64(key ^ i)
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    c = u - np.float32(0.5)                      # exact in fp32
    if kind in GAIN_KINDS:
        v = np.float32(1.0) + c * C_GAIN         # two fp32 roundings, no FMA
    else:
        v = c * C_MAT
    return bf16_round(v.astype(np.float32))


def gen_tensor(seed: int, layer_slot: int, kind: str, shape) -> np.ndarray:
    n = int(np.prod(shape))
    return gen_values(seed, tensor_id(layer_slot, kind), n, kind).reshape(shape)


def decoder_only_weights(spec, seed: int, dtype=np.float64) -> Dict:
    """All parameters of a decoder-only (OPT / GPT-3 style) model in the
    canonical layout: W[in][out].  Values are bf16-exact."""
    d, inner, ff, V, P = spec.d_model, spec.inner, spec.d_ff, spec.vocab, spec.max_pos
    W = {"tok_emb": gen_tensor(seed, 0, "tok_emb", (V, d)).astype(dtype),
         "pos_emb": gen_tensor(seed, 0, "pos_emb", (P, d)).astype(dtype),
         "lnf_g": gen_tensor(seed, 0, "lnf_g", (d,)).astype(dtype),
         "lnf_b": gen_tensor(seed, 0, "lnf_b", (d,)).astype(dtype),
         "layers": []}
    for l in range(spec.n_dec_layers):
        s = dec_slot(l)
        W["layers"].append(decoder_layer_weights(spec, seed, s, dtype))
    return W


def decoder_layer_weights(spec, seed: int, slot: int, dtype=np.float64) -> Dict:
    d, inner, ff = spec.d_model, spec.inner, spec.d_ff
    shapes = {"ln1_g": (d,), "ln1_b": (d,), "W_qkv": (d, 3 * inner), "b_qkv": (3 * inner,),
              "W_o": (inner, d), "b_o": (d,), "ln2_g": (d,), "ln2_b": (d,),
              "W_1": (d, ff), "b_1": (ff,), "W_2": (ff, d), "b_2": (d,)}
    return {k: gen_tensor(seed, slot, k, shp).astype(dtype) for k, shp in shapes.items()}
