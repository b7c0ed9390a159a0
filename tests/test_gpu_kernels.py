"""Kernel-level parity of the sm_100a kernels (through the op-level C-ABI,
include/exegpt_ops.h) against plain fp64 definitions on the same bf16
inputs.  Tolerances: bf16 outputs within one bf16
rounding of the fp64 value plus fp32-accumulation slack; fp32 outputs within
1e-4 * sum|x||w|; integer/index work bit-exact."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from gpu_util import bf16_round_np, bf16_tensor, blocked, dev, ptr, stream, to_np  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2404_07947_b200 import _lib
    _lib.lib()
    return _lib


def _run(L, fn, *args):
    L.check(getattr(L.lib(), fn)(*args))


# ------------------------------------------------------------------- GEMM --
GEMM_CASES = [
    # tokens, features, K, decode   (decode uses stream-K over the weight stream)
    (1, 64, 64, True), (5, 200, 256, True), (33, 1024, 1000, True), (64, 192, 512, True),
    (130, 320, 128, True), (256, 256, 256, True), (300, 128, 192, True), (20, 5120, 5120, True),
    (513, 384, 4096, True), (7, 20480, 320, True),
    (1, 64, 64, False), (100, 300, 320, False), (257, 512, 64, False), (1000, 96, 136, False),
    (700, 2048, 1024, False),
]


def _ws(L, features, K, tokens):
    n = L.lib().exg_op_decode_workspace(features, K, tokens)
    assert n >= 0
    return torch.zeros(max(int(n), 1), dtype=torch.float32, device=dev()), int(n)


@pytest.mark.parametrize("tokens,features,K,decode", GEMM_CASES)
@pytest.mark.parametrize("mode,act", [(0, 0), (1, 1), (1, 2), (2, 0), (3, 0)])
def test_linear_parity(L, tokens, features, K, decode, mode, act):
    rng = np.random.default_rng(tokens * 7 + features + K)
    X = bf16_round_np(rng.standard_normal((tokens, K)) * 0.5)
    W = bf16_round_np(rng.standard_normal((features, K)) * 0.05)
    b = bf16_round_np(rng.standard_normal(features) * 0.1)
    acc = X @ W.T + b
    mag = np.abs(X) @ np.abs(W).T + np.abs(b)
    tX, tW, tb = bf16_tensor(X), bf16_tensor(W), bf16_tensor(b)
    tWb = blocked(L, tW)
    ws, nws = _ws(L, features, K, tokens)
    if mode in (0, 1):
        out = torch.zeros((tokens, features), dtype=torch.bfloat16, device=dev())
        _run(L, "exg_op_linear", ptr(tX), K, ptr(tWb), tokens, features, K, mode, act, ptr(tb), ptr(out),
             features, None, 0, int(decode), ptr(ws), nws, stream())
        torch.cuda.synchronize()
        ref = acc if mode == 0 else (np.maximum(acc, 0) if act == 1 else
                                     0.5 * acc * (1 + np.tanh(math.sqrt(2 / math.pi) * (acc + 0.044715 * acc ** 3))))
        got = to_np(out)
        tol = 2.0 ** -8 * np.abs(ref) + 1e-4 * mag + 1e-6
        assert np.all(np.abs(got - ref) <= tol), np.max(np.abs(got - ref) - tol)
    elif mode == 2:
        r0 = rng.standard_normal((tokens, features)).astype(np.float32)
        resid = torch.from_numpy(r0).to(dev())
        _run(L, "exg_op_linear", ptr(tX), K, ptr(tWb), tokens, features, K, 2, 0, ptr(tb), None, 0,
             ptr(resid), features, int(decode), ptr(ws), nws, stream())
        torch.cuda.synchronize()
        ref = r0.astype(np.float64) + acc
        assert np.all(np.abs(resid.cpu().numpy() - ref) <= 1e-4 * mag + 1e-5 * np.abs(ref) + 1e-6)
    else:
        out = torch.zeros((tokens, features), dtype=torch.float32, device=dev())
        _run(L, "exg_op_linear", ptr(tX), K, ptr(tWb), tokens, features, K, 3, 0, ptr(tb), ptr(out), features,
             None, 0, int(decode), ptr(ws), nws, stream())
        torch.cuda.synchronize()
        assert np.all(np.abs(out.cpu().numpy() - acc) <= 1e-4 * mag + 1e-6)


def test_linear_strided_operands(L):
    """ldx/ldw larger than K (TP-slice style views) and ldo > features."""
    rng = np.random.default_rng(3)
    tokens, features, K, ld = 40, 128, 192, 320
    Xf = bf16_round_np(rng.standard_normal((tokens, ld)))
    Wf = bf16_round_np(rng.standard_normal((features, ld)) * 0.05)
    tX, tW = bf16_tensor(Xf), bf16_tensor(Wf)
    tWb = blocked(L, tW[:, :K])
    ws, nws = _ws(L, features, K, tokens)
    for decode in (0, 1):
        out = torch.zeros((tokens, 256), dtype=torch.float32, device=dev())
        _run(L, "exg_op_linear", ptr(tX), ld, ptr(tWb), tokens, features, K, 3, 0, None, ptr(out), 256, None, 0,
             decode, ptr(ws), nws, stream())
        torch.cuda.synchronize()
        ref = Xf[:, :K] @ Wf[:, :K].T
        assert np.abs(out.cpu().numpy()[:, :features] - ref).max() < 1e-3
        assert np.all(out.cpu().numpy()[:, features:] == 0)


@pytest.mark.parametrize("tokens,features,K", [(300, 300, 320), (777, 1024, 5120), (256, 512, 64), (1, 260, 128),
                                               (513, 2560, 960)])
def test_prefill_pair_kernel_matches_single_cta(L, tokens, features, K):
    """The CTA-pair prefill GEMM (cta_group::2, M=256 tiles) computes every
    output element with the same K order and MMA K steps as the 1-CTA kernel
    (diagnostics flag bit 6): outputs are bit-identical, ragged token and
    feature tails included, in every epilogue mode."""
    rng = np.random.default_rng(tokens + features + K)
    tX = bf16_tensor(bf16_round_np(rng.standard_normal((tokens, K)) * 0.5))
    tWb = blocked(L, bf16_tensor(bf16_round_np(rng.standard_normal((features, K)) * 0.05)))
    tb = bf16_tensor(bf16_round_np(rng.standard_normal(features) * 0.1))
    r0 = torch.from_numpy(rng.standard_normal((tokens, features)).astype(np.float32)).to(dev())
    try:
        for mode, act in ((0, 0), (1, 1), (1, 2), (2, 0), (3, 0)):
            outs = []
            for flag in (0, 64):
                L.lib().exg_diag_gemm_flags(flag)
                if mode in (0, 1):
                    out = torch.zeros((tokens, features), dtype=torch.bfloat16, device=dev())
                    _run(L, "exg_op_linear", ptr(tX), K, ptr(tWb), tokens, features, K, mode, act, ptr(tb), ptr(out),
                         features, None, 0, 0, None, 0, stream())
                elif mode == 2:
                    out = r0.clone()
                    _run(L, "exg_op_linear", ptr(tX), K, ptr(tWb), tokens, features, K, 2, 0, ptr(tb), None, 0,
                         ptr(out), features, 0, None, 0, stream())
                else:
                    out = torch.zeros((tokens, features), dtype=torch.float32, device=dev())
                    _run(L, "exg_op_linear", ptr(tX), K, ptr(tWb), tokens, features, K, 3, 0, ptr(tb), ptr(out),
                         features, None, 0, 0, None, 0, stream())
                torch.cuda.synchronize()
                outs.append(out)
            assert torch.equal(outs[0], outs[1]), (mode, act)
    finally:
        L.lib().exg_diag_gemm_flags(0)


def test_decode_gemm_batch_invariant(L):
    """T13: a token row's decode-GEMM bits do not depend on its batch-mates
    or its row position (tokens ride the MMA N axis)."""
    rng = np.random.default_rng(9)
    K, features = 2048, 1280       # stream-K with tiles cut between CTAs
    W = blocked(L, bf16_tensor(bf16_round_np(rng.standard_normal((features, K)) * 0.05)))
    X = bf16_round_np(rng.standard_normal((200, K)))
    ws, nws = _ws(L, features, K, 200)

    def run(rows):
        x = bf16_tensor(X[rows])
        out = torch.zeros((len(rows), features), dtype=torch.float32, device=dev())
        _run(L, "exg_op_linear", ptr(x), K, ptr(W), len(rows), features, K, 3, 0, None, ptr(out), features, None,
             0, 1, ptr(ws), nws, stream())
        torch.cuda.synchronize()
        return out.cpu().numpy()

    full = run(list(range(200)))
    for rows in ([17], [3, 17, 150], list(range(100, 160)), list(range(199, -1, -1))):
        part = run(rows)
        assert np.array_equal(part, full[rows])


# --------------------------------------------------------- decode attention --
@pytest.mark.parametrize("dh", [16, 64, 128])
def test_decode_attention_parity(L, dh):
    rng = np.random.default_rng(dh)
    H, max_ctx, slots = 3, 1100, 16
    n_keys = np.array([1, 2, 31, 32, 33, 127, 128, 129, 511, 512, 513, 1000, 1100, 7], dtype=np.int32)
    B = len(n_keys)
    slot = rng.permutation(slots)[:B].astype(np.int32)
    K = bf16_round_np(rng.standard_normal((slots, H, max_ctx, dh)))
    V = bf16_round_np(rng.standard_normal((slots, H, max_ctx, dh)))
    q = bf16_round_np(rng.standard_normal((B, 3 * H * dh)))     # q block at columns [0, H*dh)
    scale = float(np.float32(1 / math.sqrt(dh)))
    tK, tV, tq = bf16_tensor(K), bf16_tensor(V), bf16_tensor(q)
    tslot = torch.from_numpy(slot).to(dev())
    tnk = torch.from_numpy(n_keys).to(dev())
    split_len = 512
    max_splits = int(math.ceil(n_keys.max() / split_len))
    part = torch.zeros(B * H * max_splits * (dh + 2), dtype=torch.float32, device=dev())
    out = torch.zeros((B, H * dh), dtype=torch.bfloat16, device=dev())
    _run(L, "exg_op_decode_attention", ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tslot), ptr(tnk), ptr(out),
         H * dh, B, H, dh, max_ctx, scale, split_len, max_splits, ptr(part), None, 0, 0, stream())
    torch.cuda.synchronize()
    got = to_np(out)
    for i in range(B):
        for h in range(H):
            qv = q[i, h * dh:(h + 1) * dh]
            k = K[slot[i], h, :n_keys[i]]
            v = V[slot[i], h, :n_keys[i]]
            s = (k @ qv) * scale
            p = np.exp(s - s.max())
            p /= p.sum()
            ref = p @ v
            g = got[i, h * dh:(h + 1) * dh]
            assert np.all(np.abs(g - ref) <= 2.0 ** -8 * np.abs(ref) + 2e-3), (i, h, np.abs(g - ref).max())


def test_decode_attention_constant_keys_give_mean(L):
    """All keys equal => softmax uniform => output = mean of V rows."""
    dh, H, max_ctx = 128, 2, 600
    rng = np.random.default_rng(5)
    K = np.zeros((1, H, max_ctx, dh)); K[...] = bf16_round_np(rng.standard_normal(dh))
    V = bf16_round_np(rng.standard_normal((1, H, max_ctx, dh)))
    q = bf16_round_np(rng.standard_normal((1, 3 * H * dh)))
    tK, tV, tq = bf16_tensor(K), bf16_tensor(V), bf16_tensor(q)
    nk = 555
    tslot = torch.zeros(1, dtype=torch.int32, device=dev())
    tnk = torch.full((1,), nk, dtype=torch.int32, device=dev())
    part = torch.zeros(H * 2 * (dh + 2), dtype=torch.float32, device=dev())
    out = torch.zeros((1, H * dh), dtype=torch.bfloat16, device=dev())
    _run(L, "exg_op_decode_attention", ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tslot), ptr(tnk), ptr(out),
         H * dh, 1, H, dh, max_ctx, 0.088388, 512, 2, ptr(part), None, 0, 0, stream())
    torch.cuda.synchronize()
    ref = V[0, :, :nk].mean(axis=1).reshape(-1)
    assert np.abs(to_np(out)[0] - ref).max() < 2e-3


def test_decode_attention_batch_invariant(L):
    dh, H, max_ctx, slots = 128, 4, 700, 8
    rng = np.random.default_rng(6)
    tK = bf16_tensor(bf16_round_np(rng.standard_normal((slots, H, max_ctx, dh))))
    tV = bf16_tensor(bf16_round_np(rng.standard_normal((slots, H, max_ctx, dh))))
    q = bf16_round_np(rng.standard_normal((slots, H * dh)))
    nk = np.array([700, 3, 513, 64, 129, 1, 600, 300], dtype=np.int32)
    part = torch.zeros(slots * H * 2 * (dh + 2), dtype=torch.float32, device=dev())

    def run(rows):
        tq = bf16_tensor(q[rows])
        ts = torch.from_numpy(np.array(rows, dtype=np.int32)).to(dev())
        tn = torch.from_numpy(nk[rows]).to(dev())
        out = torch.zeros((len(rows), H * dh), dtype=torch.bfloat16, device=dev())
        _run(L, "exg_op_decode_attention", ptr(tq), H * dh, ptr(tK), ptr(tV), ptr(ts), ptr(tn), ptr(out), H * dh,
             len(rows), H, dh, max_ctx, 0.088388, 512, 2, ptr(part), None, 0, 0, stream())
        torch.cuda.synchronize()
        return out.cpu()

    full = run(list(range(slots)))
    for rows in ([0], [6, 2], [7, 5, 3, 1]):
        assert torch.equal(run(rows), full[rows])


# -------------------------------------------------------- prefill attention --
@pytest.mark.parametrize("dh", [16, 128])
def test_prefill_attention_parity(L, dh):
    """dh = 16: SIMT kernel (fp32 P); dh = 128: tcgen05 FMHA (P rounded to
    bf16 for P.V, so its tolerance is one bf16 step wider).  Lengths span
    several 128-key tiles, a ragged tail and the one-token case."""
    rng = np.random.default_rng(dh + 1)
    H, max_ctx = 2, 400
    lens = [1, 5, 32, 33, 100, 150, 128, 129, 257, 383]
    R = len(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    slot = np.array([4, 0, 2, 5, 1, 3, 9, 7, 6, 8], dtype=np.int32)
    n_slots = 10
    pos0 = np.zeros(R, dtype=np.int32)
    qkv = bf16_round_np(rng.standard_normal((T, 3 * H * dh)))
    K = np.zeros((n_slots, H, max_ctx, dh)); V = np.zeros((n_slots, H, max_ctx, dh))
    for r in range(R):
        for j in range(lens[r]):
            t = cu[r] + j
            K[slot[r], :, j] = qkv[t, H * dh:2 * H * dh].reshape(H, dh)
            V[slot[r], :, j] = qkv[t, 2 * H * dh:].reshape(H, dh)
    tK, tV = bf16_tensor(K), bf16_tensor(V)
    tq = bf16_tensor(qkv)
    tcu, tsl, tp0 = (torch.from_numpy(a).to(dev()) for a in (cu, slot, pos0))
    out = torch.zeros((T, H * dh), dtype=torch.bfloat16, device=dev())
    scale = float(np.float32(1 / math.sqrt(dh)))
    _run(L, "exg_op_prefill_attention", ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tcu), ptr(tsl), ptr(tp0), R,
         max(lens), ptr(out), H * dh, H, dh, max_ctx, n_slots, T, scale, 1, None, 0, 0, stream())
    torch.cuda.synchronize()
    got = to_np(out)
    rel, ab = (2.0 ** -8, 2e-3) if dh != 128 else (2.0 ** -7, 4e-3)
    for r in range(R):
        for h in range(H):
            k = K[slot[r], h, :lens[r]]
            v = V[slot[r], h, :lens[r]]
            qv = qkv[cu[r]:cu[r + 1], h * dh:(h + 1) * dh]
            s = (qv @ k.T) * scale
            s = np.where(np.tril(np.ones_like(s)) > 0, s, -np.inf)
            p = np.exp(s - s.max(axis=1, keepdims=True))
            p /= p.sum(axis=1, keepdims=True)
            ref = p @ v
            g = got[cu[r]:cu[r + 1], h * dh:(h + 1) * dh]
            assert np.all(np.abs(g - ref) <= rel * np.abs(ref) + ab), (r, h, np.abs(g - ref).max())


# ------------------------------------------------------------ small kernels --
def test_kv_scatter_exact(L):
    rng = np.random.default_rng(1)
    H, dh, max_ctx, T = 4, 16, 32, 10
    qkv = bf16_round_np(rng.standard_normal((T, 3 * H * dh)))
    slot = rng.integers(0, 3, T).astype(np.int32)
    pos = rng.permutation(max_ctx)[:T].astype(np.int32)
    kc = torch.zeros((3, H, max_ctx, dh), dtype=torch.bfloat16, device=dev())
    vc = torch.zeros_like(kc)
    tq = bf16_tensor(qkv)
    ts, tp = torch.from_numpy(slot).to(dev()), torch.from_numpy(pos).to(dev())   # keep alive
    _run(L, "exg_op_kv_scatter", ptr(kc), ptr(vc), ptr(tq), ptr(ts), ptr(tp), T, H, dh, max_ctx, stream())
    torch.cuda.synchronize()
    K, V = to_np(kc), to_np(vc)
    for t in range(T):
        assert np.array_equal(K[slot[t], :, pos[t]].reshape(-1), qkv[t, H * dh:2 * H * dh])
        assert np.array_equal(V[slot[t], :, pos[t]].reshape(-1), qkv[t, 2 * H * dh:])


def test_layernorm_parity(L):
    rng = np.random.default_rng(2)
    for T, d in [(1, 64), (7, 5120), (33, 12288)]:
        x = (rng.standard_normal((T, d)) * 2 + 0.3).astype(np.float32)
        g = bf16_round_np(1 + 0.1 * rng.standard_normal(d))
        b = bf16_round_np(0.02 * rng.standard_normal(d))
        y = torch.zeros((T, d), dtype=torch.bfloat16, device=dev())
        tx, tg, tb = torch.from_numpy(x).to(dev()), bf16_tensor(g), bf16_tensor(b)
        _run(L, "exg_op_layernorm", ptr(y), d, ptr(tx), d, ptr(tg), ptr(tb), T, d, 1e-5, stream())
        torch.cuda.synchronize()
        xd = x.astype(np.float64)
        mu = xd.mean(1, keepdims=True)
        ref = (xd - mu) / np.sqrt(((xd - mu) ** 2).mean(1, keepdims=True) + 1e-5) * g + b
        assert np.all(np.abs(to_np(y) - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-5)


def test_embed_exact(L):
    rng = np.random.default_rng(4)
    V, P, d, T = 50, 20, 64, 9
    te = bf16_round_np(rng.standard_normal((V, d)) * 0.02)
    pe = bf16_round_np(rng.standard_normal((P, d)) * 0.02)
    ids = rng.integers(0, V, T).astype(np.int32)
    pos = rng.integers(0, P, T).astype(np.int32)
    x = torch.zeros((T, d), dtype=torch.float32, device=dev())
    keep = [torch.from_numpy(ids).to(dev()), torch.from_numpy(pos).to(dev()), bf16_tensor(te), bf16_tensor(pe)]
    _run(L, "exg_op_embed", ptr(x), *[ptr(k) for k in keep], T, d, stream())
    torch.cuda.synchronize()
    ref = (te[ids].astype(np.float32) + pe[pos].astype(np.float32))
    assert np.array_equal(x.cpu().numpy(), ref)


def test_argmax_lowest_index_on_ties_and_nan_flag(L):
    rng = np.random.default_rng(8)
    B, V = 6, 50272
    lg = rng.standard_normal((B, V)).astype(np.float32)
    lg[1, [7, 300, 50000]] = 9.0          # tie -> 7
    lg[2, :] = 1.0                         # all equal -> 0
    lg[3, V - 1] = 100.0
    t = torch.from_numpy(lg).to(dev())
    out = torch.zeros(B, dtype=torch.int32, device=dev())
    err = torch.zeros(1, dtype=torch.int32, device=dev())
    _run(L, "exg_op_argmax", ptr(out), ptr(t), V, B, V, ptr(err), stream())
    torch.cuda.synchronize()
    assert out.cpu().tolist() == [int(np.argmax(r)) for r in lg]
    assert out.cpu().tolist()[1:4] == [7, 0, V - 1] and err.item() == 0
    lg[4, 11] = np.nan
    t = torch.from_numpy(lg).to(dev())
    _run(L, "exg_op_argmax", ptr(out), ptr(t), V, B, V, ptr(err), stream())
    torch.cuda.synchronize()
    assert err.item() == 1


@pytest.mark.parametrize("kind,transposed,rows,cols,canon", [("W_qkv", 1, 192, 64, 192), ("tok_emb", 0, 512, 64, 64),
                                                             ("ln1_g", 0, 1, 5120, 5120), ("W_2", 1, 64, 256, 64)])
def test_weightgen_bit_identical_to_oracle(L, kind, transposed, rows, cols, canon):
    from oracle import weights as wg
    seed = 0xE6E00001
    tid = wg.tensor_id(1001 if kind not in ("tok_emb",) else 0, kind)
    out = torch.zeros((rows, cols), dtype=torch.bfloat16, device=dev())
    _run(L, "exg_op_weightgen", ptr(out), rows, cols, cols, seed, tid, int(kind in wg.GAIN_KINDS), transposed, canon,
         0, 0, 0, stream())
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    vals = wg.gen_values(seed, tid, rows * cols, kind)
    ref = vals.reshape(cols, rows).T if transposed else vals.reshape(rows, cols)
    assert np.array_equal(got.view(np.uint32), np.ascontiguousarray(ref).view(np.uint32))
    # blocked layout: generating in place == packing the row-major tensor
    blk = torch.zeros(int(L.lib().exg_op_blocked_elems(rows, cols)), dtype=torch.bfloat16, device=dev())
    _run(L, "exg_op_weightgen", ptr(blk), rows, cols, cols, seed, tid, int(kind in wg.GAIN_KINDS), transposed, canon,
         0, 0, 1, stream())
    packed = blocked(L, out)
    torch.cuda.synchronize()
    assert torch.equal(blk, packed)


# ------------------------------------------------------ paged KV (NEXT-2) --
def _to_pages(C, lens, P, rng):
    """Slot cache C [slots][H][ctx][dh] -> page pool [n_pages][H][P][dh] and
    a page table [rows][maxp] (pages shuffled, unused entries -> page 0)."""
    slots, H, ctx, dh = C.shape
    maxp = (ctx + P - 1) // P
    n_pages = slots * maxp + 3
    perm = rng.permutation(n_pages)
    pool = np.zeros((n_pages, H, P, dh))
    tab = np.zeros((slots, maxp), dtype=np.int32)
    k = 0
    for s in range(slots):
        for j in range((lens[s] + P - 1) // P):
            pg = perm[k]; k += 1
            tab[s, j] = pg
            w = min(P, ctx - j * P)
            pool[pg, :, :w] = C[s, :, j * P:j * P + w]
    return pool, tab, n_pages, maxp


@pytest.mark.parametrize("dh,P", [(16, 64), (64, 128), (128, 64), (128, 512)])
def test_decode_attention_paged_matches_slots(L, dh, P):
    """The paged kernel on a shuffled page pool gives bitwise the slot
    kernel's output (same keys, same arithmetic), new-key append included."""
    rng = np.random.default_rng(100 + dh + P)
    H, max_ctx = 3, 1100
    n_keys = np.array([1, 2, 63, 64, 65, 127, 128, 129, 511, 512, 513, 1000, 1100, 7], dtype=np.int32)
    B = len(n_keys)
    K = bf16_round_np(rng.standard_normal((B, H, max_ctx, dh)))
    V = bf16_round_np(rng.standard_normal((B, H, max_ctx, dh)))
    q = bf16_round_np(rng.standard_normal((B, 3 * H * dh)))
    scale = float(np.float32(1 / math.sqrt(dh)))
    slot = np.arange(B, dtype=np.int32)
    split_len, max_splits = 512, 3
    tq, tslot, tnk = bf16_tensor(q), torch.from_numpy(slot).to(dev()), torch.from_numpy(n_keys).to(dev())
    part = torch.zeros(B * H * max_splits * (dh + 2), dtype=torch.float32, device=dev())
    out_s = torch.zeros((B, H * dh), dtype=torch.bfloat16, device=dev())
    tK, tV = bf16_tensor(K), bf16_tensor(V)   # kept alive until the launches complete
    _run(L, "exg_op_decode_attention", ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tslot),
         ptr(tnk), ptr(out_s), H * dh, B, H, dh, max_ctx, scale, split_len, max_splits, ptr(part), None, 0, 0,
         stream())
    Kp, tab, n_pages, maxp = _to_pages(K, n_keys, P, rng)
    Vp = np.zeros_like(Kp)   # V in the pages of the K table
    for s in range(B):
        for j in range((n_keys[s] + P - 1) // P):
            w = min(P, max_ctx - j * P)
            Vp[tab[s, j], :, :w] = V[s, :, j * P:j * P + w]
    ttab = torch.from_numpy(tab).to(dev())
    out_p = torch.zeros_like(out_s)
    tKp, tVp = bf16_tensor(Kp), bf16_tensor(Vp)
    _run(L, "exg_op_decode_attention_paged", ptr(tq), 3 * H * dh, ptr(tKp), ptr(tVp),
         ptr(tslot), ptr(tnk), ptr(out_p), H * dh, B, H, dh, P, scale, split_len, max_splits, ptr(part), None, 0, 0,
         ptr(ttab), maxp, stream())
    torch.cuda.synchronize()
    assert torch.equal(out_s.cpu(), out_p.cpu())
    # and against the fp64 definition on a few rows
    got = to_np(out_p)
    for i in (0, 4, 11, 12):
        for h in range(H):
            s_ = (K[i, h, :n_keys[i]] @ q[i, h * dh:(h + 1) * dh]) * scale
            p_ = np.exp(s_ - s_.max()); p_ /= p_.sum()
            ref = p_ @ V[i, h, :n_keys[i]]
            assert np.all(np.abs(got[i, h * dh:(h + 1) * dh] - ref) <= 2.0 ** -8 * np.abs(ref) + 2e-3)


@pytest.mark.parametrize("dh,P", [(16, 64), (128, 64), (128, 128)])
def test_prefill_attention_paged_matches_slots(L, dh, P):
    """Paged prefill attention (SIMT dh=16, tcgen05 FMHA dh=128, 128-key
    tiles split across 64-key pages) is bitwise the slot kernel."""
    rng = np.random.default_rng(200 + dh + P)
    H, max_ctx = 2, 448
    lens = [1, 5, 63, 64, 65, 100, 128, 129, 257, 383, 448]
    R = len(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    slot = np.arange(R, dtype=np.int32)
    pos0 = np.zeros(R, dtype=np.int32)
    qkv = bf16_round_np(rng.standard_normal((T, 3 * H * dh)))
    K = np.zeros((R, H, max_ctx, dh)); V = np.zeros((R, H, max_ctx, dh))
    for r in range(R):
        for j in range(lens[r]):
            t = cu[r] + j
            K[r, :, j] = qkv[t, H * dh:2 * H * dh].reshape(H, dh)
            V[r, :, j] = qkv[t, 2 * H * dh:].reshape(H, dh)
    tq = bf16_tensor(qkv)
    tcu, tsl, tp0 = (torch.from_numpy(a).to(dev()) for a in (cu, slot, pos0))
    scale = float(np.float32(1 / math.sqrt(dh)))
    out_s = torch.zeros((T, H * dh), dtype=torch.bfloat16, device=dev())
    tK, tV = bf16_tensor(K), bf16_tensor(V)   # kept alive until the launches complete
    _run(L, "exg_op_prefill_attention", ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tcu),
         ptr(tsl), ptr(tp0), R, max(lens), ptr(out_s), H * dh, H, dh, max_ctx, R, T, scale, 1, None, 0, 0, stream())
    Kp, tab, n_pages, maxp = _to_pages(K, lens, P, rng)
    Vp = np.zeros_like(Kp)
    for s in range(R):
        for j in range((lens[s] + P - 1) // P):
            w = min(P, max_ctx - j * P)
            Vp[tab[s, j], :, :w] = V[s, :, j * P:j * P + w]
    ttab = torch.from_numpy(tab).to(dev())
    out_p = torch.zeros_like(out_s)
    tKp, tVp = bf16_tensor(Kp), bf16_tensor(Vp)
    _run(L, "exg_op_prefill_attention_paged", ptr(tq), 3 * H * dh, ptr(tKp), ptr(tVp),
         ptr(tcu), ptr(tsl), ptr(tp0), R, max(lens), ptr(out_p), H * dh, H, dh, P, n_pages, T, scale, 1, None, 0, 0,
         ptr(ttab), maxp, stream())
    torch.cuda.synchronize()
    assert torch.equal(out_s.cpu(), out_p.cpu())
    # and against the fp64 definition on a few requests (causal)
    got = to_np(out_p)
    rel, ab = (2.0 ** -8, 2e-3) if dh != 128 else (2.0 ** -7, 4e-3)
    for r in (0, 4, 9, 10):
        for h in range(H):
            qv = qkv[cu[r]:cu[r + 1], h * dh:(h + 1) * dh]
            s_ = (qv @ K[r, h, :lens[r]].T) * scale
            s_ = np.where(np.tril(np.ones_like(s_)) > 0, s_, -np.inf)
            p_ = np.exp(s_ - s_.max(axis=1, keepdims=True))
            p_ /= p_.sum(axis=1, keepdims=True)
            ref = p_ @ V[r, h, :lens[r]]
            g = got[cu[r]:cu[r + 1], h * dh:(h + 1) * dh]
            assert np.all(np.abs(g - ref) <= rel * np.abs(ref) + ab), (r, h, np.abs(g - ref).max())


@pytest.mark.parametrize("causal", [1, 0])
def test_prefill_attention_tc_repeatable(L, causal):
    """Race check of the tcgen05 FMHA (P kept in TMEM over its S buffer):
    items of up to 4 key tiles, run 12 times -- every output finite and
    bitwise equal across runs."""
    rng = np.random.default_rng(31 + causal)
    H, dh, max_ctx = 4, 128, 512
    lens = [512, 300, 257, 129, 511, 384, 200, 65]
    R = len(lens)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    qkv = bf16_round_np(rng.standard_normal((T, 3 * H * dh)) * 2.0)
    K = bf16_round_np(rng.standard_normal((R, H, max_ctx, dh)) * 2.0)
    V = bf16_round_np(rng.standard_normal((R, H, max_ctx, dh)))
    tq, tK, tV = bf16_tensor(qkv), bf16_tensor(K), bf16_tensor(V)
    tcu = torch.from_numpy(cu).to(dev())
    tsl = torch.arange(R, dtype=torch.int32, device=dev())
    tp0 = torch.zeros(R, dtype=torch.int32, device=dev())
    first = None
    for _ in range(12):
        out = torch.zeros((T, H * dh), dtype=torch.bfloat16, device=dev())
        _run(L, "exg_op_prefill_attention", ptr(tq), 3 * H * dh, ptr(tK), ptr(tV), ptr(tcu), ptr(tsl), ptr(tp0), R,
             max(lens), ptr(out), H * dh, H, dh, max_ctx, R, T, float(np.float32(1 / np.sqrt(dh))), causal, None, 0,
             0, stream())
        torch.cuda.synchronize()
        o = out.float().cpu()
        assert torch.isfinite(o).all()
        if first is None:
            first = o
        else:
            assert torch.equal(o, first)
