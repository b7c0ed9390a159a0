// tcgen05 / TMEM / TMA GEMM for the prefill GEMMs (K3), decode projections
// (K5, swap-AB) and LM head (K8).  Y[token][feature] = X[token][K] .
// W[feature][K]^T, bf16 in, fp32 accumulate in TMEM, fused epilogues.
//
// Weights live in HBM in a pre-tiled, pre-swizzled blocked layout: the
// 128-row x 64-column tile (m, kb) of W is one contiguous 16 KB block at
// element offset (m * nkb + kb) * 8192, holding row r's 16-byte chunk c at
// r*64 + ((c ^ (r & 7)) * 8) -- byte-for-byte the shared-memory image a
// SWIZZLE_128B TMA box would produce.  A CTA therefore streams its weight
// range with 1-D bulk copies of whole contiguous blocks (decode is a pure
// HBM stream) instead of 128 scattered 128-byte rows per box.
#pragma once
#include "common.cuh"

namespace exg {

enum EpiMode : int {
  EPI_BF16 = 0,        // out_bf16 = bf16(acc + bias)
  EPI_BF16_ACT = 1,    // out_bf16 = bf16(act(acc + bias))      (FFN1, T4(h))
  EPI_RESID = 2,       // resid   += acc + bias                 (O-proj / FFN2, fp32, T4(a,i))
  EPI_F32 = 3,         // out_f32  = acc + bias                 (logits, T4(j))
};
enum ActKind : int { ACT_NONE = 0, ACT_RELU = 1, ACT_GELU = 2 };

struct EpiParams {
  int mode = EPI_BF16;
  int act = ACT_NONE;
  const bf16* bias = nullptr;  // [features] or null
  bf16* out_bf16 = nullptr;
  float* out_f32 = nullptr;
  int64_t ldo = 0;
  float* resid = nullptr;
  int64_t ldr = 0;
  int tokens = 0, features = 0;
  // prefill QKV (EPI_BF16, row orientation): also store output features
  // [kv_inner, 3 kv_inner) -- K then V -- of token t into the KV cache at
  // (kv_slot[t], head, kv_pos[t]) (K7 fused into the producing GEMM); the
  // qkv output then holds Q only
  bf16* kv_k = nullptr;
  bf16* kv_v = nullptr;
  const int32_t* kv_slot = nullptr;
  const int32_t* kv_pos = nullptr;
  int kv_inner = 0, kv_H = 0, kv_dh = 0, kv_ctx = 0;
  // decode (swap-AB) only -- deferred stream-K reduction: every work unit
  // stores its raw fp32 accumulator segment to defer_out[seg][token][feature]
  // (seg = the unit's segment index within its 128-feature tile) and the
  // kernel ends there: no partial round trip, counters or fixup tail.  The
  // consumer kernel sums a feature's segments in segment order, adds the
  // bias and applies the epilogue (seg_count / SegInfo below) -- the same
  // arithmetic as the in-kernel fixup, so results are bit-identical.
  float* defer_out = nullptr;
};

// Stream-K cut of a decode GEMM's weight shape (tiles of 128 features x 64-k
// blocks over G CTAs): a function of the weight shape only (T13).  Feature
// tile m has seg_count(m) segments, summed in order by the consumer of a
// deferred reduction.
struct SegInfo {
  int nkb = 0, G = 0;
  int64_t I = 0;   // tiles_m * nkb
};
__host__ __device__ inline int seg_count(const SegInfo& s, int m) {
  const int64_t x0 = (int64_t)m * s.nkb, x1 = x0 + s.nkb - 1;
  auto owner = [&](int64_t x) { return (int)(((x + 1) * s.G + s.I - 1) / s.I) - 1; };
  return owner(x1) - owner(x0) + 1;
}
SegInfo decode_seg_info(int features, int K);
constexpr int DEFER_QKV = 1, DEFER_RESID = 2;
// default: the residual GEMMs only -- A/B on OPT-13B (tools/ab_deferred.py): the
// deferred QKV sums cost the attention kernel more than they save the GEMM
constexpr int DEFER_DEFAULT = DEFER_RESID;
int& deferred_enabled();    // mask of deferred decode GEMMs (exg_diag_deferred)
bool& chain_enabled();      // decode GEMM chain (exg_diag_chain)
// floats a deferred decode GEMM writes: max segments x tokens x features
size_t deferred_floats(int features, int K, int tokens);

// ---- blocked weight layout ---------------------------------------------------
inline int64_t blocked_elems(int64_t rows, int64_t K) {
  return ((rows + 127) / 128) * ((K + 63) / 64) * 128 * 64;
}
// element offset of W[row][k] in the blocked layout
__host__ __device__ inline int64_t blocked_index(int64_t row, int64_t k, int64_t K) {
  const int64_t nkb = (K + 63) / 64;
  const int64_t m = row >> 7, r = row & 127, kb = k >> 6, c = k & 63;
  return ((m * nkb + kb) << 13) + (r << 6) + ((((c >> 3) ^ (r & 7))) << 3) + (c & 7);
}
// pack a row-major W [rows][ld] (first K columns) into the blocked layout
// (zero padding to whole tiles)
void pack_blocked(bf16* dst, const bf16* src, int64_t rows, int64_t K, int64_t ld, cudaStream_t st);

CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows);

// fp32 workspace (floats) a decode (stream-K) GEMM of this weight shape
// needs for partial segments + fixup counters, for up to max_tokens tokens.
size_t decode_ws_floats(int features, int K, int max_tokens);

// Y = X . W^T with epilogue.  X: row-major [tokens][ldx]; W: blocked layout
// of a [features][K] matrix.  decode = true selects swap-AB with stream-K
// (tokens on the MMA N axis); `ws` must hold decode_ws_floats() floats and
// be zero-initialised once (its fixup counters return to zero after use).
struct LinearArgs {
  const bf16* X = nullptr;
  int64_t ldx = 0;
  const bf16* Wb = nullptr;   // blocked
  int K = 0;
  EpiParams ep;
  bool decode = false;
  float* ws = nullptr;
  size_t ws_floats = 0;
  int bn = 0;                 // 0 -> auto
};
void linear(const LinearArgs& a, cudaStream_t st);

int decode_bn(int tokens);

// Decode GEMM chain (gemm_tc.cu decode_chain_kernel): up to 4 decode GEMMs
// (same token count) in one persistent launch, each with its own stream-K
// cut, epilogue and in-kernel fixup -- bit-identical to separate launches --
// with an optional LayerNorm of x into h after a phase (ln_after = index
// into ln_g / ln_b).  Phase q's activations X must be complete once phase
// q-1 (and its LayerNorm) is; phase 0 waits for the previous kernel (PDL).
struct ChainSpec {
  struct Phase {
    const bf16* X = nullptr;
    int64_t ldx = 0;
    const bf16* Wb = nullptr;
    int features = 0, K = 0;
    EpiParams ep;
    int ln_after = -1;
  } ph[4];
  int n = 0, tokens = 0;
  const bf16* ln_g[2] = {nullptr, nullptr};
  const bf16* ln_b[2] = {nullptr, nullptr};
  float* x = nullptr;      // fp32 residual [tokens][d] (the LayerNorm input)
  bf16* h = nullptr;       // bf16 [tokens][d] (the LayerNorm output)
  int d = 0;
  float eps = 1e-5f;
  float* ws = nullptr;     // chain_ws_floats() floats, zero-initialised once
  size_t ws_floats = 0;
  unsigned* sync = nullptr;   // 8 zero-initialised counters, owned by the caller
  unsigned epoch = 0;         // 1, 2, ... per launch on the same sync counters
};
size_t chain_ws_floats(const ChainSpec& c);
void decode_chain(const ChainSpec& c, cudaStream_t st);

}  // namespace exg
