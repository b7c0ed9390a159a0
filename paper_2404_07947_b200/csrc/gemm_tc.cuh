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
};

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

}  // namespace exg
