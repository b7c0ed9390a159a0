// tcgen05 / TMEM / TMA GEMM for the prefill GEMMs (K3), decode projections
// (K5, swap-AB) and LM head (K8).  D[M][N] = A[M][K] . B[N][K]^T, bf16 in,
// fp32 accumulate in TMEM, fused epilogues (bias / activation / residual).
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

// Output orientation is always Y[token][feature]; `swap` says whether the
// GEMM's M axis is tokens (swap = 0: A = activations, B = weights) or
// features (swap = 1: A = weights, B = activations; decode).
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
};

struct GemmTmaps {
  CUtensorMap a, b;
};

// Build a 2-D TMA map over a row-major bf16 matrix [rows][ld] using the
// first `cols` columns; box = 64 columns x box_rows rows, 128B swizzle.
CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows);

// Choose the split-K factor for a decode (swap-AB) GEMM from the weight
// shape only (never the batch), so results are batch invariant (T13).
int decode_split_k(int features, int K);

// Y = X . W^T with epilogue.  X: [tokens][K] (ldx), W: [features][K] (ldw).
// decode = true selects swap-AB (tokens on the MMA N axis).  `ws` is an fp32
// workspace for split-K partials of at least split*tokens*features floats.
struct LinearArgs {
  const bf16* X = nullptr;
  int64_t ldx = 0;
  const bf16* W = nullptr;
  int64_t ldw = 0;
  int K = 0;
  EpiParams ep;
  bool decode = false;
  int split = 1;
  float* ws = nullptr;
  const GemmTmaps* cached = nullptr;   // optional prebuilt maps (A,B as the kernel sees them)
  int bn = 0;                         // 0 -> auto
};
void linear(const LinearArgs& a, cudaStream_t st);

// token tile (MMA N) used for a decode GEMM with `tokens` rows
int decode_bn(int tokens);

}  // namespace exg
