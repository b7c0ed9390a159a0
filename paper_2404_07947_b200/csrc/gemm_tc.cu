// tcgen05 GEMM (K3 prefill, K5 decode swap-AB, K8 LM head).
//
// One 128 x BN output tile per CTA, K in 64-wide blocks through an
// STAGES-deep TMA -> shared ring (SWIZZLE_128B, K-major), single-thread
// tcgen05.mma issue with the fp32 accumulator in TMEM, 4 epilogue warps
// draining TMEM with tcgen05.ld.  Warp roles: 0 = TMA producer, 1 = MMA
// issuer, 2 = TMEM allocator, 4..7 = epilogue.
#include <cuda.h>

#include <mutex>

#include "gemm_tc.cuh"

namespace exg {

namespace {
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                      CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    EXG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  });
  return fn;
}

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f;  // sqrt(2/pi)
  return 0.5f * x * (1.0f + tanhf(k0 * (x + 0.044715f * x * x * x)));
}

__device__ __forceinline__ void epi_store(const EpiParams& ep, int tok, int feat, float acc) {
  float v = acc;
  if (ep.bias) v += bf2f(ep.bias[feat]);
  switch (ep.mode) {
    case EPI_BF16:
      ep.out_bf16[(int64_t)tok * ep.ldo + feat] = f2bf(v);
      break;
    case EPI_BF16_ACT:
      v = ep.act == ACT_RELU ? fmaxf(v, 0.0f) : (ep.act == ACT_GELU ? gelu_tanh(v) : v);
      ep.out_bf16[(int64_t)tok * ep.ldo + feat] = f2bf(v);
      break;
    case EPI_RESID: {
      float* r = ep.resid + (int64_t)tok * ep.ldr + feat;
      *r = *r + v;
      break;
    }
    default:
      ep.out_f32[(int64_t)tok * ep.ldo + feat] = v;
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(256, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                   int K, int kb_per_split, int swap, EpiParams ep, float* __restrict__ partial) {
  constexpr int B_BYTES = BN * BK * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nkb_total = (K + BK - 1) / BK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = min(kb_per_split, nkb_total - kb0);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_holder, BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        if (kb >= STAGES) mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
        tma_load_2d(sA + s * A_BYTES, &tmA, &full[s], (kb0 + kb) * BK, m0);
        tma_load_2d(sB + s * B_BYTES, &tmB, &full[s], (kb0 + kb) * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_base = smem_u32(sA + s * A_BYTES);
        const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          umma_bf16(tmem, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                    (kb | k) != 0);
        }
        umma_commit(&empty[s]);
      }
      umma_commit(tfull);
    }
  } else if (warp >= 4) {
    mbar_wait(tfull, 0);
    tc_fence_after();
    const int q = warp - 4;
    const int r = q * 32 + lane;  // accumulator row == TMEM lane
    const int gm = m0 + r;
    const bool row_ok = gm < M;
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
      if (!row_ok) continue;
      if (nkb <= 0) {  // empty K range (last split): contributes zeros
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.0f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int gn = n0 + c + j;
        if (gn >= N) break;
        const int tok = swap ? gn : gm;
        const int feat = swap ? gm : gn;
        if (partial) {
          partial[((int64_t)blockIdx.z * ep.tokens + tok) * ep.features + feat] = v[j];
        } else {
          epi_store(ep, tok, feat, v[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, BN);
  }
}

// split-K reduction in split order, then the epilogue (deterministic)
__global__ void splitk_reduce_kernel(const float* __restrict__ partial, int split, EpiParams ep) {
  const int64_t n = (int64_t)ep.tokens * ep.features;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int s = 0; s < split; ++s) acc += partial[(int64_t)s * n + i];
    epi_store(ep, (int)(i / ep.features), (int)(i % ep.features), acc);
  }
}

template <int BN>
constexpr int stages_for() {
  return (BN * BK * 2 + A_BYTES) * 8 <= 200 * 1024 ? 8 : (200 * 1024) / (BN * BK * 2 + A_BYTES);
}

template <int BN>
size_t smem_bytes() {
  constexpr int S = stages_for<BN>();
  return 1024 + (size_t)S * (A_BYTES + BN * BK * 2) + (2 * S + 1) * 8 + 16;
}

template <int BN>
void launch(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, int split, int swap,
            const EpiParams& ep, float* partial, cudaStream_t st) {
  constexpr int S = stages_for<BN>();
  static bool attr_set = false;
  const size_t smem = smem_bytes<BN>();
  if (!attr_set) {
    EXG_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  const int nkb = (K + BK - 1) / BK;
  const int kbps = (nkb + split - 1) / split;
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN, split);
  gemm_tc_kernel<BN, S><<<grid, 256, smem, st>>>(ta, tb, M, N, K, kbps, swap, ep, partial);
  EXG_CHECK_LAUNCH();
}
}  // namespace

CUtensorMap make_tmap_bf16(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ") rows=" + std::to_string(rows) +
                    " cols=" + std::to_string(cols) + " ld=" + std::to_string(ld));
  return m;
}

int decode_split_k(int features, int K) {
  const int tiles = (features + BM - 1) / BM;
  const int nkb = (K + BK - 1) / BK;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= 16; ++s) {
    if (nkb / s < 4) break;
    const double ctas = (double)tiles * s;
    const double waves = std::ceil(ctas / 148.0);
    const double eff = ctas / (waves * 148.0);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

int decode_bn(int tokens) {
  if (tokens <= 32) return 32;
  if (tokens <= 64) return 64;
  if (tokens <= 128) return 128;
  return 256;
}

void linear(const LinearArgs& a, cudaStream_t st) {
  const int tokens = a.ep.tokens, features = a.ep.features;
  if (tokens <= 0 || features <= 0) return;
  int BN;
  CUtensorMap ta, tb;
  int M, N;
  if (a.decode) {
    BN = a.bn ? a.bn : decode_bn(tokens);
    M = features;
    N = tokens;
    if (a.cached) {
      ta = a.cached->a;
      tb = a.cached->b;
    } else {
      ta = make_tmap_bf16(a.W, features, a.K, a.ldw, BM);
      tb = make_tmap_bf16(a.X, tokens, a.K, a.ldx, BN);
    }
  } else {
    BN = a.bn ? a.bn : (features >= 256 ? 256 : (features > 64 ? 128 : 64));
    M = tokens;
    N = features;
    if (a.cached) {
      ta = a.cached->a;
      tb = a.cached->b;
    } else {
      ta = make_tmap_bf16(a.X, tokens, a.K, a.ldx, BM);
      tb = make_tmap_bf16(a.W, features, a.K, a.ldw, BN);
    }
  }
  const int split = a.split > 1 ? a.split : 1;
  float* partial = split > 1 ? a.ws : nullptr;
  if (split > 1 && !partial) throw CudaError("split-K GEMM without workspace");
  const int swap = a.decode ? 1 : 0;
  switch (BN) {
    case 32: launch<32>(ta, tb, M, N, a.K, split, swap, a.ep, partial, st); break;
    case 64: launch<64>(ta, tb, M, N, a.K, split, swap, a.ep, partial, st); break;
    case 128: launch<128>(ta, tb, M, N, a.K, split, swap, a.ep, partial, st); break;
    case 256: launch<256>(ta, tb, M, N, a.K, split, swap, a.ep, partial, st); break;
    default: throw CudaError("bad BN");
  }
  if (split > 1) {
    const int64_t n = (int64_t)tokens * features;
    const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(partial, split, a.ep);
    EXG_CHECK_LAUNCH();
  }
}

}  // namespace exg
