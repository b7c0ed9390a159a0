// tcgen05 GEMM (K3 prefill, K5 decode swap-AB, K8 LM head).
//
// Persistent kernel, one CTA per SM.  128 x BN accumulator tiles in TMEM,
// double buffered so the epilogue of one work unit overlaps the MMAs of the
// next.  K streams in 64-wide blocks through an S-deep shared-memory ring
// (SWIZZLE_128B, K-major): activations arrive by 2-D TMA, weights by 1-D bulk
// copies of whole pre-swizzled 16 KB blocks (see gemm_tc.cuh).  Warp roles:
// 0 = producer, 1 = MMA issuer (one thread), 2 = TMEM allocator,
// 4..7 = epilogue (TMEM lanes 32*(w%4)..).
//
// Work decomposition
//  * prefill (data-parallel): unit = whole tile, tiles t = cta, cta+G, ...
//  * decode (stream-K): per BN-column chunk of tokens, the iteration space
//    tiles_m x k-blocks is cut into G equal contiguous ranges (G = min(#SMs,
//    iterations): a function of the weight shape only).  A tile cut by a range
//    boundary leaves fp32 partial segments; the CTA that completes a tile's
//    last segment (atomic counter) sums the segments in segment order and
//    runs the epilogue.  Cut points never depend on the batch, so a token's
//    bits do not depend on its batch-mates (T13).
#include <cuda.h>

#include <mutex>

#include <vector>

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

// diagnostics only (exg_diag_gemm_flags): bit 0 = skip the MMAs, bit 6 = prefill on
// the 1-CTA kernel instead of CTA pairs, bit 7 = no early stream-K fixup
int& gemm_debug_flags() {
  static int f = 0;
  return f;
}

// prefill raster: A slab (MB) kept L2-resident per group (diagnostics override)
int64_t& gemm_slab_mb() {
  static int64_t mb = 32;
  return mb;
}

// diagnostics: stream-K CTA count cap (0 = one per SM)
int& gemm_sk_ctas() {
  static int n = 0;
  return n;
}

// g_dbg kernel argument: the flags, plus the launch sequence number when
// span recording (bit 4) is on
int& gemm_span_seq() {
  static int n = 0;
  return n;
}
int gemm_dbg_arg(bool decode) {
  const int f = gemm_debug_flags();
  if (!(f & 16)) return f;
  if (!decode || gemm_span_seq() >= 4096) return f & ~16;   // decode launches only, first 4096
  const int seq = gemm_span_seq()++;
  return (f & 0xff) | (seq << 8);
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    EXG_CUDA(cudaGetDevice(&dev));
    EXG_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int A_BYTES = BM * BK * 2;     // one 16 KB block
constexpr int BLK_ELEMS = BM * BK;

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f;  // sqrt(2/pi)
  return 0.5f * x * (1.0f + tanhf(k0 * (x + 0.044715f * x * x * x)));
}

__device__ __forceinline__ float epi_value(const EpiParams& ep, int feat, float acc) {
  float v = acc;
  if (ep.bias) v += bf2f(ep.bias[feat]);
  if (ep.mode == EPI_BF16_ACT) v = ep.act == ACT_RELU ? fmaxf(v, 0.0f) : (ep.act == ACT_GELU ? gelu_tanh(v) : v);
  return v;
}

__device__ __forceinline__ void epi_store(const EpiParams& ep, int tok, int feat, float acc) {
  const float v = epi_value(ep, feat, acc);
  switch (ep.mode) {
    case EPI_BF16:
    case EPI_BF16_ACT:
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

// 16 consecutive tokens t0.. of one feature (decode swap-AB orientation).
// All global loads (bias, residual) are issued before any store: a per-element
// read-modify-write would serialise 16 memory round trips, since the compiler
// cannot prove the stores do not alias the next load.
__device__ __forceinline__ void epi_store_col16(const EpiParams& ep, int t0, int feat, int N, const float* v) {
  const int n = min(16, N - t0);
  const float b = ep.bias ? bf2f(ep.bias[feat]) : 0.f;
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    x[j] = v[j];
    if (ep.bias) x[j] += b;
  }
  switch (ep.mode) {
    case EPI_BF16_ACT:
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = ep.act == ACT_RELU ? fmaxf(x[j], 0.0f) : (ep.act == ACT_GELU ? gelu_tanh(x[j]) : x[j]);
      // fall through
    case EPI_BF16:
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < n) ep.out_bf16[(int64_t)(t0 + j) * ep.ldo + feat] = f2bf(x[j]);
      break;
    case EPI_RESID: {
      float* r = ep.resid + (int64_t)t0 * ep.ldr + feat;
      float old[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) old[j] = j < n ? r[(int64_t)j * ep.ldr] : 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < n) r[(int64_t)j * ep.ldr] = old[j] + x[j];
      break;
    }
    default:
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < n) ep.out_f32[(int64_t)(t0 + j) * ep.ldo + feat] = x[j];
  }
}

// 16 consecutive features of one token row (prefill orientation), vectorised
__device__ __forceinline__ void epi_store_row16(const EpiParams& ep, int tok, int f0, int N, const float* v) {
  if (f0 + 16 <= N) {
    if (ep.mode == EPI_BF16 || ep.mode == EPI_BF16_ACT) {
      if ((ep.ldo & 7) == 0) {
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat162 h2 =
              __floats2bfloat162_rn(epi_value(ep, f0 + 2 * j, v[2 * j]), epi_value(ep, f0 + 2 * j + 1, v[2 * j + 1]));
          pk[j] = *reinterpret_cast<uint32_t*>(&h2);
        }
        if (ep.kv_k && f0 >= ep.kv_inner) {
          // K / V columns: straight into the cache row (slot, head, pos); the
          // 16 features lie in one head (dh % 16 == 0)
          const int which = (f0 - ep.kv_inner) / ep.kv_inner, hd = (f0 - ep.kv_inner) % ep.kv_inner;
          const int h = hd / ep.kv_dh, j = hd % ep.kv_dh;
          bf16* base = which ? ep.kv_v : ep.kv_k;
          uint4* dst = reinterpret_cast<uint4*>(
              base + (((int64_t)ep.kv_slot[tok] * ep.kv_H + h) * ep.kv_ctx + ep.kv_pos[tok]) * ep.kv_dh + j);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          return;
        }
        uint4* dst = reinterpret_cast<uint4*>(ep.out_bf16 + (int64_t)tok * ep.ldo + f0);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        return;
      }
    } else if (ep.mode == EPI_RESID) {
      if ((ep.ldr & 3) == 0) {
        float4* r = reinterpret_cast<float4*>(ep.resid + (int64_t)tok * ep.ldr + f0);
        float4 old[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) old[q] = r[q];   // all loads before any store
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 x = old[q];
          x.x += epi_value(ep, f0 + 4 * q, v[4 * q]);
          x.y += epi_value(ep, f0 + 4 * q + 1, v[4 * q + 1]);
          x.z += epi_value(ep, f0 + 4 * q + 2, v[4 * q + 2]);
          x.w += epi_value(ep, f0 + 4 * q + 3, v[4 * q + 3]);
          r[q] = x;
        }
        return;
      }
    } else if ((ep.ldo & 3) == 0) {
      float4* o = reinterpret_cast<float4*>(ep.out_f32 + (int64_t)tok * ep.ldo + f0);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        o[q] = make_float4(epi_value(ep, f0 + 4 * q, v[4 * q]), epi_value(ep, f0 + 4 * q + 1, v[4 * q + 1]),
                           epi_value(ep, f0 + 4 * q + 2, v[4 * q + 2]), epi_value(ep, f0 + 4 * q + 3, v[4 * q + 3]));
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < 16; ++j)
    if (f0 + j < N) epi_store(ep, tok, f0 + j, v[j]);
}

// ---- work units -------------------------------------------------------------
struct Work {
  int dp;          // 1 = data-parallel tiles, 0 = stream-K
  int tiles_m, tiles_n, nkb, G, max_segs;
  int gm;          // data-parallel raster group (m-tiles)
  int64_t I;       // stream-K iterations per chunk = tiles_m * nkb
};

struct Unit {
  int m, n, kb0, kb1, seg;
  bool full;
};

__host__ __device__ __forceinline__ int64_t sk_start(const Work& w, int c) { return (int64_t)c * w.I / w.G; }
// CTA whose range contains iteration x
__host__ __device__ __forceinline__ int sk_owner(const Work& w, int64_t x) {
  return (int)(((x + 1) * w.G + w.I - 1) / w.I) - 1;
}

struct UnitIter {
  Work w;
  int c, t, chunk;
  int64_t x, xe;
  __device__ void init(const Work& w_, int cta) {
    w = w_;
    c = cta;
    t = cta;
    chunk = 0;
    x = sk_start(w, c);
    xe = sk_start(w, c + 1);
  }
  __device__ bool next(Unit& u) {
    if (w.dp) {
      if (t >= w.tiles_m * w.tiles_n) return false;
      // grouped raster: GM m-tiles (a ~32 MB slab of A) sweep all n-tiles
      // before the next slab, so A stays L2-resident while B streams
      const int per_group = w.gm * w.tiles_n;
      const int g = t / per_group, within = t % per_group;
      const int gm_count = min(w.gm, w.tiles_m - g * w.gm);
      u.m = g * w.gm + within % gm_count;
      u.n = within / gm_count;
      u.kb0 = 0;
      u.kb1 = w.nkb;
      u.seg = 0;
      u.full = true;
      t += w.G;
      return true;
    }
    while (x >= xe) {
      if (++chunk >= w.tiles_n) return false;
      x = sk_start(w, c);
      xe = sk_start(w, c + 1);
    }
    u.m = (int)(x / w.nkb);
    u.kb0 = (int)(x % w.nkb);
    const int64_t e = min((int64_t)(u.m + 1) * w.nkb, xe);
    u.kb1 = u.kb0 + (int)(e - x);
    u.n = chunk;
    u.full = (u.kb0 == 0 && u.kb1 == w.nkb);
    u.seg = c - sk_owner(w, (int64_t)u.m * w.nkb);
    x = e;
    return true;
  }
};

// 8 epilogue warps (two per TMEM lane quarter, each half of the columns).
// Under PDL the producer streams its first weight blocks before the grid
// dependency resolves.
template <int SWAP>
struct EpiCfg {
  static constexpr int WARPS = 8;
  static constexpr int THREADS = 128 + 32 * WARPS;
};

// diagnostics (exg_diag_gemm_flags bit 2): per-CTA %globaltimer marks
//   0 entry, 1 setup done, 2 producer past griddepcontrol.wait, 3 first full
//   stage at the MMA warp, 4 last MMA commit, 5 epilogue done, 6 exit
__device__ unsigned long long g_gemm_tl[256 * 8];
// flag bit 4: in-situ launch spans -- earliest CTA entry / latest CTA exit of
// launch number (g_dbg >> 8) & 4095 (exg_diag_gemm_spans)
__device__ unsigned long long g_span_start[4096], g_span_end[4096], g_span_dep[4096];
__device__ __forceinline__ void tl_mark(int dbg, int k) {
  if (dbg & 4) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 256) g_gemm_tl[blockIdx.x * 8 + k] = t;
  }
}

// SWAP = 1 (decode): A = weights (blocked), B = activations (TMA 2-D).
// SWAP = 0 (prefill): A = activations (TMA 2-D), B = weights (blocked).
template <int BN, int STAGES, int SWAP>
__global__ void __launch_bounds__(EpiCfg<SWAP>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmX, const bf16* __restrict__ Wb, int M, int N, int n_wblk,
                   Work work, EpiParams ep, float* __restrict__ partial, int* __restrict__ counters,
                   int inkernel_fixup, int g_dbg) {
  constexpr int EPI_WARPS = EpiCfg<SWAP>::WARPS;
  auto epi_bar = [] { asm volatile("bar.sync 1, %0;" ::"n"(32 * EpiCfg<SWAP>::WARPS) : "memory"); };
  griddep_launch_dependents();
  if (threadIdx.x == 0) tl_mark(g_dbg, 0);
  if ((g_dbg & 16) && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(&g_span_start[(g_dbg >> 8) & 4095], t);
  }
  constexpr int B_BYTES = BN * BK * 2;
  constexpr uint32_t TMEM_COLS =
      (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;      // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_last = reinterpret_cast<int*>(tmem_holder + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_holder, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (threadIdx.x == 0) tl_mark(g_dbg, 1);

  UnitIter it;
  it.init(work, blockIdx.x);
  Unit u;
  if (warp == 0) {
    if (lane == 0) {
      // Weights never depend on the previous kernel: the first STAGES weight
      // loads are issued before griddepcontrol.wait; the activation loads of
      // those stages follow once the previous grid has completed.
      auto wbytes_of = [&](int n) {
        if (SWAP) return A_BYTES;
        int bytes = 0;
        for (int rr = 0; rr < BN; rr += BM)
          if ((n * BN + rr) / BM < n_wblk) bytes += (BN < BM ? BN : BM) * BK * 2;
        return bytes;
      };
      auto issue_w = [&](uint32_t s, int m, int n, int kb) {
        if (SWAP) {
          bulk_load(sA + s * A_BYTES, Wb + ((int64_t)m * work.nkb + kb) * BLK_ELEMS, A_BYTES, &full[s]);
        } else {
          // weight rows [n*BN, n*BN+BN) = blocks (n*BN)/128 ..; BN = 64 uses half a block
          for (int rr = 0; rr < BN; rr += BM) {
            const int blk = (n * BN + rr) / BM;
            if (blk >= n_wblk) break;
            const int sub = (n * BN + rr) % BM;
            bulk_load(sB + s * B_BYTES + rr * BK * 2, Wb + ((int64_t)blk * work.nkb + kb) * BLK_ELEMS + (int64_t)sub * BK,
                      (uint32_t)((BN < BM ? BN : BM) * BK * 2), &full[s]);
          }
        }
      };
      auto issue_x = [&](uint32_t s, int m, int n, int kb) {
        if (SWAP)
          tma_load_2d(sB + s * B_BYTES, &tmX, &full[s], kb * BK, n * BN);
        else
          tma_load_2d(sA + s * A_BYTES, &tmX, &full[s], kb * BK, m * BM);
      };
      int pend[STAGES][3];
      int npend = 0;
      bool waited = false;
      uint32_t g = 0;
      while (it.next(u)) {
        for (int kb = u.kb0; kb < u.kb1; ++kb, ++g) {
          const uint32_t s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          if (!waited && g >= STAGES) {
            griddep_wait();
            tl_mark(g_dbg, 2);
            if (g_dbg & 16) {
              unsigned long long t;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
              atomicMin(&g_span_dep[(g_dbg >> 8) & 4095], t);
            }
            for (int i = 0; i < npend; ++i) issue_x(i, pend[i][0], pend[i][1], pend[i][2]);
            waited = true;
          }
          if (g >= STAGES) mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], wbytes_of(u.n) + (SWAP ? B_BYTES : A_BYTES));
          issue_w(s, u.m, u.n, kb);
          if (waited) {
            issue_x(s, u.m, u.n, kb);
          } else {
            pend[npend][0] = u.m;
            pend[npend][1] = u.n;
            pend[npend][2] = kb;
            ++npend;
          }
        }
      }
      if (!waited) {
        griddep_wait();
        tl_mark(g_dbg, 2);
        if (g_dbg & 16) {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          atomicMin(&g_span_dep[(g_dbg >> 8) & 4095], t);
        }
        for (int i = 0; i < npend; ++i) issue_x(i, pend[i][0], pend[i][1], pend[i][2]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      uint32_t g = 0, ui = 0;
      while (it.next(u)) {
        const uint32_t a = ui & 1;
        if (ui >= 2) mbar_wait(&tempty[a], ((ui >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + a * BN;
        for (int kb = u.kb0; kb < u.kb1; ++kb, ++g) {
          const uint32_t s = g % STAGES;
          const uint32_t ph = (g / STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (g == 0) tl_mark(g_dbg, 3);
          if (g_dbg & 1) {  // diagnostics: memory pipeline only (no MMA)
            mbar_arrive(&empty[s]);
            continue;
          }
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                      (kb != u.kb0 || k) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[a]);
        ++ui;
      }
      tl_mark(g_dbg, 4);
    }
  } else if (warp >= 4) {
    // 8 epilogue warps: warp w reads TMEM lanes 32*(w%4).. (hardware rule)
    // and one half of the accumulator columns
    const int q = warp & 3;
    constexpr int PARTS = EPI_WARPS / 4;  // column parts per TMEM lane quarter
    const int part = (warp - 4) >> 2;
    const int c_lo = part * (BN / PARTS), c_hi = c_lo + BN / PARTS;
    griddep_wait();  // outputs / residual may still be in use by the previous kernel
    const int r = q * 32 + lane;
    uint32_t ui = 0;
    while (it.next(u)) {
      const uint32_t a = ui & 1;
      mbar_wait(&tfull[a], (ui >> 1) & 1);
      tc_fence_after();
      const int gm = u.m * BM + r;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + a * BN;
      const bool row_ok = gm < M;
      float* pp = nullptr;
      // stream-K: a CTA that reaches a split tile after every other segment
      // of it has landed (the usual case for a CTA's last unit: the tile's
      // other segments opened the next CTAs' ranges) sums them with its own
      // segment straight from TMEM -- in segment order, the fixup's
      // arithmetic -- instead of storing its segment, counting in and
      // reading it back
      const bool fixup = !u.full && inkernel_fixup && !(SWAP && ep.defer_out);
      bool early = false;
      int* cnt = nullptr;
      int nseg = 0;
      if (fixup && !(g_dbg & 128)) {   // diagnostics bit 7: always count in (A/B)
        const int64_t x0 = (int64_t)u.m * work.nkb;
        nseg = sk_owner(work, x0 + work.nkb - 1) - sk_owner(work, x0) + 1;
        cnt = counters + (u.n * work.tiles_m + u.m);
        if (threadIdx.x == 128) {
          int v;
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
          *s_last = (v == nseg - 1);
        }
        epi_bar();
        early = *s_last;
        epi_bar();   // every thread has read s_last before it is written again
      }
      if (early) {
        __threadfence();
        const float* base = partial + ((int64_t)u.n * work.tiles_m + u.m) * work.max_segs * (int64_t)(BM * BN);
        for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
          float own[16], acc[16];
          tmem_ld16(taddr + c0, own);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = 0.f;
          for (int s0 = 0; s0 < nseg; s0 += 4) {
            float v[4][16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float* src = base + (int64_t)(s0 + q) * BM * BN + (int64_t)c0 * BM + r;
              const bool other = s0 + q < nseg && s0 + q != u.seg;
#pragma unroll
              for (int j = 0; j < 16; ++j) v[q][j] = other ? __ldcg(src + (int64_t)j * BM) : own[j];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (s0 + q < nseg) acc[j] += v[q][j];
          }
          if (!row_ok) continue;
          if (SWAP) {
            if (u.n * BN + c0 < N) epi_store_col16(ep, u.n * BN + c0, gm, N, acc);
          } else {
            epi_store_row16(ep, gm, u.n * BN + c0, N, acc);
          }
        }
        if (threadIdx.x == 128) *cnt = 0;
      } else if (SWAP && ep.defer_out) {
        // deferred reduction: the raw segment, [seg][token][feature]
        // (a warp's 32 features of one token are one 128-byte line)
        float* dst = ep.defer_out + ((int64_t)u.seg * N) * M + gm;
        for (int c = c_lo; c < c_hi; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
          const int t0 = u.n * BN + c;
          if (row_ok)
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (t0 + j < N) dst[(int64_t)(t0 + j) * M] = v[j];
        }
      } else if (!u.full) {
        // fp32 partial segment, column-major [BN][128] per (chunk, tile, seg)
        pp = partial + (((int64_t)u.n * work.tiles_m + u.m) * work.max_segs + u.seg) * (int64_t)(BM * BN);
        for (int c = c_lo; c < c_hi; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) pp[(int64_t)(c + j) * BM + r] = v[j];
        }
      } else if (SWAP) {
        // rows = features, columns = tokens
        for (int c = c_lo; c < c_hi; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
          if (row_ok && u.n * BN + c < N) epi_store_col16(ep, u.n * BN + c, gm, N, v);
        }
      } else {
        for (int c = c_lo; c < c_hi; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
          if (row_ok) epi_store_row16(ep, gm, u.n * BN + c, N, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
      ++ui;
      if (fixup && !early) {
        // stream-K fixup: the CTA completing the tile's last segment reduces
        if (g_dbg & 128) {
          const int64_t x0 = (int64_t)u.m * work.nkb;
          nseg = sk_owner(work, x0 + work.nkb - 1) - sk_owner(work, x0) + 1;
          cnt = counters + (u.n * work.tiles_m + u.m);
        }
        __threadfence();
        epi_bar();
        if (threadIdx.x == 128) *s_last = (atomicAdd(cnt, 1) == nseg - 1);
        epi_bar();
        if (*s_last) {
          __threadfence();
          const float* base = partial + ((int64_t)u.n * work.tiles_m + u.m) * work.max_segs * (int64_t)(BM * BN);
          // 16 columns at a time; the loads of up to 4 segments issue back to
          // back (one L2 round trip instead of one per segment), segments
          // summed in segment order
          for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
            float acc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = 0.f;
            for (int s0 = 0; s0 < nseg; s0 += 4) {
              float v[4][16];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float* src = base + (int64_t)(s0 + q) * BM * BN + (int64_t)c0 * BM + r;
#pragma unroll
                for (int j = 0; j < 16; ++j) v[q][j] = (s0 + q < nseg) ? __ldcg(src + (int64_t)j * BM) : 0.f;
              }
#pragma unroll
              for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (s0 + q < nseg) acc[j] += v[q][j];
            }
            if (!row_ok) continue;
            if (SWAP) {
              if (u.n * BN + c0 < N) epi_store_col16(ep, u.n * BN + c0, gm, N, acc);
            } else {
              epi_store_row16(ep, gm, u.n * BN + c0, N, acc);
            }
          }
          if (threadIdx.x == 128) *cnt = 0;
        }
        epi_bar();
      }
    }
    if (threadIdx.x == 128) tl_mark(g_dbg, 5);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
  if (threadIdx.x == 0) tl_mark(g_dbg, 6);
  if ((g_dbg & 16) && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&g_span_end[(g_dbg >> 8) & 4095], t);
  }
}

// ============================================================================
// Decode GEMM chain (one persistent launch per decoder layer): the
// O-projection (+ residual), LN2, FFN1 (+ act), FFN2 (+ residual) and -- when
// another layer follows -- that layer's LN1 and QKV, between two decode
// attention launches.  Every GEMM phase keeps its own stream-K cut (Work of
// its weight shape, G_p = min(#SMs, I_p)), epilogues and in-kernel fixups --
// the arithmetic of the separate launches, so results are bit-identical --
// but the weight stream never stops at a phase boundary: the producer keeps
// issuing the next phase's weight blocks into the ring while that phase's
// activations are not ready yet (their TMA loads are queued and issued once
// the phase's inputs are complete), and the epilogue warps overlap a phase's
// fixups / LayerNorm with the next phase's mainloop.  Readiness between
// phases is a grid-wide counter per phase in global memory (every CTA adds
// one when its epilogue has finished the phase; LN phases add a second
// counter), monotonic across launches (targets grid x epoch).
// ============================================================================
constexpr int CHAIN_MAX = 4;
struct ChainPhase {
  const bf16* Wb;
  Work w;
  EpiParams ep;
  float* partial;
  int* counters;
  int M, N, n_wblk;
  int ln_after;          // LayerNorm of x into h once this phase is complete (index into ln[]), -1: none
};
struct ChainLN {
  const bf16 *g, *b;
};
struct ChainArgs {
  int n;
  ChainPhase ph[CHAIN_MAX];
  ChainLN ln[2];
  float* x;
  bf16* h;
  int d;
  float eps;
  unsigned* sync;        // [2 * CHAIN_MAX]: done[p], ln_done[p]
  unsigned epoch;        // this launch's number (>= 1): counters reach grid * epoch
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// spin until *p reaches target (wrap-around compare); traps after ~4 s
__device__ __forceinline__ void wait_counter(const unsigned* p, unsigned target) {
  if ((int)(ld_acquire_u32(p) - target) >= 0) return;
  const long long t0 = clock64();
  while ((int)(ld_acquire_u32(p) - target) < 0) {
    __nanosleep(128);
    if (clock64() - t0 > 8000000000LL) {
      printf("exg: chain counter wait timeout block %d thread %d\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

struct ChainIter {
  const ChainArgs* a;
  UnitIter it;
  int p;
  __device__ void init(const ChainArgs* args) {
    a = args;
    p = 0;
    it.init(a->ph[0].w, blockIdx.x);
  }
  // next unit of this CTA; phase index in *ph.  Returns false at the end.
  __device__ bool next(Unit& u, int* ph) {
    while (p < a->n) {
      if ((int)blockIdx.x < a->ph[p].w.G && it.next(u)) {
        *ph = p;
        return true;
      }
      if (++p < a->n) it.init(a->ph[p].w, blockIdx.x);
    }
    return false;
  }
};

// diagnostics (exg_diag_chain_timeline): per-CTA %globaltimer marks of the
// last chain launch -- [0] entry, [1+q] producer: inputs of phase q ready,
// [5+q] epilogue: phase q finished on this CTA, [9+q] LayerNorm after q done,
// [13] producer: last load issued, [14] epilogue exit
__device__ unsigned long long g_chain_tl[256 * 32];
__device__ int g_chain_tl_on;
__device__ __forceinline__ void chain_mark(int k) {
  if (g_chain_tl_on) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 256) g_chain_tl[blockIdx.x * 32 + k] = t;
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(EpiCfg<1>::THREADS, 1)
    decode_chain_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
                        const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3,
                        const __grid_constant__ ChainArgs ca) {
  constexpr int EPI_WARPS = EpiCfg<1>::WARPS;
  auto epi_bar = [] { asm volatile("bar.sync 1, %0;" ::"n"(32 * EpiCfg<1>::WARPS) : "memory"); };
  griddep_launch_dependents();
  constexpr int B_BYTES = BN * BK * 2;
  constexpr uint32_t TMEM_COLS =
      (2 * BN <= 32) ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;      // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_last = reinterpret_cast<int*>(tmem_holder + 1);
  float* red = reinterpret_cast<float*>(s_last + 1) + 2;   // [8] LayerNorm partial sums

  const CUtensorMap* tms[CHAIN_MAX] = {&tm0, &tm1, &tm2, &tm3};
  const unsigned G = gridDim.x;
  unsigned* done = ca.sync;
  unsigned* ln_done = ca.sync + CHAIN_MAX;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int q = 0; q < ca.n; ++q) prefetch_tmap(tms[q]);
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], 1);
    }
    for (int a2 = 0; a2 < 2; ++a2) {
      mbar_init(&tfull[a2], 1);
      mbar_init(&tempty[a2], EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_holder, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (threadIdx.x == 0) chain_mark(0);

  // the inputs of phase q are complete: q = 0 -> the previous kernel (PDL);
  // else the previous phase (or the LayerNorm that follows it) on every CTA
  auto inputs_ready = [&](int q) {
    if (q == 0) {
      griddep_wait();
    } else {
      const int pq = q - 1;
      wait_counter(ca.ph[pq].ln_after >= 0 ? &ln_done[pq] : &done[pq], G * ca.epoch);
    }
    fence_proxy_async_global();   // generic-proxy writes of other CTAs -> this CTA's TMA reads
    chain_mark(1 + q);
  };

  ChainIter it;
  it.init(&ca);
  Unit u;
  int ph;
  if (warp == 0) {
    if (lane == 0) {
      // weight blocks stream ahead of their activations: a stage's activation
      // load waits in a FIFO until its phase's inputs are ready
      int pend_s[STAGES], pend_ph[STAGES], pend_n[STAGES], pend_kb[STAGES];
      int ph_head = 0, ph_tail = 0;
      int ready = -1;   // highest phase whose inputs are known ready
      auto flush = [&](bool block) {
        while (ph_head != ph_tail) {
          const int k = ph_head % STAGES;
          const int q = pend_ph[k];
          if (q > ready) {
            if (!block) return;
            inputs_ready(q);
            ready = q;
          }
          tma_load_2d(sB + pend_s[k] * B_BYTES, tms[q], &full[pend_s[k]], pend_kb[k] * BK, pend_n[k] * BN);
          ++ph_head;
        }
      };
      uint32_t g = 0;
      while (it.next(u, &ph)) {
        const ChainPhase& P = ca.ph[ph];
        for (int kb = u.kb0; kb < u.kb1; ++kb, ++g) {
          const uint32_t s = g % STAGES;
          const uint32_t par = (g / STAGES) & 1;
          if (g >= STAGES) {
            // a stage is reused only after the MMA consumed it, which needs
            // its activation: queued loads of older stages go out first
            if (ph_tail - ph_head == STAGES) flush(true);
            mbar_wait(&empty[s], par ^ 1);
          }
          mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
          bulk_load(sA + s * A_BYTES, P.Wb + ((int64_t)u.m * P.w.nkb + kb) * BLK_ELEMS, A_BYTES, &full[s]);
          if (ph <= ready && ph_head == ph_tail) {
            tma_load_2d(sB + s * B_BYTES, tms[ph], &full[s], kb * BK, u.n * BN);
          } else {
            const int k = ph_tail % STAGES;
            pend_s[k] = s, pend_ph[k] = ph, pend_n[k] = u.n, pend_kb[k] = kb;
            ++ph_tail;
            flush(false);
          }
        }
      }
      flush(true);
      chain_mark(13);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      uint32_t g = 0, ui = 0;
      int last_ph = -1;
      while (it.next(u, &ph)) {
        const uint32_t a2 = ui & 1;
        if (ui >= 2) mbar_wait(&tempty[a2], ((ui >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem + a2 * BN;
        for (int kb = u.kb0; kb < u.kb1; ++kb, ++g) {
          const uint32_t s = g % STAGES;
          mbar_wait(&full[s], (g / STAGES) & 1);
          tc_fence_after();
          if (ph != last_ph) {
            if (last_ph >= 0) chain_mark(20 + last_ph);
            chain_mark(16 + ph);
            last_ph = ph;
          }
          const uint32_t a_base = smem_u32(sA + s * A_BYTES);
          const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(dtm, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                      (kb != u.kb0 || k) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[a2]);
        ++ui;
      }
      if (last_ph >= 0) chain_mark(20 + last_ph);
    }
  } else if (warp >= 4) {
    const int q4 = warp & 3;
    constexpr int PARTS = EPI_WARPS / 4;
    const int part = (warp - 4) >> 2;
    const int c_lo = part * (BN / PARTS), c_hi = c_lo + BN / PARTS;
    const int et = threadIdx.x - 128;      // 0..255 within the epilogue group
    const int r = q4 * 32 + lane;
    griddep_wait();   // outputs / residual may still be in use by the previous kernel
    uint32_t ui = 0;
    int cur = -1;     // phase whose units this group is storing
    // end of phase q for this CTA: publish, then the LayerNorm rows of this CTA
    auto finish_phase = [&](int q) {
      __threadfence();
      epi_bar();
      if (et == 0) red_release_add(&done[q], 1u);
      if (et == 0) chain_mark(5 + q);
      const int li = ca.ph[q].ln_after;
      if (li < 0) {
        // every counter advances by one per CTA per launch (targets grid x epoch)
        if (et == 0) red_release_add(&ln_done[q], 1u);
        return;
      }
      // LayerNorm of x into h (rows blockIdx.x, +G, ..): the arithmetic of
      // norm_reg_kernel (256 threads, fp32 statistics, two block sums)
      if (et == 0) wait_counter(&done[q], G * ca.epoch);
      epi_bar();
      const int rows = ca.ph[q].ep.tokens;
      const int d = ca.d, n4 = d >> 2;
      const int nv = (n4 + 255) / 256;
      for (int row = blockIdx.x; row < rows; row += G) {
        const float4* xr = reinterpret_cast<const float4*>(ca.x + (int64_t)row * d);
        float4 v[16];
        float sm = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (k >= nv) break;
          const int i = et + k * 256;
          v[k] = i < n4 ? __ldcg(xr + i) : make_float4(0.f, 0.f, 0.f, 0.f);
          sm += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        }
        auto block_sum = [&](float val) {
          val = warp_sum(val);
          epi_bar();
          if (lane == 0) red[et >> 5] = val;
          epi_bar();
          float t = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < 8; ++w2) t += red[w2];
          return t;
        };
        const float mean = block_sum(sm) / (float)d;
        float qq = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (k >= nv) break;
          if (et + k * 256 >= n4) continue;
          const float a0 = v[k].x - mean, b0 = v[k].y - mean, c0 = v[k].z - mean, e0 = v[k].w - mean;
          qq += (a0 * a0 + b0 * b0) + (c0 * c0 + e0 * e0);
        }
        const float rstd = rsqrtf(block_sum(qq) / (float)d + ca.eps);
        bf16* yr = ca.h + (int64_t)row * d;
        const ChainLN& L = ca.ln[li];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (k >= nv) break;
          const int i = et + k * 256;
          if (i >= n4) continue;
          const uint2 gr = reinterpret_cast<const uint2*>(L.g)[i];
          const float2 g01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gr.x));
          const float2 g23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gr.y));
          const uint2 br = reinterpret_cast<const uint2*>(L.b)[i];
          const float2 b01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.x));
          const float2 b23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.y));
          const float o0 = (v[k].x - mean) * rstd * g01.x + b01.x;
          const float o1 = (v[k].y - mean) * rstd * g01.y + b01.y;
          const float o2 = (v[k].z - mean) * rstd * g23.x + b23.x;
          const float o3 = (v[k].w - mean) * rstd * g23.y + b23.y;
          __nv_bfloat162 p0 = __floats2bfloat162_rn(o0, o1), p1 = __floats2bfloat162_rn(o2, o3);
          uint2 outv;
          outv.x = *reinterpret_cast<uint32_t*>(&p0);
          outv.y = *reinterpret_cast<uint32_t*>(&p1);
          reinterpret_cast<uint2*>(yr)[i] = outv;
        }
      }
      __threadfence();
      epi_bar();
      if (et == 0) red_release_add(&ln_done[q], 1u);
      if (et == 0) chain_mark(9 + q);
    };
    while (it.next(u, &ph)) {
      while (cur < ph) {   // phases before this unit's are complete on this CTA
        if (cur >= 0) finish_phase(cur);
        ++cur;
      }
      const ChainPhase& P = ca.ph[ph];
      const EpiParams& ep = P.ep;
      const uint32_t a2 = ui & 1;
      mbar_wait(&tfull[a2], (ui >> 1) & 1);
      tc_fence_after();
      const int gm = u.m * BM + r;
      const uint32_t taddr = tmem + ((uint32_t)(q4 * 32) << 16) + a2 * BN;
      const bool row_ok = gm < P.M;
      if (!u.full) {
        float* pp = P.partial + (((int64_t)u.n * P.w.tiles_m + u.m) * P.w.max_segs + u.seg) * (int64_t)(BM * BN);
        for (int c = c_lo; c < c_hi; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) pp[(int64_t)(c + j) * BM + r] = v[j];
        }
      } else {
        for (int c = c_lo; c < c_hi; c += 16) {
          float v[16];
          tmem_ld16(taddr + c, v);
          if (row_ok && u.n * BN + c < P.N) epi_store_col16(ep, u.n * BN + c, gm, P.N, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a2]);
      ++ui;
      if (!u.full) {
        // stream-K fixup: the CTA completing the tile's last segment reduces
        const int64_t x0 = (int64_t)u.m * P.w.nkb;
        const int nseg = sk_owner(P.w, x0 + P.w.nkb - 1) - sk_owner(P.w, x0) + 1;
        int* cnt = P.counters + (u.n * P.w.tiles_m + u.m);
        __threadfence();
        epi_bar();
        if (et == 0) *s_last = (atomicAdd(cnt, 1) == nseg - 1);
        epi_bar();
        if (*s_last) {
          __threadfence();
          const float* base = P.partial + ((int64_t)u.n * P.w.tiles_m + u.m) * P.w.max_segs * (int64_t)(BM * BN);
          for (int c0 = c_lo; c0 < c_hi; c0 += 16) {
            float acc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = 0.f;
            for (int s0 = 0; s0 < nseg; s0 += 4) {
              float v[4][16];
#pragma unroll
              for (int qv = 0; qv < 4; ++qv) {
                const float* src = base + (int64_t)(s0 + qv) * BM * BN + (int64_t)c0 * BM + r;
#pragma unroll
                for (int j = 0; j < 16; ++j) v[qv][j] = (s0 + qv < nseg) ? __ldcg(src + (int64_t)j * BM) : 0.f;
              }
#pragma unroll
              for (int qv = 0; qv < 4; ++qv)
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  if (s0 + qv < nseg) acc[j] += v[qv][j];
            }
            if (!row_ok) continue;
            if (u.n * BN + c0 < P.N) epi_store_col16(ep, u.n * BN + c0, gm, P.N, acc);
          }
          if (et == 0) *cnt = 0;
        }
        epi_bar();
      }
    }
    // the remaining phases (including ones with no units on this CTA)
    while (cur < ca.n) {
      if (cur >= 0) finish_phase(cur);
      ++cur;
    }
    if (et == 0) chain_mark(14);
    // counters of the phases this launch does not have
    if (et == 0)
      for (int q = ca.n; q < CHAIN_MAX; ++q) {
        red_release_add(&done[q], 1u);
        red_release_add(&ln_done[q], 1u);
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, TMEM_COLS);
  }
}

// Ring depth: up to 8 stages within ~200 KB (one CTA per SM).  Measured: a
// half-SM ring (2 CTAs/SM so the next GEMM co-resides under PDL) loses more
// weight-stream depth than the overlap gains.
template <int BN, int SWAP>
constexpr int stages_for() {
  constexpr int budget = 200 * 1024;
  constexpr int per = BN * BK * 2 + A_BYTES;
  return budget / per > 8 ? 8 : budget / per;
}

template <int BN, int SWAP>
size_t smem_bytes() {
  constexpr int S = stages_for<BN, SWAP>();
  return 1024 + (size_t)S * (A_BYTES + BN * BK * 2) + (2 * S + 4) * 8 + 16;
}

Work make_work(int M, int N, int K, int BN, bool streamk) {
  Work w;
  w.tiles_m = (M + BM - 1) / BM;
  w.tiles_n = (N + BN - 1) / BN;
  w.nkb = (K + BK - 1) / BK;
  w.I = (int64_t)w.tiles_m * w.nkb;
  // raster group: m-tiles whose A slab is ~32 MB (kept L2-resident)
  w.gm = (int)std::max<int64_t>(1, std::min<int64_t>(w.tiles_m, (gemm_slab_mb() << 20) / ((int64_t)BM * K * 2)));
  const int sms = num_sms();
  if (streamk) {
    w.dp = 0;
    const int cap = gemm_sk_ctas() > 0 ? std::min(gemm_sk_ctas(), sms) : sms;
    w.G = (int)std::min<int64_t>(cap, w.I);
    const int64_t per = w.I / w.G;  // >= 1
    w.max_segs = (int)((w.nkb + per - 1) / per) + 2;
  } else {
    w.dp = 1;
    w.G = std::min(sms, w.tiles_m * w.tiles_n);
    w.max_segs = 1;
  }
  return w;
}

// Grid-wide stream-K reduction: block (tile, 32-column slice), thread = row;
// segments summed in segment order (same arithmetic as the in-kernel fixup).
template <int BN, int SWAP>
__global__ void __launch_bounds__(128) streamk_reduce_kernel(const float* __restrict__ partial, int M, int N, Work w,
                                                             EpiParams ep) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  const int tile = blockIdx.x, m = tile % w.tiles_m, n = tile / w.tiles_m;
  const int64_t x0 = (int64_t)m * w.nkb;
  const int nseg = sk_owner(w, x0 + w.nkb - 1) - sk_owner(w, x0) + 1;
  if (nseg <= 1) return;  // whole tile: stored by its CTA
  const int r = threadIdx.x, gm = m * BM + r;
  const float* base = partial + ((int64_t)n * w.tiles_m + m) * w.max_segs * (int64_t)(BM * BN);
  for (int c0 = blockIdx.y * 32; c0 < blockIdx.y * 32 + 32; c0 += 16) {
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.f;
    for (int s0 = 0; s0 < nseg; s0 += 4) {   // up to 4 segments' loads in flight
      float v[4][16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* src = base + (int64_t)(s0 + q) * BM * BN + (int64_t)c0 * BM + r;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[q][j] = (s0 + q < nseg) ? __ldcg(src + (int64_t)j * BM) : 0.f;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (s0 + q < nseg) acc[j] += v[q][j];
    }
    if (gm >= M) continue;
    if (SWAP) {
      if (n * BN + c0 < N) epi_store_col16(ep, n * BN + c0, gm, N, acc);
    } else {
      epi_store_row16(ep, gm, n * BN + c0, N, acc);
    }
  }
}

// Workspace layout: [fixup counters: CNT_CAP ints][partial segments].  The
// counter region sits at a fixed offset for every shape and token tile so
// the zero state each fixup leaves behind is where the next launch looks.
constexpr size_t CNT_CAP = 16384;
size_t ws_need(const Work& w, int BN) {
  const size_t parts = (size_t)w.tiles_n * w.tiles_m * w.max_segs * BM * BN;
  return CNT_CAP + parts;
}

template <int BN, int SWAP>
void launch(const CUtensorMap& tx, const bf16* Wb, int M, int N, int K, int n_wblk, const EpiParams& ep, float* ws,
            size_t ws_floats, cudaStream_t st) {
  constexpr int S = stages_for<BN, SWAP>();
  static bool attr_set = false;
  const size_t smem = smem_bytes<BN, SWAP>();
  if (!attr_set) {
    EXG_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, S, SWAP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    attr_set = true;
  }
  Work w = make_work(M, N, K, BN, SWAP != 0);
  float* partial = nullptr;
  int* counters = nullptr;
  if (SWAP) {
    const size_t need = ws_need(w, BN);
    if (!ws || need > ws_floats) throw CudaError("stream-K workspace too small");
    if ((size_t)w.tiles_n * w.tiles_m > CNT_CAP) throw CudaError("stream-K: too many tiles for the counter region");
    counters = reinterpret_cast<int*>(ws);
    partial = ws + CNT_CAP;
  }
  // small token tiles: the last CTA of a split tile reduces in-kernel; wide
  // tiles (>= 128 columns): a grid-wide reduce kernel spreads the segment sums
  // over all SMs instead of serialising a whole tile on one CTA's tail
  const bool inkernel = BN < 128;
  // programmatic dependent launch: the kernel may start while the previous
  // one drains; it prefetches weights, then griddepcontrol.wait()s
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(w.G);
  cfg.blockDim = dim3(EpiCfg<SWAP>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  EXG_CUDA(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, S, SWAP>, tx, Wb, M, N, n_wblk, w, ep, partial, counters,
                              inkernel ? 1 : 0, gemm_dbg_arg(SWAP)));
  EXG_CHECK_LAUNCH();
  if (SWAP && !inkernel && !ep.defer_out) {
    dim3 grid(w.tiles_m * w.tiles_n, BN / 32);
    launch_pdl(streamk_reduce_kernel<BN, SWAP>, dim3(grid), dim3(128), 0, st, partial, M, N, w, ep);
    EXG_CHECK_LAUNCH();
  }
}

// ============================================================================
// Prefill GEMM on CTA pairs (tcgen05 cta_group::2).  A cluster of two CTAs on
// one TPC computes a 256-token x 256-feature tile with one M=256 N=256 MMA
// per 16-wide K step issued by the leader CTA: each CTA stages its own 128
// tokens of A and its own 128 features of W per 64-wide k-block (32 KB per
// stage instead of the 48 KB a 1-CTA 128x256 tile needs, so the per-SM L2 ->
// shared-memory stream drops by a third), and each holds its 128 rows x 256
// columns of the fp32 accumulator in its own TMEM (double-buffered, 512
// columns).  Both CTAs' TMA loads complete on the leader's `full` barrier; the
// leader's commits arrive on both CTAs' `empty` / `tfull` barriers
// (multicast); both CTAs' epilogue warps release a TMEM buffer on the
// leader's `tempty`.  Weights stream as verbatim 16 KB blocks of the blocked
// layout (a 2-D TMA box of 128 rows x 128 B, no swizzle: the block already
// is the SWIZZLE_128B shared-memory image).  Per output element the K loop,
// MMA K steps and epilogue are those of the 1-CTA kernel.
// ============================================================================
constexpr int P2_STAGES = 6;
// shared::cluster address of this shared variable's copy in the leader CTA (rank 0)
__device__ __forceinline__ uint32_t leader_addr(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(p)));
  return r;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const CUtensorMap* tmap, uint64_t* bar, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(leader_addr(bar))
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this offset in both CTAs once the issued MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(leader_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  const long long t0 = clock64();
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (clock64() - t0 > 8000000000LL) {
      printf("exg: pair mbarrier wait timeout block %d thread %d\n", blockIdx.x, threadIdx.x);
      __trap();
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(EpiCfg<0>::THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, int M, int N,
                     int nkb, int tiles_m, int tiles_n, int gm_group, EpiParams ep) {
  constexpr int EPI_WARPS = EpiCfg<0>::WARPS;
  constexpr int TN = 256;                     // features per pair tile (= tokens per pair tile)
  constexpr int HALF = 16384;                 // one CTA's A or B share of a k-block
  constexpr uint32_t TMEM_COLS = 512;
  griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + P2_STAGES * HALF;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + P2_STAGES * HALF);
  uint64_t* empty = full + P2_STAGES;
  uint64_t* tfull = empty + P2_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t rank = cluster_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    for (int s = 0; s < P2_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();      // the CTA's own view of the allocation (racecheck does not model barrier.cluster)
  cluster_sync_all();   // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  const int tiles = tiles_m * tiles_n;
  auto tile_mn = [&](int t, int& m, int& n) {
    // grouped raster: gm_group m-tiles (an L2-resident slab of A) sweep all n-tiles
    const int per_group = gm_group * tiles_n;
    const int g = t / per_group, within = t % per_group;
    const int gm_count = min(gm_group, tiles_m - g * gm_group);
    m = g * gm_group + within % gm_count;
    n = within / gm_count;
  };

  if (warp == 0) {
    if (lane == 0) {
      griddep_wait();   // activations are the previous kernel's output
      uint32_t g = 0;
      for (int t = cid; t < tiles; t += ncl) {
        int m, n;
        tile_mn(t, m, n);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const uint32_t s = g % P2_STAGES;
          const uint32_t ph = (g / P2_STAGES) & 1;
          if (g >= P2_STAGES) mbar_wait(&empty[s], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 4 * HALF);
          tma_load_2d_pair(sA + s * HALF, &tmX, &full[s], kb * BK, m * TN + (int)rank * BM);
          tma_load_2d_pair(sB + s * HALF, &tmW, &full[s], 0, ((n * 2 + (int)rank) * nkb + kb) * BM);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * BM, TN);
      uint32_t g = 0, ui = 0;
      for (int t = cid; t < tiles; t += ncl, ++ui) {
        const uint32_t a = ui & 1;
        if (ui >= 2) mbar_wait_cluster(&tempty[a], ((ui >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + a * TN;
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const uint32_t s = g % P2_STAGES;
          mbar_wait(&full[s], (g / P2_STAGES) & 1);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + s * HALF), b_base = smem_u32(sB + s * HALF);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16_pair(d, umma_desc_sw128(a_base + k * 32), umma_desc_sw128(b_base + k * 32), idesc,
                           (kb || k) ? 1u : 0u);
          umma_commit_pair(&empty[s]);
        }
        umma_commit_pair(&tfull[a]);
      }
    }
  } else if (warp >= 4) {
    // warp w reads TMEM lanes 32*(w%4).. and one half of the 256 columns
    const int q = warp & 3;
    const int part = (warp - 4) >> 2;
    const int c_lo = part * (TN / 2), c_hi = c_lo + TN / 2;
    griddep_wait();   // outputs / residual may still be in use by the previous kernel
    const int r = q * 32 + lane;
    uint32_t ui = 0;
    for (int t = cid; t < tiles; t += ncl, ++ui) {
      int m, n;
      tile_mn(t, m, n);
      const uint32_t a = ui & 1;
      mbar_wait(&tfull[a], (ui >> 1) & 1);
      tc_fence_after();
      const int gm = m * TN + (int)rank * BM + r;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + a * TN;
      for (int c = c_lo; c < c_hi; c += 16) {
        float v[16];
        tmem_ld16(taddr + c, v);
        if (gm < M && n * TN + c < N) epi_store_row16(ep, gm, n * TN + c, N, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(&tempty[a]);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();   // both CTAs done with TMEM and with each other's shared memory
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

constexpr size_t P2_SMEM = 1024 + (size_t)P2_STAGES * 2 * 16384 + (2 * P2_STAGES + 4) * 8 + 16;

// weights (blocked layout) as a 2-D tensor of 128-byte rows: block (nb, kb) is
// rows [(nb*nkb + kb)*128, +128), copied verbatim (no swizzle)
CUtensorMap make_tmap_blocked(const bf16* Wb, int64_t n_wblk, int64_t nkb) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)BK, (cuuint64_t)(n_wblk * nkb * BM)};
  cuuint64_t strides[1] = {(cuuint64_t)BK * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<bf16*>(Wb), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (blocked weights) failed " + std::to_string((int)r));
  return m;
}

void launch_pair(const CUtensorMap& tx, const bf16* Wb, int M, int N, int K, int n_wblk, const EpiParams& ep,
                 cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    EXG_CUDA(cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P2_SMEM));
    attr_set = true;
  }
  const int nkb = (K + BK - 1) / BK;
  const int tiles_m = (M + 255) / 256, tiles_n = (N + 255) / 256;
  const int gm = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_m, (gemm_slab_mb() << 20) / ((int64_t)256 * K * 2)));
  const int clusters = std::min(num_sms() / 2, tiles_m * tiles_n);
  const CUtensorMap tw = make_tmap_blocked(Wb, n_wblk, nkb);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters);
  cfg.blockDim = dim3(EpiCfg<0>::THREADS);
  cfg.dynamicSmemBytes = P2_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  EXG_CUDA(cudaLaunchKernelEx(&cfg, gemm_pair_kernel, tx, tw, M, N, nkb, tiles_m, tiles_n, gm, ep));
  EXG_CHECK_LAUNCH();
}

__global__ void pack_blocked_kernel(bf16* __restrict__ dst, const bf16* __restrict__ src, int64_t rows, int64_t K,
                                    int64_t ld) {
  const int64_t rp = (rows + 127) / 128 * 128, kp = (K + 63) / 64 * 64;
  const int64_t n = rp * kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / kp, k = e % kp;
    dst[blocked_index(r, k, K)] = (r < rows && k < K) ? src[r * ld + k] : __float2bfloat16_rn(0.f);
  }
}
}  // namespace

void pack_blocked(bf16* dst, const bf16* src, int64_t rows, int64_t K, int64_t ld, cudaStream_t st) {
  const int64_t n = blocked_elems(rows, K);
  pack_blocked_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(dst, src, rows, K, ld);
  EXG_CHECK_LAUNCH();
}

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

// off by default: measured on OPT-13B task S (tools/ab_deferred.py, mode 10)
// the chain is slower than PDL-chained separate launches (decode phase 3.65 vs
// 2.99 s): a one-phase chain launch is ~7 us slower than exg_op_linear and a
// phase boundary costs as much as a kernel boundary (the fixup tail and the
// grid-wide readiness wait are still serial); kept as an option
bool& chain_enabled() {
  static bool on = false;
  return on;
}

int& deferred_enabled() {
  static int on = DEFER_DEFAULT;
  return on;
}

SegInfo decode_seg_info(int features, int K) {
  const Work w = make_work(features, 1, K, 32, true);   // the cut does not depend on tokens / BN
  SegInfo s;
  s.nkb = w.nkb;
  s.G = w.G;
  s.I = w.I;
  return s;
}

size_t deferred_floats(int features, int K, int tokens) {
  const Work w = make_work(features, 1, K, 32, true);
  return (size_t)(w.max_segs) * tokens * features;
}

int decode_bn(int tokens) {
  if (tokens <= 32) return 32;
  if (tokens <= 64) return 64;
  if (tokens <= 128) return 128;
  return 256;
}

size_t decode_ws_floats(int features, int K, int max_tokens) {
  size_t best = 0;
  for (int bn : {32, 64, 128, 256}) {
    const int n = bn == 256 ? std::max(max_tokens, 1) : bn;
    best = std::max(best, ws_need(make_work(features, n, K, bn, true), bn));
  }
  return best;
}

void linear(const LinearArgs& a, cudaStream_t st) {
  const int tokens = a.ep.tokens, features = a.ep.features;
  if (tokens <= 0 || features <= 0) return;
  const int n_wblk = (features + BM - 1) / BM;
  if (a.decode) {
    const int BN = a.bn ? a.bn : decode_bn(tokens);
    const CUtensorMap tx = make_tmap_bf16(a.X, tokens, a.K, a.ldx, BN);
    switch (BN) {
      case 32: launch<32, 1>(tx, a.Wb, features, tokens, a.K, n_wblk, a.ep, a.ws, a.ws_floats, st); break;
      case 64: launch<64, 1>(tx, a.Wb, features, tokens, a.K, n_wblk, a.ep, a.ws, a.ws_floats, st); break;
      case 128: launch<128, 1>(tx, a.Wb, features, tokens, a.K, n_wblk, a.ep, a.ws, a.ws_floats, st); break;
      case 256: launch<256, 1>(tx, a.Wb, features, tokens, a.K, n_wblk, a.ep, a.ws, a.ws_floats, st); break;
      default: throw CudaError("bad BN");
    }
  } else {
    const int BN = a.bn ? a.bn : (features > 128 ? 256 : (features > 64 ? 128 : 64));
    const CUtensorMap tx = make_tmap_bf16(a.X, tokens, a.K, a.ldx, BM);
    // CTA pairs (cta_group::2) for the wide prefill GEMMs; diagnostics flag
    // bit 6 forces the 1-CTA kernel
    if (BN == 256 && !(gemm_debug_flags() & 64)) {
      launch_pair(tx, a.Wb, tokens, features, a.K, n_wblk, a.ep, st);
      return;
    }
    switch (BN) {
      case 64: launch<64, 0>(tx, a.Wb, tokens, features, a.K, n_wblk, a.ep, nullptr, 0, st); break;
      case 128: launch<128, 0>(tx, a.Wb, tokens, features, a.K, n_wblk, a.ep, nullptr, 0, st); break;
      case 256: launch<256, 0>(tx, a.Wb, tokens, features, a.K, n_wblk, a.ep, nullptr, 0, st); break;
      default: throw CudaError("bad BN");
    }
  }
}

// chain workspace: [CHAIN_MAX counter regions of CNT_CAP ints][partials of
// phase 0][partials of phase 1]..  The counter regions sit at fixed offsets
// for every token tile (the partials' layout changes with BN), so the zero
// state the fixups leave behind is where the next launch looks
size_t chain_ws_floats(const ChainSpec& c) {
  const int BN = decode_bn(c.tokens);
  size_t total = (size_t)CHAIN_MAX * CNT_CAP;
  for (int q = 0; q < c.n; ++q)
    total += ws_need(make_work(c.ph[q].features, c.tokens, c.ph[q].K, BN, true), BN) - CNT_CAP;
  return total;
}

namespace {
template <int BN>
void launch_chain(const ChainSpec& c, cudaStream_t st) {
  constexpr int S = stages_for<BN, 1>();
  const size_t smem = smem_bytes<BN, 1>() + 64;
  static bool attr_set = false;
  if (!attr_set) {
    EXG_CUDA(cudaFuncSetAttribute(decode_chain_kernel<BN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = true;
  }
  ChainArgs a = {};
  a.n = c.n;
  CUtensorMap tm[CHAIN_MAX];
  float* ws = c.ws;
  size_t used = (size_t)CHAIN_MAX * CNT_CAP;
  for (int q = 0; q < CHAIN_MAX; ++q) {
    const int qq = q < c.n ? q : c.n - 1;   // unused maps: any valid one
    tm[q] = make_tmap_bf16(c.ph[qq].X, c.tokens, c.ph[qq].K, c.ph[qq].ldx, BN);
  }
  for (int q = 0; q < c.n; ++q) {
    ChainPhase& P = a.ph[q];
    P.Wb = c.ph[q].Wb;
    P.M = c.ph[q].features;
    P.N = c.tokens;
    P.n_wblk = (P.M + BM - 1) / BM;
    P.w = make_work(P.M, c.tokens, c.ph[q].K, BN, true);
    P.ep = c.ph[q].ep;
    P.ep.tokens = c.tokens;
    P.ep.features = P.M;
    P.ln_after = c.ph[q].ln_after;
    const size_t need = ws_need(P.w, BN) - CNT_CAP;   // partials
    if ((size_t)P.w.tiles_n * P.w.tiles_m > CNT_CAP) throw CudaError("decode chain: too many tiles for the counter region");
    if (used + need > c.ws_floats) throw CudaError("decode chain workspace too small");
    P.counters = reinterpret_cast<int*>(ws + (size_t)q * CNT_CAP);
    P.partial = ws + used;
    used += need;
  }
  for (int i = 0; i < 2; ++i) a.ln[i] = ChainLN{c.ln_g[i], c.ln_b[i]};
  a.x = c.x;
  a.h = c.h;
  a.d = c.d;
  a.eps = c.eps;
  a.sync = c.sync;
  a.epoch = c.epoch;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(num_sms());
  cfg.blockDim = dim3(EpiCfg<1>::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  EXG_CUDA(cudaLaunchKernelEx(&cfg, decode_chain_kernel<BN, S>, tm[0], tm[1], tm[2], tm[3], a));
  EXG_CHECK_LAUNCH();
}
}  // namespace

void decode_chain(const ChainSpec& c, cudaStream_t st) {
  if (c.n < 1 || c.n > CHAIN_MAX) throw CudaError("decode chain: 1..4 phases");
  if (c.tokens <= 0) return;
  if ((c.d & 3) || c.d > 16384) throw CudaError("decode chain: LayerNorm width");
  switch (decode_bn(c.tokens)) {
    case 32: launch_chain<32>(c, st); break;
    case 64: launch_chain<64>(c, st); break;
    case 128: launch_chain<128>(c, st); break;
    default: launch_chain<256>(c, st); break;
  }
}

}  // namespace exg

extern "C" void exg_diag_gemm_flags(int flags) { exg::gemm_debug_flags() = flags; }
// one-phase chain (EPI_BF16, no bias) for A/B against exg_op_linear
extern "C" int exg_diag_chain_gemm(const void* X, int64_t ldx, const void* Wb, int tokens, int features, int K,
                                   void* out, int64_t ldo, float* ws, int64_t ws_floats, unsigned* sync,
                                   unsigned epoch, int n_rep, void* stream) {
  try {
    exg::ChainSpec c;
    c.n = std::max(1, std::min(4, n_rep));
    for (int q = 0; q < c.n; ++q) {
      c.ph[q].X = (const exg::bf16*)X;
      c.ph[q].ldx = ldx;
      c.ph[q].Wb = (const exg::bf16*)Wb;
      c.ph[q].features = features;
      c.ph[q].K = K;
      c.ph[q].ep.mode = exg::EPI_BF16;
      c.ph[q].ep.out_bf16 = (exg::bf16*)out;
      c.ph[q].ep.ldo = ldo;
    }
    c.tokens = tokens;
    c.d = 4;
    c.ws = ws;
    c.ws_floats = (size_t)ws_floats;
    c.sync = sync;
    c.epoch = epoch;
    if (!ws) return (int)exg::chain_ws_floats(c);
    exg::decode_chain(c, (cudaStream_t)stream);
    return 0;
  } catch (...) {
    return -1;
  }
}

extern "C" int exg_diag_chain_timeline(int on, unsigned long long* out) {
  if (on >= 0) cudaMemcpyToSymbol(exg::g_chain_tl_on, &on, sizeof(int));
  if (out) return cudaMemcpyFromSymbol(out, exg::g_chain_tl, sizeof(unsigned long long) * 256 * 32) == cudaSuccess ? 0 : 1;
  return 0;
}
// decode GEMM chain for engines created after the call (1 = on; 0 = separate launches, default)
extern "C" void exg_diag_chain(int on) { exg::chain_enabled() = on != 0; }
// deferred stream-K reductions for engines created after the call: bit 0 =
// QKV (summed by the decode attention), bit 1 = O-projection / FFN2 (summed by
// the following LayerNorm); -1 restores the default
extern "C" void exg_diag_deferred(int mask) { exg::deferred_enabled() = mask < 0 ? exg::DEFER_DEFAULT : mask; }
extern "C" void exg_diag_gemm_sk_ctas(int n) { exg::gemm_sk_ctas() = n; }
extern "C" void exg_diag_gemm_slab_mb(int mb) { exg::gemm_slab_mb() = mb; }
// span recording: reset clears the arrays and the launch counter; read copies
// min(n, 4096) spans (ns) and returns the number of launches recorded
extern "C" int exg_diag_gemm_spans_reset() {
  std::vector<unsigned long long> lo(4096, ~0ull), hi(4096, 0ull);
  exg::gemm_span_seq() = 0;
  if (cudaMemcpyToSymbol(exg::g_span_start, lo.data(), sizeof(unsigned long long) * 4096) != cudaSuccess) return 1;
  if (cudaMemcpyToSymbol(exg::g_span_dep, lo.data(), sizeof(unsigned long long) * 4096) != cudaSuccess) return 1;
  return cudaMemcpyToSymbol(exg::g_span_end, hi.data(), sizeof(unsigned long long) * 4096) == cudaSuccess ? 0 : 1;
}
extern "C" int exg_diag_gemm_spans(unsigned long long* start, unsigned long long* end, unsigned long long* dep) {
  cudaMemcpyFromSymbol(dep, exg::g_span_dep, sizeof(unsigned long long) * 4096);
  cudaMemcpyFromSymbol(start, exg::g_span_start, sizeof(unsigned long long) * 4096);
  cudaMemcpyFromSymbol(end, exg::g_span_end, sizeof(unsigned long long) * 4096);
  return exg::gemm_span_seq();
}
// per-CTA timeline marks of the last GEMM run with flag bit 2 ([256][8] ns)
extern "C" int exg_diag_gemm_timeline(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, exg::g_gemm_tl, sizeof(unsigned long long) * 256 * 8) == cudaSuccess ? 0 : 1;
}
