// K4 prefill attention on the 5th-gen tensor cores (dh = 128).
//
// Persistent: one CTA per SM walks the work items (128 queries of one
// (request, head)) -- longest causal items first, item id strided by the grid
// -- so TMEM allocation, barrier set-up and the first Q / K / V loads of an
// item overlap the previous item's softmax and P.V.  Per 128-key tile j:
//   S_j = Q . K_j^T        tcgen05.mma kind::f16, M=128 N=128 K=128, fp32 in TMEM
//   P_j = exp(s - m_j)     8 softmax warps: one query row per thread pair, each
//                          thread of the pair exponentiates one 64-key half of
//                          the tile (both take the row max over all 128 keys,
//                          so no exchange per tile); online max / half sums;
//                          P_j -> TMEM as bf16, over S_j's own buffer
//   O  += P_j . V_j        tcgen05.mma, A = P read from TMEM, B = V (MN-major),
//                          fp32, accumulated in TMEM across the item's tiles
//                          (a shared-memory P variant stays for A/B)
// Lazy rescaling: P_j is exponentiated against the row's running reference
// max m_ref, which moves (and O in TMEM is rescaled by the softmax warps) only
// when a tile's max exceeds it by more than 8 in log2 units -- so p <= 2^8 and
// the fp32 O / row sums stay far from overflow; mathematically the same
// softmax (the final 1/l uses the same reference).  About a quarter of the
// exponentials run as a degree-3 polynomial on the FMA pipe (relative error
// 1.9e-4, far below P's bf16 rounding) beside the SFU ex2.
// S is double-buffered in TMEM (2 x 128 columns) so the softmax of tile j+1
// overlaps the P.V of tile j; Q is double-buffered in shared memory so the
// next item's Q lands while the current one finishes.  Buffer indices and
// mbarrier phases run on per-CTA counters across items.  Q, K, V arrive by
// 2-D TMA (SWIZZLE_128B) straight from the packed qkv buffer and the KV cache.
// Scores follow T4(e): fp32(q.k) * fp32(scale); P is rounded to bf16 for the
// P.V MMA.  The arithmetic per query row is the same as a
// one-item-per-CTA launch: results do not depend on the item order.
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace exg {

namespace {
int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    EXG_CUDA(cudaGetDevice(&dev));
    EXG_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

constexpr int FQ = 128;          // queries per CTA
constexpr int FK = 128;          // keys per tile
constexpr int FD = 128;          // head dim
constexpr int TILE_BYTES = 128 * 64 * 2;            // one 128-row x 64-col SW128 box
constexpr int Q_BYTES = 2 * TILE_BYTES;             // [128][128]
constexpr int KV_BYTES = 2 * TILE_BYTES;            // K or V tile
constexpr int P_BYTES = 2 * TILE_BYTES;
constexpr int KV_STAGES = 2;
constexpr int Q_STAGES = 2;
constexpr int SM_WARPS = 8;      // softmax warps (two per TMEM lane quarter)
constexpr size_t FMHA_SMEM = 1024 + Q_STAGES * Q_BYTES + KV_STAGES * 2 * KV_BYTES + P_BYTES + 256 + 2 * FQ * 4;
static_assert(FMHA_SMEM <= 232448, "FMHA shared memory over the sm_100 per-CTA limit");

__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t smem_addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// 2^x on the SFU (flush-to-zero: a P below 2^-126 is 0 either way once
// rounded into the row sum)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe: Cody-Waite split x = i + f, f in [0, 1), degree-3
// polynomial for 2^f (max relative error 1.9e-4), i added to the exponent
// field; 0 below 2^-126 like ex2.approx.ftz
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float xi = floorf(x);
  const float f = x - xi;
  float p = fmaf(f, 0.07619732618331909f, 0.22820299863815308f);
  p = fmaf(p, f, 0.6952236294746399f);
  p = fmaf(p, f, 1.0f);
  const int e = (int)xi;
  return e < -126 ? 0.f : __int_as_float(__float_as_int(p) + (e << 23));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// O += P . V with P (the A operand) read from TMEM: 128 lanes = query rows,
// bf16 pairs packed per 32-bit column (K-major), B from shared memory
__device__ __forceinline__ void umma_bf16_tmem_a(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

struct FmhaParams {
  const int32_t* cu_seqlens;
  const int32_t* slot;
  const int32_t* pos0;
  int H, max_ctx, R, QT;   // QT = query tiles of the longest request
  float scale_log2;     // fp32(scale) * log2(e)
  float scale;
  bf16* out;
  int64_t ldo;
  int causal;
  const float* bias;    // T5 relative bias: score += bias[h * bias_ld + bias_off + kpos - qpos]
  int bias_ld, bias_off;
  KvMap kv;             // paged mode: page table of the requests
  int pf_ahead;         // L2 prefetch distance in items (0 = off)
};

// Work item `id` -> (request, head, query tile); false if the tile is past
// the request's length.  Query tiles are enumerated last-first (the causal
// cost of a tile grows with its index), so the grid stride deals the
// expensive items out first.
struct Item {
  int r, h, qb, t0, len, pos0, ntiles, slot, last_key;
};
__device__ __forceinline__ bool item_of(const FmhaParams& p, int id, Item& it) {
  const int rh = p.R * p.H;
  const int qt = p.QT - 1 - id / rh;
  const int rem = id % rh;
  it.r = rem / p.H;
  it.h = rem % p.H;
  it.t0 = p.cu_seqlens[it.r];
  it.len = p.cu_seqlens[it.r + 1] - it.t0;
  it.qb = qt * FQ;
  if (it.qb >= it.len) return false;
  it.pos0 = p.pos0[it.r];
  const int last_key = p.causal ? it.pos0 + min(it.len, it.qb + FQ) - 1 : it.pos0 + it.len - 1;  // inclusive
  it.ntiles = last_key / FK + 1;
  it.last_key = last_key;
  it.slot = p.slot[it.r];
  return true;
}

// PT: P kept in TMEM (written over its S buffer by the softmax warps, read by
// the P.V MMA as the A operand) instead of shared memory -- the softmax of
// tile j+1 then never waits for the P.V of tile j (only a lazy rescale of O
// does), and the P buffer's 32 KB of shared memory go unused
template <bool PT>
__global__ void __launch_bounds__(128 + 32 * SM_WARPS, 1) fmha_prefill_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                              const __grid_constant__ CUtensorMap tmK,
                                                              const __grid_constant__ CUtensorMap tmV,
                                                              FmhaParams p) {
  griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                               // [q stage]
  uint8_t* sK = sQ + Q_STAGES * Q_BYTES;            // [kv stage]
  uint8_t* sV = sK + KV_STAGES * KV_BYTES;          // [kv stage]
  uint8_t* sP = sV + KV_STAGES * KV_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + P_BYTES);
  uint64_t* q_full = bars;              // 2
  uint64_t* q_empty = bars + 2;         // 2
  uint64_t* kv_full = bars + 4;         // 2
  uint64_t* kv_empty = bars + 6;        // 2
  uint64_t* s_full = bars + 8;          // 2
  uint64_t* s_free = bars + 10;         // 2
  uint64_t* p_full = bars + 12;         // P of tile gj written: p_full[gj & 1] (slots 12 and 15)
  uint64_t* o_full = bars + 13;         // 2: P.V of a tile done (parity by tile)
  uint64_t* p_full1 = bars + 15;        // the second p_full (by tile parity; 16 unused)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 17);
  float* lx = reinterpret_cast<float*>(sP + P_BYTES + 256);   // [2][FQ] row-sum halves

  const int n_items = p.QT * p.R * p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], SM_WARPS);
      mbar_init(&o_full[i], 1);
      if (i == 0) mbar_init(p_full1, SM_WARPS);
    }
    mbar_init(p_full, SM_WARPS);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  // TMEM columns: S buffers at 0 / 128, O buffers at 256 / 384
  griddep_wait();  // launched with PDL: predecessors complete + visible

  if (warp == 0) {
    if (lane == 0) {
      // cache rows of the two 64-key halves of K/V tile j of an item (a half
      // entirely past the item's last key reads the first half's rows)
      auto kv_rows2 = [&](const Item& it, int j, int& row0, int& row1) {
        row0 = (int)kv_row(p.kv, it.r, it.slot, p.H, it.h, p.max_ctx, j * FK);
        const int k1 = j * FK + 64;
        row1 = k1 <= it.last_key ? (int)kv_row(p.kv, it.r, it.slot, p.H, it.h, p.max_ctx, k1) : row0;
      };
      // L2 prefetch of the items pf_ahead ahead of the one being loaded: at
      // task-S lengths the kernel is bound by HBM latency / bytes in flight
      // (DESIGN.md §6), the prefetch keeps more of them in flight than the
      // shared-memory stages can
      int pf_id = blockIdx.x, pf_n = 0;
      auto prefetch_upto = [&](int count) {
        while (pf_n < count && pf_id < n_items) {
          Item f;
          const int id = pf_id;
          pf_id += gridDim.x;
          if (!item_of(p, id, f)) continue;
          ++pf_n;
          tma_prefetch_2d(&tmQ, f.h * FD, f.t0 + f.qb);
          tma_prefetch_2d(&tmQ, f.h * FD + 64, f.t0 + f.qb);
          for (int j = 0; j < f.ntiles; ++j) {
            int r0, r1;
            kv_rows2(f, j, r0, r1);
            for (int hf = 0; hf < (r1 == r0 ? 1 : 2); ++hf) {
              const int row = hf ? r1 : r0;
              tma_prefetch_2d(&tmK, 0, row);
              tma_prefetch_2d(&tmK, 64, row);
              tma_prefetch_2d(&tmV, 0, row);
              tma_prefetch_2d(&tmV, 64, row);
            }
          }
        }
      };
      uint32_t nq = 0, g = 0;   // items loaded, K/V tiles loaded by this CTA
      for (int id = blockIdx.x; id < n_items; id += gridDim.x) {
        Item it;
        if (!item_of(p, id, it)) continue;
        if (p.pf_ahead > 0) {
          if (nq == 0) pf_n = 1, pf_id = id + gridDim.x;   // this item's loads are issued now
          prefetch_upto((int)nq + 1 + p.pf_ahead);
        }
        const int qs = nq & 1;
        if (nq >= Q_STAGES) mbar_wait(&q_empty[qs], ((nq >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qs], Q_BYTES);
        tma_load_2d(sQ + qs * Q_BYTES, &tmQ, &q_full[qs], it.h * FD, it.t0 + it.qb);
        tma_load_2d(sQ + qs * Q_BYTES + TILE_BYTES, &tmQ, &q_full[qs], it.h * FD + 64, it.t0 + it.qb);
        ++nq;
        for (int j = 0; j < it.ntiles; ++j, ++g) {
          const int s = g & 1;
          if (g >= KV_STAGES) mbar_wait(&kv_empty[s], ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&kv_full[s], 2 * KV_BYTES);
          // two 64-key halves (each inside one KV block: 64 | page length);
          // a half entirely past the item's last key is loaded from the
          // first half's rows (masked, finite)
          int row0, row1;
          kv_rows2(it, j, row0, row1);
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            const int row = hf ? row1 : row0;
            const uint32_t o = hf * (TILE_BYTES / 2);
            tma_load_2d(sK + s * KV_BYTES + o, &tmK, &kv_full[s], 0, row);
            tma_load_2d(sK + s * KV_BYTES + TILE_BYTES + o, &tmK, &kv_full[s], 64, row);
            tma_load_2d(sV + s * KV_BYTES + o, &tmV, &kv_full[s], 0, row);
            tma_load_2d(sV + s * KV_BYTES + TILE_BYTES + o, &tmV, &kv_full[s], 64, row);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = umma_idesc_bf16(FQ, FK);                   // K-major A and B
      constexpr uint32_t idesc_o = umma_idesc_bf16(FQ, FD) | (1u << 16);      // B (V) MN-major
      // S_j of (item, its Q stage, global tile index gj)
      auto issue_s = [&](const Item& it, int qs, uint32_t gj, bool last) {
        const int s = gj & 1;
        mbar_wait(&kv_full[s], (gj >> 1) & 1);
        if (gj >= 2) mbar_wait(&s_free[s], ((gj >> 1) & 1) ^ 1);
        // TMEM P: S buffer s still holds P of tile gj-2 -- its P.V must have
        // read it before this S overwrites it (the MMA pipe does not order a
        // TMEM read of one MMA before the TMEM write of a later one)
        if (PT && gj >= 2) mbar_wait(&o_full[(gj - 2) & 1], ((gj - 2) >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + s * 128;
        const uint32_t qa = smem_u32(sQ + qs * Q_BYTES), kb = smem_u32(sK + s * KV_BYTES);
#pragma unroll
        for (int k = 0; k < FD / 16; ++k) {
          const uint32_t off = (k >> 2) * TILE_BYTES + (k & 3) * 32;
          umma_bf16(d, umma_desc_sw128(qa + off), umma_desc_sw128(kb + off), idesc_s, k ? 1u : 0u);
        }
        umma_commit(&s_full[s]);
        if (last) umma_commit(&q_empty[qs]);   // last read of this Q
      };
      auto next_item = [&](int from, Item& it) {
        for (int id = from; id < n_items; id += gridDim.x)
          if (item_of(p, id, it)) return id;
        return n_items;
      };
      uint32_t nq = 0, base = 0;   // items, tiles before the current item
      Item cur, nxt;
      int id = next_item(blockIdx.x, cur);
      if (id < n_items) {
        mbar_wait(&q_full[0], 0);
        issue_s(cur, 0, 0, cur.ntiles == 1);
      }
      while (id < n_items) {
        const int qs = nq & 1;
        const int id_next = next_item(id + gridDim.x, nxt);
        for (int j = 0; j < cur.ntiles; ++j) {
          if (j + 1 < cur.ntiles) {
            issue_s(cur, qs, base + j + 1, j + 2 == cur.ntiles);
          } else if (id_next < n_items) {
            // look ahead: the next item's first S while this item's last
            // softmax and epilogue run
            const uint32_t nqn = nq + 1;
            mbar_wait(&q_full[nqn & 1], (nqn >> 1) & 1);
            issue_s(nxt, nqn & 1, base + cur.ntiles, nxt.ntiles == 1);
          }
          // O += P_j . V_j (one TMEM accumulator per item; the softmax warps
          // signal p_full after any lazy rescale of O and, for an item's
          // first tile, after reading out the previous item's O)
          const uint32_t gj = base + j;
          const int s = gj & 1;
          mbar_wait((gj & 1) ? p_full1 : p_full, (gj >> 1) & 1);
          tc_fence_after();
          const uint32_t d = tmem + 256;
          const uint32_t pa = smem_u32(sP), vb = smem_u32(sV + s * KV_BYTES);
#pragma unroll
          for (int k = 0; k < FK / 16; ++k) {
            // B (V, MN-major): 16 keys = two 8-key core groups of 1024 B
            const uint32_t b_off = k * 2048;
            if constexpr (PT) {
              // A (P) in TMEM over S buffer s: 16 keys = 8 packed columns
              umma_bf16_tmem_a(d, tmem + s * 128 + k * 8, desc_mn_sw128(vb + b_off, TILE_BYTES, 1024), idesc_o,
                               (j || k) ? 1u : 0u);
            } else {
              // A (P, K-major): 64-key blocks of 16 KB, 32 B per 16 keys
              const uint32_t a_off = (k >> 2) * TILE_BYTES + (k & 3) * 32;
              umma_bf16(d, umma_desc_sw128(pa + a_off), desc_mn_sw128(vb + b_off, TILE_BYTES, 1024), idesc_o,
                        (j || k) ? 1u : 0u);
            }
          }
          umma_commit(&o_full[gj & 1]);
          umma_commit(&kv_empty[s]);
        }
        base += cur.ntiles;
        ++nq;
        id = id_next;
        cur = nxt;
      }
    }
  } else if (warp >= 4) {
    // warp w reads TMEM lanes 32*(w%4).. (hardware rule); hf = key / dim half
    const int q = warp & 3, hf = (warp - 4) >> 2;
    const int r = q * 32 + lane;                    // query row of the tile = TMEM lane
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    auto pair_bar = [q] { asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory"); };
    uint32_t base = 0;
    for (int id = blockIdx.x; id < n_items; id += gridDim.x) {
      Item it;
      if (!item_of(p, id, it)) continue;
      const int qpos = it.pos0 + it.qb + r;                  // absolute position of this query
      const int kmax = p.causal ? qpos : it.pos0 + it.len - 1;  // last key this query sees
      const float* brow =
          (p.bias && it.qb + r < it.len) ? p.bias + (int64_t)it.h * p.bias_ld + p.bias_off - qpos : nullptr;
      constexpr int HD = FD / 2;                      // output dims / keys per half
      constexpr float LOG2E = 1.4426950408889634f;
      constexpr float RESCALE_LOG2 = 8.f;             // move m_ref when a tile max exceeds it by > 2^8
      float m = -INFINITY, l = 0.f;                   // m: reference max the P's are taken against
      const uint32_t oa = tmem + lane_base + 256 + hf * HD;
      for (int j = 0; j < it.ntiles; ++j) {
        const uint32_t gj = base + j;
        const int s = gj & 1;
        mbar_wait(&s_full[s], (gj >> 1) & 1);
        tc_fence_after();
        // pass 1: this half's 64 scores (scaled, biased, masked) into
        // registers and their max; the row max over the tile is the max of
        // the two halves' (exchanged through shared memory)
        const uint32_t sa = tmem + lane_base + s * 128 + hf * HD;
        const int k0 = j * FK + hf * HD;
        float sc[HD];
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < HD; c += 16) tmem_ld16(sa + c, sc + c);
        if (k0 + HD - 1 <= kmax && !brow) {      // no key of this half is masked
#pragma unroll
          for (int e = 0; e < HD; ++e) {
            sc[e] = __fmul_rn(sc[e], p.scale);
            mx = fmaxf(mx, sc[e]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < HD; ++e) {
            const int kpos = k0 + e;
            float x = (kpos <= kmax) ? __fmul_rn(sc[e], p.scale) : -INFINITY;
            if (brow && kpos <= kmax) x = __fadd_rn(x, brow[kpos]);
            sc[e] = x;
            mx = fmaxf(mx, x);
          }
        }
        lx[hf * FQ + r] = mx;
        pair_bar();
        mx = fmaxf(lx[r], lx[FQ + r]);
        pair_bar();   // both halves have read lx before it is written again
        // smem P: the previous tile's P.V has completed before P is overwritten
        // (and O read); TMEM P lives in this tile's own S buffer, so only a
        // rescale of O below waits for it
        if (!PT && j >= 1) mbar_wait(&o_full[(gj - 1) & 1], ((gj - 1) >> 1) & 1);
        // lazy rescale: the reference max moves only when this tile's max
        // exceeds it by more than 2^RESCALE_LOG2 (both threads of a row take the
        // same decision); the TMEM accesses are warp-collective, so a warp
        // rescales when any of its rows must (alpha = 1 for the others)
        const bool move = m == -INFINITY || (mx - m) * LOG2E > RESCALE_LOG2;
        const float m_new = move ? fmaxf(m, mx) : m;
        const bool resc = move && j >= 1 && m != -INFINITY;
        if (__any_sync(0xffffffffu, resc)) {
          const float alpha = resc ? ex2((m - m_new) * LOG2E) : 1.f;
          if (PT) mbar_wait(&o_full[(gj - 1) & 1], ((gj - 1) >> 1) & 1);   // O holds P.V up to tile j-1
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < HD; c += 16) {
            float v[16];
            tmem_ld16(oa + c, v);
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] *= alpha;
            tmem_st16(oa + c, v);
          }
          tmem_st_wait();
          l *= alpha;
        }
        m = m_new;
        // p = 2^(s log2 e - m log2 e): one FFMA + an SFU op (or, for a quarter
        // of the keys, the FMA-pipe polynomial) per score
        const float nml = (m == -INFINITY) ? 0.f : -m * LOG2E;
        float sum = 0.f;
#pragma unroll
        float pw[16];   // TMEM P: 32 keys = 16 packed columns per store
        for (int c = 0; c < HD; c += 16) {
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float a0 = fmaf(sc[c + e], LOG2E, nml), a1 = fmaf(sc[c + e + 1], LOG2E, nml);
            const float p0 = ex2(a0);
            const float p1 = (e % 4 == 2) ? ex2_poly(a1) : ex2(a1);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
            sum += __low2float(b2) + __high2float(b2);   // the sum uses the bf16 P that feeds P.V
            pk[e / 2] = *reinterpret_cast<uint32_t*>(&b2);
          }
          if constexpr (PT) {
            // row r, keys hf*64+c..+15 -> packed columns hf*32 + c/2 .. +8 of S buffer s
#pragma unroll
            for (int q = 0; q < 8; ++q) pw[(c & 16) / 2 + q] = __uint_as_float(pk[q]);
            if (c & 16) tmem_st16(tmem + lane_base + s * 128 + hf * 32 + (c - 16) / 2, pw);
          } else {
            // row r, keys hf*64+c..+15: two 16-byte chunks in the SW128 K-major image
            uint8_t* blk = sP + hf * TILE_BYTES;
            const int ch = c >> 3;
            *reinterpret_cast<uint4*>(blk + r * 128 + (((ch) ^ (r & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            *reinterpret_cast<uint4*>(blk + r * 128 + (((ch + 1) ^ (r & 7)) << 4)) =
                make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
        }
        l += sum;
        if (PT)
          tmem_st_wait();
        else
          fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&s_free[s]);
          mbar_arrive((gj & 1) ? p_full1 : p_full);
        }
      }
      // the item's last P.V, then O out of TMEM: normalised by the row sum
      {
        const uint32_t gl = base + it.ntiles - 1;
        mbar_wait(&o_full[gl & 1], (gl >> 1) & 1);
      }
      tc_fence_after();
      base += it.ntiles;
      // row sum = the two halves' sums (low half + high half)
      lx[hf * FQ + r] = l;
      pair_bar();
      const float lt = lx[r] + lx[FQ + r];
      pair_bar();   // both halves have read lx before the next item writes it
      const float inv = 1.f / lt;
      bf16* dst = p.out + (int64_t)(it.t0 + it.qb + r) * p.ldo + it.h * FD + hf * HD;
#pragma unroll
      for (int c = 0; c < HD; c += 16) {
        float v[16];
        tmem_ld16(oa + c, v);
        if (it.qb + r < it.len) {
          uint32_t pk[8];
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[e] * inv, v[e + 1] * inv);
            pk[e / 2] = *reinterpret_cast<uint32_t*>(&b2);
          }
          *reinterpret_cast<uint4*>(dst + c) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4*>(dst + c + 8) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      // O has been read: the next item's first P.V may overwrite it (it is
      // issued after this CTA's softmax warps signal the next p_full)
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}
}  // namespace

// P in TMEM (1) or shared memory (0) (exg_diag_fmha_p_tmem, A/B): TMEM P is
// 6 % faster on the task-S mix (tools/probe_kernels.py pmix_pt: 270 vs 287
// us).  With it the softmax warps can run two tiles ahead of the P.V issue, so
// p_full is double-buffered by tile parity (a single barrier aliased phases
// and corrupted rows in the T5 relative-bias test; tools/fmha_pt_check.py)
int& fmha_p_tmem() {
  static int on = 1;
  return on;
}

// L2 prefetch distance of the FMHA producer in items (exg_diag_fmha_prefetch);
// off: measured slower at the task-S mix (tools/probe_kernels.py pmix_pf:
// 280.6 us without, 294.9 / 310.2 / 311.3 us with 1 / 2 / 4 items ahead)
int& fmha_prefetch_ahead() {
  static int n = 0;
  return n;
}

// diagnostics: 1 = route dh = 128 to the SIMT kernel (exg_diag_prefill_simt)
int& prefill_force_simt() {
  static int f = 0;
  return f;
}

bool prefill_attention_tc(const PrefillAttnArgs& a, cudaStream_t st) {
  if (a.dh != FD || prefill_force_simt()) return false;
  static bool attr = false;
  if (!attr) {
    EXG_CUDA(cudaFuncSetAttribute(fmha_prefill_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)FMHA_SMEM));
    EXG_CUDA(cudaFuncSetAttribute(fmha_prefill_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)FMHA_SMEM));
    attr = true;
  }
  // Q: the packed qkv buffer [q_rows][ldq] (rows past the last token are
  // zero-filled by TMA and never stored); K/V: the cache viewed as
  // [kv_rows = slots*H*max_ctx][dh]
  const int QT = (a.max_len + FQ - 1) / FQ;
  FmhaParams p{a.cu_seqlens, a.slot, a.pos0, a.H, a.max_ctx, a.R, QT,
               a.scale * 1.4426950408889634f, a.scale, a.out, a.ldo, a.causal, a.bias, a.bias_ld, a.bias_off, a.kv,
               fmha_prefetch_ahead()};
  const int n_items = QT * a.R * a.H;
  if (n_items <= 0) return true;
  const CUtensorMap tq = make_tmap_bf16(a.q, a.q_rows, a.ldq, a.ldq, 128);
  // K / V boxes of 64 keys: a 128-key tile is two boxes per 64-column half
  const CUtensorMap tk = make_tmap_bf16(a.kc, a.kv_rows, FD, FD, 64);
  const CUtensorMap tv = make_tmap_bf16(a.vc, a.kv_rows, FD, FD, 64);
  // persistent grid: one CTA per SM (227 KB of shared memory, 512 TMEM columns)
  const int grid = std::min(n_items, sm_count());
  if (fmha_p_tmem())
    launch_pdl(fmha_prefill_kernel<true>, dim3(grid), dim3(128 + 32 * SM_WARPS), FMHA_SMEM, st, tq, tk, tv, p);
  else
    launch_pdl(fmha_prefill_kernel<false>, dim3(grid), dim3(128 + 32 * SM_WARPS), FMHA_SMEM, st, tq, tk, tv, p);
  EXG_CHECK_LAUNCH();
  return true;
}

}  // namespace exg

extern "C" void exg_diag_prefill_simt(int on) { exg::prefill_force_simt() = on; }
extern "C" void exg_diag_fmha_prefetch(int ahead) { exg::fmha_prefetch_ahead() = ahead > 0 ? ahead : 0; }
extern "C" void exg_diag_fmha_p_tmem(int on) { exg::fmha_p_tmem() = on; }
