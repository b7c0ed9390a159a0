// Non-GEMM kernels (see kernels.cuh for the contracts).
#include "kernels.cuh"
#include "gemm_tc.cuh"

namespace exg {

// ============================================================================
// K14 weight generator
// ============================================================================
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void weightgen_kernel(bf16* __restrict__ dst, int64_t rows, int64_t cols, int64_t ld, GenParams p) {
  // blocked: scatter rows [dst_row0, dst_row0 + rows) of the blocked layout
  // (padding is not written: the destination is zero-filled beforehand);
  // else the plain row-major [rows][ld]
  const int64_t n = rows * cols;
  const uint64_t key = p.seed ^ (p.tensor_id << 40);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    const int64_t i = p.transposed ? (c + p.col_off) * p.canon_cols + (r + p.row_off)
                                   : (r + p.row_off) * p.canon_cols + (c + p.col_off);
    const uint64_t h = splitmix64(key ^ (uint64_t)i);
    const float u = __fmul_rn((float)(uint32_t)(h >> 40), 5.9604644775390625e-08f);  // * 2^-24, exact
    const float cen = __fsub_rn(u, 0.5f);                                           // exact
    const float v = p.gain ? __fadd_rn(1.0f, __fmul_rn(cen, p.c_gain)) : __fmul_rn(cen, p.c_mat);
    dst[p.blocked ? blocked_index(r + p.dst_row0, c, cols) : r * ld + c] = __float2bfloat16_rn(v);
  }
}

void weightgen(bf16* dst, int64_t rows, int64_t cols, int64_t ld, const GenParams& p, cudaStream_t st) {
  const int64_t n = rows * cols;
  if (n <= 0) return;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  weightgen_kernel<<<blocks, 256, 0, st>>>(dst, rows, cols, ld, p);
  EXG_CHECK_LAUNCH();
}

// ============================================================================
// K1 embedding
// ============================================================================
__global__ void embed_kernel(float* __restrict__ x, const int32_t* __restrict__ ids, const int32_t* __restrict__ pos,
                             const bf16* __restrict__ tok, const bf16* __restrict__ pe, int d, int tok_blocked) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  const int t = blockIdx.x;
  const int64_t id = ids[t];
  const bf16* b = pe ? pe + (int64_t)pos[t] * d : nullptr;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const bf16 a = tok[tok_blocked ? blocked_index(id, j, d) : id * d + j];
    x[(int64_t)t * d + j] = b ? __fadd_rn(bf2f(a), bf2f(b[j])) : bf2f(a);
  }
}

void embed(float* x, const int32_t* ids, const int32_t* pos, const bf16* tok_emb, const bf16* pos_emb, int T, int d,
           cudaStream_t st, int tok_blocked) {
  if (T <= 0) return;
  launch_pdl(embed_kernel, dim3(T), dim3(256), 0, st, x, ids, pos, tok_emb, pos_emb, d, tok_blocked);
  EXG_CHECK_LAUNCH();
}

// ============================================================================
// K2 LayerNorm (fp32 statistics, biased variance)
// ============================================================================
__device__ __forceinline__ float block_sum_256(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += red[i];
  return s;
}

__global__ void __launch_bounds__(256) layernorm_kernel(bf16* __restrict__ y, int64_t ldy, const float* __restrict__ x,
                                                        int64_t ldx, const bf16* __restrict__ g,
                                                        const bf16* __restrict__ b, int d, float eps) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  __shared__ float red[8];
  const float* xr = x + (int64_t)blockIdx.x * ldx;
  float s = 0.f;
  for (int j = threadIdx.x; j < d; j += 256) s += xr[j];
  const float mean = block_sum_256(s, red) / (float)d;
  float q = 0.f;
  for (int j = threadIdx.x; j < d; j += 256) {
    const float c = xr[j] - mean;
    q += c * c;
  }
  const float var = block_sum_256(q, red) / (float)d;
  const float rstd = rsqrtf(var + eps);
  bf16* yr = y + (int64_t)blockIdx.x * ldy;
  for (int j = threadIdx.x; j < d; j += 256) yr[j] = f2bf((xr[j] - mean) * rstd * bf2f(g[j]) + bf2f(b[j]));
}

// Row held in registers (NV float4 per thread): one global read of x, the
// statistics from registers -- the decode-time LayerNorm is latency-bound
// (a few dozen rows), so one load round trip instead of three matters.
// RMS = 1: T5 RMSNorm with output scale (b unused).
template <int NV, int RMS>
__global__ void __launch_bounds__(256) norm_reg_kernel(bf16* __restrict__ y, int64_t ldy, const float* __restrict__ x,
                                                       int64_t ldx, const bf16* __restrict__ g,
                                                       const bf16* __restrict__ b, int d, float eps, float out_scale) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  __shared__ float red[8];
  const float4* xr = reinterpret_cast<const float4*>(x + (int64_t)blockIdx.x * ldx);
  const int n4 = d >> 2;
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = threadIdx.x + k * 256;
    v[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += RMS ? (v[k].x * v[k].x + v[k].y * v[k].y) + (v[k].z * v[k].z + v[k].w * v[k].w)
             : (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  float mean = 0.f, rstd;
  if (RMS) {
    rstd = rsqrtf(block_sum_256(s, red) / (float)d + eps);
  } else {
    mean = block_sum_256(s, red) / (float)d;
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      if (threadIdx.x + k * 256 >= n4) continue;
      const float a = v[k].x - mean, bb = v[k].y - mean, c = v[k].z - mean, e = v[k].w - mean;
      q += (a * a + bb * bb) + (c * c + e * e);
    }
    rstd = rsqrtf(block_sum_256(q, red) / (float)d + eps);
  }
  bf16* yr = y + (int64_t)blockIdx.x * ldy;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = threadIdx.x + k * 256;
    if (i >= n4) continue;
    const uint2 gr = reinterpret_cast<const uint2*>(g)[i];
    const float2 g01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gr.x));
    const float2 g23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gr.y));
    float o0, o1, o2, o3;
    if (RMS) {
      o0 = v[k].x * rstd * g01.x * out_scale;
      o1 = v[k].y * rstd * g01.y * out_scale;
      o2 = v[k].z * rstd * g23.x * out_scale;
      o3 = v[k].w * rstd * g23.y * out_scale;
    } else {
      const uint2 br = reinterpret_cast<const uint2*>(b)[i];
      const float2 b01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.x));
      const float2 b23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.y));
      o0 = (v[k].x - mean) * rstd * g01.x + b01.x;
      o1 = (v[k].y - mean) * rstd * g01.y + b01.y;
      o2 = (v[k].z - mean) * rstd * g23.x + b23.x;
      o3 = (v[k].w - mean) * rstd * g23.y + b23.y;
    }
    __nv_bfloat162 p0 = __floats2bfloat162_rn(o0, o1), p1 = __floats2bfloat162_rn(o2, o3);
    uint2 out;
    out.x = *reinterpret_cast<uint32_t*>(&p0);
    out.y = *reinterpret_cast<uint32_t*>(&p1);
    reinterpret_cast<uint2*>(yr)[i] = out;
  }
}

// dispatch: register-resident rows up to d = 16384 (x, y row strides and d
// multiples of 4 floats / bf16), the strided kernels otherwise
template <int RMS>
static bool norm_reg(bf16* y, int64_t ldy, const float* x, int64_t ldx, const bf16* g, const bf16* b, int T, int d,
                     float eps, float out_scale, cudaStream_t st) {
  if ((d & 3) || (ldx & 3) || (ldy & 3) || d > 16384) return false;
  const int nv = (d / 4 + 255) / 256;
  auto go = [&](auto kern) {
    launch_pdl(kern, dim3(T), dim3(256), 0, st, y, ldy, x, ldx, g, b, d, eps, out_scale);
    EXG_CHECK_LAUNCH();
  };
  if (nv <= 1) go(norm_reg_kernel<1, RMS>);
  else if (nv <= 2) go(norm_reg_kernel<2, RMS>);
  else if (nv <= 4) go(norm_reg_kernel<4, RMS>);
  else if (nv <= 5) go(norm_reg_kernel<5, RMS>);
  else if (nv <= 8) go(norm_reg_kernel<8, RMS>);
  else if (nv <= 9) go(norm_reg_kernel<9, RMS>);
  else if (nv <= 12) go(norm_reg_kernel<12, RMS>);
  else go(norm_reg_kernel<16, RMS>);
  return true;
}

// Deferred stream-K reduction folded into the LayerNorm (decode, tp = 1):
// x[row] += (sum_seg P[seg][row][:] + bias) -- the residual update of the
// preceding O-projection / FFN2, whose GEMM stored only its raw segments --
// written back to x, then the LayerNorm of norm_reg_kernel on the updated row
// (same arithmetic, bit-identical to the in-kernel fixup + LayerNorm).
template <int NV, int MS = (NV <= 5 ? 6 : (NV <= 9 ? 3 : 1))>
__global__ void __launch_bounds__(256) resid_reduce_ln_kernel(bf16* __restrict__ y, int64_t ldy, float* __restrict__ x,
                                                              int64_t ldx, const float* __restrict__ P, int tokens,
                                                              SegInfo si, const bf16* __restrict__ rbias,
                                                              const bf16* __restrict__ g, const bf16* __restrict__ b,
                                                              int d, float eps) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  __shared__ float red[8];
  const int row = blockIdx.x;
  float4* xr = reinterpret_cast<float4*>(x + (int64_t)row * ldx);
  const int n4 = d >> 2;
  float4 v[NV];
  float s = 0.f;
  // every segment load of this thread's NV chunks is issued before any sum
  // (one memory round trip instead of NV x segments of them); the sums then
  // run in segment order -- the fixup's arithmetic
  constexpr int MAXS = MS;
  const int64_t segstride4 = (int64_t)tokens * d / 4;
  float4 pre[NV][MAXS], old[NV];
  int nsk[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = threadIdx.x + k * 256;
    nsk[k] = i < n4 ? seg_count(si, (4 * i) >> 7) : 0;
    old[k] = i < n4 ? xr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4* p = reinterpret_cast<const float4*>(P + (int64_t)row * d + 4 * i);
#pragma unroll
    for (int sg = 0; sg < MAXS; ++sg)
      pre[k][sg] = sg < nsk[k] ? __ldcg(p + sg * segstride4) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = threadIdx.x + k * 256;
    if (i < n4) {
      const int f0 = 4 * i;
      const int ns = nsk[k];
      const float4* p = reinterpret_cast<const float4*>(P + (int64_t)row * d + f0);
      float4 acc = pre[k][0];
#pragma unroll
      for (int sg = 1; sg < MAXS; ++sg) {
        if (sg < ns) {
          acc.x += pre[k][sg].x;
          acc.y += pre[k][sg].y;
          acc.z += pre[k][sg].z;
          acc.w += pre[k][sg].w;
        }
      }
      for (int sg = MAXS; sg < ns; ++sg) {   // rare: more segments than preloaded
        const float4 q = __ldcg(p + sg * segstride4);
        acc.x += q.x;
        acc.y += q.y;
        acc.z += q.z;
        acc.w += q.w;
      }
      if (rbias) {
        const uint2 br = reinterpret_cast<const uint2*>(rbias)[i];
        const float2 b01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.x));
        const float2 b23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.y));
        acc.x += b01.x;
        acc.y += b01.y;
        acc.z += b23.x;
        acc.w += b23.y;
      }
      v[k] = make_float4(old[k].x + acc.x, old[k].y + acc.y, old[k].z + acc.z, old[k].w + acc.w);
      xr[i] = v[k];
    } else {
      v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
  }
  const float mean = block_sum_256(s, red) / (float)d;
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    if (threadIdx.x + k * 256 >= n4) continue;
    const float a = v[k].x - mean, bb = v[k].y - mean, c = v[k].z - mean, e = v[k].w - mean;
    q += (a * a + bb * bb) + (c * c + e * e);
  }
  const float rstd = rsqrtf(block_sum_256(q, red) / (float)d + eps);
  bf16* yr = y + (int64_t)row * ldy;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int i = threadIdx.x + k * 256;
    if (i >= n4) continue;
    const uint2 gr = reinterpret_cast<const uint2*>(g)[i];
    const float2 g01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gr.x));
    const float2 g23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gr.y));
    const uint2 br = reinterpret_cast<const uint2*>(b)[i];
    const float2 b01 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.x));
    const float2 b23 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&br.y));
    const float o0 = (v[k].x - mean) * rstd * g01.x + b01.x;
    const float o1 = (v[k].y - mean) * rstd * g01.y + b01.y;
    const float o2 = (v[k].z - mean) * rstd * g23.x + b23.x;
    const float o3 = (v[k].w - mean) * rstd * g23.y + b23.y;
    __nv_bfloat162 p0 = __floats2bfloat162_rn(o0, o1), p1 = __floats2bfloat162_rn(o2, o3);
    uint2 out;
    out.x = *reinterpret_cast<uint32_t*>(&p0);
    out.y = *reinterpret_cast<uint32_t*>(&p1);
    reinterpret_cast<uint2*>(yr)[i] = out;
  }
}

// diagnostics (exg_diag_ln_preload): 0 = preload only the first segment (A/B)
int& ln_preload_segments() {
  static int on = 1;
  return on;
}

bool layernorm_deferred(bf16* y, int64_t ldy, float* x, int64_t ldx, const float* P, const SegInfo& si,
                        const bf16* rbias, const bf16* g, const bf16* b, int T, int d, float eps, cudaStream_t st) {
  if ((d & 3) || (ldx & 3) || (ldy & 3) || d > 16384) return false;
  if (T <= 0) return true;
  const int nv = (d / 4 + 255) / 256;
  auto go = [&](auto kern) {
    launch_pdl(kern, dim3(T), dim3(256), 0, st, y, ldy, x, ldx, P, T, si, rbias, g, b, d, eps);
    EXG_CHECK_LAUNCH();
  };
  if (nv <= 1) go(resid_reduce_ln_kernel<1>);
  else if (nv <= 2) go(resid_reduce_ln_kernel<2>);
  else if (nv <= 4) go(resid_reduce_ln_kernel<4>);
  else if (nv <= 5 && ln_preload_segments()) go(resid_reduce_ln_kernel<5>);
  else if (nv <= 5) go(resid_reduce_ln_kernel<5, 1>);
  else if (nv <= 8) go(resid_reduce_ln_kernel<8>);
  else if (nv <= 9) go(resid_reduce_ln_kernel<9>);
  else if (nv <= 12) go(resid_reduce_ln_kernel<12>);
  else go(resid_reduce_ln_kernel<16>);
  return true;
}

void layernorm(bf16* y, int64_t ldy, const float* x, int64_t ldx, const bf16* g, const bf16* b, int T, int d,
               float eps, cudaStream_t st) {
  if (T <= 0) return;
  if (norm_reg<0>(y, ldy, x, ldx, g, b, T, d, eps, 1.f, st)) return;
  launch_pdl(layernorm_kernel, dim3(T), dim3(256), 0, st, y, ldy, x, ldx, g, b, d, eps);
  EXG_CHECK_LAUNCH();
}

// T5 RMSNorm: y = bf16(x * rsqrt(mean(x^2) + eps) * g * out_scale)
__global__ void __launch_bounds__(256) rmsnorm_kernel(bf16* __restrict__ y, int64_t ldy, const float* __restrict__ x,
                                                      int64_t ldx, const bf16* __restrict__ g, int d, float eps,
                                                      float out_scale) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  __shared__ float red[8];
  const float* xr = x + (int64_t)blockIdx.x * ldx;
  float q = 0.f;
  for (int j = threadIdx.x; j < d; j += 256) q += xr[j] * xr[j];
  const float ms = block_sum_256(q, red) / (float)d;
  const float rstd = rsqrtf(ms + eps);
  bf16* yr = y + (int64_t)blockIdx.x * ldy;
  for (int j = threadIdx.x; j < d; j += 256) yr[j] = f2bf(xr[j] * rstd * bf2f(g[j]) * out_scale);
}

void rmsnorm(bf16* y, int64_t ldy, const float* x, int64_t ldx, const bf16* g, int T, int d, float eps,
             float out_scale, cudaStream_t st) {
  if (T <= 0) return;
  if (norm_reg<1>(y, ldy, x, ldx, g, nullptr, T, d, eps, out_scale, st)) return;
  launch_pdl(rmsnorm_kernel, dim3(T), dim3(256), 0, st, y, ldy, x, ldx, g, d, eps, out_scale);
  EXG_CHECK_LAUNCH();
}

// fp32 relative-bias table: tab[h][j] = rel[bucket[j]][h0 + h] (bf16 weights,
// rel is [n_buckets][H_total])
__global__ void rel_bias_table_kernel(float* __restrict__ tab, const bf16* __restrict__ rel,
                                      const int32_t* __restrict__ bucket, int n, int Hl, int H_total, int h0) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)n * Hl) return;
  const int h = (int)(e / n), j = (int)(e % n);
  tab[e] = bf2f(rel[(int64_t)bucket[j] * H_total + h0 + h]);
}

void rel_bias_table(float* tab, const bf16* rel, const int32_t* bucket, int n, int Hl, int H_total, int h0,
                    cudaStream_t st) {
  const int64_t tot = (int64_t)n * Hl;
  if (tot <= 0) return;
  rel_bias_table_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(tab, rel, bucket, n, Hl, H_total, h0);
  EXG_CHECK_LAUNCH();
}

// ============================================================================
// K7 KV scatter
// ============================================================================
__global__ void kv_scatter_kernel(bf16* __restrict__ kc, bf16* __restrict__ vc, const bf16* __restrict__ qkv,
                                  const int32_t* __restrict__ slot, const int32_t* __restrict__ pos, int T, int H,
                                  int dh, int max_ctx) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  const int inner = H * dh;
  const int chunks = inner / 8;  // 16-byte chunks per K (or V) row
  const int64_t n = (int64_t)T * 2 * chunks;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(e / (2 * chunks));
    const int rem = (int)(e % (2 * chunks));
    const int which = rem / chunks, c = rem % chunks;
    const int h = (c * 8) / dh, j = (c * 8) % dh;
    const int4 v = *reinterpret_cast<const int4*>(qkv + (int64_t)t * 3 * inner + (1 + which) * inner + c * 8);
    bf16* dst = (which ? vc : kc) + (((int64_t)slot[t] * H + h) * max_ctx + pos[t]) * dh + j;
    *reinterpret_cast<int4*>(dst) = v;
  }
}

void kv_scatter(bf16* kc, bf16* vc, const bf16* qkv, const int32_t* slot, const int32_t* pos, int T, int H, int dh,
                int max_ctx, cudaStream_t st) {
  if (T <= 0) return;
  const int64_t n = (int64_t)T * 2 * (H * dh / 8);
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  launch_pdl(kv_scatter_kernel, dim3(blocks), dim3(256), 0, st, kc, vc, qkv, slot, pos, T, H, dh, max_ctx);
  EXG_CHECK_LAUNCH();
}

// ============================================================================
// K6 ragged decode attention
//
// One CTA (4 warps) per (row, head, split).  Thread 0 streams the split's K
// and V rows (contiguous per (slot, head)) through a 2-stage ring of
// cp.async.bulk copies completing on mbarriers (32 KB, 7 CTAs per SM: at the
// bench's context mix the per-CTA tile loop, not the ring depth, limits
// throughput, so more resident CTAs beat deeper rings -- measured 4.5 ->
// 5.1 TB/s at B=56, 5.5 -> 6.5 TB/s at B=256); every warp owns a fixed
// subset of keys of each tile, keeps its own online-softmax state, and the
// four warp states are merged at the end in warp order.
// ============================================================================
template <int DH, int ST = 4>
struct DecodeCfg {
  static constexpr int CH = DH / 8;                 // 16-byte chunks per key row
  static constexpr int LPK = CH >= 4 ? 4 : CH;      // lanes per key (dot product)
  static constexpr int CPL = CH / LPK;              // chunks per lane
  static constexpr int KPW = 32 / LPK;              // keys per warp per tile
  static constexpr int KT = 4 * KPW;                // keys per tile
  static constexpr int ROWB = DH * 2;               // bytes per key row
  static constexpr int STAGES = ST;
  static constexpr int DPL = DH >= 32 ? DH / 32 : 1;  // output dims per lane (P.V)
  static constexpr size_t SMEM = (size_t)STAGES * KT * ROWB * 2;
};

// feature f of row i of a deferred QKV GEMM: its segments summed in order +
// bias (the in-kernel fixup's arithmetic), before the bf16 rounding point
__device__ __forceinline__ float deferred_qkv(const DecodeAttnArgs& a, int i, int f) {
  const int ns = seg_count(a.qkv_si, f >> 7);
  const int64_t F = 3LL * a.qkv_inner;
  const float* p = a.qkv_part + (int64_t)i * F + f;
  const int64_t ss = (int64_t)a.B * F;
  // up to 8 segment loads in flight, summed in segment order
  float acc = 0.f;
  for (int s0 = 0; s0 < ns; s0 += 8) {
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = s0 + q < ns ? __ldcg(p + (s0 + q) * ss) : 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (s0 + q < ns) acc = (s0 + q == 0) ? v[q] : acc + v[q];
  }
  if (a.qkv_bias) acc += bf2f(a.qkv_bias[f]);
  return acc;
}

template <int DH, int ST, int MB = 1>
__global__ void __launch_bounds__(128, MB) decode_attn_kernel(DecodeAttnArgs a) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  using C = DecodeCfg<DH, ST>;
  extern __shared__ __align__(128) uint8_t dsm[];
  uint8_t* sk = dsm;
  uint8_t* sv = dsm + C::STAGES * C::KT * C::ROWB;
  __shared__ uint64_t bar[C::STAGES];
  __shared__ float qs[DH];
  __shared__ float wm[4], wl[4];
  __shared__ float wo[4][DH];

  const int i = blockIdx.x / a.H, h = blockIdx.x % a.H;
  const int sp = blockIdx.y;
  const int nk = a.n_keys[i];
  const int k_begin = sp * a.split_len;
  if (k_begin >= nk) return;
  const int n = min(nk - k_begin, a.split_len);
  const int ntiles = (n + C::KT - 1) / C::KT;
  const int nsplit = (nk + a.split_len - 1) / a.split_len;
  const int slot_i = a.slot[i];
  // cache row of key k_begin + t*KT (tile t never crosses a page: KT | P | split_len)
  auto tile_row = [&](int t) { return kv_row(a.kv, i, slot_i, a.H, h, a.max_ctx, k_begin + t * C::KT); };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
  }
  // fused KV append: this split holds the new key nk-1 -> write its K / V row
  // to the cache, and patch it into its shared-memory tile after the bulk copy
  // of that tile (which may carry the stale cache row) has landed
  const int r_new = nk - 1 - k_begin;
  const bool app = (a.knew != nullptr || a.qkv_part != nullptr) && r_new < n;
  __shared__ __align__(16) bf16 kvn[2][DH];   // deferred QKV: the new K / V rows
  if (a.qkv_part) {
    // q, and (appending CTA) the new K / V rows: each thread sums the
    // segments of a few features, rounded at the T4(d) point
    if (tid < DH) qs[tid] = bf2f(f2bf(deferred_qkv(a, i, h * DH + tid)));
    if (app)
      for (int e = tid; e < 2 * DH; e += 128)
        kvn[e / DH][e % DH] = f2bf(deferred_qkv(a, i, (1 + e / DH) * a.qkv_inner + h * DH + e % DH));
    __syncthreads();
  } else if (tid < DH) {
    qs[tid] = bf2f(a.q[(int64_t)i * a.ldq + h * DH + tid]);
  }
  int4 new_chunk = make_int4(0, 0, 0, 0);
  if (app && tid < 2 * C::CH) {
    const int which = tid / C::CH, c = tid % C::CH;
    if (a.qkv_part) {
      new_chunk = *reinterpret_cast<const int4*>(&kvn[which][c * 8]);
    } else {
      new_chunk = *reinterpret_cast<const int4*>((which ? a.vnew : a.knew) + (int64_t)i * a.ldnew + h * DH + c * 8);
    }
    const int64_t row = kv_row(a.kv, i, slot_i, a.H, h, a.max_ctx, nk - 1);
    bf16* dst = const_cast<bf16*>(which ? a.vc : a.kc) + row * DH + c * 8;
    *reinterpret_cast<int4*>(dst) = new_chunk;
  }
  __syncthreads();

  auto issue = [&](int t) {
    const int s = t % C::STAGES;
    const int nkt = min(C::KT, n - t * C::KT);
    const uint32_t bytes = (uint32_t)nkt * C::ROWB;
    const int64_t off = tile_row(t) * DH;
    mbar_arrive_expect_tx(&bar[s], 2 * bytes);
    bulk_load(sk + s * C::KT * C::ROWB, a.kc + off, bytes, &bar[s]);
    bulk_load(sv + s * C::KT * C::ROWB, a.vc + off, bytes, &bar[s]);
  };
  if (tid == 0)
    for (int t = 0; t < min(C::STAGES, ntiles); ++t) issue(t);

  const int part = lane % C::LPK;
  const int g = lane / C::LPK;                     // key slot inside this warp's group
  const int key_local = warp * C::KPW + g;         // key index inside a tile
  const int rot = (C::CPL > 1) ? (g & 1) : 0;      // bank-conflict rotation
  float qreg[C::CPL * 8];
#pragma unroll
  for (int j = 0; j < C::CPL; ++j) {
    const int chunk = ((j + rot) % C::CPL) * C::LPK + part;
#pragma unroll
    for (int e = 0; e < 8; ++e) qreg[j * 8 + e] = qs[chunk * 8 + e];
  }

  float m = -INFINITY, l = 0.f;
  float o[C::DPL];
#pragma unroll
  for (int d = 0; d < C::DPL; ++d) o[d] = 0.f;
  const bool pv_lane = lane * C::DPL < DH;

  for (int t = 0; t < ntiles; ++t) {
    const int s = t % C::STAGES;
    mbar_wait(&bar[s], (t / C::STAGES) & 1);
    if (app && t == r_new / C::KT) {   // CTA-uniform
      if (tid < 2 * C::CH) {
        const int which = tid / C::CH, c = tid % C::CH;
        uint8_t* row = (which ? sv : sk) + s * C::KT * C::ROWB + (r_new % C::KT) * C::ROWB;
        *reinterpret_cast<int4*>(row + c * 16) = new_chunk;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // before the stage is refilled by a bulk copy
      }
      __syncthreads();
    }
    const int nkt = min(C::KT, n - t * C::KT);
    const uint8_t* krow = sk + s * C::KT * C::ROWB;
    const uint8_t* vrow = sv + s * C::KT * C::ROWB;
    float dot = 0.f;
    const bool valid = key_local < nkt;
    if (valid) {
#pragma unroll
      for (int j = 0; j < C::CPL; ++j) {
        const int chunk = ((j + rot) % C::CPL) * C::LPK + part;
        const int4 raw = *reinterpret_cast<const int4*>(krow + key_local * C::ROWB + chunk * 16);
        const __nv_bfloat162* kv2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 f = __bfloat1622float2(kv2[e]);
          dot = fmaf(qreg[j * 8 + 2 * e], f.x, dot);
          dot = fmaf(qreg[j * 8 + 2 * e + 1], f.y, dot);
        }
      }
    }
#pragma unroll
    for (int o2 = 1; o2 < C::LPK; o2 <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o2);
    float score = valid ? __fmul_rn(dot, a.scale) : -INFINITY;
    if (a.bias && valid)  // T5 relative bias of distance key - query (query = newest key)
      score = __fadd_rn(score, a.bias[(int64_t)h * a.bias_ld + a.bias_off + (k_begin + t * C::KT + key_local) - (nk - 1)]);
    const float tmax = warp_max(score);
    const float m_new = fmaxf(m, tmax);
    const float alpha = (m == -INFINITY) ? 0.f : __expf(m - m_new);
    const float p = valid ? __expf(score - m_new) : 0.f;
    const float psum = warp_sum(part == 0 ? p : 0.f);
    l = l * alpha + psum;
#pragma unroll
    for (int d = 0; d < C::DPL; ++d) o[d] *= alpha;
    const int kw = min(C::KPW, nkt - warp * C::KPW);
    for (int kk = 0; kk < kw; ++kk) {
      const float pk = __shfl_sync(0xffffffffu, p, kk * C::LPK);
      if (pv_lane) {
        const bf16* vr = reinterpret_cast<const bf16*>(vrow + (warp * C::KPW + kk) * C::ROWB) + lane * C::DPL;
        if constexpr (C::DPL == 4) {
          const uint2 raw = *reinterpret_cast<const uint2*>(vr);
          const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.x));
          const float2 f1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&raw.y));
          o[0] = fmaf(pk, f0.x, o[0]);
          o[1] = fmaf(pk, f0.y, o[1]);
          o[2] = fmaf(pk, f1.x, o[2]);
          o[3] = fmaf(pk, f1.y, o[3]);
        } else {
#pragma unroll
          for (int d = 0; d < C::DPL; ++d) o[d] = fmaf(pk, bf2f(vr[d]), o[d]);
        }
      }
    }
    m = m_new;
    __syncthreads();  // every warp is done with stage s
    if (tid == 0 && t + C::STAGES < ntiles) issue(t + C::STAGES);
  }

  if (lane == 0) {
    wm[warp] = m;
    wl[warp] = l;
  }
  if (pv_lane) {
#pragma unroll
    for (int d = 0; d < C::DPL; ++d) wo[warp][lane * C::DPL + d] = o[d];
  }
  __syncthreads();
  if (tid < DH) {
    float M = wm[0];
#pragma unroll
    for (int w = 1; w < 4; ++w) M = fmaxf(M, wm[w]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float c = (wm[w] == -INFINITY) ? 0.f : __expf(wm[w] - M);
      L += wl[w] * c;
      O += wo[w][tid] * c;
    }
    if (nsplit == 1) {
      a.out[(int64_t)i * a.ldo + h * DH + tid] = f2bf(O / L);
    } else {
      float* pp = a.partial + (((int64_t)i * a.H + h) * a.max_splits + sp) * (DH + 2);
      if (tid == 0) {
        pp[0] = M;
        pp[1] = L;
      }
      pp[2 + tid] = O;
    }
  }
  if (nsplit > 1 && a.counters) {
    // the last split CTA of this (row, head) merges the splits in split order
    // -- the arithmetic of decode_combine_kernel, without its launch
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&a.counters[(int64_t)i * a.H + h], 1) == nsplit - 1);
    __syncthreads();
    if (s_last) {
      __threadfence();
      const float* base = a.partial + ((int64_t)i * a.H + h) * a.max_splits * (DH + 2);
      float M = -INFINITY;
      for (int s2 = 0; s2 < nsplit; ++s2) M = fmaxf(M, __ldcg(base + s2 * (DH + 2)));
      if (tid < DH) {
        float L = 0.f, O = 0.f;
        for (int s2 = 0; s2 < nsplit; ++s2) {
          const float* pp = base + s2 * (DH + 2);
          const float c = __expf(__ldcg(pp) - M);
          L += __ldcg(pp + 1) * c;
          O += __ldcg(pp + 2 + tid) * c;
        }
        a.out[(int64_t)i * a.ldo + h * DH + tid] = f2bf(O / L);
      }
      if (tid == 0) a.counters[(int64_t)i * a.H + h] = 0;
    }
  }
}

template <int DH>
__global__ void decode_combine_kernel(DecodeAttnArgs a) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  const int i = blockIdx.x / a.H, h = blockIdx.x % a.H;
  const int nk = a.n_keys[i];
  const int nsplit = (nk + a.split_len - 1) / a.split_len;
  if (nsplit <= 1) return;
  const float* base = a.partial + ((int64_t)i * a.H + h) * a.max_splits * (DH + 2);
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, base[s * (DH + 2)]);
  for (int d = threadIdx.x; d < DH; d += blockDim.x) {
    float L = 0.f, O = 0.f;
    for (int s = 0; s < nsplit; ++s) {
      const float* pp = base + s * (DH + 2);
      const float c = __expf(pp[0] - M);
      L += pp[1] * c;
      O += pp[2 + d] * c;
    }
    a.out[(int64_t)i * a.ldo + h * DH + d] = f2bf(O / L);
  }
}

// decode-attention key split length (diagnostics override via
// exg_diag_decode_split; 0 = the engine's default); >= 128
int& decode_split_override() {
  static int s = 0;
  return s;
}

// ring depth (diagnostics override via exg_diag_decode_stages; 0 = default)
int& decode_stages_override() {
  static int s = 0;
  return s;
}

template <int DH, int ST, int MB = 1>
void decode_attention_st(const DecodeAttnArgs& a, cudaStream_t st) {
  using C = DecodeCfg<DH, ST>;
  static bool attr = false;
  if (!attr) {
    EXG_CUDA(cudaFuncSetAttribute(decode_attn_kernel<DH, ST, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)C::SMEM));
    attr = true;
  }
  dim3 grid(a.B * a.H, a.max_splits);
  launch_pdl(decode_attn_kernel<DH, ST, MB>, dim3(grid), dim3(128), C::SMEM, st, a);
  EXG_CHECK_LAUNCH();
}

template <int DH>
void decode_attention_t(const DecodeAttnArgs& a, cudaStream_t st) {
  switch (decode_stages_override()) {
    case 1: decode_attention_st<DH, 1, 8>(a, st); break;
    case 2: decode_attention_st<DH, 2>(a, st); break;
    case 3: decode_attention_st<DH, 3>(a, st); break;
    case 4: decode_attention_st<DH, 4>(a, st); break;
    case 27: decode_attention_st<DH, 2, 7>(a, st); break;
    case 16: decode_attention_st<DH, 1, 6>(a, st); break;
    default: decode_attention_st<DH, 2, 7>(a, st); break;
  }
  if (a.max_splits > 1 && !a.counters) {
    launch_pdl(decode_combine_kernel<DH>, dim3(a.B * a.H), dim3(DH < 32 ? 32 : DH), 0, st, a);
    EXG_CHECK_LAUNCH();
  }
}

// diagnostics (exg_diag_decode_merge): 1 = merge splits in the separate
// combine kernel even when counters are given
int& decode_force_combine() {
  static int f = 0;
  return f;
}

void decode_attention(const DecodeAttnArgs& a_in, cudaStream_t st) {
  if (a_in.B <= 0) return;
  DecodeAttnArgs a = a_in;
  if (decode_force_combine()) a.counters = nullptr;
  if (a.kv.ptab && (a.max_ctx % 64 != 0 || a.split_len % a.max_ctx != 0))
    throw CudaError("decode_attention: the page length must be a multiple of 64 dividing the split length");
  switch (a.dh) {
    case 16: decode_attention_t<16>(a, st); break;
    case 64: decode_attention_t<64>(a, st); break;
    case 128: decode_attention_t<128>(a, st); break;
    default: throw CudaError("decode_attention: unsupported head dim " + std::to_string(a.dh));
  }
}

// ============================================================================
// K4 causal prefill attention (SIMT, fp32 softmax and P.V)
//
// CTA = 32 queries x 4 lanes of one (request, head); K/V tiles of 32 keys are
// staged in shared memory; each lane owns DH/4 dims of q and of the output.
// ============================================================================
template <int DH>
__global__ void __launch_bounds__(128) prefill_attn_kernel(PrefillAttnArgs a) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  constexpr int QPB = 32, LPQ = 4, DPL = DH / LPQ, KTILE = 32;
  __shared__ __align__(16) bf16 ks[KTILE][DH];
  __shared__ __align__(16) bf16 vs[KTILE][DH];
  const int r = blockIdx.z, h = blockIdx.y;
  const int t0 = a.cu_seqlens[r], len = a.cu_seqlens[r + 1] - t0;
  const int qb = blockIdx.x * QPB;
  if (qb >= len) return;
  const int tid = threadIdx.x, qi = tid / LPQ, part = tid % LPQ;
  const int qidx = qb + qi;
  const bool qvalid = qidx < len;
  const int p0 = a.pos0[r];
  const int my_pos = p0 + qidx;
  const int slot_r = a.slot[r];

  float q[DPL], o[DPL];
#pragma unroll
  for (int d = 0; d < DPL; ++d) {
    q[d] = qvalid ? bf2f(a.q[(int64_t)(t0 + qidx) * a.ldq + h * DH + part * DPL + d]) : 0.f;
    o[d] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const int last_key = a.causal ? p0 + min(len, qb + QPB) - 1 : p0 + len - 1;  // inclusive, for the whole CTA
  const float* brow = a.bias ? a.bias + (int64_t)h * a.bias_ld + a.bias_off - my_pos : nullptr;
  for (int kt = 0; kt <= last_key; kt += KTILE) {
    const int nkt = min(KTILE, last_key + 1 - kt);
    __syncthreads();
    // the 32-key tile lies inside one page (32 | P)
    const int64_t toff = kv_row(a.kv, r, slot_r, a.H, h, a.max_ctx, kt) * DH;
    for (int e = tid; e < nkt * DH / 8; e += blockDim.x) {
      const int row = e / (DH / 8), c = e % (DH / 8);
      *reinterpret_cast<int4*>(&ks[row][c * 8]) = *reinterpret_cast<const int4*>(a.kc + toff + (int64_t)row * DH + c * 8);
      *reinterpret_cast<int4*>(&vs[row][c * 8]) = *reinterpret_cast<const int4*>(a.vc + toff + (int64_t)row * DH + c * 8);
    }
    __syncthreads();
    float sc[KTILE];
    float tmax = -INFINITY;
#pragma unroll 4
    for (int j = 0; j < KTILE; ++j) {
      float dot = 0.f;
      if (j < nkt) {
#pragma unroll
        for (int d = 0; d < DPL; ++d) dot = fmaf(q[d], bf2f(ks[j][part * DPL + d]), dot);
      }
      dot += __shfl_xor_sync(0xffffffffu, dot, 1);
      dot += __shfl_xor_sync(0xffffffffu, dot, 2);
      const bool ok = qvalid && j < nkt && (!a.causal || (kt + j) <= my_pos);
      sc[j] = ok ? __fmul_rn(dot, a.scale) : -INFINITY;
      if (brow && ok) sc[j] = __fadd_rn(sc[j], brow[kt + j]);
      tmax = fmaxf(tmax, sc[j]);
    }
    if (tmax == -INFINITY) continue;
    const float m_new = fmaxf(m, tmax);
    const float alpha = (m == -INFINITY) ? 0.f : __expf(m - m_new);
    l *= alpha;
#pragma unroll
    for (int d = 0; d < DPL; ++d) o[d] *= alpha;
#pragma unroll 4
    for (int j = 0; j < KTILE; ++j) {
      if (sc[j] == -INFINITY) continue;
      const float p = __expf(sc[j] - m_new);
      l += p;
#pragma unroll
      for (int d = 0; d < DPL; ++d) o[d] = fmaf(p, bf2f(vs[j][part * DPL + d]), o[d]);
    }
    m = m_new;
  }
  if (qvalid) {
    const float inv = 1.f / l;
#pragma unroll
    for (int d = 0; d < DPL; ++d) a.out[(int64_t)(t0 + qidx) * a.ldo + h * DH + part * DPL + d] = f2bf(o[d] * inv);
  }
}

void prefill_attention(const PrefillAttnArgs& a, cudaStream_t st) {
  if (a.R <= 0 || a.max_len <= 0) return;
  if (a.kv.ptab && a.max_ctx % 64 != 0) throw CudaError("prefill_attention: the page length must be a multiple of 64");
  if (prefill_attention_tc(a, st)) return;
  dim3 grid((a.max_len + 31) / 32, a.H, a.R);
  switch (a.dh) {
    case 16: launch_pdl(prefill_attn_kernel<16>, grid, dim3(128), 0, st, a); break;
    case 64: launch_pdl(prefill_attn_kernel<64>, grid, dim3(128), 0, st, a); break;
    case 128: launch_pdl(prefill_attn_kernel<128>, grid, dim3(128), 0, st, a); break;
    default: throw CudaError("prefill_attention: unsupported head dim");
  }
  EXG_CHECK_LAUNCH();
}

// ============================================================================
// K8 argmax (lowest index on ties)
// ============================================================================
__global__ void __launch_bounds__(256) argmax_kernel(int32_t* __restrict__ out, const float* __restrict__ logits,
                                                      int64_t ld, int V, int32_t* err) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  __shared__ float sv[256];
  __shared__ int si[256];
  const float* row = logits + (int64_t)blockIdx.x * ld;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  bool nan = false;
  for (int j = threadIdx.x; j < V; j += 256) {
    const float v = row[j];
    if (v != v) nan = true;
    if (v > best || (v == best && j < bi)) {
      best = v;
      bi = j;
    }
  }
  if (nan && err) atomicExch(err, 1);
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const float ov = sv[threadIdx.x + s];
      const int oi = si[threadIdx.x + s];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = si[0] == 0x7fffffff ? 0 : si[0];
}

void argmax_rows(int32_t* out, const float* logits, int64_t ld, int B, int V, int32_t* err_flag, cudaStream_t st) {
  if (B <= 0) return;
  launch_pdl(argmax_kernel, dim3(B), dim3(256), 0, st, out, logits, ld, V, err_flag);
  EXG_CHECK_LAUNCH();
}

}  // namespace exg

extern "C" void exg_diag_decode_stages(int s) { exg::decode_stages_override() = s; }
extern "C" void exg_diag_decode_split(int s) { exg::decode_split_override() = s >= 128 ? s : 0; }
extern "C" void exg_diag_decode_merge(int force_combine) { exg::decode_force_combine() = force_combine; }
extern "C" void exg_diag_ln_preload(int on) { exg::ln_preload_segments() = on; }
