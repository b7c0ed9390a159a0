// fp32 parity path (north_star: logits within 1e-4 of
// the fp64 oracle, mode (ii)).  PAPER.md computes in FP16 throughout
// (PAPER.md:431-434); this path exists so the method's result -- greedy
// decoding of each request in isolation (R1) -- can be checked against the
// plain fp64 definition without the bf16 rounding points of T4.
//
// Everything is fp32 end to end: residual, norm outputs, q/k/v, the KV
// cache, attention context, FFN activations, logits.  The weights are the
// same bf16-representable values as the bf16 path (T3), read from the same
// blocked HBM layout and widened exactly.  tcgen05 has no fp32 MMA kind and
// TF32 would lose 13 mantissa bits, so the contractions are FFMA (SIMT) with
// fp32 accumulation; softmax uses precise expf, GELU precise tanhf (the
// library is built without fast-math).  Speed is not the point of this path:
// it serves the config-1 parity run.
#include <cmath>

#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace exg {

namespace {
constexpr int F32_TT = 64, F32_TF = 64, F32_TK = 16;   // GEMM tile: tokens x features x k

// y[t][:] = (x[t] - mean) / sqrt(var + eps) * g + b  (biased variance, two
// passes over the row, fp32)
__global__ void __launch_bounds__(256) ln_f32_kernel(float* __restrict__ y, int64_t ldy, const float* __restrict__ x,
                                                     int64_t ldx, const bf16* __restrict__ g,
                                                     const bf16* __restrict__ b, int d, float eps) {
  __shared__ float red[256];
  const float* xr = x + (int64_t)blockIdx.x * ldx;
  float s = 0.f;
  for (int j = threadIdx.x; j < d; j += 256) s += xr[j];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  const float mean = red[0] / (float)d;
  __syncthreads();
  float v = 0.f;
  for (int j = threadIdx.x; j < d; j += 256) {
    const float c = xr[j] - mean;
    v += c * c;
  }
  red[threadIdx.x] = v;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  const float inv = 1.0f / sqrtf(red[0] / (float)d + eps);
  float* yr = y + (int64_t)blockIdx.x * ldy;
  for (int j = threadIdx.x; j < d; j += 256) yr[j] = (xr[j] - mean) * inv * bf2f(g[j]) + bf2f(b[j]);
}

__device__ __forceinline__ float act_f32(float v, int act) {
  if (act == ACT_RELU) return fmaxf(v, 0.f);
  if (act == ACT_GELU) {
    const float k0 = 0.7978845608028654f;   // sqrt(2/pi)
    return 0.5f * v * (1.f + tanhf(k0 * (v + 0.044715f * v * v * v)));
  }
  return v;
}

// Y[t][f] = sum_k X[t][k] W[f][k] (+ bias[f]) with W in the blocked bf16
// layout of a [F][K] matrix.  mode: EPI_F32 (out = acc + bias), EPI_BF16_ACT
// reused as "fp32 out = act(acc + bias)", EPI_RESID (resid += acc + bias).
__global__ void __launch_bounds__(256) gemm_f32_kernel(const float* __restrict__ X, int64_t ldx,
                                                       const bf16* __restrict__ Wb, int T, int F, int K,
                                                       const bf16* __restrict__ bias, int mode, int act,
                                                       float* __restrict__ out, int64_t ldo) {
  __shared__ float As[F32_TK][F32_TT + 4];
  __shared__ float Ws[F32_TK][F32_TF + 4];
  const int t0 = blockIdx.y * F32_TT, f0 = blockIdx.x * F32_TF;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;   // 16 x 16 threads, 4 x 4 outputs each
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += F32_TK) {
    for (int e = threadIdx.x; e < F32_TT * F32_TK; e += 256) {
      const int r = e / F32_TK, c = e % F32_TK;
      const int t = t0 + r, k = k0 + c;
      As[c][r] = (t < T && k < K) ? X[(int64_t)t * ldx + k] : 0.f;
      const int f = f0 + r;
      Ws[c][r] = (f < F && k < K) ? bf2f(Wb[blocked_index(f, k, K)]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < F32_TK; ++c) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[c][ty * 4 + i];
        w[i] = Ws[c][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int t = t0 + ty * 4 + i;
    if (t >= T) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int f = f0 + tx * 4 + j;
      if (f >= F) continue;
      float v = acc[i][j] + (bias ? bf2f(bias[f]) : 0.f);
      float* o = out + (int64_t)t * ldo + f;
      if (mode == EPI_RESID)
        *o = *o + v;
      else
        *o = mode == EPI_BF16_ACT ? act_f32(v, act) : v;
    }
  }
}

// K,V columns of qkv row t -> cache (slot[t], head, pos[t])
__global__ void kv_scatter_f32_kernel(float* __restrict__ kc, float* __restrict__ vc, const float* __restrict__ qkv,
                                      int64_t ldqkv, int inner, const int32_t* __restrict__ slot,
                                      const int32_t* __restrict__ pos, int H, int dh, int ctx) {
  const int t = blockIdx.x;
  const int64_t base = (int64_t)slot[t] * H * ctx;
  for (int j = threadIdx.x; j < inner; j += blockDim.x) {
    const int h = j / dh, c = j % dh;
    const int64_t o = ((base + (int64_t)h * ctx) + pos[t]) * dh + c;
    kc[o] = qkv[(int64_t)t * ldqkv + inner + j];
    vc[o] = qkv[(int64_t)t * ldqkv + 2 * inner + j];
  }
}

// One warp per (query row i, head h): scores over keys 0..pos[i] of slot[i]
// (causal: a request's keys sit at positions 0..its own in its slot), s =
// fp32(q.k) * scale, p = expf(s - max), out = sum_j p_j v_j / sum_j p_j.
constexpr int ATT_WARPS = 4;
__global__ void __launch_bounds__(32 * ATT_WARPS) attn_f32_kernel(const float* __restrict__ q, int64_t ldq,
                                                                  const float* __restrict__ kc,
                                                                  const float* __restrict__ vc,
                                                                  const int32_t* __restrict__ slot,
                                                                  const int32_t* __restrict__ pos, int rows, int H,
                                                                  int dh, int ctx, float scale,
                                                                  float* __restrict__ out, int64_t ldo) {
  extern __shared__ float sc[];   // [ATT_WARPS][ctx]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * ATT_WARPS + warp;
  if (item >= rows * H) return;
  const int i = item / H, h = item % H;
  float* s = sc + (int64_t)warp * ctx;
  const int nk = pos[i] + 1;
  const float* qr = q + (int64_t)i * ldq + (int64_t)h * dh;
  const int64_t kv0 = ((int64_t)slot[i] * H + h) * ctx * dh;
  float mx = -INFINITY;
  for (int j = lane; j < nk; j += 32) {
    const float* kr = kc + kv0 + (int64_t)j * dh;
    float dot = 0.f;
    for (int c = 0; c < dh; ++c) dot = fmaf(qr[c], kr[c], dot);
    const float v = dot * scale;
    s[j] = v;
    mx = fmaxf(mx, v);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
  for (int j = lane; j < nk; j += 32) {
    const float p = expf(s[j] - mx);
    s[j] = p;
    sum += p;
  }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncwarp();
  float* orow = out + (int64_t)i * ldo + (int64_t)h * dh;
  for (int c = lane; c < dh; c += 32) {
    float a = 0.f;
    for (int j = 0; j < nk; ++j) a = fmaf(s[j], vc[kv0 + (int64_t)j * dh + c], a);
    orow[c] = a / sum;
  }
}
}  // namespace

void layernorm_f32(float* y, int64_t ldy, const float* x, int64_t ldx, const bf16* g, const bf16* b, int T, int d,
                   float eps, cudaStream_t st) {
  if (T <= 0) return;
  ln_f32_kernel<<<T, 256, 0, st>>>(y, ldy, x, ldx, g, b, d, eps);
  EXG_CHECK_LAUNCH();
}

void linear_f32(const float* X, int64_t ldx, const bf16* Wb, int T, int F, int K, const bf16* bias, int mode, int act,
                float* out, int64_t ldo, cudaStream_t st) {
  if (T <= 0 || F <= 0) return;
  dim3 grid((F + F32_TF - 1) / F32_TF, (T + F32_TT - 1) / F32_TT);
  gemm_f32_kernel<<<grid, 256, 0, st>>>(X, ldx, Wb, T, F, K, bias, mode, act, out, ldo);
  EXG_CHECK_LAUNCH();
}

void kv_scatter_f32(float* kc, float* vc, const float* qkv, int64_t ldqkv, int inner, const int32_t* slot,
                    const int32_t* pos, int T, int H, int dh, int ctx, cudaStream_t st) {
  if (T <= 0) return;
  kv_scatter_f32_kernel<<<T, 128, 0, st>>>(kc, vc, qkv, ldqkv, inner, slot, pos, H, dh, ctx);
  EXG_CHECK_LAUNCH();
}

void attention_f32(const float* q, int64_t ldq, const float* kc, const float* vc, const int32_t* slot,
                   const int32_t* pos, int rows, int H, int dh, int ctx, float scale, float* out, int64_t ldo,
                   cudaStream_t st) {
  if (rows <= 0) return;
  const size_t smem = sizeof(float) * ATT_WARPS * (size_t)ctx;
  if (smem > 48 * 1024) EXG_CUDA(cudaFuncSetAttribute(attn_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int items = rows * H;
  attn_f32_kernel<<<(items + ATT_WARPS - 1) / ATT_WARPS, 32 * ATT_WARPS, smem, st>>>(q, ldq, kc, vc, slot, pos, rows,
                                                                                     H, dh, ctx, scale, out, ldo);
  EXG_CHECK_LAUNCH();
}

}  // namespace exg
