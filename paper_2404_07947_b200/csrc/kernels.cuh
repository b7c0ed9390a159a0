// Non-GEMM kernels of the hot path: K14 weight generator,
// K1 embedding, K2 LayerNorm, K7 KV scatter/append, K6 ragged decode
// attention, K4 prefill attention, K8 argmax, K9 row compaction.
#pragma once
#include "common.cuh"
#include "gemm_tc.cuh"

namespace exg {

// ---- K14: seeded weights -----------------------------
// dst is a [rows][cols] bf16 matrix (leading dim ld).  Element (r, c) takes
// the canonical index
//   transposed = 0: i = (r + row_off) * canon_cols + (c + col_off)
//   transposed = 1: i = (c + col_off) * canon_cols + (r + row_off)
// (transposed = 1 stores W^T[out][in] of a canonical W[in][out]).
struct GenParams {
  uint64_t seed;
  uint64_t tensor_id;
  int gain;            // 1: 1 + U(+-0.1); 0: U(+-sqrt(3) sigma)
  float c_mat;         // fp32(2 sqrt(3) sigma)
  float c_gain;        // fp32(0.2)
  int transposed;
  int64_t canon_cols;
  int64_t row_off, col_off;
  int blocked;         // 1: write the GEMM blocked layout (gemm_tc.cuh) of a matrix
                       //    with `cols` columns (padding left as is: zero-fill first)
  int64_t dst_row0;    // blocked: first destination row
};
void weightgen(bf16* dst, int64_t rows, int64_t cols, int64_t ld, const GenParams& p, cudaStream_t st);

// ---- K1: x[t] = tok_emb[ids[t]] + pos_emb[pos[t]]  (fp32 residual) ---------
// tok_blocked = 1: tok_emb is in the GEMM blocked layout ([V][d] blocks).
void embed(float* x, const int32_t* ids, const int32_t* pos, const bf16* tok_emb, const bf16* pos_emb, int T,
           int d, cudaStream_t st, int tok_blocked = 0);

// ---- K2: y = bf16(LN(x) * g + b), fp32 statistics, eps 1e-5 ----------------
void layernorm(bf16* y, int64_t ldy, const float* x, int64_t ldx, const bf16* g, const bf16* b, int T, int d,
               float eps, cudaStream_t st);
// the same after folding a deferred residual GEMM (gemm_tc.cuh SegInfo):
// x += sum_seg P[seg][row][:] + rbias, written back, then LN.  Returns false
// (nothing launched) when the shape needs the strided kernels.
bool layernorm_deferred(bf16* y, int64_t ldy, float* x, int64_t ldx, const float* P, const SegInfo& si,
                        const bf16* rbias, const bf16* g, const bf16* b, int T, int d, float eps, cudaStream_t st);

// ---- T5 RMSNorm: y = bf16(x rsqrt(mean(x^2) + eps) g out_scale) ----------
void rmsnorm(bf16* y, int64_t ldy, const float* x, int64_t ldx, const bf16* g, int T, int d, float eps,
             float out_scale, cudaStream_t st);
// fp32 table tab[h][j] = rel[bucket[j]][h0 + h], h < Hl, j < n (T5 relative
// attention bias, bucket[] precomputed on the host, T9)
void rel_bias_table(float* tab, const bf16* rel, const int32_t* bucket, int n, int Hl, int H_total, int h0,
                    cudaStream_t st);

// ---- KV blocks: slots or pages -----------------------------------------------
// The cache of a layer is an array of blocks [block][H][max_ctx][dh] (K and V
// separately).  Slot mode (ptab == nullptr): block = the row's slot, max_ctx
// = the slot length, key k at offset k.  Paged mode (NEXT-2):
// max_ctx = the page length P (a multiple of 64), the row's page table
// ptab[row * maxp + j] holds the page of keys [jP, (j+1)P), key k at offset
// k mod P.  Every tile the kernels stream (32 / 64 / 128 keys, aligned to
// its size from key 0) lies inside one page.
struct KvMap {
  const int32_t* ptab = nullptr;   // [rows][maxp] (row = decode row / encode request)
  int maxp = 0;
};
// cache row index (in units of dh elements) of key k of (row, head h)
__device__ __forceinline__ int64_t kv_row(const KvMap& m, int row, int slot, int H, int h, int max_ctx, int k) {
  if (!m.ptab) return ((int64_t)slot * H + h) * max_ctx + k;
  const int pg = __ldg(m.ptab + (int64_t)row * m.maxp + k / max_ctx);
  return ((int64_t)pg * H + h) * max_ctx + k % max_ctx;
}

// ---- K7: scatter the K,V columns of a fused qkv buffer into cache slots -----
// qkv: [T][3*inner] bf16; token t goes to block slot[t], offset pos[t] (slot
// mode: its slot and position; paged mode: its page and position mod P).
// Cache layout per layer: [block][H][max_ctx][dh] for K and for V.
void kv_scatter(bf16* kc, bf16* vc, const bf16* qkv, const int32_t* slot, const int32_t* pos, int T, int H,
                int dh, int max_ctx, cudaStream_t st);

// ---- K6: ragged decode attention -------------------------------------------
// Row i attends with q_i (head h at q + i*ldq + h*dh) over keys 0..n_keys[i]-1
// of slot[i].  out[i][h*dh..] = bf16(softmax(fp32(q.k) * scale) . V).
// Keys are processed in fixed chunks of `split_len` (a constant of the
// model, never the batch) -- splits > 1 are merged by a combine pass in
// split order, so a row's bits never depend on its batch-mates (T13).
struct DecodeAttnArgs {
  const bf16* q;
  int64_t ldq;
  const bf16* kc;
  const bf16* vc;
  const int32_t* slot;
  const int32_t* n_keys;
  bf16* out;
  int64_t ldo;
  int B, H, dh, max_ctx;   // max_ctx: slot length, or the page length when paged
  float scale;
  int split_len;           // a multiple of the page length when paged
  int max_splits;      // >= ceil(max_i n_keys[i] / split_len)
  float* partial;      // [B][H][max_splits][dh + 2] when max_splits > 1
  // optional [B][H] zeroed counters: the last split CTA of a (row, head)
  // merges the splits in-kernel (no combine launch); null -> combine kernel
  int32_t* counters = nullptr;
  // optional additive score bias (T5 relative position bias): the score of
  // key k of row i, head h gets bias[h * bias_ld + bias_off + k - (n_keys[i]-1)]
  const float* bias = nullptr;
  int bias_ld = 0, bias_off = 0;
  // optional fused KV append (K7): the new token of row i -- key n_keys[i]-1
  // -- is read from knew / vnew [B][ldnew] (head h at h * dh) instead of the
  // cache, and written to the cache at that position by the CTA whose split
  // holds it (the cache need not contain it before the launch)
  const bf16* knew = nullptr;
  const bf16* vnew = nullptr;
  int64_t ldnew = 0;
  // deferred QKV reduction (gemm_tc.cuh): when qkv_part is set, q / knew /
  // vnew of row i are bf16(sum_seg qkv_part[seg][i][f] + qkv_bias[f]) with f
  // = h*dh + j, inner + h*dh + j, 2 inner + h*dh + j (q, knew, vnew ignored)
  const float* qkv_part = nullptr;
  SegInfo qkv_si;
  const bf16* qkv_bias = nullptr;
  int qkv_inner = 0;
  KvMap kv;   // paged mode: page table of the decode rows (max_ctx = page length)
};
void decode_attention(const DecodeAttnArgs& a, cudaStream_t st);
int& decode_split_override();   // diagnostics: key split length (0 = default)

// ---- K4: causal prefill attention over packed variable-length requests -----
// Token t of request r (cu_seqlens[r] <= t < cu_seqlens[r+1]) sits at
// position pos0[r] + (t - cu_seqlens[r]) of slot[r]; it attends to cached
// keys 0..its own position (the keys must already be scattered).
struct PrefillAttnArgs {
  const bf16* q;
  int64_t ldq;
  const bf16* kc;
  const bf16* vc;
  const int32_t* cu_seqlens;   // [R+1]
  const int32_t* slot;         // [R]
  const int32_t* pos0;         // [R]
  int R, max_len;
  bf16* out;
  int64_t ldo;
  int H, dh, max_ctx;  // max_ctx: slot length, or the page length when paged
  float scale;
  int64_t q_rows;      // rows of the qkv buffer (tokens)
  int64_t kv_rows;     // blocks * H * max_ctx
  // causal = 0: every query attends to all keys pos0 .. pos0+len-1 of its
  // request (T5 encoder); bias: score(q, k) += bias[h * bias_ld + bias_off + kpos - qpos]
  int causal = 1;
  const float* bias = nullptr;
  int bias_ld = 0, bias_off = 0;
  KvMap kv;   // paged mode: page table of the requests, row = r (max_ctx = page length)
};
// dh = 128: tcgen05 FMHA (attn_prefill_tc.cu); other head dims: SIMT kernel
void prefill_attention(const PrefillAttnArgs& a, cudaStream_t st);
bool prefill_attention_tc(const PrefillAttnArgs& a, cudaStream_t st);

// ---- fp32 parity path (fp32_path.cu) -------------------
// y = LN(x) * g + b in fp32 (biased variance, eps)
void layernorm_f32(float* y, int64_t ldy, const float* x, int64_t ldx, const bf16* g, const bf16* b, int T, int d,
                   float eps, cudaStream_t st);
// FFMA GEMM: out[t][f] (=, += for EPI_RESID) X[t][:] . W[f][:] + bias[f] with W
// the blocked bf16 [F][K] layout; mode EPI_F32 | EPI_BF16_ACT (fp32 act(.)) |
// EPI_RESID
void linear_f32(const float* X, int64_t ldx, const bf16* Wb, int T, int F, int K, const bf16* bias, int mode, int act,
                float* out, int64_t ldo, cudaStream_t st);
// K, V columns [inner, 3 inner) of qkv row t -> fp32 cache (slot[t], h, pos[t])
void kv_scatter_f32(float* kc, float* vc, const float* qkv, int64_t ldqkv, int inner, const int32_t* slot,
                    const int32_t* pos, int T, int H, int dh, int ctx, cudaStream_t st);
// row i attends over keys 0..pos[i] of slot[i] (causal), fp32 softmax with expf
void attention_f32(const float* q, int64_t ldq, const float* kc, const float* vc, const int32_t* slot,
                   const int32_t* pos, int rows, int H, int dh, int ctx, float scale, float* out, int64_t ldo,
                   cudaStream_t st);

// ---- K8: greedy argmax per row (lowest index wins ties; NaN -> err flag) ---
void argmax_rows(int32_t* out, const float* logits, int64_t ld, int B, int V, int32_t* err_flag, cudaStream_t st);

}  // namespace exg
