/*
 * exegpt_ops.h -- op-level C-ABI of libexegpt.so: the individual sm_100a
 * kernels of the hot path, exposed for kernel parity tests and for timing
 * the dominant kernel in bench.py.  Same conventions as exegpt.h, except:
 *
 *  - every data pointer here is a DEVICE pointer (cudaMalloc'd or a torch
 *    CUDA tensor's data_ptr) owned by the caller;
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream); the call only enqueues work (asynchronous);
 *  - bf16 tensors are passed as void* holding IEEE bfloat16 values.
 *
 * Operation definitions cite PAPER.md / SURVEY.md §8(c); shapes below.
 */
#ifndef EXEGPT_OPS_H
#define EXEGPT_OPS_H

#include <stdint.h>

#include "exegpt.h"

#ifdef __cplusplus
extern "C" {
#endif

/* K14 -- seeded weights.  dst: bf16 [rows][ld]; element
 * (r,c) is value index i = transposed ? (c+col_off)*canon_cols + (r+row_off)
 * : (r+row_off)*canon_cols + (c+col_off) of tensor `tensor_id`;
 * gain = 1 for norm gains 1+U(+-0.1), else U(+-sqrt(3)*0.02).  blocked = 1
 * writes the GEMM blocked layout (below) of the [rows][cols] matrix instead
 * (ld ignored, exg_op_blocked_elems(rows, cols) elements; the padding of the
 * last tiles is not written -- zero-fill the destination first). */
exg_status exg_op_weightgen(void* dst, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint64_t tensor_id,
                            int32_t gain, int32_t transposed, int64_t canon_cols, int64_t row_off, int64_t col_off,
                            int32_t blocked, void* stream);

/* GEMM weight layout: W [rows][K] is stored as 128 x 64 tiles, tile (m, kb)
 * a contiguous 16 KB block at element (m*ceil(K/64) + kb) * 8192 holding
 * row r's 8-element chunk c at r*64 + ((c ^ (r & 7)) * 8) (the SWIZZLE_128B
 * shared-memory image), zero padded to whole tiles.  pack: row-major src
 * [rows][ld] -> blocked dst. */
exg_status exg_op_pack_weight(void* dst, const void* src, int64_t rows, int64_t K, int64_t ld, void* stream);
int64_t exg_op_blocked_elems(int64_t rows, int64_t K);

/* K3/K5/K8 -- Y[tokens][features] = X[tokens][K] . W[features][K]^T, X
 * row-major with leading dim ldx, W given as Wb in the blocked layout, with
 * epilogue `mode`: 0 bf16(acc+bias) -> out; 1 bf16(act(acc+bias)) -> out
 * (act 1 = ReLU, 2 = GELU-tanh); 2 resid(fp32) += acc+bias; 3 fp32 acc+bias
 * -> out.  bias: bf16 [features] or NULL.  decode = 1 selects the swap-AB
 * tcgen05 path (tokens on the MMA N axis) with a deterministic stream-K split
 * of the weight stream (cut points depend on the weight shape only; ws:
 * fp32 scratch of exg_op_decode_workspace(features, K, tokens) floats), else
 * the data-parallel prefill path (ws unused). */
exg_status exg_op_linear(const void* X, int64_t ldx, const void* Wb, int32_t tokens, int32_t features, int32_t K,
                         int32_t mode, int32_t act, const void* bias, void* out, int64_t ldo, float* resid,
                         int64_t ldr, int32_t decode, float* ws, int64_t ws_floats, void* stream);

/* K2 -- y bf16 [T][ldy] = LN(x fp32 [T][ldx]) * g + b, eps, fp32 statistics. */
exg_status exg_op_layernorm(void* y, int64_t ldy, const float* x, int64_t ldx, const void* g, const void* b, int32_t T,
                            int32_t d, float eps, void* stream);

/* T5 RMSNorm (SURVEY.md §8(c) T1 T5 reading): y bf16 [T][d] =
 * bf16(x rsqrt(mean_j x^2 + eps) g out_scale), fp32 statistics.  out_scale
 * folds the tied LM head's d^-1/2 into the final norm. */
exg_status exg_op_rmsnorm(void* y, int64_t ldy, const float* x, int64_t ldx, const void* g, int32_t T, int32_t d,
                          float eps, float out_scale, void* stream);

/* K1 -- x fp32 [T][d] = tok_emb[ids[t]] + pos_emb[pos[t]] (bf16 tables;
 * pos_emb NULL: no position term, T5). */
exg_status exg_op_embed(float* x, const int32_t* ids, const int32_t* pos, const void* tok_emb, const void* pos_emb,
                        int32_t T, int32_t d, void* stream);

/* K7 -- copy the K and V column blocks of qkv bf16 [T][3*H*dh] into cache
 * [slot][H][max_ctx][dh] at (slot[t], pos[t]). */
exg_status exg_op_kv_scatter(void* kc, void* vc, const void* qkv, const int32_t* slot, const int32_t* pos, int32_t T,
                             int32_t H, int32_t dh, int32_t max_ctx, void* stream);

/* K6 -- ragged decode attention (incremental decoding):
 * out[i][h] = bf16( softmax_j( fp32(q_i,h . K[slot_i][h][j]) * scale ) . V )
 * over j < n_keys[i].  q: bf16 rows of stride ldq (head h at h*dh); out:
 * bf16 [B][ldo].  Keys are split in fixed chunks of split_len; partial: fp32
 * [B][H][max_splits][dh+2] scratch when max_splits > 1.  bias (may be NULL):
 * fp32 additive score bias, key j of row i / head h gets
 * bias[h*bias_ld + bias_off + j - (n_keys[i]-1)] after the scale (T5 relative
 * position bias; the query is the newest key). */
exg_status exg_op_decode_attention(const void* q, int64_t ldq, const void* kc, const void* vc, const int32_t* slot,
                                   const int32_t* n_keys, void* out, int64_t ldo, int32_t B, int32_t H, int32_t dh,
                                   int32_t max_ctx, float scale, int32_t split_len, int32_t max_splits, float* partial,
                                   const float* bias, int32_t bias_ld, int32_t bias_off, void* stream);

/* K4 -- causal prefill attention over packed requests (cu_seqlens [R+1],
 * T = cu_seqlens[R] tokens, q rows [T][ldq]); request r's tokens sit at
 * positions pos0[r].. of slot[r] and attend to cached keys 0..own position
 * (keys scattered beforehand); cache [n_slots][H][max_ctx][dh].  dh = 128
 * runs on tcgen05 (S and O in TMEM, P rounded to bf16 for P.V); other head
 * dims on a SIMT kernel with fp32 P.  causal = 0: every query sees all keys
 * of its request (T5 encoder).  bias (may be NULL): score(q, k) +=
 * bias[h*bias_ld + bias_off + kpos - qpos] after the scale. */
exg_status exg_op_prefill_attention(const void* q, int64_t ldq, const void* kc, const void* vc,
                                    const int32_t* cu_seqlens, const int32_t* slot, const int32_t* pos0, int32_t R,
                                    int32_t max_len, void* out, int64_t ldo, int32_t H, int32_t dh, int32_t max_ctx,
                                    int32_t n_slots, int32_t T, float scale, int32_t causal, const float* bias,
                                    int32_t bias_ld, int32_t bias_off, void* stream);

/* Paged KV variants of K6 / K4: the
 * cache is [n_pages][H][max_ctx][dh] with max_ctx = the page length P (a
 * multiple of 64; for K6 it divides split_len), and key k of row i (K6: decode
 * row; K4: request r) lives in page page_table[i*maxp + k/P] at offset k mod
 * P.  page_table: device int32 [rows][maxp], caller-owned; every entry a row's
 * keys reach must name a page of the cache (K4 reads whole 64-key halves of
 * its 128-key tiles up to the row's last key).  slot[] must still be valid
 * device memory of B (K6) / R (K4) entries but does not address the cache.
 * Same arithmetic as the slot variants: identical results for identical key
 * values.  EXG_E_INPUT on a null page_table, maxp < 1 or a page length that is
 * not a multiple of 64 (K6: also one that does not divide split_len). */
exg_status exg_op_decode_attention_paged(const void* q, int64_t ldq, const void* kc, const void* vc,
                                         const int32_t* slot, const int32_t* n_keys, void* out, int64_t ldo,
                                         int32_t B, int32_t H, int32_t dh, int32_t max_ctx, float scale,
                                         int32_t split_len, int32_t max_splits, float* partial, const float* bias,
                                         int32_t bias_ld, int32_t bias_off, const int32_t* page_table, int32_t maxp,
                                         void* stream);
exg_status exg_op_prefill_attention_paged(const void* q, int64_t ldq, const void* kc, const void* vc,
                                          const int32_t* cu_seqlens, const int32_t* slot, const int32_t* pos0,
                                          int32_t R, int32_t max_len, void* out, int64_t ldo, int32_t H, int32_t dh,
                                          int32_t max_ctx, int32_t n_slots, int32_t T, float scale, int32_t causal,
                                          const float* bias, int32_t bias_ld, int32_t bias_off,
                                          const int32_t* page_table, int32_t maxp, void* stream);

/* K8 -- out[i] = argmax_v logits[i][v] (fp32 [B][ld]), lowest index on ties;
 * *err_flag (device int32, may be NULL) set to 1 on a NaN. */
exg_status exg_op_argmax(int32_t* out, const float* logits, int64_t ld, int32_t B, int32_t V, int32_t* err_flag,
                         void* stream);

/* fp32 scratch (floats) a decode GEMM of this weight shape needs for up to
 * `tokens` rows (stream-K partial segments). */
int64_t exg_op_decode_workspace(int32_t features, int32_t K, int32_t tokens);

#ifdef __cplusplus
}
#endif
#endif /* EXEGPT_OPS_H */
