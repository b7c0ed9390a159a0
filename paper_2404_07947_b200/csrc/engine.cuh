// Device-side model shard: seeded weights in HBM, activation workspace, KV
// slot pool, and the encode (prefill) / decode forward passes built from the
// sm_100a kernels.
//
// An Engine holds the layers [l0, l1) of the model, tensor-parallel rank
// tp_rank of tp (heads and FFN columns split as in Megatron),
// plus the embeddings if it is a first stage and the final norm + LM head if
// it is a last stage.  A single-GPU model is the shard {0, L, 1, 0, true,
// true}.  Pipelines, TP groups and WAA encoder/decoder sets are built from
// several Engines by the executors (runner.cu, multi.cu).
#pragma once
#include <memory>
#include <vector>

#include "../../include/exegpt.h"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace exg {

struct LayerW {
  bf16 *ln1_g = nullptr, *ln1_b = nullptr, *Wqkv = nullptr, *bqkv = nullptr, *Wo = nullptr, *bo = nullptr;
  bf16 *ln2_g = nullptr, *ln2_b = nullptr, *W1 = nullptr, *b1 = nullptr, *W2 = nullptr, *b2 = nullptr;
  // T5 decoder cross-attention: RMS gain, W_q_x^T, W_kv_x^T, W_o_x^T
  bf16 *lnx_g = nullptr, *Wqx = nullptr, *Wkvx = nullptr, *Wox = nullptr;
};

struct Dims {
  int arch, L, d, H, dh, inner, ff, V, max_pos, act;
  bool f32 = false;   // fp32 parity path (fp32_path.cu)
  uint64_t seed;
  // local (tensor-parallel shard) sizes
  int Hl, inner_l, ffl;
};

struct EngineShard {
  int l0 = 0, l1 = -1;        // layer range (l1 = -1: all layers)
  int tp = 1, tp_rank = 0;    // tensor-parallel degree and rank
  bool embed = true;          // first stage: token + position embeddings
  bool head = true;           // last stage: final LayerNorm + tied LM head + argmax
  // T5 (tp = 1): 0 = encoder and decoder layers [l0, l1) (single GPU);
  // 1 = WAA encoder side: encoder layers [l0, l1), and if enc_last the final
  //     encoder norm + the cross K/V projections of every decoder layer (K13);
  // 2 = WAA decoder side: decoder layers [l0, l1) with their cross caches
  int t5_role = 0;
  bool enc_last = true;
};

// TP reduction of fp32 partial sums (O-projection / FFN2 outputs, T4(i)).
struct Reducer {
  virtual ~Reducer() = default;
  // in-place sum over the TP group; called by every rank of the group
  virtual void allreduce_sum(float* buf, int64_t n, cudaStream_t st) = 0;
};

// Packed encode batch, device arrays (see Engine::encode).
struct EncodeBatch {
  int T = 0, R = 0, max_len = 0;
  double attn_pairs = 0;   // sum_r n_r (n_r + 1) / 2   (prefill-attention work)
  const int32_t *ids = nullptr, *pos = nullptr, *tslot = nullptr;      // [T]
  const int32_t *cu = nullptr, *rslot = nullptr, *pos0 = nullptr;      // [R+1], [R], [R]
  // paged KV (NEXT-2): token t's K / V go to page kv_blk[t] at offset
  // kv_off[t] (= pos mod P) and request r's keys are found through kv.ptab
  // row r; null / empty = slot mode (tslot, pos)
  const int32_t *kv_blk = nullptr, *kv_off = nullptr;                  // [T]
  KvMap kv;
};

// Decode batch: B active rows, device arrays.
struct DecodeBatch {
  int B = 0, max_keys = 0;
  double sum_keys = 0;     // sum_i n_keys[i]   (decode-attention work)
  const int32_t *slot = nullptr, *pos = nullptr, *nkeys = nullptr, *out_off = nullptr;
  int32_t* out_tokens = nullptr;   // device [sum S] (last stage)
  // encoder-decoder: cross-attention key counts (= input lengths) per row
  const int32_t* xkeys = nullptr;
  int max_xkeys = 0;
  double sum_xkeys = 0;
  // paged KV (NEXT-2): row i's self-attention keys through kv.ptab row i
  KvMap kv;
};

class Engine {
 public:
  // stream == nullptr: the engine creates its own non-blocking stream
  Engine(const exg_model_spec& spec, int device, const EngineShard& shard = EngineShard(),
         cudaStream_t stream = nullptr);
  ~Engine();
  Engine(const Engine&) = delete;

  const Dims& dims() const { return D; }
  const EngineShard& shard() const { return S_; }
  int n_layers() const { return S_.l1 - S_.l0; }
  int device() const { return dev_; }
  cudaStream_t stream() const { return st_; }
  void set_reducer(Reducer* r) { red_ = r; }

  void ensure_workspace(int max_tokens, int max_rows);
  // decoder self-attention KV (slot_ctx keys per slot); encoder-decoder
  // models also get the cross K/V cache of every decoder layer (xctx keys)
  // Paged mode: slots = pages, slot_ctx = the page length (the cache is
  // [block][Hl][block_len][dh] either way; batches carry the page tables).
  void ensure_kv(int slots, int slot_ctx, int layers = -1, int xctx = 0);
  // T5-style encoder-decoder: encode = encoder over all
  // n input tokens + cross K/V projections (K13); decode starts from token 0
  bool encdec() const { return t5_; }
  int t5_role() const { return S_.t5_role; }
  // decoder layers whose cross K/V this engine holds (xkc / xvc index range)
  int n_cross_layers() const { return t5_ ? (S_.t5_role == 1 ? (S_.enc_last ? D.L : 1) : n_layers()) : 0; }
  int xctx() const { return xctx_; }
  bf16* xkc(int l) const { return xkv_ + (size_t)l * 2 * xkv_layer_elems(); }
  bf16* xvc(int l) const { return xkc(l) + xkv_layer_elems(); }
  // K13: cross K/V of decoder layer l (all layers held: cross_kv_all) from
  // the encoder output (bf16 in h())
  void cross_kv(int l, const EncodeBatch& eb);
  void cross_kv_all(const EncodeBatch& eb);
  bf16* h() { return h_; }
  int kv_slots() const { return kv_slots_; }
  int slot_ctx() const { return slot_ctx_; }
  int32_t* last_tok() { return last_tok_; }
  // residual stream x [rows][d] fp32: the stage input (non-first stages) and
  // output (non-last stages)
  float* x() { return x_; }
  // KV cache of local layer l: [slot][Hl][slot_ctx][dh] (bf16; fp32 on the
  // fp32 path: kcf / vcf)
  bf16* kc(int l) const { return kv_ + (size_t)l * 2 * kv_layer_elems(); }
  bf16* vc(int l) const { return kc(l) + kv_layer_elems(); }
  float* kcf(int l) const { return reinterpret_cast<float*>(kv_) + (size_t)l * 2 * kv_layer_elems(); }
  float* vcf(int l) const { return kcf(l) + kv_layer_elems(); }
  bool fp32() const { return D.f32; }

  // prefill of the packed tokens through this shard's layers; writes K/V into
  // slots.  First stage: embeds eb.ids; otherwise x() holds the input rows.
  void encode(const EncodeBatch& eb);
  // one decode iteration for B rows.  First stage embeds last_tok[slot];
  // last stage: next ids -> last_tok[slot] and out_tokens[out_off[i]],
  // logits left in logits() ([B][V] fp32).
  void decode(const DecodeBatch& db);
  const float* logits() const { return logits_; }

  // single-layer helpers: XProfiler timing (part 0: attention and / or the
  // rest of layer l) and the blocks a lockstep TP group drives (part 1: up
  // to the attention output; part 2: the FFN)
  void layer_encode(int l, const EncodeBatch& eb, bool attn, bool rest, int part = 0);
  void layer_decode(int l, const DecodeBatch& db, bool attn, bool rest, int part = 0);

  // stage pieces, for executors that drive several engines
  void embed_encode(const EncodeBatch& eb);
  void embed_decode(const DecodeBatch& db);
  void head_decode(const DecodeBatch& db);
  // layer l around its two TP reductions: attention block (LN1 .. O-proj),
  // FFN block (LN2 .. FFN2).  tp > 1 without a reducer leaves the fp32
  // partial in part() for the group to sum; finish_pending() then adds it
  // and the bias to the residual.
  void enc_attn_block(int l, const EncodeBatch& eb);
  void enc_ffn_block(int l, const EncodeBatch& eb);
  void dec_attn_block(int l, const DecodeBatch& db);
  void dec_ffn_block(int l, const DecodeBatch& db);
  void finish_pending();
  float* part() { return part_; }

  int32_t* err_flag() { return err_; }
  // the runner's host-side state kept across runs (pinned staging ring,
  // events, table buffers): allocating and pinning it per run costs host
  // time that the end-to-end number pays
  std::shared_ptr<void>& run_cache() { return run_cache_; }
  size_t weight_bytes() const { return wbytes_; }

  // per-launch CUDA-event timing of the kernel classes of exegpt.h
  void set_kernel_timing(bool on);
  // after a stream sync: accumulate into t/w/n [EXG_K_CLASSES] and reset
  void collect_kernel_timing(double* t, double* w, int64_t* n);

 private:
  struct KRec {
    int cls, ev;
    double work;
  };
  bool ktiming_ = false;
  std::vector<cudaEvent_t> kev_;
  std::vector<KRec> krec_;
  int kbegin();
  void kend(int idx, int cls, double work);
  void gen_weights();
  void gen_weights_t5();
  void encode_t5(const EncodeBatch& eb);
  // fp32 parity path: the same layer, every intermediate in fp32
  void encode_f32(const EncodeBatch& eb);
  void decode_f32(const DecodeBatch& db);
  void layer_f32(int l, int rows, const int32_t* slot, const int32_t* pos);
  void enc_layer_t5(int l, const EncodeBatch& eb, bool attn, bool rest);
  void dec_layer_t5(int l, const DecodeBatch& db, bool attn, bool rest);
  void dattn(const bf16* q, int64_t ldq, const bf16* kc, const bf16* vc, int ctx, const DecodeBatch& db,
             const int32_t* nkeys, int max_keys, double sum_keys, const float* bias, bool append = false,
             KvMap kv = KvMap());
  void linear_dec(const bf16* X, int64_t ldx, int tokens, const bf16* W, int features, int K, EpiParams ep);
  void linear_pre(const bf16* X, int64_t ldx, int tokens, const bf16* W, int features, int K, EpiParams ep);
  // residual update x += W.act + b: fused epilogue (tp = 1) or partial ->
  // TP all-reduce -> add (tp > 1)
  void resid_update(bool decode, const bf16* X, int64_t ldx, int tokens, const bf16* W, int K, const bf16* bias);

  Dims D;
  EngineShard S_;
  int dev_;
  bool own_stream_ = false;
  cudaStream_t st_ = nullptr;
  Reducer* red_ = nullptr;
  const bf16* pend_bias_ = nullptr;
  int pend_rows_ = 0;
  uint8_t* wbuf_ = nullptr;
  size_t wbytes_ = 0;
  bf16 *tok_emb_ = nullptr, *pos_emb_ = nullptr, *lnf_g_ = nullptr, *lnf_b_ = nullptr;
  std::vector<LayerW> layers_;
  // encoder-decoder (T5)
  bool t5_ = false;
  std::vector<LayerW> enc_layers_;
  std::vector<bf16*> xproj_;   // role 1, enc_last: W_kv_x^T of every decoder layer
  bf16 *enc_lnf_g_ = nullptr, *enc_rel_ = nullptr, *dec_rel_ = nullptr;
  float *enc_bias_ = nullptr, *dec_bias_ = nullptr;   // fp32 [Hl][2 max_pos - 1], centre max_pos - 1
  int bias_ld_ = 0, bias_off_ = 0;
  bf16* xkv_ = nullptr;
  int xctx_ = 0;
  size_t xkv_layer_elems() const { return (size_t)kv_slots_ * D.Hl * xctx_ * D.dh; }
  // workspace
  int cap_tokens_ = 0, cap_rows_ = 0;
  float* x_ = nullptr;
  float* part_ = nullptr;        // TP partial sums [T][d]
  bf16 *h_ = nullptr, *qkv_ = nullptr, *ctx_ = nullptr, *ff_ = nullptr;
  float* logits_ = nullptr;
  // fp32 path activations: norm output, q|k|v, attention context, FFN1 output
  float *hf_ = nullptr, *qkvf_ = nullptr, *ctxf_ = nullptr, *fff_ = nullptr;
  // deferred stream-K reductions of the decode GEMMs (gemm_tc.cuh): QKV
  // segments summed by the decode attention, O-projection / FFN2 segments by
  // the following LayerNorm (decoder-only, tp = 1, bf16)
  int defer_ = 0;   // DEFER_QKV | DEFER_RESID
  float *defer_qkv_ = nullptr, *defer_res_ = nullptr;
  struct PendingResid {
    const float* P = nullptr;
    SegInfo si;
    const bf16* bias = nullptr;
  } pend_res_;
  // LayerNorm of x into h_, folding a pending deferred residual update first
  void ln_decode(const bf16* g, const bf16* b, int rows);
  // decode GEMM chain (gemm_tc.cuh decode_chain): one launch per layer for
  // O-proj, LN2, FFN1, FFN2 (+ LN1 and QKV of layer next_l when >= 0);
  // decoder-only, tp = 1, bf16
  bool chain_ = false;
  float* chain_ws_ = nullptr;
  size_t chain_ws_cap_ = 0;
  unsigned* chain_sync_ = nullptr;
  unsigned chain_epoch_ = 0;
  void dec_attention(int l, const DecodeBatch& db);
  void dec_rest_chain(int l, const DecodeBatch& db, int next_l);
  ChainSpec chain_spec(int l, int B, int next_l) const;
  float* splitk_ws_ = nullptr;
  size_t splitk_cap_ = 0;
  float* attn_part_ = nullptr;
  int32_t* attn_cnt_ = nullptr;
  int split_len_ = 512, max_splits_cap_ = 0;
  int split_len() const { return decode_split_override() ? decode_split_override() : split_len_; }
  int32_t* err_ = nullptr;
  // KV
  bf16* kv_ = nullptr;
  int kv_slots_ = 0, slot_ctx_ = 0, kv_layers_ = 0;
  int32_t* last_tok_ = nullptr;
  std::shared_ptr<void> run_cache_;

  size_t kv_layer_elems() const { return (size_t)kv_slots_ * D.Hl * slot_ctx_ * D.dh; }
};

// x[i][:] += p[i][:] + bias   (fp32 residual, bf16 bias), n = rows * d
void add_bias_resid(float* x, const float* p, const bf16* bias, int rows, int d, cudaStream_t st);

}  // namespace exg
