// Device-side model: seeded weights in HBM, activation workspace, KV slot
// pool, and the encode (prefill) / decode forward passes built from the
// sm_100a kernels.  One Engine per GPU (rank).
#pragma once
#include <vector>

#include "../../include/exegpt.h"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels.cuh"

namespace exg {

struct LayerW {
  bf16 *ln1_g, *ln1_b, *Wqkv, *bqkv, *Wo, *bo, *ln2_g, *ln2_b, *W1, *b1, *W2, *b2;
};

struct Dims {
  int arch, L, d, H, dh, inner, ff, V, max_pos, act;
  uint64_t seed;
};

// Packed encode batch, device arrays (see Engine::encode).
struct EncodeBatch {
  int T = 0, R = 0, max_len = 0;
  double attn_pairs = 0;   // sum_r n_r (n_r + 1) / 2   (prefill-attention work)
  const int32_t *ids = nullptr, *pos = nullptr, *tslot = nullptr;      // [T]
  const int32_t *cu = nullptr, *rslot = nullptr, *pos0 = nullptr;      // [R+1], [R], [R]
};

// Decode batch: B active rows, device arrays.
struct DecodeBatch {
  int B = 0, max_keys = 0;
  double sum_keys = 0;     // sum_i n_keys[i]   (decode-attention work)
  const int32_t *slot = nullptr, *pos = nullptr, *nkeys = nullptr, *out_off = nullptr;
  int32_t* out_tokens = nullptr;   // device [sum S]
  float* logits_keep = nullptr;    // optional: logits stay in Engine::logits
};

class Engine {
 public:
  Engine(const exg_model_spec& spec, int device);
  ~Engine();
  Engine(const Engine&) = delete;

  const Dims& dims() const { return D; }
  int device() const { return dev_; }
  cudaStream_t stream() const { return st_; }

  void ensure_workspace(int max_tokens, int max_rows);
  void ensure_kv(int slots, int slot_ctx, int layers = -1);
  int kv_slots() const { return kv_slots_; }
  int slot_ctx() const { return slot_ctx_; }
  int32_t* last_tok() { return last_tok_; }

  // prefill of the packed tokens through every layer; writes K/V into slots
  void encode(const EncodeBatch& eb);
  // one decode iteration for B rows: next token ids -> last_tok[slot],
  // out_tokens[out_off[i]]; logits left in logits() ([B][V] fp32)
  void decode(const DecodeBatch& db);
  const float* logits() const { return logits_; }

  // single-layer timing helpers for XProfiler (one encoder / decoder layer)
  void layer_encode(int l, const EncodeBatch& eb, bool attn, bool rest);
  void layer_decode(int l, const DecodeBatch& db, bool attn, bool rest);
  void fill_tables_for_profile();

  int32_t* err_flag() { return err_; }
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
  void linear_dec(const bf16* X, int64_t ldx, int tokens, const bf16* W, int features, int K, EpiParams ep);
  void linear_pre(const bf16* X, int64_t ldx, int tokens, const bf16* W, int features, int K, EpiParams ep);

  Dims D;
  int dev_;
  cudaStream_t st_ = nullptr;
  uint8_t* wbuf_ = nullptr;
  size_t wbytes_ = 0;
  bf16 *tok_emb_ = nullptr, *pos_emb_ = nullptr, *lnf_g_ = nullptr, *lnf_b_ = nullptr;
  std::vector<LayerW> layers_;
  // workspace
  int cap_tokens_ = 0, cap_rows_ = 0;
  float* x_ = nullptr;
  bf16 *h_ = nullptr, *qkv_ = nullptr, *ctx_ = nullptr, *ff_ = nullptr;
  float* logits_ = nullptr;
  float* splitk_ws_ = nullptr;
  size_t splitk_cap_ = 0;
  float* attn_part_ = nullptr;
  int split_len_ = 512, max_splits_cap_ = 0;
  int32_t* err_ = nullptr;
  // KV
  bf16* kv_ = nullptr;
  int kv_slots_ = 0, slot_ctx_ = 0, kv_layers_ = 0;
  int32_t* last_tok_ = nullptr;
  // profiler scratch tables
  int32_t* prof_tables_ = nullptr;

  bf16* kc(int l) const { return kv_ + (size_t)l * 2 * kv_layer_elems(); }
  bf16* vc(int l) const { return kc(l) + kv_layer_elems(); }
  size_t kv_layer_elems() const { return (size_t)kv_slots_ * D.H * slot_ctx_ * D.dh; }
};

}  // namespace exg
