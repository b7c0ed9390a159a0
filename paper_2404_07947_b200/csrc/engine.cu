// Engine: seeded weights, workspace, encode / decode forward passes of one
// model shard (layers [l0, l1), TP rank of tp).
//
// Layer (pre-LN) with the rounding points of T4:
//   h   = bf16(LN1(x))                 x: fp32 residual
//   qkv = bf16(h W_qkv + b)            -> K,V scattered into the row's slot
//   ctx = bf16(attention(q, K, V))     fp32 scores / softmax / P.V
//   x  += ctx W_o + b_o                fp32 (TP: fp32 partials all-reduced, T4(i))
//   h   = bf16(LN2(x))
//   f   = bf16(act(h W_1 + b_1))       act in fp32
//   x  += f W_2 + b_2                  fp32 (TP: as above)
// final (last stage): logits = bf16(LN_f(x)) E^T (fp32), argmax.
//
// Tensor parallelism (Megatron): rank r of t holds heads
// [r H/t, (r+1) H/t) of Q, K, V and W_o's matching input rows, and FFN
// columns [r F/t, (r+1) F/t); the two residual updates of a layer are the
// layer's two all-reduces.
#include <cmath>
#include <cstring>

#include "engine.cuh"

namespace exg {

namespace {
enum Kind {
  K_TOK = 0, K_POS = 1, K_LN1G = 2, K_LN1B = 3, K_WQKV = 4, K_BQKV = 5, K_WO = 6, K_BO = 7, K_LN2G = 8,
  K_LN2B = 9, K_W1 = 10, K_B1 = 11, K_W2 = 12, K_B2 = 13, K_LNFG = 14, K_LNFB = 15,
  K_RELB = 16, K_WQX = 17, K_WKVX = 18, K_WOX = 19, K_LNXG = 20
};
constexpr int T5_BUCKETS = 32, T5_MAX_DIST = 128;
constexpr float T5_EPS = 1e-6f;

// T5 relative position bucket of rel = key_pos - query_pos (double-precision
// log, truncation)
int t5_bucket(int rel, bool bidirectional) {
  int ret = 0, n = T5_BUCKETS;
  if (bidirectional) {
    n /= 2;
    if (rel > 0) ret += n;
    rel = std::abs(rel);
  } else {
    rel = -std::min(rel, 0);
  }
  const int max_exact = n / 2;
  if (rel < max_exact) return ret + rel;
  const int large = max_exact + (int)(std::log((double)rel / max_exact) / std::log((double)T5_MAX_DIST / max_exact) *
                                      (n - max_exact));
  return ret + std::min(large, n - 1);
}
inline uint64_t tid_of(int slot, int kind) { return (uint64_t)slot * 64 + kind; }

__global__ void embed_decode_kernel(float* __restrict__ x, const int32_t* __restrict__ last_tok,
                                    const int32_t* __restrict__ slot, const int32_t* __restrict__ pos,
                                    const bf16* __restrict__ tok, const bf16* __restrict__ pe, int d) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  const int i = blockIdx.x;
  const int64_t id = last_tok[slot[i]];
  const bf16* b = pe ? pe + (int64_t)pos[i] * d : nullptr;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    const float e = bf2f(tok[blocked_index(id, j, d)]);
    x[(int64_t)i * d + j] = b ? __fadd_rn(e, bf2f(b[j])) : e;
  }
}

// argmax over a logits row, lowest index on ties, result scattered to the
// request's output slot and to last_tok[slot] (the next iteration's input)
__global__ void __launch_bounds__(256) argmax_scatter_kernel(const float* __restrict__ logits, int V,
                                                              const int32_t* __restrict__ slot,
                                                              const int32_t* __restrict__ out_off,
                                                              int32_t* __restrict__ last_tok,
                                                              int32_t* __restrict__ out_tokens, int32_t* err) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  __shared__ float sv[256];
  __shared__ int si[256];
  const float* row = logits + (int64_t)blockIdx.x * V;
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
  if (nan) atomicExch(err, 1);
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
  if (threadIdx.x == 0) {
    const int y = si[0] == 0x7fffffff ? 0 : si[0];
    last_tok[slot[blockIdx.x]] = y;
    if (out_tokens) out_tokens[out_off[blockIdx.x]] = y;
  }
}

__global__ void add_bias_resid_kernel(float* __restrict__ x, const float* __restrict__ p,
                                      const bf16* __restrict__ bias, int64_t n, int d) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = x[i] + (bias ? p[i] + bf2f(bias[i % d]) : p[i]);
}

template <typename T>
T* carve(uint8_t*& p, size_t n) {
  T* r = reinterpret_cast<T*>(p);
  p += (n * sizeof(T) + 255) & ~size_t(255);
  return r;
}
}  // namespace

void add_bias_resid(float* x, const float* p, const bf16* bias, int rows, int d, cudaStream_t st) {
  const int64_t n = (int64_t)rows * d;
  if (n <= 0) return;
  launch_pdl(add_bias_resid_kernel, dim3((int)std::min<int64_t>((n + 255) / 256, 148 * 8)), dim3(256), 0, st, x, p, bias, n, d);
  EXG_CHECK_LAUNCH();
}

Engine::Engine(const exg_model_spec& s, int device, const EngineShard& shard, cudaStream_t stream)
    : S_(shard), dev_(device) {
  t5_ = s.arch == EXG_ARCH_T5;
  if (t5_) {
    if (s.n_enc_layers != s.n_dec_layers) throw std::invalid_argument("T5: n_enc_layers must equal n_dec_layers");
    if (shard.tp != 1) throw std::invalid_argument("T5: tensor-parallel shards are not built yet");
    if (shard.t5_role == 1 && shard.head) throw std::invalid_argument("T5 encoder-side shards hold no LM head");
    if (shard.t5_role < 0 || shard.t5_role > 2) throw std::invalid_argument("bad T5 role");
  } else if (s.n_enc_layers != 0) {
    throw std::invalid_argument("decoder-only architectures have no encoder layers");
  }
  D.arch = s.arch;
  D.L = s.n_dec_layers;
  D.d = s.d_model;
  D.H = s.n_heads;
  D.dh = s.d_head;
  D.inner = s.n_heads * s.d_head;
  D.ff = s.d_ff;
  D.V = s.vocab;
  D.max_pos = s.max_pos;
  D.seed = s.weight_seed;
  D.act = (s.arch == EXG_ARCH_OPT || t5_) ? ACT_RELU : ACT_GELU;
  if (s.dtype != EXG_BF16 && s.dtype != EXG_FP32) throw std::invalid_argument("unknown dtype");
  D.f32 = s.dtype == EXG_FP32;
  if (D.f32 && (t5_ || shard.tp != 1 || !shard.embed || !shard.head || shard.l0 != 0 ||
                (shard.l1 >= 0 && shard.l1 != s.n_dec_layers)))
    throw std::invalid_argument("the fp32 path runs decoder-only models on one GPU (whole model, no TP / PP)");
  defer_ = (!t5_ && !D.f32 && shard.tp == 1 && s.d_model % 4 == 0 && s.d_model <= 16384) ? deferred_enabled() : 0;
  chain_ = !t5_ && !D.f32 && shard.tp == 1 && s.d_model % 4 == 0 && s.d_model <= 16384 && chain_enabled();
  if (S_.l1 < 0) S_.l1 = D.L;
  if (S_.l0 < 0 || S_.l1 > D.L || S_.l0 >= S_.l1) throw std::invalid_argument("bad shard layer range");
  if (S_.tp < 1 || D.H % S_.tp || D.ff % S_.tp || S_.tp_rank < 0 || S_.tp_rank >= S_.tp)
    throw std::invalid_argument("n_heads and d_ff must be divisible by the TP degree");
  D.Hl = D.H / S_.tp;
  D.inner_l = D.Hl * D.dh;
  D.ffl = D.ff / S_.tp;
  if (D.d % 64 || D.inner % 64 || D.ff % 64) throw std::invalid_argument("d, H*dh, d_ff must be multiples of 64");
  if (D.inner_l % 8 || D.ffl % 8) throw std::invalid_argument("TP shard widths must be multiples of 8");
  if (D.dh != 16 && D.dh != 64 && D.dh != 128) throw std::invalid_argument("d_head must be 16, 64 or 128");
  EXG_CUDA(cudaSetDevice(dev_));
  if (stream) {
    st_ = stream;
  } else {
    EXG_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    own_stream_ = true;
  }
  EXG_CUDA(cudaMalloc(&err_, sizeof(int32_t)));
  EXG_CUDA(cudaMemsetAsync(err_, 0, sizeof(int32_t), st_));
  if (t5_)
    gen_weights_t5();
  else
    gen_weights();
}

Engine::~Engine() {
  cudaSetDevice(dev_);
  cudaStreamSynchronize(st_);
  run_cache_.reset();
  for (void* p : {(void*)wbuf_, (void*)x_, (void*)kv_, (void*)xkv_, (void*)last_tok_, (void*)err_,
                  (void*)enc_bias_, (void*)chain_ws_, (void*)chain_sync_})
    if (p) cudaFree(p);
  for (cudaEvent_t e : kev_) cudaEventDestroy(e);
  if (own_stream_ && st_) cudaStreamDestroy(st_);
}

void Engine::gen_weights() {
  const size_t d = D.d, il = D.inner_l, fl = D.ffl;
  const int64_t inner = D.inner, ff = D.ff;
  const int r = S_.tp_rank;
  auto al = [](size_t n) { return (n * 2 + 255) & ~size_t(255); };
  auto bl = [&](size_t rows, size_t K) { return al((size_t)blocked_elems(rows, K)); };
  const size_t per_layer =
      al(d) * 4 + bl(3 * il, d) + al(3 * il) + bl(d, il) + al(d) + bl(fl, d) + al(fl) + bl(d, fl) + al(d);
  const bool need_tok = S_.embed || S_.head;
  wbytes_ = (need_tok ? bl(D.V, d) : 0) + (S_.embed ? al((size_t)D.max_pos * d) : 0) + (S_.head ? 2 * al(d) : 0) +
            per_layer * n_layers();
  EXG_CUDA(cudaMalloc(&wbuf_, wbytes_));
  EXG_CUDA(cudaMemsetAsync(wbuf_, 0, wbytes_, st_));  // zero padding of the blocked tiles
  uint8_t* p = wbuf_;
  const float c_mat = (float)(2.0 * std::sqrt(3.0) * 0.02);
  const float c_gain = 0.2f;
  // generate rows x cols of tensor (slot, kind) with canonical index offsets
  // (row_off, col_off) into dst (plain row-major, or blocked starting at
  // destination row dst_row0 of a matrix with `cols` columns)
  auto gen = [&](bf16* dst, int64_t rows, int64_t cols, int slot, int kind, int gain, int transposed,
                 int64_t canon_cols, int blocked = 0, int64_t row_off = 0, int64_t col_off = 0,
                 int64_t dst_row0 = 0) {
    GenParams g{D.seed, tid_of(slot, kind), gain, c_mat, c_gain, transposed, canon_cols, row_off, col_off, blocked,
                dst_row0};
    weightgen(dst, rows, cols, cols, g, st_);
  };
  auto carve_blk = [&](size_t rows, size_t K) { return carve<bf16>(p, (size_t)blocked_elems(rows, K)); };
  if (need_tok) {
    // token embedding in the GEMM blocked layout: the A operand of the tied
    // LM head (decode swap-AB); the embedding gather indexes it directly
    tok_emb_ = carve_blk(D.V, d);
    gen(tok_emb_, D.V, d, 0, K_TOK, 0, 0, d, 1);
  }
  if (S_.embed) {
    pos_emb_ = carve<bf16>(p, (size_t)D.max_pos * d);
    gen(pos_emb_, D.max_pos, d, 0, K_POS, 0, 0, d);
  }
  if (S_.head) {
    lnf_g_ = carve<bf16>(p, d);
    gen(lnf_g_, 1, d, 0, K_LNFG, 1, 0, d);
    lnf_b_ = carve<bf16>(p, d);
    gen(lnf_b_, 1, d, 0, K_LNFB, 0, 0, d);
  }
  layers_.resize(n_layers());
  for (int l = 0; l < n_layers(); ++l) {
    const int s = 1001 + S_.l0 + l;
    LayerW& w = layers_[l];
    w.ln1_g = carve<bf16>(p, d);  gen(w.ln1_g, 1, d, s, K_LN1G, 1, 0, d);
    w.ln1_b = carve<bf16>(p, d);  gen(w.ln1_b, 1, d, s, K_LN1B, 0, 0, d);
    w.ln2_g = carve<bf16>(p, d);  gen(w.ln2_g, 1, d, s, K_LN2G, 1, 0, d);
    w.ln2_b = carve<bf16>(p, d);  gen(w.ln2_b, 1, d, s, K_LN2B, 0, 0, d);
    // matrices stored W^T [out][in] (K-major for tcgen05) in the blocked,
    // pre-swizzled GEMM layout; canonical index from the unsharded W[in][out]
    w.Wqkv = carve_blk(3 * il, d);
    w.bqkv = carve<bf16>(p, 3 * il);
    for (int sec = 0; sec < 3; ++sec) {  // q, k, v rows of this rank's heads
      gen(w.Wqkv, il, d, s, K_WQKV, 0, 1, 3 * inner, 1, sec * inner + r * (int64_t)il, 0, sec * (int64_t)il);
      gen(w.bqkv + sec * il, 1, il, s, K_BQKV, 0, 0, 3 * inner, 0, 0, sec * inner + r * (int64_t)il);
    }
    w.Wo = carve_blk(d, il);   gen(w.Wo, d, il, s, K_WO, 0, 1, d, 1, 0, r * (int64_t)il);
    w.bo = carve<bf16>(p, d);  gen(w.bo, 1, d, s, K_BO, 0, 0, d);
    w.W1 = carve_blk(fl, d);   gen(w.W1, fl, d, s, K_W1, 0, 1, ff, 1, r * (int64_t)fl, 0);
    w.b1 = carve<bf16>(p, fl); gen(w.b1, 1, fl, s, K_B1, 0, 0, ff, 0, 0, r * (int64_t)fl);
    w.W2 = carve_blk(d, fl);   gen(w.W2, d, fl, s, K_W2, 0, 1, d, 1, 0, r * (int64_t)fl);
    w.b2 = carve<bf16>(p, d);  gen(w.b2, 1, d, s, K_B2, 0, 0, d);
  }
  EXG_CUDA(cudaStreamSynchronize(st_));
}

// T5: no biases, RMS gains, relative-bias tables at
// the first encoder / decoder layer slots, encoder final norm = (slot 0, lnx_g)
void Engine::gen_weights_t5() {
  const size_t d = D.d, in = D.inner, f = D.ff;
  const int role = S_.t5_role, nl = n_layers();
  const bool has_enc = role != 2, has_dec = role != 1;
  const bool enc_last = role != 2 && S_.enc_last;   // holds the encoder's final norm
  const int n_xproj = (role == 1 && S_.enc_last) ? D.L : 0;
  auto al = [](size_t n) { return (n * 2 + 255) & ~size_t(255); };
  auto bl = [&](size_t rows, size_t K) { return al((size_t)blocked_elems(rows, K)); };
  const size_t enc_layer = al(d) * 2 + bl(3 * in, d) + bl(d, in) + bl(f, d) + bl(d, f);
  const size_t dec_layer = enc_layer + al(d) + bl(in, d) + bl(2 * in, d) + bl(d, in);
  const bool need_tok = S_.embed || S_.head;
  wbytes_ = (need_tok ? bl(D.V, d) : 0) + 2 * al(d) + 2 * al((size_t)T5_BUCKETS * D.H) +
            (has_enc ? nl * enc_layer : 0) + (has_dec ? nl * dec_layer : 0) + n_xproj * bl(2 * in, d);
  EXG_CUDA(cudaMalloc(&wbuf_, wbytes_));
  EXG_CUDA(cudaMemsetAsync(wbuf_, 0, wbytes_, st_));
  uint8_t* p = wbuf_;
  const float c_mat = (float)(2.0 * std::sqrt(3.0) * 0.02);
  const float c_gain = 0.2f;
  auto gen = [&](bf16* dst, int64_t rows, int64_t cols, int slot, int kind, int gain, int transposed,
                 int64_t canon_cols, int blocked = 0, int64_t row_off = 0, int64_t col_off = 0,
                 int64_t dst_row0 = 0) {
    GenParams g{D.seed, tid_of(slot, kind), gain, c_mat, c_gain, transposed, canon_cols, row_off, col_off, blocked,
                dst_row0};
    weightgen(dst, rows, cols, cols, g, st_);
  };
  auto carve_blk = [&](size_t rows, size_t K) { return carve<bf16>(p, (size_t)blocked_elems(rows, K)); };
  auto vec = [&](int slot, int kind, int gain) {
    bf16* v = carve<bf16>(p, d);
    gen(v, 1, d, slot, kind, gain, 0, d);
    return v;
  };
  // W^T [out][in] blocked from the canonical W[in][out] (columns col0.. of it)
  auto mat = [&](int slot, int kind, int64_t out, int64_t K, int64_t canon_cols, int64_t col0 = 0) {
    bf16* m = carve_blk(out, K);
    gen(m, out, K, slot, kind, 0, 1, canon_cols, 1, col0, 0);
    return m;
  };
  if (need_tok) {
    tok_emb_ = carve_blk(D.V, d);
    gen(tok_emb_, D.V, d, 0, K_TOK, 0, 0, d, 1);
  }
  if (S_.head) lnf_g_ = vec(0, K_LNFG, 1);
  if (enc_last) enc_lnf_g_ = vec(0, K_LNXG, 1);
  if (has_enc) {
    enc_rel_ = carve<bf16>(p, (size_t)T5_BUCKETS * D.H);
    gen(enc_rel_, T5_BUCKETS, D.H, 1, K_RELB, 0, 0, D.H);
  }
  if (has_dec) {
    dec_rel_ = carve<bf16>(p, (size_t)T5_BUCKETS * D.H);
    gen(dec_rel_, T5_BUCKETS, D.H, 1001, K_RELB, 0, 0, D.H);
  }
  if (has_enc) enc_layers_.resize(nl);
  if (has_dec) layers_.resize(nl);
  for (int side = 0; side < 2; ++side) {
    if (side == 0 ? !has_enc : !has_dec) continue;
    for (int l = 0; l < nl; ++l) {
      const int s = side ? 1001 + S_.l0 + l : 1 + S_.l0 + l;
      LayerW& w = side ? layers_[l] : enc_layers_[l];
      w.ln1_g = vec(s, K_LN1G, 1);
      w.ln2_g = vec(s, K_LN2G, 1);
      w.Wqkv = mat(s, K_WQKV, 3 * in, d, 3 * in);
      w.Wo = mat(s, K_WO, d, in, d);
      w.W1 = mat(s, K_W1, f, d, f);
      w.W2 = mat(s, K_W2, d, f, d);
      if (side) {
        w.lnx_g = vec(s, K_LNXG, 1);
        w.Wqx = mat(s, K_WQX, in, d, in);
        w.Wkvx = mat(s, K_WKVX, 2 * in, d, 2 * in);
        w.Wox = mat(s, K_WOX, d, in, d);
      }
    }
  }
  for (int l = 0; l < n_xproj; ++l) xproj_.push_back(mat(1001 + l, K_WKVX, 2 * in, d, 2 * in));
  // fp32 bias tables over every signed distance -(P-1) .. P-1
  const int P = D.max_pos;
  bias_ld_ = 2 * P - 1;
  bias_off_ = P - 1;
  std::vector<int32_t> bk(2 * (size_t)bias_ld_);
  for (int j = 0; j < bias_ld_; ++j) {
    bk[j] = t5_bucket(j - bias_off_, true);
    bk[bias_ld_ + j] = t5_bucket(j - bias_off_, false);
  }
  int32_t* dbk = nullptr;
  EXG_CUDA(cudaMalloc(&enc_bias_, sizeof(float) * 2 * (size_t)D.Hl * bias_ld_));
  dec_bias_ = enc_bias_ + (size_t)D.Hl * bias_ld_;
  EXG_CUDA(cudaMalloc(&dbk, sizeof(int32_t) * bk.size()));
  EXG_CUDA(cudaMemcpyAsync(dbk, bk.data(), sizeof(int32_t) * bk.size(), cudaMemcpyHostToDevice, st_));
  if (enc_rel_) rel_bias_table(enc_bias_, enc_rel_, dbk, bias_ld_, D.Hl, D.H, 0, st_);
  if (dec_rel_) rel_bias_table(dec_bias_, dec_rel_, dbk + bias_ld_, bias_ld_, D.Hl, D.H, 0, st_);
  EXG_CUDA(cudaStreamSynchronize(st_));
  EXG_CUDA(cudaFree(dbk));
}

void Engine::ensure_workspace(int max_tokens, int max_rows) {
  max_tokens = std::max(max_tokens, max_rows);
  if (max_tokens <= cap_tokens_ && max_rows <= cap_rows_) return;
  EXG_CUDA(cudaStreamSynchronize(st_));
  if (x_) EXG_CUDA(cudaFree(x_));
  cap_tokens_ = std::max(max_tokens, cap_tokens_);
  cap_rows_ = std::max(max_rows, cap_rows_);
  const size_t T = cap_tokens_, R = cap_rows_;
  size_t sk = 0;
  for (auto fk : {std::make_pair(3 * D.inner_l, D.d), std::make_pair(D.d, D.inner_l), std::make_pair(D.ffl, D.d),
                  std::make_pair(D.inner_l, D.d),
                  std::make_pair(D.d, D.ffl), std::make_pair(D.V, D.d)})
    sk = std::max(sk, decode_ws_floats(fk.first, fk.second, (int)R));
  splitk_cap_ = sk;
  max_splits_cap_ = (D.max_pos + 127) / 128;   // any split length >= 128 (diagnostics override)
  const size_t parts = R * D.Hl * (size_t)max_splits_cap_ * (D.dh + 2);
  const size_t tp_part = S_.tp > 1 ? T * D.d : 0;
  const size_t logit_rows = S_.head ? R : 0;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t f32_act = D.f32 ? al(T * D.d * 4) + al(T * 3 * D.inner_l * 4) + al(T * D.inner_l * 4) +
                                     al(T * D.ffl * 4)
                               : 0;
  const size_t dq = (defer_ & DEFER_QKV) ? deferred_floats(3 * D.inner_l, D.d, (int)R) : 0;
  const size_t dr = (defer_ & DEFER_RESID)
                        ? std::max(deferred_floats(D.d, D.inner_l, (int)R), deferred_floats(D.d, D.ffl, (int)R))
                        : 0;
  const size_t bytes = al(T * D.d * 4) + al(tp_part * 4) + al(T * D.d * 2) + al(T * 3 * D.inner_l * 2) +
                       al(T * D.inner_l * 2) + al(T * D.ffl * 2) + al(logit_rows * D.V * 4) + al(sk * 4) +
                       al(parts * 4) + al(R * D.Hl * 4) + f32_act + al(dq * 4) + al(dr * 4);
  uint8_t* p;
  EXG_CUDA(cudaMalloc(&p, bytes));
  x_ = carve<float>(p, T * D.d);
  part_ = tp_part ? carve<float>(p, tp_part) : nullptr;
  h_ = carve<bf16>(p, T * D.d);
  qkv_ = carve<bf16>(p, T * 3 * D.inner_l);
  ctx_ = carve<bf16>(p, T * D.inner_l);
  ff_ = carve<bf16>(p, T * D.ffl);
  logits_ = logit_rows ? carve<float>(p, logit_rows * D.V) : nullptr;
  splitk_ws_ = carve<float>(p, sk);
  attn_part_ = carve<float>(p, parts);
  attn_cnt_ = carve<int32_t>(p, R * D.Hl);   // split-merge counters: zero, left at zero by each merge
  defer_qkv_ = dq ? carve<float>(p, dq) : nullptr;
  defer_res_ = dr ? carve<float>(p, dr) : nullptr;
  pend_res_ = PendingResid();
  if (D.f32) {
    hf_ = carve<float>(p, T * D.d);
    qkvf_ = carve<float>(p, T * 3 * D.inner_l);
    ctxf_ = carve<float>(p, T * D.inner_l);
    fff_ = carve<float>(p, T * D.ffl);
  }
  EXG_CUDA(cudaMemsetAsync(x_, 0, bytes, st_));
  if (chain_) {
    // decode chain workspace: the largest need over the token tiles up to R
    size_t need = 0;
    for (int t : {32, 64, 128, 256, (int)R}) {
      if (t > (int)R && t != 32) continue;
      need = std::max(need, chain_ws_floats(chain_spec(0, std::min<int>(t, (int)R), n_layers() > 1 ? 1 : -1)));
    }
    if (need > chain_ws_cap_) {
      if (chain_ws_) EXG_CUDA(cudaFree(chain_ws_));
      EXG_CUDA(cudaMalloc(&chain_ws_, need * sizeof(float)));
      EXG_CUDA(cudaMemsetAsync(chain_ws_, 0, need * sizeof(float), st_));   // fixup counters start at 0
      chain_ws_cap_ = need;
    }
    if (!chain_sync_) {
      EXG_CUDA(cudaMalloc(&chain_sync_, 16 * sizeof(unsigned)));
      EXG_CUDA(cudaMemsetAsync(chain_sync_, 0, 16 * sizeof(unsigned), st_));
      chain_epoch_ = 0;
    }
  }
}

void Engine::ensure_kv(int slots, int slot_ctx, int layers, int xctx) {
  if (slot_ctx > D.max_pos || xctx > D.max_pos) throw std::invalid_argument("slot_ctx exceeds max_pos");
  if (t5_ && xctx < 1) throw std::invalid_argument("encoder-decoder model: cross-attention context xctx must be >= 1");
  if (!t5_) xctx = 0;
  if (layers < 0) layers = n_layers();
  // T5 encoder side: no self-attention cache; cross caches per n_cross_layers
  const int self_layers = (t5_ && S_.t5_role == 1) ? 0 : layers;
  const int x_layers = !t5_ ? 0 : (S_.t5_role == 1 ? n_cross_layers() : layers);
  if (slots <= kv_slots_ && slot_ctx == slot_ctx_ && layers <= kv_layers_ && xctx == xctx_) return;
  EXG_CUDA(cudaStreamSynchronize(st_));
  if (kv_) EXG_CUDA(cudaFree(kv_));
  if (xkv_) EXG_CUDA(cudaFree(xkv_));
  if (last_tok_) EXG_CUDA(cudaFree(last_tok_));
  kv_ = nullptr;
  xkv_ = nullptr;
  last_tok_ = nullptr;
  kv_slots_ = std::max(slots, 1);
  slot_ctx_ = slot_ctx;
  xctx_ = xctx;
  kv_layers_ = layers;
  const size_t bytes = (size_t)self_layers * 2 * kv_layer_elems() * (D.f32 ? sizeof(float) : sizeof(bf16));
  const size_t xbytes = (size_t)x_layers * 2 * xkv_layer_elems() * sizeof(bf16);
  cudaError_t e = bytes ? cudaMalloc(&kv_, bytes) : cudaSuccess;
  if (e == cudaSuccess && xbytes) e = cudaMalloc(&xkv_, xbytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (kv_) cudaFree(kv_);
    kv_ = nullptr;
    kv_slots_ = 0;
    kv_layers_ = 0;
    throw std::bad_alloc();
  }
  if (bytes) EXG_CUDA(cudaMemsetAsync(kv_, 0, bytes, st_));
  if (xbytes) EXG_CUDA(cudaMemsetAsync(xkv_, 0, xbytes, st_));
  EXG_CUDA(cudaMalloc(&last_tok_, sizeof(int32_t) * kv_slots_));
  EXG_CUDA(cudaMemsetAsync(last_tok_, 0, sizeof(int32_t) * kv_slots_, st_));
}

void Engine::linear_dec(const bf16* X, int64_t ldx, int tokens, const bf16* W, int features, int K, EpiParams ep) {
  LinearArgs a;
  a.X = X;
  a.ldx = ldx;
  a.Wb = W;
  a.K = K;
  ep.tokens = tokens;
  ep.features = features;
  a.ep = ep;
  a.decode = true;
  a.ws = splitk_ws_;
  a.ws_floats = splitk_cap_;
  const int k = kbegin();
  linear(a, st_);
  const double out_b = ep.mode == EPI_RESID ? 8.0 : (ep.mode == EPI_F32 ? 4.0 : 2.0);
  kend(k, EXG_K_DECODE_GEMM, 2.0 * features * K + 2.0 * tokens * K + out_b * tokens * features);
}

void Engine::linear_pre(const bf16* X, int64_t ldx, int tokens, const bf16* W, int features, int K, EpiParams ep) {
  LinearArgs a;
  a.X = X;
  a.ldx = ldx;
  a.Wb = W;
  a.K = K;
  ep.tokens = tokens;
  ep.features = features;
  a.ep = ep;
  a.decode = false;
  const int k = kbegin();
  linear(a, st_);
  kend(k, EXG_K_PREFILL_GEMM, 2.0 * tokens * features * K);
}

int Engine::kbegin() {
  if (!ktiming_) return -1;
  const int idx = (int)krec_.size();
  while ((int)kev_.size() < 2 * (idx + 1)) {
    cudaEvent_t e;
    EXG_CUDA(cudaEventCreate(&e));
    kev_.push_back(e);
  }
  EXG_CUDA(cudaEventRecord(kev_[2 * idx], st_));
  krec_.push_back(KRec{-1, idx, 0.0});
  return idx;
}

void Engine::kend(int idx, int cls, double work) {
  if (idx < 0) return;
  EXG_CUDA(cudaEventRecord(kev_[2 * idx + 1], st_));
  krec_[idx].cls = cls;
  krec_[idx].work = work;
}

void Engine::set_kernel_timing(bool on) {
  ktiming_ = on;
  krec_.clear();
}

void Engine::collect_kernel_timing(double* t, double* w, int64_t* n) {
  for (const KRec& r : krec_) {
    if (r.cls < 0) continue;
    float ms = 0.f;
    EXG_CUDA(cudaEventElapsedTime(&ms, kev_[2 * r.ev], kev_[2 * r.ev + 1]));
    t[r.cls] += ms * 1e-3;
    w[r.cls] += r.work;
    n[r.cls] += 1;
  }
  krec_.clear();
}

static EpiParams epi_bf16(const bf16* bias, bf16* out, int64_t ldo, int act = ACT_NONE) {
  EpiParams e;
  e.mode = act == ACT_NONE ? EPI_BF16 : EPI_BF16_ACT;
  e.act = act;
  e.bias = bias;
  e.out_bf16 = out;
  e.ldo = ldo;
  return e;
}

void Engine::resid_update(bool decode, const bf16* X, int64_t ldx, int tokens, const bf16* W, int K,
                          const bf16* bias) {
  EpiParams e;
  if (S_.tp == 1) {
    e.mode = EPI_RESID;
    e.bias = bias;
    e.resid = x_;
    e.ldr = D.d;
  } else {
    e.mode = EPI_F32;
    e.out_f32 = part_;
    e.ldo = D.d;
  }
  if (decode)
    linear_dec(X, ldx, tokens, W, D.d, K, e);
  else
    linear_pre(X, ldx, tokens, W, D.d, K, e);
  if (S_.tp > 1) {
    if (red_) {
      red_->allreduce_sum(part_, (int64_t)tokens * D.d, st_);
      add_bias_resid(x_, part_, bias, tokens, D.d, st_);
    } else {
      // lockstep TP group on one device: the group sums every rank's part_
      // (sum_tp_parts) and then calls finish_pending()
      pend_bias_ = bias;
      pend_rows_ = tokens;
    }
  }
}

void Engine::finish_pending() {
  if (!pend_bias_) return;
  add_bias_resid(x_, part_, pend_bias_, pend_rows_, D.d, st_);
  pend_bias_ = nullptr;
}

void Engine::enc_attn_block(int l, const EncodeBatch& eb) {
  const LayerW& w = layers_[l];
  layer_encode(l, eb, true, false, 1);
  resid_update(false, ctx_, D.inner_l, eb.T, w.Wo, D.inner_l, w.bo);
}

void Engine::enc_ffn_block(int l, const EncodeBatch& eb) { layer_encode(l, eb, false, true, 2); }

void Engine::dec_attn_block(int l, const DecodeBatch& db) {
  const LayerW& w = layers_[l];
  layer_decode(l, db, true, false, 1);
  resid_update(true, ctx_, D.inner_l, db.B, w.Wo, D.inner_l, w.bo);
}

void Engine::dec_ffn_block(int l, const DecodeBatch& db) { layer_decode(l, db, false, true, 2); }

// part 0: the whole layer (attention and / or the rest, for the profiler);
// part 1: LN1, QKV, KV scatter, attention (up to, excluding, the O-proj);
// part 2: LN2, FFN1, FFN2 (after the attention residual update).
void Engine::layer_encode(int l, const EncodeBatch& eb, bool attn, bool rest, int part) {
  if (t5_) {
    if (part != 0) throw std::logic_error("T5: no TP blocks");
    enc_layer_t5(l, eb, attn, rest);
    return;
  }
  const LayerW& w = layers_[l];
  const int T = eb.T, d = D.d, il = D.inner_l;
  const float scale = (float)(1.0 / std::sqrt((double)D.dh));
  if (part == 2) {
    layernorm(h_, d, x_, d, w.ln2_g, w.ln2_b, T, d, 1e-5f, st_);
    linear_pre(h_, d, T, w.W1, D.ffl, d, epi_bf16(w.b1, ff_, D.ffl, D.act));
    resid_update(false, ff_, D.ffl, T, w.W2, D.ffl, w.b2);
    return;
  }
  if (part == 1) attn = rest = true;
  if (rest) {
    layernorm(h_, d, x_, d, w.ln1_g, w.ln1_b, T, d, 1e-5f, st_);
    // K7 fused into the QKV GEMM epilogue: K / V rows go straight into the
    // cache at (tslot, pos); qkv_ keeps Q (the FMHA's A operand)
    EpiParams e = epi_bf16(w.bqkv, qkv_, 3 * il);
    e.kv_k = kc(l);
    e.kv_v = vc(l);
    e.kv_slot = eb.kv_blk ? eb.kv_blk : eb.tslot;
    e.kv_pos = eb.kv_blk ? eb.kv_off : eb.pos;
    e.kv_inner = il;
    e.kv_H = D.Hl;
    e.kv_dh = D.dh;
    e.kv_ctx = slot_ctx_;
    if (D.dh % 16 == 0 && (3 * il) % 8 == 0) {
      linear_pre(h_, d, T, w.Wqkv, 3 * il, d, e);
    } else {
      linear_pre(h_, d, T, w.Wqkv, 3 * il, d, epi_bf16(w.bqkv, qkv_, 3 * il));
      kv_scatter(kc(l), vc(l), qkv_, eb.kv_blk ? eb.kv_blk : eb.tslot, eb.kv_blk ? eb.kv_off : eb.pos, T, D.Hl,
                 D.dh, slot_ctx_, st_);
    }
  }
  if (attn) {
    PrefillAttnArgs pa{qkv_, 3 * il, kc(l), vc(l), eb.cu, eb.rslot, eb.pos0, eb.R, eb.max_len,
                       ctx_, il, D.Hl, D.dh, slot_ctx_, scale,
                       (int64_t)eb.T, (int64_t)kv_slots_ * D.Hl * slot_ctx_};
    pa.kv = eb.kv;
    const int k = kbegin();
    prefill_attention(pa, st_);
    kend(k, EXG_K_PREFILL_ATTN, 4.0 * D.Hl * D.dh * eb.attn_pairs);
  }
  if (part == 1) return;
  if (rest) {
    resid_update(false, ctx_, il, T, w.Wo, il, w.bo);
    layernorm(h_, d, x_, d, w.ln2_g, w.ln2_b, T, d, 1e-5f, st_);
    linear_pre(h_, d, T, w.W1, D.ffl, d, epi_bf16(w.b1, ff_, D.ffl, D.act));
    resid_update(false, ff_, D.ffl, T, w.W2, D.ffl, w.b2);
  }
}

void Engine::embed_encode(const EncodeBatch& eb) {
  if (eb.T > cap_tokens_) throw std::invalid_argument("encode batch exceeds workspace");
  if (S_.embed && eb.T > 0) embed(x_, eb.ids, eb.pos, tok_emb_, pos_emb_, eb.T, D.d, st_, 1);
}

void Engine::encode(const EncodeBatch& eb) {
  if (eb.T <= 0) return;
  if (D.f32) {
    encode_f32(eb);
    return;
  }
  if (t5_) {
    encode_t5(eb);
    return;
  }
  if (S_.tp > 1 && !red_) throw std::logic_error("TP shard without a reducer: drive it through a TP group");
  embed_encode(eb);
  for (int l = 0; l < n_layers(); ++l) layer_encode(l, eb, true, true);
}

void Engine::layer_decode(int l, const DecodeBatch& db, bool attn, bool rest, int part) {
  if (t5_) {
    if (part != 0) throw std::logic_error("T5: no TP blocks");
    dec_layer_t5(l, db, attn, rest);
    return;
  }
  const LayerW& w = layers_[l];
  const int B = db.B, d = D.d, il = D.inner_l;
  const float scale = (float)(1.0 / std::sqrt((double)D.dh));
  if (chain_ && part == 0) {
    // one layer's work as the chained decode runs it: the attention, then one
    // chain launch (O-proj .. FFN2 and this layer's LN1 + QKV in place of the
    // next layer's)
    if (attn) dec_attention(l, db);
    if (rest) dec_rest_chain(l, db, l);
    return;
  }
  if (part == 2) {
    layernorm(h_, d, x_, d, w.ln2_g, w.ln2_b, B, d, 1e-5f, st_);
    linear_dec(h_, d, B, w.W1, D.ffl, d, epi_bf16(w.b1, ff_, D.ffl, D.act));
    resid_update(true, ff_, D.ffl, B, w.W2, D.ffl, w.b2);
    return;
  }
  if (part == 1) attn = rest = true;
  const bool defer_qkv = (defer_ & DEFER_QKV) && part == 0, defer = (defer_ & DEFER_RESID) && part == 0;
  if (rest) {
    ln_decode(w.ln1_g, w.ln1_b, B);
    EpiParams e = epi_bf16(w.bqkv, qkv_, 3 * il);
    if (defer_qkv) e.defer_out = defer_qkv_;   // q / k / v summed by the attention kernel
    linear_dec(h_, d, B, w.Wqkv, 3 * il, d, e);
  }
  if (attn) {
    // K7 fused: the attention kernel appends the new token's K / V (from the
    // qkv buffer, or the deferred QKV segments) to the cache at position
    // n_keys - 1
    DecodeAttnArgs da;
    da.knew = qkv_ + il;
    da.vnew = qkv_ + 2 * il;
    da.ldnew = 3 * il;
    da.q = qkv_;
    da.ldq = 3 * il;
    if (defer_qkv) {
      da.qkv_part = defer_qkv_;
      da.qkv_si = decode_seg_info(3 * il, d);
      da.qkv_bias = w.bqkv;
      da.qkv_inner = il;
    }
    da.kc = kc(l);
    da.vc = vc(l);
    da.slot = db.slot;
    da.n_keys = db.nkeys;
    da.out = ctx_;
    da.ldo = il;
    da.B = B;
    da.H = D.Hl;
    da.dh = D.dh;
    da.max_ctx = slot_ctx_;
    da.kv = db.kv;
    da.scale = scale;
    const int sl = split_len();
    da.split_len = sl;
    da.max_splits = std::max(1, (db.max_keys + sl - 1) / sl);
    da.partial = attn_part_;
    da.counters = attn_cnt_;
    const int k = kbegin();
    decode_attention(da, st_);
    kend(k, EXG_K_DECODE_ATTN, db.sum_keys * 2.0 * D.Hl * D.dh * 2.0 + (double)B * D.Hl * D.dh * 2.0 * 2.0 +
                                   (double)B * 2.0 * D.Hl * D.dh * 2.0);
  }
  if (part == 1) return;
  if (rest) {
    if (defer) {
      // O-projection: segments only; the residual update + LN2 in one kernel
      EpiParams e;
      e.mode = EPI_RESID;
      e.defer_out = defer_res_;
      linear_dec(ctx_, il, B, w.Wo, d, il, e);
      pend_res_ = PendingResid{defer_res_, decode_seg_info(d, il), w.bo};
    } else {
      resid_update(true, ctx_, il, B, w.Wo, il, w.bo);
    }
    ln_decode(w.ln2_g, w.ln2_b, B);
    linear_dec(h_, d, B, w.W1, D.ffl, d, epi_bf16(w.b1, ff_, D.ffl, D.act));
    // FFN2 deferred when a LayerNorm of this engine follows (the next layer's
    // LN1 or the final norm); a non-last pipeline stage hands x on as is
    if (defer && (l + 1 < n_layers() || S_.head)) {
      EpiParams e;
      e.mode = EPI_RESID;
      e.defer_out = defer_res_;
      linear_dec(ff_, D.ffl, B, w.W2, d, D.ffl, e);
      pend_res_ = PendingResid{defer_res_, decode_seg_info(d, D.ffl), w.b2};
    } else {
      resid_update(true, ff_, D.ffl, B, w.W2, D.ffl, w.b2);
    }
  }
}

ChainSpec Engine::chain_spec(int l, int B, int next_l) const {
  const LayerW& w = layers_[l];
  const int d = D.d, il = D.inner_l;
  ChainSpec c;
  c.tokens = B;
  c.d = d;
  c.x = x_;
  c.h = h_;
  c.eps = 1e-5f;
  auto resid = [&](const bf16* bias) {
    EpiParams e;
    e.mode = EPI_RESID;
    e.bias = bias;
    e.resid = x_;
    e.ldr = d;
    return e;
  };
  c.ph[0].X = ctx_, c.ph[0].ldx = il, c.ph[0].Wb = w.Wo, c.ph[0].features = d, c.ph[0].K = il;
  c.ph[0].ep = resid(w.bo);
  c.ph[0].ln_after = 0;
  c.ln_g[0] = w.ln2_g, c.ln_b[0] = w.ln2_b;
  c.ph[1].X = h_, c.ph[1].ldx = d, c.ph[1].Wb = w.W1, c.ph[1].features = D.ffl, c.ph[1].K = d;
  c.ph[1].ep = epi_bf16(w.b1, ff_, D.ffl, D.act);
  c.ph[2].X = ff_, c.ph[2].ldx = D.ffl, c.ph[2].Wb = w.W2, c.ph[2].features = d, c.ph[2].K = D.ffl;
  c.ph[2].ep = resid(w.b2);
  c.n = 3;
  if (next_l >= 0) {
    const LayerW& nx = layers_[next_l];
    c.ph[2].ln_after = 1;
    c.ln_g[1] = nx.ln1_g, c.ln_b[1] = nx.ln1_b;
    c.ph[3].X = h_, c.ph[3].ldx = d, c.ph[3].Wb = nx.Wqkv, c.ph[3].features = 3 * il, c.ph[3].K = d;
    c.ph[3].ep = epi_bf16(nx.bqkv, qkv_, 3 * il);
    c.n = 4;
  }
  return c;
}

void Engine::dec_rest_chain(int l, const DecodeBatch& db, int next_l) {
  ChainSpec c = chain_spec(l, db.B, next_l);
  c.ws = chain_ws_;
  c.ws_floats = chain_ws_cap_;
  c.sync = chain_sync_;
  c.epoch = ++chain_epoch_;
  double bytes = 0;
  for (int q = 0; q < c.n; ++q) {
    const double out_b = c.ph[q].ep.mode == EPI_RESID ? 8.0 : 2.0;
    bytes += 2.0 * c.ph[q].features * c.ph[q].K + 2.0 * db.B * c.ph[q].K + out_b * db.B * c.ph[q].features;
  }
  const int k = kbegin();
  decode_chain(c, st_);
  kend(k, EXG_K_DECODE_GEMM, bytes);
}

void Engine::dec_attention(int l, const DecodeBatch& db) {
  const int B = db.B, il = D.inner_l;
  DecodeAttnArgs da;
  da.knew = qkv_ + il;
  da.vnew = qkv_ + 2 * il;
  da.ldnew = 3 * il;
  da.q = qkv_;
  da.ldq = 3 * il;
  da.kc = kc(l);
  da.vc = vc(l);
  da.slot = db.slot;
  da.n_keys = db.nkeys;
  da.out = ctx_;
  da.ldo = il;
  da.B = B;
  da.H = D.Hl;
  da.dh = D.dh;
  da.max_ctx = slot_ctx_;
  da.kv = db.kv;
  da.scale = (float)(1.0 / std::sqrt((double)D.dh));
  const int sl = split_len();
  da.split_len = sl;
  da.max_splits = std::max(1, (db.max_keys + sl - 1) / sl);
  da.partial = attn_part_;
  da.counters = attn_cnt_;
  const int k = kbegin();
  decode_attention(da, st_);
  kend(k, EXG_K_DECODE_ATTN, db.sum_keys * 2.0 * D.Hl * D.dh * 2.0 + (double)B * D.Hl * D.dh * 2.0 * 2.0 +
                                 (double)B * 2.0 * D.Hl * D.dh * 2.0);
}

void Engine::ln_decode(const bf16* g, const bf16* b, int rows) {
  if (pend_res_.P) {
    const PendingResid pr = pend_res_;
    pend_res_ = PendingResid();
    if (layernorm_deferred(h_, D.d, x_, D.d, pr.P, pr.si, pr.bias, g, b, rows, D.d, 1e-5f, st_)) return;
    throw std::logic_error("deferred LayerNorm: unsupported shape");
  }
  layernorm(h_, D.d, x_, D.d, g, b, rows, D.d, 1e-5f, st_);
}

void Engine::embed_decode(const DecodeBatch& db) {
  const int B = db.B;
  pend_res_ = PendingResid();   // a new iteration's residual stream starts here
  if (B > cap_rows_) throw std::invalid_argument("decode batch exceeds workspace");
  if (S_.embed && B > 0) {
    // T5: no position embedding (pos_emb_ null)
    launch_pdl(embed_decode_kernel, dim3(B), dim3(256), 0, st_, x_, last_tok_, db.slot, db.pos, tok_emb_, pos_emb_, D.d);
    EXG_CHECK_LAUNCH();
  }
}

void Engine::decode(const DecodeBatch& db) {
  if (db.B <= 0) return;
  if (D.f32) {
    decode_f32(db);
    return;
  }
  if (t5_ && S_.t5_role == 1) throw std::logic_error("T5 encoder-side shard: no decoder layers");
  if (S_.tp > 1 && !red_) throw std::logic_error("TP shard without a reducer: drive it through a TP group");
  embed_decode(db);
  if (chain_) {
    // layer 0's LN1 + QKV, then per layer: the attention and one chain launch
    // (O-proj, LN2, FFN1, FFN2 and the next layer's LN1 + QKV)
    const LayerW& w0 = layers_[0];
    layernorm(h_, D.d, x_, D.d, w0.ln1_g, w0.ln1_b, db.B, D.d, 1e-5f, st_);
    linear_dec(h_, D.d, db.B, w0.Wqkv, 3 * D.inner_l, D.d, epi_bf16(w0.bqkv, qkv_, 3 * D.inner_l));
    for (int l = 0; l < n_layers(); ++l) {
      dec_attention(l, db);
      dec_rest_chain(l, db, l + 1 < n_layers() ? l + 1 : -1);
    }
  } else {
    for (int l = 0; l < n_layers(); ++l) layer_decode(l, db, true, true);
  }
  head_decode(db);
}

void Engine::head_decode(const DecodeBatch& db) {
  const int B = db.B;
  if (S_.head && B > 0) {
    if (t5_)  // tied head of T5: logits = (RMS_f(x) d^-1/2) E^T (the scale folded into the norm output)
      rmsnorm(h_, D.d, x_, D.d, lnf_g_, B, D.d, T5_EPS, (float)(1.0 / std::sqrt((double)D.d)), st_);
    else
      ln_decode(lnf_g_, lnf_b_, B);
    EpiParams e;
    e.mode = EPI_F32;
    e.out_f32 = logits_;
    e.ldo = D.V;
    linear_dec(h_, D.d, B, tok_emb_, D.V, D.d, e);
    launch_pdl(argmax_scatter_kernel, dim3(B), dim3(256), 0, st_, logits_, D.V, db.slot, db.out_off, last_tok_, db.out_tokens, err_);
    EXG_CHECK_LAUNCH();
  }
}

// ---------------------------------------------------------------------------
// fp32 parity path (fp32_path.cu): the layer of the file
// header with every rounding point of T4 removed -- fp32 norm output, q/k/v,
// KV cache, context, FFN activation and logits; FFMA contractions.
// ---------------------------------------------------------------------------
void Engine::layer_f32(int l, int rows, const int32_t* slot, const int32_t* pos) {
  const LayerW& w = layers_[l];
  const int d = D.d, il = D.inner_l;
  const float scale = (float)(1.0 / std::sqrt((double)D.dh));
  layernorm_f32(hf_, d, x_, d, w.ln1_g, w.ln1_b, rows, d, 1e-5f, st_);
  linear_f32(hf_, d, w.Wqkv, rows, 3 * il, d, w.bqkv, EPI_F32, ACT_NONE, qkvf_, 3 * il, st_);
  // K7: the rows' K / V into their slots, then causal attention over keys
  // 0..pos of each row's slot
  kv_scatter_f32(kcf(l), vcf(l), qkvf_, 3 * il, il, slot, pos, rows, D.Hl, D.dh, slot_ctx_, st_);
  attention_f32(qkvf_, 3 * il, kcf(l), vcf(l), slot, pos, rows, D.Hl, D.dh, slot_ctx_, scale, ctxf_, il, st_);
  linear_f32(ctxf_, il, w.Wo, rows, d, il, w.bo, EPI_RESID, ACT_NONE, x_, d, st_);
  layernorm_f32(hf_, d, x_, d, w.ln2_g, w.ln2_b, rows, d, 1e-5f, st_);
  linear_f32(hf_, d, w.W1, rows, D.ffl, d, w.b1, EPI_BF16_ACT, D.act, fff_, D.ffl, st_);
  linear_f32(fff_, D.ffl, w.W2, rows, d, D.ffl, w.b2, EPI_RESID, ACT_NONE, x_, d, st_);
}

void Engine::encode_f32(const EncodeBatch& eb) {
  if (eb.kv.ptab) throw std::invalid_argument("paged KV is not supported on the fp32 path");
  embed_encode(eb);
  for (int l = 0; l < n_layers(); ++l) layer_f32(l, eb.T, eb.tslot, eb.pos);
}

void Engine::decode_f32(const DecodeBatch& db) {
  if (db.kv.ptab) throw std::invalid_argument("paged KV is not supported on the fp32 path");
  embed_decode(db);
  for (int l = 0; l < n_layers(); ++l) layer_f32(l, db.B, db.slot, db.pos);
  layernorm_f32(hf_, D.d, x_, D.d, lnf_g_, lnf_b_, db.B, D.d, 1e-5f, st_);
  linear_f32(hf_, D.d, tok_emb_, db.B, D.V, D.d, nullptr, EPI_F32, ACT_NONE, logits_, D.V, st_);
  launch_pdl(argmax_scatter_kernel, dim3(db.B), dim3(256), 0, st_, logits_, D.V, db.slot, db.out_off, last_tok_,
             db.out_tokens, err_);
  EXG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// T5 encoder-decoder (SURVEY.md §8(c) T1 T5 reading; oracle/t5.py)
//   encoder layer:  h = bf16(RMS(x)); qkv; bidirectional attention + relative
//                   bias (scale 1); x += ctx W_o; h = bf16(RMS(x));
//                   x += bf16(relu(h W_1)) W_2
//   encode phase:   encoder over all n input tokens, e = bf16(RMS_enc(x)),
//                   cross K/V of every decoder layer = bf16(e W_kv_x) -> xkv
//   decoder layer:  self-attention (causal relative bias) over the decoder
//                   KV, cross-attention over xkv, ReLU FFN; no biases.
// The encoder's own K/V are staged in decoder layer 0's cross cache at the
// request's slot; the cross K/V projection of layer 0 overwrites them.
// ---------------------------------------------------------------------------
void Engine::enc_layer_t5(int l, const EncodeBatch& eb, bool attn, bool rest) {
  const LayerW& w = enc_layers_[l];
  const int T = eb.T, d = D.d, il = D.inner_l;
  if (rest) {
    rmsnorm(h_, d, x_, d, w.ln1_g, T, d, T5_EPS, 1.f, st_);
    linear_pre(h_, d, T, w.Wqkv, 3 * il, d, epi_bf16(nullptr, qkv_, 3 * il));
    kv_scatter(xkc(0), xvc(0), qkv_, eb.tslot, eb.pos, T, D.Hl, D.dh, xctx_, st_);
  }
  if (attn) {
    PrefillAttnArgs pa{qkv_, 3 * il, xkc(0), xvc(0), eb.cu, eb.rslot, eb.pos0, eb.R, eb.max_len,
                       ctx_, il, D.Hl, D.dh, xctx_, 1.0f,
                       (int64_t)eb.T, (int64_t)kv_slots_ * D.Hl * xctx_, 0, enc_bias_, bias_ld_, bias_off_};
    const int k = kbegin();
    prefill_attention(pa, st_);
    kend(k, EXG_K_PREFILL_ATTN, 4.0 * D.Hl * D.dh * eb.attn_pairs);
  }
  if (rest) {
    resid_update(false, ctx_, il, T, w.Wo, il, nullptr);
    rmsnorm(h_, d, x_, d, w.ln2_g, T, d, T5_EPS, 1.f, st_);
    linear_pre(h_, d, T, w.W1, D.ffl, d, epi_bf16(nullptr, ff_, D.ffl, ACT_RELU));
    resid_update(false, ff_, D.ffl, T, w.W2, D.ffl, nullptr);
  }
}

// the encode phase of this shard: its encoder layers, then (last encoder
// shard) the final norm -> h() and the cross K/V it holds.  A non-last shard of
// an RRA pipeline (role 0) gets the encoder output broadcast into h() by the
// executor and then runs cross_kv_all() for its decoder layers.
void Engine::encode_t5(const EncodeBatch& eb) {
  const int T = eb.T, d = D.d;
  if (S_.t5_role == 2) throw std::logic_error("T5 decoder-side shard: no encoder layers");
  if (T > cap_tokens_) throw std::invalid_argument("encode batch exceeds workspace");
  if (S_.embed) embed(x_, eb.ids, eb.pos, tok_emb_, nullptr, T, d, st_, 1);
  for (int l = 0; l < n_layers(); ++l) enc_layer_t5(l, eb, true, true);
  if (!S_.enc_last) return;   // the residual stream x() continues on the next stage
  rmsnorm(h_, d, x_, d, enc_lnf_g_, T, d, T5_EPS, 1.f, st_);
  cross_kv_all(eb);
}

// K13: cross K/V of every decoder layer held here from the encoder output in
// h(): K at columns [il, 2il) and V at [2il, 3il) of the qkv buffer, then
// scattered to the slots
void Engine::cross_kv_all(const EncodeBatch& eb) {
  for (int l = 0; l < n_cross_layers(); ++l) cross_kv(l, eb);
}

void Engine::cross_kv(int l, const EncodeBatch& eb) {
  const int il = D.inner_l;
  const bf16* W = S_.t5_role == 1 ? xproj_[l] : layers_[l].Wkvx;
  linear_pre(h_, D.d, eb.T, W, 2 * il, D.d, epi_bf16(nullptr, qkv_ + il, 3 * il));
  kv_scatter(xkc(l), xvc(l), qkv_, eb.tslot, eb.pos, eb.T, D.Hl, D.dh, xctx_, st_);
}

void Engine::dattn(const bf16* q, int64_t ldq, const bf16* kc, const bf16* vc, int ctx, const DecodeBatch& db,
                   const int32_t* nkeys, int max_keys, double sum_keys, const float* bias, bool append,
                   KvMap kv) {
  DecodeAttnArgs da;
  da.kv = kv;
  if (append) {   // fused KV append of the new token (K7): K / V follow q in the qkv buffer
    da.knew = q + D.inner_l;
    da.vnew = q + 2 * D.inner_l;
    da.ldnew = ldq;
  }
  da.q = q;
  da.ldq = ldq;
  da.kc = kc;
  da.vc = vc;
  da.slot = db.slot;
  da.n_keys = nkeys;
  da.out = ctx_;
  da.ldo = D.inner_l;
  da.B = db.B;
  da.H = D.Hl;
  da.dh = D.dh;
  da.max_ctx = ctx;
  da.scale = 1.0f;
  const int sl = split_len();
  da.split_len = sl;
  da.max_splits = std::max(1, (max_keys + sl - 1) / sl);
  da.partial = attn_part_;
  da.counters = attn_cnt_;
  da.bias = bias;
  da.bias_ld = bias_ld_;
  da.bias_off = bias_off_;
  const int k = kbegin();
  decode_attention(da, st_);
  kend(k, EXG_K_DECODE_ATTN, sum_keys * 2.0 * D.Hl * D.dh * 2.0 + (double)db.B * D.Hl * D.dh * 2.0 * 2.0 +
                                (append ? (double)db.B * 2.0 * D.Hl * D.dh * 2.0 : 0.0));
}

void Engine::dec_layer_t5(int l, const DecodeBatch& db, bool attn, bool rest) {
  const LayerW& w = layers_[l];
  const int B = db.B, d = D.d, il = D.inner_l;
  if (rest) {
    rmsnorm(h_, d, x_, d, w.ln1_g, B, d, T5_EPS, 1.f, st_);
    linear_dec(h_, d, B, w.Wqkv, 3 * il, d, epi_bf16(nullptr, qkv_, 3 * il));
  }
  // the self-attention appends the new token's K / V to the cache itself
  if (attn)
    dattn(qkv_, 3 * il, kc(l), vc(l), slot_ctx_, db, db.nkeys, db.max_keys, db.sum_keys, dec_bias_, true, db.kv);
  if (rest) {
    resid_update(true, ctx_, il, B, w.Wo, il, nullptr);
    rmsnorm(h_, d, x_, d, w.lnx_g, B, d, T5_EPS, 1.f, st_);
    linear_dec(h_, d, B, w.Wqx, il, d, epi_bf16(nullptr, qkv_, 3 * il));
  }
  if (attn) dattn(qkv_, 3 * il, xkc(l), xvc(l), xctx_, db, db.xkeys, db.max_xkeys, db.sum_xkeys, nullptr);
  if (rest) {
    resid_update(true, ctx_, il, B, w.Wox, il, nullptr);
    rmsnorm(h_, d, x_, d, w.ln2_g, B, d, T5_EPS, 1.f, st_);
    linear_dec(h_, d, B, w.W1, D.ffl, d, epi_bf16(nullptr, ff_, D.ffl, ACT_RELU));
    resid_update(true, ff_, D.ffl, B, w.W2, D.ffl, nullptr);
  }
}

namespace {
__global__ void set_last_tokens_kernel(int32_t* last_tok, const int32_t* rslot, const int32_t* tok, int n) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) last_tok[rslot[k]] = tok[k];
}
}  // namespace

void set_last_tokens(int32_t* last_tok, const int32_t* rslot, const int32_t* tok, int n, cudaStream_t st) {
  if (n <= 0) return;
  set_last_tokens_kernel<<<(n + 127) / 128, 128, 0, st>>>(last_tok, rslot, tok, n);
  EXG_CHECK_LAUNCH();
}

}  // namespace exg
