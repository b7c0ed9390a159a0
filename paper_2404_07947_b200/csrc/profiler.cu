// XProfiler: "for a single encoding and decoding layer,
// the profiler separately measures the execution times of the attention
// kernel and the rest of the encoding/decoding layer ... sweeps across batch
// sizes and, for each batch size, ... over possible sequence lengths.  For
// the latter, ... sweeping input sizes (batch x input length)."
//
// Each point runs the real sm_100a kernels of one layer (layer 0) on
// synthetic tables, 1 warm-up + `reps` timed repetitions, CUDA events on the
// engine stream, median kept.  TP degree 1 on a single-GPU context (TP>1
// all-reduce and PP send timings need a multi-rank context).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <vector>

#include "profiler.h"

namespace exg {

namespace {
// Reads a buffer larger than L2 so every timed repetition starts with the
// layer's weights and KV cold, as they are inside a real step (each layer's
// weights are streamed once per iteration).
__global__ void l2_flush_kernel(const int4* __restrict__ p, int64_t n, int* sink) {
  int acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc ^= __ldcs(p + i).x;
  if (acc == 0x7fffffff) *sink = acc;
}

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t st;
  int4* flush = nullptr;
  int64_t flush_n = 0;
  explicit Timer(cudaStream_t s) : st(s) {
    EXG_CUDA(cudaEventCreate(&a));
    EXG_CUDA(cudaEventCreate(&b));
    flush_n = (256ll << 20) / sizeof(int4);
    EXG_CUDA(cudaMalloc(&flush, flush_n * sizeof(int4) + 16));
    EXG_CUDA(cudaMemsetAsync(flush, 0, flush_n * sizeof(int4) + 16, st));
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (flush) cudaFree(flush);
  }
  // median over `reps` of (time of `burst` back-to-back runs of f) / burst,
  // L2 flushed before each rep.  burst = 1: one cold run (attention tables);
  // burst > 1: the layer as it runs inside a step -- consecutive layers
  // chained under PDL, the clock in its sustained state (the "rest" tables;
  // a large model's layer weights exceed L2, so repeats stream from HBM)
  template <class F>
  double median(int reps, F&& f, int burst = 1) {
    f();  // warm-up
    std::vector<double> v;
    for (int r = 0; r < reps; ++r) {
      l2_flush_kernel<<<148 * 4, 256, 0, st>>>(flush, flush_n, reinterpret_cast<int*>(flush + flush_n));
      EXG_CHECK_LAUNCH();
      EXG_CUDA(cudaEventRecord(a, st));
      for (int k = 0; k < burst; ++k) f();
      EXG_CUDA(cudaEventRecord(b, st));
      EXG_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      EXG_CUDA(cudaEventElapsedTime(&ms, a, b));
      v.push_back(ms * 1e-3 / burst);
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  }
  // the clock's sustained (power-capped) state of a long phase: f back to
  // back for >= warm_s unmeasured, then >= meas_s timed (no host sync in
  // between); median over reps
  template <class F>
  double sustained(int reps, F&& f, double warm_s = 0.05, double meas_s = 0.05) {
    EXG_CUDA(cudaEventRecord(a, st));
    f();
    EXG_CUDA(cudaEventRecord(b, st));
    EXG_CUDA(cudaEventSynchronize(b));
    float ms1 = 0;
    EXG_CUDA(cudaEventElapsedTime(&ms1, a, b));
    const double t1 = std::max(1e-6, ms1 * 1e-3);
    const int kw = (int)std::min(4000.0, std::ceil(warm_s / t1));
    const int k = (int)std::max(2.0, std::min(4000.0, std::ceil(meas_s / t1)));
    std::vector<double> v;
    for (int r = 0; r < reps; ++r) {
      for (int i = 0; i < kw; ++i) f();
      EXG_CUDA(cudaEventRecord(a, st));
      for (int i = 0; i < k; ++i) f();
      EXG_CUDA(cudaEventRecord(b, st));
      EXG_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      EXG_CUDA(cudaEventElapsedTime(&ms, a, b));
      v.push_back(ms * 1e-3 / k);
    }
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  }
};
}  // namespace

constexpr int kBurst = 8, kBurstEnc = 4;

// diagnostics (exg_diag_profile_insitu): 1 = the decode attention table is
// the in-situ increment of a PDL-chained burst of full layers over the rest
// burst (it then also charges the kernel boundaries around the attention
// launches); 0 = the attention launches timed alone (default)
int& profile_insitu() {
  static int on = 0;
  return on;
}

// attention and "rest" tables of one layer of engine E under key t (+ the
// decode head table when E holds the LM head and t = 1)
static void profile_one(Engine& E, int t, const exg_profile_grid& g, plan::Profile& P) {
  const Dims& D = E.dims();
  const int reps = std::max(1, g.reps);
  std::vector<int> bs(g.batch, g.batch + g.n_batch), cs(g.ctx, g.ctx + g.n_ctx), ts(g.tokens, g.tokens + g.n_tokens);
  for (auto* v : {&bs, &cs, &ts})
    for (size_t i = 0; i < v->size(); ++i)
      if ((*v)[i] < 1 || (i && (*v)[i] <= (*v)[i - 1])) throw std::invalid_argument("grid axes must be increasing, >= 1");
  const int max_b = bs.back(), max_c = std::min(cs.back(), D.max_pos), max_t = ts.back();
  // encode-attention points with b*c > max_t tokens are timed at
  // b' = max_t / c requests and scaled by b / b' (requests are independent)
  const int max_enc_tokens = std::max(max_t, max_c);
  const int ctx_cap = max_c;
  const int slots = std::max(max_b, (max_enc_tokens + ctx_cap - 1) / ctx_cap);
  E.ensure_kv(slots, ctx_cap, 1, E.encdec() ? ctx_cap : 0);
  E.ensure_workspace(max_enc_tokens, max_b);
  cudaStream_t st = E.stream();

  // synthetic tables: token t -> (slot t / ctx_cap, pos t % ctx_cap)
  const int n_tok = max_enc_tokens;
  std::vector<int32_t> h_ids(n_tok), h_pos(n_tok), h_slot(n_tok);
  for (int t = 0; t < n_tok; ++t) {
    h_ids[t] = t % D.V;
    h_pos[t] = t % ctx_cap;
    h_slot[t] = t / ctx_cap;
  }
  int32_t* d;
  const size_t nints = (size_t)3 * n_tok + 3 * (slots + 1) + 2 * max_b;
  EXG_CUDA(cudaMalloc(&d, nints * sizeof(int32_t)));
  int32_t *d_ids = d, *d_pos = d + n_tok, *d_slot = d + 2 * n_tok;
  int32_t *d_cu = d + 3 * n_tok, *d_rs = d_cu + slots + 1, *d_p0 = d_rs + slots + 1, *d_aux = d_p0 + slots + 1;
  EXG_CUDA(cudaMemcpy(d_ids, h_ids.data(), n_tok * 4, cudaMemcpyHostToDevice));
  EXG_CUDA(cudaMemcpy(d_pos, h_pos.data(), n_tok * 4, cudaMemcpyHostToDevice));
  EXG_CUDA(cudaMemcpy(d_slot, h_slot.data(), n_tok * 4, cudaMemcpyHostToDevice));
  std::vector<int32_t> h_rs(slots + 1), h_p0(slots + 1, 0);
  for (int i = 0; i <= slots; ++i) h_rs[i] = i;
  EXG_CUDA(cudaMemcpy(d_rs, h_rs.data(), (slots + 1) * 4, cudaMemcpyHostToDevice));
  EXG_CUDA(cudaMemcpy(d_p0, h_p0.data(), (slots + 1) * 4, cudaMemcpyHostToDevice));

  Timer tm(st);
  plan::Table2D ae, ad;
  ae.b.assign(bs.begin(), bs.end());
  ae.c.assign(cs.begin(), cs.end());
  ad = ae;
  ae.t.assign(bs.size(), std::vector<double>(cs.size()));
  ad.t.assign(bs.size(), std::vector<double>(cs.size()));
  std::vector<int32_t> h_cu(slots + 1), h_nk(2 * max_b);
  std::vector<std::vector<double>> full_dec(bs.size(), std::vector<double>(cs.size(), 0.0));
  for (size_t ib = 0; ib < bs.size(); ++ib) {
    const int b = bs[ib];
    for (size_t ic = 0; ic < cs.size(); ++ic) {
      const int c = std::min(cs[ic], ctx_cap);
      // encode attention: be requests of c tokens each, request k in slot k
      const int be = std::max(1, std::min(b, max_enc_tokens / c));
      for (int k = 0; k <= be; ++k) h_cu[k] = k * c;
      EXG_CUDA(cudaMemcpy(d_cu, h_cu.data(), (be + 1) * 4, cudaMemcpyHostToDevice));
      EncodeBatch eb;
      eb.T = be * c;
      eb.R = be;
      eb.max_len = c;
      eb.ids = d_ids;
      eb.pos = d_pos;
      eb.tslot = d_slot;
      eb.cu = d_cu;
      eb.rslot = d_rs;
      eb.pos0 = d_p0;
      ae.t[ib][ic] = tm.median(reps, [&] { E.layer_encode(0, eb, true, false); }) * ((double)b / be);
      // decode attention: b rows, c keys each, row i in slot i
      // (encoder-decoder: c keys split between self- and cross-attention,
      // ceil(c/2) encoder keys -- the simulator's context is S_e + S_d / 2)
      const int c_self = E.encdec() ? std::max(1, c / 2) : c, c_x = std::max(1, c - c / 2);
      for (int i = 0; i < b; ++i) h_nk[i] = c_self;
      for (int i = 0; i < b; ++i) h_nk[max_b + i] = c_x;
      EXG_CUDA(cudaMemcpy(d_aux, h_nk.data(), 2 * max_b * 4, cudaMemcpyHostToDevice));
      DecodeBatch db;
      db.B = b;
      db.max_keys = c_self;
      db.slot = d_rs;
      db.pos = d_p0;
      db.nkeys = d_aux;
      db.xkeys = d_aux + max_b;
      db.max_xkeys = c_x;
      ad.t[ib][ic] = tm.median(reps, [&] { E.layer_decode(0, db, true, false); });
      if (profile_insitu()) full_dec[ib][ic] = tm.median(reps, [&] { E.layer_decode(0, db, true, true); }, kBurst);
    }
  }
  P.attn[{"enc", t}] = ae;
  P.attn[{"dec", t}] = ad;
  plan::Table1D re, rd;
  // decode rest (timed before the encode heater below: memory-bound decode
  // iterations run between encode phases at the recovered clock): input
  // size = batch rows, swept over the batch axis
  for (int b : bs) {
    DecodeBatch db;
    db.B = b;
    db.max_keys = 1;
    db.slot = d_rs;
    db.pos = d_p0;
    db.nkeys = d_aux;
    db.xkeys = d_aux + max_b;
    db.max_xkeys = 1;
    rd.x.push_back(b);
    rd.t.push_back(tm.median(reps, [&] { E.layer_decode(0, db, false, true); }, kBurst));
  }
  if (profile_insitu()) {
    for (size_t ib = 0; ib < bs.size(); ++ib)
      for (size_t ic = 0; ic < cs.size(); ++ic)
        ad.t[ib][ic] = std::max(0.05 * full_dec[ib][ic], full_dec[ib][ic] - rd.t[ib]);
    P.attn[{"dec", t}] = ad;
  }
  // head of a decode iteration on the last stage (final norm + tied LM head +
  // argmax), per decode batch: the model-level part of an iteration that the
  // per-layer tables do not hold (DESIGN.md reading)
  plan::Table1D hd;
  if (t == 1 && E.shard().head) {
    std::vector<int32_t> h_off(max_b);
    for (int i = 0; i < max_b; ++i) h_off[i] = i;
    int32_t* d_tok = nullptr;
    EXG_CUDA(cudaMalloc(&d_tok, sizeof(int32_t) * 2 * max_b));
    EXG_CUDA(cudaMemcpy(d_tok, h_off.data(), max_b * 4, cudaMemcpyHostToDevice));
    for (int b : bs) {
      DecodeBatch db;
      db.B = b;
      db.max_keys = 1;
      db.slot = d_rs;
      db.pos = d_p0;
      db.nkeys = d_aux;
      db.out_off = d_tok;
      db.out_tokens = d_tok + max_b;   // scratch: the argmax writes ids there
      hd.x.push_back(b);
      hd.t.push_back(tm.median(reps, [&] { E.head_decode(db); }, kBurst));
    }
    EXG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_tok);
  }
  // Sustained-load state (reading): a real encode phase runs
  // back-to-back prefill GEMMs for ~0.1-0.3 s, long enough for the power
  // limiter to settle the SM clock below its boost; bring the GPU there
  // before timing the "rest" tables (compute-bound prefill GEMMs follow the
  // clock).  Runs the largest encode point for >= 0.5 s.
  {
    EncodeBatch hb;
    hb.T = ts.back();
    hb.R = 1;
    hb.max_len = hb.T;
    hb.ids = d_ids;
    hb.pos = d_pos;
    hb.tslot = d_slot;
    const auto t0 = std::chrono::steady_clock::now();
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 0.5) {
      for (int k = 0; k < 4; ++k) E.layer_encode(0, hb, false, true);
      EXG_CUDA(cudaStreamSynchronize(st));
    }
  }
  for (int T : ts) {
    EncodeBatch eb;
    eb.T = T;
    eb.R = 1;
    eb.max_len = T;
    eb.ids = d_ids;
    eb.pos = d_pos;
    eb.tslot = d_slot;
    re.x.push_back(T);
    // encoder-decoder: the encode phase also projects the cross K/V of each
    // decoder layer (K13), charged to the layer
    // a real encode phase is 0.1-0.3 s of back-to-back prefill GEMMs: the
    // clock is the power-capped sustained one (DESIGN.md reading)
    re.t.push_back(tm.sustained(reps, [&] {
      E.layer_encode(0, eb, false, true);
      if (E.encdec()) E.cross_kv(0, eb);
    }));
  }
  // encode -> decode switch: after an encode phase the clock recovers from
  // the power cap over the first decode iterations.  Per decode batch b (a
  // subset of the batch axis, its ends included): k = 1..16 back-to-back
  // iterations (L decode layers of layer 0's weights and KV + the head) right
  // after a sustained encode burst, minus the same at the recovered clock;
  // the table holds the cumulative extra time of the first k iterations
  plan::Table2D swt;
  if (t == 1) {
    const int n_sw = E.dims().L;
    const int c_sw = cs[cs.size() / 2] < ctx_cap ? cs[cs.size() / 2] : ctx_cap;
    std::vector<int32_t> h_k(2 * max_b);
    for (int i = 0; i < max_b; ++i) h_k[i] = c_sw, h_k[max_b + i] = std::max(1, c_sw / 2);
    EXG_CUDA(cudaMemcpy(d_aux, h_k.data(), 2 * max_b * 4, cudaMemcpyHostToDevice));
    int32_t* d_tok = nullptr;
    EXG_CUDA(cudaMalloc(&d_tok, sizeof(int32_t) * 2 * max_b));
    std::vector<int32_t> h_off(max_b);
    for (int i = 0; i < max_b; ++i) h_off[i] = i;
    EXG_CUDA(cudaMemcpy(d_tok, h_off.data(), max_b * 4, cudaMemcpyHostToDevice));
    EncodeBatch hb;
    hb.T = ts.back();
    hb.R = 1;
    hb.max_len = hb.T;
    hb.ids = d_ids;
    hb.pos = d_pos;
    hb.tslot = d_slot;
    const std::vector<int> ks = {1, 2, 4, 8, 16};
    const int KMAX = ks.back();
    std::vector<cudaEvent_t> ev(2 * (KMAX + 1));
    for (auto& e : ev) EXG_CUDA(cudaEventCreate(&e));
    std::vector<int> bsw;
    for (size_t i = 0; i < bs.size(); i += 3) bsw.push_back(bs[i]);
    if (bsw.back() != bs.back()) bsw.push_back(bs.back());
    swt.b.assign(bsw.begin(), bsw.end());
    swt.c.assign(ks.begin(), ks.end());
    for (int b : bsw) {
      DecodeBatch db;
      db.B = b;
      db.max_keys = c_sw;
      db.sum_keys = (double)b * c_sw;
      db.slot = d_rs;
      db.pos = d_p0;
      db.nkeys = d_aux;
      db.xkeys = d_aux + max_b;
      db.max_xkeys = std::max(1, c_sw / 2);
      db.out_off = d_tok;
      db.out_tokens = d_tok + max_b;
      auto run_k = [&](cudaEvent_t* e) {
        EXG_CUDA(cudaEventRecord(e[0], st));
        for (int k = 1; k <= KMAX; ++k) {
          for (int l = 0; l < n_sw; ++l) E.layer_decode(0, db, true, true);
          if (E.shard().head) E.head_decode(db);
          EXG_CUDA(cudaEventRecord(e[k], st));
        }
        EXG_CUDA(cudaEventSynchronize(e[KMAX]));
      };
      std::vector<std::vector<double>> ex(ks.size());
      for (int r = 0; r < std::max(2, reps - 1); ++r) {
        const auto h0 = std::chrono::steady_clock::now();   // sustained encode ...
        while (std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count() < 0.06) {
          for (int k = 0; k < 2; ++k) E.layer_encode(0, hb, false, true);
          EXG_CUDA(cudaStreamSynchronize(st));
        }
        for (int k = 0; k < 2; ++k) E.layer_encode(0, hb, false, true);   // ... still running when decode is queued
        run_k(ev.data());
        std::this_thread::sleep_for(std::chrono::milliseconds(80));       // the clock recovers
        run_k(ev.data() + KMAX + 1);
        for (size_t j = 0; j < ks.size(); ++j) {
          float ma = 0, mb = 0;
          EXG_CUDA(cudaEventElapsedTime(&ma, ev[0], ev[ks[j]]));
          EXG_CUDA(cudaEventElapsedTime(&mb, ev[KMAX + 1], ev[KMAX + 1 + ks[j]]));
          ex[j].push_back(std::max(0.0, (ma - mb) * 1e-3));
        }
      }
      std::vector<double> row;
      for (auto& v : ex) {
        std::sort(v.begin(), v.end());
        row.push_back(v[v.size() / 2]);
      }
      for (size_t j = 1; j < row.size(); ++j) row[j] = std::max(row[j], row[j - 1]);   // cumulative: non-decreasing
      swt.t.push_back(row);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    EXG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_tok);
  }
  P.rest[{"enc", t}] = re;
  P.rest[{"dec", t}] = rd;
  if (!hd.x.empty()) {
    P.head = hd;
    P.has_head = true;
  }
  if (!swt.b.empty()) {
    P.sw = swt;
    P.has_sw = true;
  }
  EXG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d);
}

// Every requested TP degree t ("all possible parallel
// configurations"): t = 1 times the context's own layer 0; t > 1 builds a
// one-layer shard engine of TP rank 0 (H/t heads, d_ff/t FFN columns -- the
// per-GPU work of a TP group) and times it the same way.  The all-reduce
// itself is the tp_sync table (exg_profile_comm_model / a multi-rank profile).
void profile_layers(Engine& E, const exg_model_spec& spec, const exg_profile_grid& g, plan::Profile* out) {
  if (g.n_batch < 1 || g.n_ctx < 1 || g.n_tokens < 1) throw std::invalid_argument("empty profile grid");
  std::vector<int> tps;
  for (int i = 0; i < g.n_tp; ++i) tps.push_back(g.tp[i]);
  if (tps.empty()) tps.push_back(1);
  for (size_t i = 0; i < tps.size(); ++i)
    if (tps[i] < 1 || (i && tps[i] <= tps[i - 1])) throw std::invalid_argument("grid TP degrees must be increasing");
  plan::Profile& P = *out;
  P = plan::Profile();
  for (int t : tps) {
    if (t == 1) {
      profile_one(E, 1, g, P);
    } else {
      if (E.encdec()) throw std::invalid_argument("T5: tensor-parallel profiles are not built yet");
      if (spec.n_heads % t || spec.d_ff % t) throw std::invalid_argument("TP degree must divide n_heads and d_ff");
      EngineShard sh;
      sh.l0 = 0;
      sh.l1 = 1;
      sh.tp = t;
      sh.tp_rank = 0;
      sh.embed = false;
      sh.head = false;
      Engine shard(spec, E.device(), sh);
      profile_one(shard, t, g, P);
    }
    P.tps.push_back(t);
  }
}

}  // namespace exg

extern "C" void exg_diag_profile_insitu(int on) { exg::profile_insitu() = on; }
