// Multi-stage execution of a schedule: pipeline stages (PP),
// partial tensor parallelism inside a stage
// and WAA's encoder / decoder split with the KV handoff.
//
// This file drives the stages of one schedule on ONE device in a single host
// thread: every (stage, TP rank) is its own Engine holding exactly the weight
// shard and KV of that GPU of the layout, TP partial sums are reduced in rank
// order by sum_tp_parts, pipeline hops and the WAA handoff are device copies
// between the engines.  It is the functional emulation used to check the
// multi-GPU data flow against the oracle on a single B200; the per-stage
// work, tables and transfers are the ones a multi-process deployment (one
// rank per GPU, NCCL in place of the copies) performs.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <vector>

#include "engine.cuh"
#include "multi.h"
#include "runner.h"

namespace exg {

namespace {
struct PartPtrs {
  float* p[8];
  int n;
};

// out[i] = sum_r part_r[i] in rank order, written back to every rank
__global__ void sum_tp_parts_kernel(PartPtrs pp, int64_t n) {
  griddep_launch_dependents();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = pp.p[0][i];
    for (int r = 1; r < pp.n; ++r) s += pp.p[r][i];
    for (int r = 0; r < pp.n; ++r) pp.p[r][i] = s;
  }
}

struct HandoffRow {
  int src_slot, dst_slot, len;
};

// copy K (or V) rows [0, len) of heads [h0, h0+Hd) of each request from an
// encoder KV layer [slot][He][ctx_e][dh] into a decoder KV layer
// [slot][Hd][ctx_d][dh]
__global__ void kv_handoff_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst, const HandoffRow* rows,
                                  int nrows, int He, int h0, int Hd, int ctx_e, int ctx_d, int dh) {
  const int rh = blockIdx.x;
  const int i = rh / Hd, h = rh % Hd;
  if (i >= nrows) return;
  const HandoffRow r = rows[i];
  const int4* s = reinterpret_cast<const int4*>(src + (((int64_t)r.src_slot * He + h0 + h) * ctx_e) * dh);
  int4* d = reinterpret_cast<int4*>(dst + (((int64_t)r.dst_slot * Hd + h) * ctx_d) * dh);
  const int n = r.len * dh / 8;
  for (int e = threadIdx.x; e < n; e += blockDim.x) d[e] = s[e];
}
}  // namespace

void sum_tp_parts(const std::vector<Engine*>& ranks, int64_t n, cudaStream_t st) {
  if (ranks.size() <= 1 || n <= 0) return;
  PartPtrs pp;
  pp.n = (int)ranks.size();
  for (int r = 0; r < pp.n; ++r) pp.p[r] = ranks[r]->part();
  sum_tp_parts_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(pp, n);
  EXG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// Stage: a TP group driven in lockstep
// ---------------------------------------------------------------------------
struct Stage {
  std::vector<std::unique_ptr<Engine>> eng;
  int l0 = 0, l1 = 0, tp = 1;
  bool first = false, last = false;
  cudaStream_t st = nullptr;

  std::vector<Engine*> ptrs() const {
    std::vector<Engine*> v;
    for (auto& e : eng) v.push_back(e.get());
    return v;
  }
  void load_x(const float* x_in, int rows, int d) {
    if (first || !x_in) return;
    for (auto& e : eng) EXG_CUDA(cudaMemcpyAsync(e->x(), x_in, sizeof(float) * rows * d, cudaMemcpyDeviceToDevice, st));
  }
  void encode(const EncodeBatch& eb, const float* x_in, int d) {
    if (eb.T <= 0) return;
    load_x(x_in, eb.T, d);
    for (auto& e : eng) e->embed_encode(eb);
    const auto v = ptrs();
    for (int l = 0; l < l1 - l0; ++l) {
      for (auto& e : eng) e->enc_attn_block(l, eb);
      if (tp > 1) {
        sum_tp_parts(v, (int64_t)eb.T * d, st);
        for (auto& e : eng) e->finish_pending();
      }
      for (auto& e : eng) e->enc_ffn_block(l, eb);
      if (tp > 1) {
        sum_tp_parts(v, (int64_t)eb.T * d, st);
        for (auto& e : eng) e->finish_pending();
      }
    }
  }
  void decode(const DecodeBatch& db, const float* x_in, int d) {
    if (db.B <= 0) return;
    load_x(x_in, db.B, d);
    for (auto& e : eng) e->embed_decode(db);
    const auto v = ptrs();
    for (int l = 0; l < l1 - l0; ++l) {
      for (auto& e : eng) e->dec_attn_block(l, db);
      if (tp > 1) {
        sum_tp_parts(v, (int64_t)db.B * d, st);
        for (auto& e : eng) e->finish_pending();
      }
      for (auto& e : eng) e->dec_ffn_block(l, db);
      if (tp > 1) {
        sum_tp_parts(v, (int64_t)db.B * d, st);
        for (auto& e : eng) e->finish_pending();
      }
    }
    if (last) eng[0]->head_decode(db);  // every TP rank holds the same x: rank 0 runs the head
  }
  float* x_out() { return eng[0]->x(); }
};

// ---------------------------------------------------------------------------
// Layout: the stages of a schedule, built once per layout and cached
// ---------------------------------------------------------------------------
struct Layout {
  std::vector<std::unique_ptr<Stage>> enc, dec;  // WAA: encoder / decoder pipelines; RRA: dec only
};

static std::string layout_key(const exg_schedule& s) {
  std::string k = std::to_string(s.strategy) + ":" + std::to_string(s.n_enc_gpus);
  for (int i = 0; i < s.n_stages; ++i)
    k += "|" + std::to_string(s.stage_n_gpus[i]) + "," + std::to_string(s.stage_layer_begin[i]) + "," +
         std::to_string(s.stage_layer_end[i]);
  return k;
}

struct MultiCtx::Impl {
  exg_model_spec spec;
  int device;
  cudaStream_t st = nullptr;
  std::map<std::string, std::unique_ptr<Layout>> layouts;
};

MultiCtx::MultiCtx(const exg_model_spec& spec, int device) : p_(new Impl) {
  p_->spec = spec;
  p_->device = device;
  EXG_CUDA(cudaSetDevice(device));
  EXG_CUDA(cudaStreamCreateWithFlags(&p_->st, cudaStreamNonBlocking));
}

MultiCtx::~MultiCtx() {
  cudaSetDevice(p_->device);
  if (p_->st) cudaStreamSynchronize(p_->st);
  p_->layouts.clear();
  if (p_->st) cudaStreamDestroy(p_->st);
  delete p_;
}

static std::unique_ptr<Stage> make_stage(const exg_model_spec& spec, int device, cudaStream_t st, int l0, int l1,
                                         int tp, bool first, bool last) {
  auto s = std::make_unique<Stage>();
  s->l0 = l0;
  s->l1 = l1;
  s->tp = tp;
  s->first = first;
  s->last = last;
  s->st = st;
  for (int r = 0; r < tp; ++r) {
    EngineShard sh;
    sh.l0 = l0;
    sh.l1 = l1;
    sh.tp = tp;
    sh.tp_rank = r;
    sh.embed = first;
    sh.head = last && r == 0;
    s->eng.push_back(std::make_unique<Engine>(spec, device, sh, st));
  }
  return s;
}

static Layout* get_layout(MultiCtx::Impl* p, const exg_schedule& s) {
  const std::string key = layout_key(s);
  auto it = p->layouts.find(key);
  if (it != p->layouts.end()) return it->second.get();
  const int L = p->spec.n_dec_layers;
  auto lay = std::make_unique<Layout>();
  std::vector<int> enc_idx, dec_idx;
  for (int i = 0; i < s.n_stages; ++i)
    (s.strategy != EXG_RRA && s.stage_first_gpu[i] < s.n_enc_gpus ? enc_idx : dec_idx).push_back(i);
  auto check_cover = [&](const std::vector<int>& idx) {
    int next = 0;
    for (int i : idx) {
      if (s.stage_layer_begin[i] != next || s.stage_layer_end[i] <= next || s.stage_n_gpus[i] < 1)
        throw std::invalid_argument("schedule stages must cover the layers contiguously");
      next = s.stage_layer_end[i];
    }
    if (next != L) throw std::invalid_argument("schedule stages must cover every layer");
  };
  if (s.strategy != EXG_RRA) check_cover(enc_idx);
  check_cover(dec_idx);
  for (size_t k = 0; k < enc_idx.size(); ++k) {
    const int i = enc_idx[k];
    if (s.stage_n_gpus[i] != 1) throw std::invalid_argument("WAA encoder stages are single-GPU");
    lay->enc.push_back(make_stage(p->spec, p->device, p->st, s.stage_layer_begin[i], s.stage_layer_end[i], 1,
                                  k == 0, false));
  }
  for (size_t k = 0; k < dec_idx.size(); ++k) {
    const int i = dec_idx[k];
    lay->dec.push_back(make_stage(p->spec, p->device, p->st, s.stage_layer_begin[i], s.stage_layer_end[i],
                                  s.stage_n_gpus[i], k == 0, k + 1 == dec_idx.size()));
  }
  Layout* out = lay.get();
  p->layouts[key] = std::move(lay);
  return out;
}

// ---------------------------------------------------------------------------
// shared run state: request bookkeeping, device tables, events
// ---------------------------------------------------------------------------
namespace {
struct Row {
  int req, slot, pos, emitted;
};

struct Tables {
  int32_t* dev = nullptr;
  int32_t* host = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool used = false;
  void ensure(size_t n) {
    if (n <= cap) return;
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
    cap = n;
    EXG_CUDA(cudaMalloc(&dev, cap * sizeof(int32_t)));
    EXG_CUDA(cudaMallocHost(&host, cap * sizeof(int32_t)));
    if (!ev) EXG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  // the host staging buffer may be rewritten once the last upload finished
  int32_t* begin() {
    if (used) EXG_CUDA(cudaEventSynchronize(ev));
    used = true;
    return host;
  }
  void upload(size_t n, cudaStream_t st) {
    EXG_CUDA(cudaMemcpyAsync(dev, host, n * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    EXG_CUDA(cudaEventRecord(ev, st));
  }
  ~Tables() {
    if (ev) cudaEventSynchronize(ev), cudaEventDestroy(ev);
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
  }
};

struct RunState {
  const exg_request* reqs;
  int n;
  std::vector<int64_t> base;
  int64_t total_out = 0;
  int max_in = 1, max_ctx = 1;
  int32_t* d_out = nullptr;
  std::vector<cudaEvent_t> evs;
  std::vector<int> ev_kind, ev_tok;
  std::vector<int> admit_ev, done_ev;
  cudaStream_t st;
  int64_t decode_iters = 0, encode_phases = 0, batch_sum = 0;
  ~RunState() {
    for (auto e : evs) cudaEventDestroy(e);
    if (d_out) cudaFree(d_out);
  }
  int record(int kind, int toks) {
    cudaEvent_t e;
    EXG_CUDA(cudaEventCreate(&e));
    EXG_CUDA(cudaEventRecord(e, st));
    evs.push_back(e);
    ev_kind.push_back(kind);
    ev_tok.push_back(toks);
    return (int)evs.size() - 1;
  }
};

void validate_requests(RunState& R, const Dims& D) {
  R.base.assign(R.n + 1, 0);
  for (int r = 0; r < R.n; ++r) {
    const exg_request& q = R.reqs[r];
    if (q.input_len < 1 || q.output_len < 1 || !q.input_ids) throw std::invalid_argument("request lengths must be >= 1");
    if (q.input_len + q.output_len > D.max_pos) throw std::invalid_argument("input_len + output_len > max_pos");
    for (int j = 0; j < q.input_len; ++j)
      if (q.input_ids[j] < 0 || q.input_ids[j] >= D.V) throw std::invalid_argument("token id out of range");
    R.max_in = std::max(R.max_in, q.input_len);
    R.max_ctx = std::max(R.max_ctx, q.input_len + q.output_len);
    R.base[r + 1] = R.base[r] + q.output_len;
  }
  R.total_out = R.base[R.n];
  EXG_CUDA(cudaMalloc(&R.d_out, sizeof(int32_t) * std::max<int64_t>(R.total_out, 1)));
}

// packed encode tables for requests [r0, r0+k) with the given slots
EncodeBatch build_encode(const RunState& R, Tables& tb, int r0, int k, const int* slots, cudaStream_t st,
                         std::vector<int32_t>* last_ids) {
  int T = 0, maxlen = 0;
  for (int j = 0; j < k; ++j) T += R.reqs[r0 + j].input_len - 1;
  tb.ensure((size_t)3 * T + 3 * (k + 1) + 8);
  int32_t* h = tb.begin();
  int32_t *ids = h, *pos = ids + T, *tsl = pos + T, *cu = tsl + T, *rsl = cu + k + 1, *p0 = rsl + k;
  int t = 0;
  cu[0] = 0;
  EncodeBatch eb;
  for (int j = 0; j < k; ++j) {
    const exg_request& q = R.reqs[r0 + j];
    for (int p = 0; p < q.input_len - 1; ++p, ++t) {
      ids[t] = q.input_ids[p];
      pos[t] = p;
      tsl[t] = slots[j];
    }
    cu[j + 1] = t;
    rsl[j] = slots[j];
    p0[j] = 0;
    maxlen = std::max(maxlen, q.input_len - 1);
    const double m = q.input_len - 1;
    eb.attn_pairs += m * (m + 1) / 2;
    if (last_ids) last_ids->push_back(q.input_ids[q.input_len - 1]);
  }
  tb.upload((size_t)3 * T + (k + 1) + 2 * k, st);
  eb.T = T;
  eb.R = k;
  eb.max_len = maxlen;
  eb.ids = tb.dev;
  eb.pos = tb.dev + T;
  eb.tslot = tb.dev + 2 * T;
  eb.cu = tb.dev + 3 * T;
  eb.rslot = eb.cu + k + 1;
  eb.pos0 = eb.rslot + k;
  return eb;
}

DecodeBatch build_decode(const RunState& R, Tables& tb, const std::vector<Row>& rows, int i0, int B,
                         cudaStream_t st) {
  tb.ensure((size_t)4 * B + 8);
  int32_t* h = tb.begin();
  DecodeBatch db;
  for (int i = 0; i < B; ++i) {
    const Row& rw = rows[i0 + i];
    h[i] = rw.slot;
    h[B + i] = rw.pos;
    h[2 * B + i] = rw.pos + 1;
    h[3 * B + i] = (int32_t)(R.base[rw.req] + rw.emitted);
    db.max_keys = std::max(db.max_keys, rw.pos + 1);
    db.sum_keys += rw.pos + 1;
  }
  tb.upload((size_t)4 * B, st);
  db.B = B;
  db.slot = tb.dev;
  db.pos = tb.dev + B;
  db.nkeys = tb.dev + 2 * B;
  db.out_off = tb.dev + 3 * B;
  db.out_tokens = R.d_out;
  return db;
}

// split n items into `parts` contiguous chunks as equal as possible
std::vector<std::pair<int, int>> chunks(int n, int parts) {
  std::vector<std::pair<int, int>> out;
  parts = std::max(1, std::min(parts, n));
  for (int p = 0, s = 0; p < parts; ++p) {
    const int len = n / parts + (p < n % parts ? 1 : 0);
    if (len > 0) out.push_back({s, len});
    s += len;
  }
  return out;
}

void finish_stats(RunState& R, Engine& any, int32_t* out_tokens, double* out_latency, exg_run_stats* stats) {
  EXG_CUDA(cudaStreamSynchronize(R.st));
  if (out_tokens) EXG_CUDA(cudaMemcpy(out_tokens, R.d_out, sizeof(int32_t) * R.total_out, cudaMemcpyDeviceToHost));
  int32_t err = 0;
  EXG_CUDA(cudaMemcpy(&err, any.err_flag(), sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (err) throw std::runtime_error("NaN logit encountered (T7)");
  const int nev = (int)R.evs.size();
  std::vector<double> t(nev, 0.0);
  for (int k = 1; k < nev; ++k) {
    float ms = 0.f;
    EXG_CUDA(cudaEventElapsedTime(&ms, R.evs[0], R.evs[k]));
    t[k] = ms * 1e-3;
  }
  std::vector<double> lat(R.n);
  for (int r = 0; r < R.n; ++r) {
    lat[r] = t[R.done_ev[r]] - t[R.admit_ev[r]];
    if (out_latency) out_latency[r] = lat[r];
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    const double wall = t[nev - 1];
    stats->wall_s = wall;
    stats->out_tokens = R.total_out;
    stats->decode_iters = R.decode_iters;
    stats->encode_phases = R.encode_phases;
    stats->tok_s = wall > 0 ? R.total_out / wall : 0;
    stats->tok_s_steady = stats->tok_s;
    stats->seq_s = wall > 0 ? R.n / wall : 0;
    std::vector<double> s = lat;
    std::sort(s.begin(), s.end());
    auto pct = [&](double q) {
      const double rr = q * (s.size() - 1);
      const size_t lo = (size_t)std::floor(rr), hi = (size_t)std::ceil(rr);
      return s[lo] + (rr - lo) * (s[hi] - s[lo]);
    };
    stats->lat_p50_s = pct(0.5);
    stats->lat_p99_s = pct(0.99);
    stats->lat_max_s = s.back();
    stats->mean_decode_batch = R.decode_iters ? (double)R.batch_sum / R.decode_iters : 0;
  }
}

// optional fp32 logits dump (exg_run_opts.logits_out / dump_mask)
struct Dump {
  const exg_run_opts* opts = nullptr;
  std::vector<int64_t> base;
  bool on() const { return opts && opts->logits_out && opts->dump_mask; }
};

// run the decode pipeline on `rows` (micro-batches through every stage)
void decode_pipeline(RunState& R, std::vector<std::unique_ptr<Stage>>& pipe, std::vector<Tables>& tabs,
                     const std::vector<Row>& rows, int n_mb, int d, const Dump& dump) {
  const int B = (int)rows.size();
  const auto mbs = chunks(B, n_mb);
  int ti = 0;
  for (const auto& mb : mbs) {
    Tables& tb = tabs[ti++ % tabs.size()];
    DecodeBatch db = build_decode(R, tb, rows, mb.first, mb.second, R.st);
    const float* x = nullptr;
    for (auto& s : pipe) {
      s->decode(db, x, d);
      x = s->x_out();
    }
    if (dump.on()) {
      Engine* head = pipe.back()->eng[0].get();
      const int V = head->dims().V;
      for (int i = 0; i < mb.second; ++i) {
        const Row& rw = rows[mb.first + i];
        if (!dump.opts->dump_mask[rw.req]) continue;
        float* dst = dump.opts->logits_out + (dump.base[rw.req] + rw.emitted) * (int64_t)V;
        EXG_CUDA(cudaMemcpyAsync(dst, head->logits() + (int64_t)i * V, sizeof(float) * V, cudaMemcpyDeviceToHost,
                                 R.st));
      }
    }
  }
}

Dump make_dump(const RunState& R, const exg_run_opts* opts) {
  Dump d;
  d.opts = opts;
  d.base.assign(R.n + 1, 0);
  if (d.on())
    for (int r = 0; r < R.n; ++r) d.base[r + 1] = d.base[r] + (opts->dump_mask[r] ? R.reqs[r].output_len : 0);
  return d;
}

// the last stage's ids become stage 0's next inputs (K15)
void return_tokens(std::vector<std::unique_ptr<Stage>>& pipe, int slots, cudaStream_t st) {
  Engine* head = pipe.back()->eng[0].get();
  for (auto& e : pipe.front()->eng)
    if (e.get() != head)
      EXG_CUDA(cudaMemcpyAsync(e->last_tok(), head->last_tok(), sizeof(int32_t) * slots, cudaMemcpyDeviceToDevice,
                               st));
}

void retire(RunState& R, std::vector<Row>& active, std::vector<int>& free_slots, int ev) {
  int w = 0;
  for (size_t i = 0; i < active.size(); ++i) {
    Row rw = active[i];
    rw.emitted += 1;
    rw.pos += 1;
    if (rw.emitted == R.reqs[rw.req].output_len) {
      R.done_ev[rw.req] = ev;
      free_slots.push_back(rw.slot);
    } else {
      active[w++] = rw;
    }
  }
  active.resize(w);
}
}  // namespace

// ---------------------------------------------------------------------------
// RRA over P pipeline stages with partial TP (S6: encode in
// P micro-batches, decode in P micro-batches)
// ---------------------------------------------------------------------------
static void run_rra_multi(MultiCtx::Impl* p, Layout* lay, const exg_schedule& s, const exg_request* reqs, int n,
                          int32_t* out_tokens, double* out_latency, exg_run_stats* stats, const exg_run_opts* opts) {
  auto& pipe = lay->dec;
  const Dims& D = pipe.front()->eng[0]->dims();
  RunState R;
  R.reqs = reqs;
  R.n = n;
  R.st = p->st;
  validate_requests(R, D);
  const int slot_ctx = (opts && opts->slot_ctx > 0) ? opts->slot_ctx : R.max_ctx;
  if (slot_ctx < R.max_ctx) throw std::invalid_argument("slot_ctx smaller than a request's input+output length");
  const int B_D = s.b_d, B_E = s.b_e, P = (int)pipe.size();
  for (auto& st : pipe)
    for (auto& e : st->eng) {
      e->ensure_kv(B_D, slot_ctx);
      e->ensure_workspace(B_E * (R.max_in - 1), B_D);
    }
  std::vector<Tables> tabs(8);
  const Dump dump = make_dump(R, opts);
  std::vector<int> free_slots(B_D);
  for (int i = 0; i < B_D; ++i) free_slots[i] = B_D - 1 - i;
  std::vector<Row> active;
  R.admit_ev.assign(n, -1);
  R.done_ev.assign(n, -1);
  int next_req = 0, ti = 0;
  R.record(0, 0);
  while (next_req < n || !active.empty()) {
    const int admit = std::min({B_E, B_D - (int)active.size(), n - next_req});
    const int ev_phase = R.record(0, 0);
    if (admit > 0) {
      std::vector<int> slots(admit);
      for (int k = 0; k < admit; ++k) {
        slots[k] = free_slots.back();
        free_slots.pop_back();
        const exg_request& q = reqs[next_req + k];
        active.push_back(Row{next_req + k, slots[k], q.input_len - 1, 0});
        R.admit_ev[next_req + k] = ev_phase;
      }
      // x[n-1] of every admitted request -> last_tok[slot] on the first stage
      for (const auto& mb : chunks(admit, P)) {
        Tables& tb = tabs[ti++ % tabs.size()];
        std::vector<int32_t> last;
        EncodeBatch eb = build_encode(R, tb, next_req + mb.first, mb.second, slots.data() + mb.first, R.st, &last);
        Tables& tl = tabs[ti++ % tabs.size()];
        tl.ensure(2 * last.size() + 2);
        int32_t* h = tl.begin();
        for (size_t j = 0; j < last.size(); ++j) {
          h[j] = slots[mb.first + j];
          h[last.size() + j] = last[j];
        }
        tl.upload(2 * last.size(), R.st);
        for (auto& e : pipe.front()->eng)
          set_last_tokens(e->last_tok(), tl.dev, tl.dev + last.size(), (int)last.size(), R.st);
        const float* x = nullptr;
        for (auto& stg : pipe) {
          stg->encode(eb, x, D.d);
          x = stg->x_out();
        }
      }
      next_req += admit;
      ++R.encode_phases;
    }
    R.record(1, 0);
    for (int u = 0; u < s.n_d && !active.empty(); ++u) {
      decode_pipeline(R, pipe, tabs, active, P, D.d, dump);
      return_tokens(pipe, B_D, R.st);
      const int ev = R.record(2, (int)active.size());
      ++R.decode_iters;
      R.batch_sum += (int64_t)active.size();
      retire(R, active, free_slots, ev);
    }
  }
  finish_stats(R, *pipe.back()->eng[0], out_tokens, out_latency, stats);
}

// ---------------------------------------------------------------------------
// WAA: encoder pipeline and decoder pipeline on disjoint
// GPUs; an encoded batch's KV is handed off layer by layer to the decoder
// stage (and TP rank heads) that owns it and the rows merge into the running
// decode batch at an iteration boundary once the decoder has free slots.
// Decoder iterations run in M = ceil(B_D / B_m) micro-batches.
// ---------------------------------------------------------------------------
static void run_waa_multi(MultiCtx::Impl* p, Layout* lay, const exg_schedule& s, const exg_request* reqs, int n,
                          int32_t* out_tokens, double* out_latency, exg_run_stats* stats, const exg_run_opts* opts) {
  auto& enc = lay->enc;
  auto& dec = lay->dec;
  const Dims& D = dec.front()->eng[0]->dims();
  RunState R;
  R.reqs = reqs;
  R.n = n;
  R.st = p->st;
  validate_requests(R, D);
  const int slot_ctx = (opts && opts->slot_ctx > 0) ? opts->slot_ctx : R.max_ctx;
  if (slot_ctx < R.max_ctx) throw std::invalid_argument("slot_ctx smaller than a request's input+output length");
  const int B_D = s.b_d, B_E = s.b_e;
  if (B_E < 1 || B_D < B_E) throw std::invalid_argument("WAA needs 1 <= B_E <= B_D");
  const int M = s.b_m > 0 ? std::max(1, (B_D + s.b_m - 1) / s.b_m) : 1;
  const int enc_ctx = std::max(1, R.max_in);
  for (auto& st : enc)
    for (auto& e : st->eng) {
      e->ensure_kv(B_E, enc_ctx);
      e->ensure_workspace(B_E * (R.max_in - 1), B_E);
    }
  for (auto& st : dec)
    for (auto& e : st->eng) {
      e->ensure_kv(B_D, slot_ctx);
      e->ensure_workspace(1, B_D);
    }
  std::vector<Tables> tabs(8);
  const Dump dump = make_dump(R, opts);
  HandoffRow* d_hrows = nullptr;
  EXG_CUDA(cudaMalloc(&d_hrows, sizeof(HandoffRow) * B_E));
  HandoffRow* h_hrows = nullptr;
  EXG_CUDA(cudaMallocHost(&h_hrows, sizeof(HandoffRow) * B_E));
  std::vector<int> free_slots(B_D);
  for (int i = 0; i < B_D; ++i) free_slots[i] = B_D - 1 - i;
  std::vector<Row> active;
  R.admit_ev.assign(n, -1);
  R.done_ev.assign(n, -1);
  int next_req = 0, pend_r0 = -1, pend_k = 0, pend_ev = -1, ti = 0;
  R.record(0, 0);
  while (next_req < n || pend_k > 0 || !active.empty()) {
    // encoder: keep one encoded batch ready (encoder slots 0..k-1)
    if (pend_k == 0 && next_req < n) {
      const int k = std::min(B_E, n - next_req);
      pend_ev = R.record(0, 0);
      std::vector<int> eslots(k);
      for (int j = 0; j < k; ++j) eslots[j] = j;
      Tables& tb = tabs[ti++ % tabs.size()];
      EncodeBatch eb = build_encode(R, tb, next_req, k, eslots.data(), R.st, nullptr);
      const float* x = nullptr;
      for (auto& stg : enc) {
        stg->encode(eb, x, D.d);
        x = stg->x_out();
      }
      R.record(1, 0);
      pend_r0 = next_req;
      pend_k = k;
      next_req += k;
      ++R.encode_phases;
    }
    // handoff + merge at an iteration boundary when the decoder has room
    if (pend_k > 0 && (int)free_slots.size() >= pend_k) {
      std::vector<int> dslots(pend_k);
      for (int j = 0; j < pend_k; ++j) {
        dslots[j] = free_slots.back();
        free_slots.pop_back();
        const exg_request& q = reqs[pend_r0 + j];
        h_hrows[j] = HandoffRow{j, dslots[j], q.input_len - 1};
        active.push_back(Row{pend_r0 + j, dslots[j], q.input_len - 1, 0});
        R.admit_ev[pend_r0 + j] = pend_ev;
      }
      EXG_CUDA(cudaMemcpyAsync(d_hrows, h_hrows, sizeof(HandoffRow) * pend_k, cudaMemcpyHostToDevice, R.st));
      for (auto& es : enc) {
        Engine* src = es->eng[0].get();
        for (int l = es->l0; l < es->l1; ++l)
          for (auto& ds : dec) {
            if (l < ds->l0 || l >= ds->l1) continue;
            for (int r = 0; r < ds->tp; ++r) {
              Engine* dst = ds->eng[r].get();
              const int Hd = dst->dims().Hl;
              for (int kv = 0; kv < 2; ++kv) {
                const bf16* sp = kv ? src->vc(l - es->l0) : src->kc(l - es->l0);
                bf16* dp = kv ? dst->vc(l - ds->l0) : dst->kc(l - ds->l0);
                kv_handoff_kernel<<<pend_k * Hd, 128, 0, R.st>>>(sp, dp, d_hrows, pend_k, D.H, r * Hd, Hd, enc_ctx,
                                                                 slot_ctx, D.dh);
                EXG_CHECK_LAUNCH();
              }
            }
          }
      }
      // x[n-1] of the merged requests -> last_tok[slot] on the decoder's first stage
      Tables& tl = tabs[ti++ % tabs.size()];
      tl.ensure(2 * pend_k + 2);
      int32_t* h = tl.begin();
      for (int j = 0; j < pend_k; ++j) {
        const exg_request& q = reqs[pend_r0 + j];
        h[j] = dslots[j];
        h[pend_k + j] = q.input_ids[q.input_len - 1];
      }
      tl.upload(2 * pend_k, R.st);
      for (auto& e : dec.front()->eng) set_last_tokens(e->last_tok(), tl.dev, tl.dev + pend_k, pend_k, R.st);
      // the handoff must finish reading encoder KV before the next encode
      pend_k = 0;
    }
    if (active.empty()) continue;
    decode_pipeline(R, dec, tabs, active, M, D.d, dump);
    return_tokens(dec, B_D, R.st);
    const int ev = R.record(2, (int)active.size());
    ++R.decode_iters;
    R.batch_sum += (int64_t)active.size();
    retire(R, active, free_slots, ev);
  }
  finish_stats(R, *dec.back()->eng[0], out_tokens, out_latency, stats);
  cudaFree(d_hrows);
  cudaFreeHost(h_hrows);
}

void MultiCtx::run(const exg_schedule& s, const exg_request* reqs, int n, int32_t* out_tokens, double* out_latency,
                   exg_run_stats* stats, const exg_run_opts* opts) {
  EXG_CUDA(cudaSetDevice(p_->device));
  if (s.n_stages < 1 || s.n_stages > EXG_MAX_STAGES) throw std::invalid_argument("schedule has no stages");
  Layout* lay = get_layout(p_, s);
  if (s.strategy == EXG_RRA)
    run_rra_multi(p_, lay, s, reqs, n, out_tokens, out_latency, stats, opts);
  else if (s.strategy == EXG_WAA_C || s.strategy == EXG_WAA_M)
    run_waa_multi(p_, lay, s, reqs, n, out_tokens, out_latency, stats, opts);
  else
    throw std::invalid_argument("unknown strategy");
}

}  // namespace exg
