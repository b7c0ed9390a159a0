// Multi-stage execution of a schedule: pipeline stages (PP),
// partial tensor parallelism inside a stage
// and WAA's encoder / decoder split with the KV handoff.
//
// SPMD: every rank runs this same host loop over the whole layout.  GPU g of
// the layout (G GPUs) belongs to rank owner(g) = g * world / G; a rank builds
// the Engines (exact weight shard + KV of that GPU) of the GPUs it owns, runs
// their kernels on its stream, and at each exchange step of the method calls
// the transport (comm.h) when the two GPUs involved belong to different ranks,
// or makes a device copy when they belong to the same one:
//   * pipeline hop: the hidden states [rows][d] fp32 from the previous stage's
//     TP rank 0 to every TP rank of the next stage;
//   * TP reduction: each TP rank's fp32 partial sums exchanged inside the group
//     and summed in rank order on every member (T4(i): bitwise identical on
//     every rank and to the single-rank run);
//   * WAA handoff: each encoded request's K/V rows of every layer, sliced by
//     the receiving TP rank's heads, into the decoder slots it was given;
//   * token return: the last stage's next-token table to the first stage.
// The control flow depends only on request lengths (forced outputs), never on
// device results, so every rank takes the same decisions and issues its sends
// and recvs in the same global order (no deadlock: the earliest pending
// exchange always has both of its ranks waiting on it).  world = 1 runs the
// whole layout in one process on one device (single-device emulation).
//
// Latency stamps: a one-thread kernel writes %globaltimer (ns, common to the
// GPUs of a node) at phase starts (on the rank owning the first encoding
// stage) and iteration ends (on the rank owning the LM head); rank 0 gathers
// them and the output tokens at the end.
#include <algorithm>
#include <functional>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <vector>

#include "comm.h"
#include "engine.cuh"
#include "multi.h"
#include "runner.h"

namespace exg {

namespace {
struct PartPtrs {
  const float* in[8];   // TP partials in rank order
  float* out[8];        // buffers receiving the sum
  int n_in, n_out;
};

__global__ void sum_parts_kernel(PartPtrs pp, int64_t n) {
  griddep_launch_dependents();
  griddep_wait();  // launched with PDL: predecessors complete + visible
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float s = pp.in[0][i];
    for (int r = 1; r < pp.n_in; ++r) s += pp.in[r][i];
    for (int r = 0; r < pp.n_out; ++r) pp.out[r][i] = s;
  }
}

void launch_sum(const PartPtrs& pp, int64_t n, cudaStream_t st) {
  launch_pdl(sum_parts_kernel, dim3((int)std::min<int64_t>((n + 255) / 256, 148 * 8)), dim3(256), 0, st, pp, n);
  EXG_CHECK_LAUNCH();
}

struct HandoffRow {
  int src_slot, dst_slot, len;
  int64_t off;   // rows before this one in the batch (packed message: [row][Hd][len][dh])
};

// K (or V) rows [0, len) of heads [h0, h0+Hd) of each request:
//   mode 0: encoder cache -> decoder cache (both on this rank)
//   mode 1: encoder cache -> packed message
//   mode 2: packed message -> decoder cache
// A paged decoder cache (dpt != nullptr; ctx_d = the page length) takes key k
// of row i at page dpt[i * maxp + k / ctx_d], offset k mod ctx_d.
__global__ void kv_handoff_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst, const HandoffRow* rows,
                                  int nrows, int He, int h0, int Hd, int ctx_e, int ctx_d, int dh, int mode,
                                  const int32_t* __restrict__ dpt = nullptr, int maxp = 0) {
  const int rh = blockIdx.x;
  const int i = rh / Hd, h = rh % Hd;
  if (i >= nrows) return;
  const HandoffRow r = rows[i];
  const int64_t pk = (r.off * Hd + (int64_t)h * r.len) * dh;
  const int4* s = reinterpret_cast<const int4*>(mode == 2 ? src + pk
                                                          : src + (((int64_t)r.src_slot * He + h0 + h) * ctx_e) * dh);
  const int n = r.len * dh / 8;
  if (mode != 1 && dpt) {
    const int cpk = dh / 8;   // 16-byte chunks per key row
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int k = e / cpk, c = e % cpk;
      const int64_t row = ((int64_t)dpt[(int64_t)i * maxp + k / ctx_d] * Hd + h) * ctx_d + k % ctx_d;
      reinterpret_cast<int4*>(dst + row * dh)[c] = s[e];
    }
    return;
  }
  int4* d = reinterpret_cast<int4*>(mode == 1 ? dst + pk : dst + (((int64_t)r.dst_slot * Hd + h) * ctx_d) * dh);
  for (int e = threadIdx.x; e < n; e += blockDim.x) d[e] = s[e];
}

__global__ void stamp_kernel(uint64_t* out) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}
}  // namespace

void sum_tp_parts(const std::vector<Engine*>& ranks, int64_t n, cudaStream_t st) {
  if (ranks.size() <= 1 || n <= 0) return;
  PartPtrs pp;
  pp.n_in = pp.n_out = (int)ranks.size();
  for (int r = 0; r < pp.n_in; ++r) pp.in[r] = pp.out[r] = ranks[r]->part();
  launch_sum(pp, n, st);
}

// ---------------------------------------------------------------------------
// Exec: this rank's view of the layout's GPUs
// ---------------------------------------------------------------------------
// Staging ring of a transfer direction between ranks: the compute stream
// and the communication stream hand buffers to each other through events, so
// a pipeline hop / token return / KV-handoff message travels on the comm
// stream while the compute stream goes on with the next micro-batch
// ("overlapping communication with computation").
struct XferRing {
  static constexpr int N = 4;
  void* buf[N] = {};
  cudaEvent_t ready[N] = {}, done[N] = {};
  bool used[N] = {};
  size_t cap = 0;
  int next = 0;
  ~XferRing() { release(); }
  void release() {
    for (int i = 0; i < N; ++i) {
      if (done[i]) cudaEventSynchronize(done[i]);
      if (buf[i]) cudaFree(buf[i]);
      if (ready[i]) cudaEventDestroy(ready[i]);
      if (done[i]) cudaEventDestroy(done[i]);
      buf[i] = nullptr;
      ready[i] = done[i] = nullptr;
      used[i] = false;
    }
    cap = 0;
  }
  int acquire(size_t bytes) {
    if (bytes > cap) {
      release();
      cap = bytes;
      for (int i = 0; i < N; ++i) {
        EXG_CUDA(cudaMalloc(&buf[i], cap));
        EXG_CUDA(cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming));
        EXG_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
      }
    }
    const int s = next;
    next = (next + 1) % N;
    return s;
  }
};

struct Exec {
  int me = 0, world = 1, G = 1;
  Comm* comm = nullptr;
  cudaStream_t st = nullptr;    // compute stream
  cudaStream_t cst = nullptr;   // communication stream (exchanges between ranks)
  XferRing* tx = nullptr;       // send staging
  XferRing* rx = nullptr;       // receive staging
  // one-rank NCCL loopback (transport test): exchanges between this rank's
  // own GPUs still go through ncclSend / ncclRecv to self
  bool loop = false;
  // parity mode (exg_run_opts.pin_nccl_algo): TP partial sums exchanged and
  // summed in member order on every rank (bitwise the one-rank sum) instead
  // of the transport's all-reduce
  bool pin = false;
  int owner(int gpu) const { return (int)((int64_t)gpu * world / G); }
  bool mine(int gpu) const { return owner(gpu) == me; }
  // bytes from (gpu a, src) to (gpu b, dst); a pointer is only valid on its owner
  void xfer(int ga, const void* src, int gb, void* dst, size_t bytes) const {
    const int oa = owner(ga), ob = owner(gb);
    if (bytes == 0) return;
    if (oa == me && ob == me) {
      if (src == dst) return;
      if (loop) {
        comm->group_start();
        comm->send(src, bytes, me, st);
        comm->recv(dst, bytes, me, st);
        comm->group_end();
      } else {
        EXG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
      }
    } else if (oa == me) {
      send_async(src, bytes, ob);
    } else if (ob == me) {
      recv_async(dst, bytes, oa);
    }
  }
  // comm stream waits for the compute stream / compute stream for the comm stream
  void fork() const {
    EXG_CUDA(cudaEventRecord(ev_fork, st));
    EXG_CUDA(cudaStreamWaitEvent(cst, ev_fork, 0));
  }
  void join() const {
    EXG_CUDA(cudaEventRecord(ev_join, cst));
    EXG_CUDA(cudaStreamWaitEvent(st, ev_join, 0));
  }
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // src (ready on the compute stream) -> peer, through a send staging buffer
  void send_async(const void* src, size_t bytes, int peer) const {
    const int s = tx->acquire(bytes);
    if (tx->used[s]) EXG_CUDA(cudaStreamWaitEvent(st, tx->done[s], 0));   // its previous send is out
    EXG_CUDA(cudaMemcpyAsync(tx->buf[s], src, bytes, cudaMemcpyDeviceToDevice, st));
    EXG_CUDA(cudaEventRecord(tx->ready[s], st));
    EXG_CUDA(cudaStreamWaitEvent(cst, tx->ready[s], 0));
    comm->send(tx->buf[s], bytes, peer, cst);
    EXG_CUDA(cudaEventRecord(tx->done[s], cst));
    tx->used[s] = true;
  }
  // peer -> dst (usable on the compute stream afterwards), through a receive staging buffer
  void recv_async(void* dst, size_t bytes, int peer) const {
    const int s = rx->acquire(bytes);
    if (rx->used[s]) EXG_CUDA(cudaStreamWaitEvent(cst, rx->done[s], 0));   // its previous copy-out is done
    comm->recv(rx->buf[s], bytes, peer, cst);
    EXG_CUDA(cudaEventRecord(rx->ready[s], cst));
    EXG_CUDA(cudaStreamWaitEvent(st, rx->ready[s], 0));
    EXG_CUDA(cudaMemcpyAsync(dst, rx->buf[s], bytes, cudaMemcpyDeviceToDevice, st));
    EXG_CUDA(cudaEventRecord(rx->done[s], st));
    rx->used[s] = true;
  }
};

// ---------------------------------------------------------------------------
// Stage: one TP group (GPUs first_gpu .. first_gpu+tp-1) driven in lockstep
// ---------------------------------------------------------------------------
struct Stage {
  std::vector<std::unique_ptr<Engine>> eng;   // [tp], nullptr for GPUs of other ranks
  int l0 = 0, l1 = 0, tp = 1, first_gpu = 0;
  bool first = false, last = false;
  std::vector<float*> tmp;                    // [tp] partial buffers of the cross-rank exchange
  size_t tmp_cap = 0;

  ~Stage() {
    for (float* p : tmp)
      if (p) cudaFree(p);
  }
  int gpu(int r) const { return first_gpu + r; }
  bool any_local() const {
    for (auto& e : eng)
      if (e) return true;
    return false;
  }

  void ensure_tmp(size_t n) {
    if (n <= tmp_cap) return;
    for (float* p : tmp)
      if (p) cudaFree(p);
    tmp.assign(tp, nullptr);
    tmp_cap = n;
    for (int r = 0; r < tp; ++r) EXG_CUDA(cudaMalloc(&tmp[r], sizeof(float) * tmp_cap));
  }

  // TP reduction of the pending fp32 partials of `rows` rows, then the
  // residual update of every local member
  // owner ranks of this TP group (ascending)
  std::vector<int> ranks(const Exec& X) const {
    std::vector<int> g;
    for (int r = 0; r < tp; ++r)
      if (g.empty() || g.back() != X.owner(gpu(r))) g.push_back(X.owner(gpu(r)));
    return g;
  }

  void tp_reduce(const Exec& X, int rows, int d) {
    if (tp == 1 || !any_local()) return;
    const int64_t n = (int64_t)rows * d;
    bool all_local = true;
    for (int r = 0; r < tp; ++r) all_local &= X.mine(gpu(r));
    std::vector<int> group;
    if (!all_local && !X.pin) group = ranks(X);   // the TP sub-communicator's ranks
    if (all_local) {
      std::vector<Engine*> v;
      for (auto& e : eng) v.push_back(e.get());
      sum_tp_parts(v, n, X.st);
    } else if (!X.pin && X.comm->has_allreduce()) {
      // the local members' partials summed in member order, all-reduced over
      // the group's ranks (NCCL all-reduce in fp32 on the TP
      // sub-communicator, T4(i)), and handed to the other local members
      int first_local = -1;
      PartPtrs pp;
      pp.n_in = 0;
      for (int r = 0; r < tp; ++r)
        if (X.mine(gpu(r))) {
          if (first_local < 0) first_local = r;
          pp.in[pp.n_in++] = eng[r]->part();
        }
      float* buf = eng[first_local]->part();
      if (pp.n_in > 1) {
        pp.n_out = 1;
        pp.out[0] = buf;
        launch_sum(pp, n, X.st);
      }
      X.comm->allreduce_sum(buf, (size_t)n, group, X.st);
      for (int r = first_local + 1; r < tp; ++r)
        if (X.mine(gpu(r)))
          EXG_CUDA(cudaMemcpyAsync(eng[r]->part(), buf, sizeof(float) * n, cudaMemcpyDeviceToDevice, X.st));
    } else {
      ensure_tmp((size_t)n);
      // ranks of this group other than this one
      std::set<int> peers;
      for (int r = 0; r < tp; ++r)
        if (!X.mine(gpu(r))) peers.insert(X.owner(gpu(r)));
      // the main communicator's operations all run on the communication
      // stream, ordered against the compute stream by events
      X.fork();
      X.comm->group_start();
      for (int a = 0; a < tp; ++a) {   // each local partial once to every other rank of the group
        if (!X.mine(gpu(a))) continue;
        for (int q : peers) X.comm->send(eng[a]->part(), sizeof(float) * n, q, X.cst);
      }
      for (int b = 0; b < tp; ++b)     // every remote member's partial, in member order
        if (!X.mine(gpu(b))) X.comm->recv(tmp[b], sizeof(float) * n, X.owner(gpu(b)), X.cst);
      X.comm->group_end();
      X.join();
      // sum in rank order into the spare buffer of the first local member,
      // then hand it to every local member
      PartPtrs pp;
      pp.n_in = tp;
      pp.n_out = 1;
      int first_local = -1;
      for (int r = 0; r < tp; ++r) {
        pp.in[r] = X.mine(gpu(r)) ? eng[r]->part() : tmp[r];
        if (first_local < 0 && X.mine(gpu(r))) first_local = r;
      }
      pp.out[0] = tmp[first_local];
      launch_sum(pp, n, X.st);
      for (int r = 0; r < tp; ++r)
        if (X.mine(gpu(r)))
          EXG_CUDA(cudaMemcpyAsync(eng[r]->part(), tmp[first_local], sizeof(float) * n, cudaMemcpyDeviceToDevice,
                                   X.st));
    }
    for (auto& e : eng)
      if (e) e->finish_pending();
  }

  bool t5() const { return eng.size() == 1 && eng[0] && eng[0]->encdec(); }
  void encode(const Exec& X, const EncodeBatch& eb, int d) {
    if (eb.T <= 0 || !any_local()) return;
    if (t5()) {  // T5 stages are single-GPU: the engine runs its whole part of the encode phase
      eng[0]->encode(eb);
      return;
    }
    for (auto& e : eng)
      if (e) e->embed_encode(eb);
    for (int l = 0; l < l1 - l0; ++l) {
      for (auto& e : eng)
        if (e) e->enc_attn_block(l, eb);
      tp_reduce(X, eb.T, d);
      for (auto& e : eng)
        if (e) e->enc_ffn_block(l, eb);
      tp_reduce(X, eb.T, d);
    }
  }
  void decode(const Exec& X, const DecodeBatch& db, int d) {
    if (db.B <= 0 || !any_local()) return;
    if (t5()) {
      eng[0]->decode(db);
      return;
    }
    for (auto& e : eng)
      if (e) e->embed_decode(db);
    for (int l = 0; l < l1 - l0; ++l) {
      for (auto& e : eng)
        if (e) e->dec_attn_block(l, db);
      tp_reduce(X, db.B, d);
      for (auto& e : eng)
        if (e) e->dec_ffn_block(l, db);
      tp_reduce(X, db.B, d);
    }
    // every TP rank holds the same x: rank 0 of the last stage runs the head
    if (last && eng[0]) eng[0]->head_decode(db);
  }
};

// hidden states of `rows` rows: previous stage's TP rank 0 -> every TP rank of the next
static void hop(const Exec& X, Stage& prev, Stage& next, int rows, int d) {
  const size_t bytes = sizeof(float) * (size_t)rows * d;
  for (int r = 0; r < next.tp; ++r)
    X.xfer(prev.gpu(0), prev.eng[0] ? prev.eng[0]->x() : nullptr, next.gpu(r),
           next.eng[r] ? next.eng[r]->x() : nullptr, bytes);
}

// ---------------------------------------------------------------------------
// Layout: the stages of a schedule, built once per layout and cached
// ---------------------------------------------------------------------------
struct Layout {
  std::vector<std::unique_ptr<Stage>> enc, dec;  // WAA: encoder / decoder pipelines; RRA: dec only
  int G = 0;                                     // GPUs of the layout
};

static std::string layout_key(const exg_schedule& s) {
  std::string k = std::to_string(s.strategy) + ":" + std::to_string(s.n_enc_gpus);
  for (int i = 0; i < s.n_stages; ++i)
    k += "|" + std::to_string(s.stage_first_gpu[i]) + "," + std::to_string(s.stage_n_gpus[i]) + "," +
         std::to_string(s.stage_layer_begin[i]) + "," + std::to_string(s.stage_layer_end[i]);
  return k;
}

struct MultiCtx::Impl {
  exg_model_spec spec;
  int device;
  cudaStream_t st = nullptr;    // compute
  cudaStream_t cst = nullptr;   // exchanges with other ranks (PAPER.md:176 overlap)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  XferRing tx, rx;
  std::unique_ptr<Comm> comm;
  int rank = 0, world = 1;
  bool loopback = false;   // a one-rank communicator: route local exchanges through it
  std::map<std::string, std::unique_ptr<Layout>> layouts;
  // the executors' table ring (device + pinned host buffers) and WAA's
  // handoff ring, kept across runs so the end-to-end path does not allocate
  // and pin per run (and released with the context, whatever a run threw)
  std::shared_ptr<void> tab_cache, hr_cache;
};

MultiCtx::MultiCtx(const exg_model_spec& spec, int device, std::unique_ptr<Comm> comm) : p_(new Impl) {
  p_->spec = spec;
  p_->device = device;
  if (comm) {
    p_->rank = comm->rank();
    p_->world = comm->world();
    p_->loopback = comm->world() == 1;
  }
  p_->comm = std::move(comm);
  EXG_CUDA(cudaSetDevice(device));
  EXG_CUDA(cudaStreamCreateWithFlags(&p_->st, cudaStreamNonBlocking));
  EXG_CUDA(cudaStreamCreateWithFlags(&p_->cst, cudaStreamNonBlocking));
  EXG_CUDA(cudaEventCreateWithFlags(&p_->ev_fork, cudaEventDisableTiming));
  EXG_CUDA(cudaEventCreateWithFlags(&p_->ev_join, cudaEventDisableTiming));
}

MultiCtx::~MultiCtx() {
  cudaSetDevice(p_->device);
  if (p_->st) cudaStreamSynchronize(p_->st);
  if (p_->cst) cudaStreamSynchronize(p_->cst);
  p_->layouts.clear();
  p_->tab_cache.reset();
  p_->hr_cache.reset();
  p_->tx.release();
  p_->rx.release();
  p_->comm.reset();
  if (p_->ev_fork) cudaEventDestroy(p_->ev_fork);
  if (p_->ev_join) cudaEventDestroy(p_->ev_join);
  if (p_->st) cudaStreamDestroy(p_->st);
  if (p_->cst) cudaStreamDestroy(p_->cst);
  delete p_;
}

int MultiCtx::rank() const { return p_->rank; }
int MultiCtx::world() const { return p_->world; }

static Exec make_exec(MultiCtx::Impl* p, int G, const exg_run_opts* opts = nullptr) {
  Exec X;
  X.me = p->rank;
  X.world = p->world;
  X.G = G;
  X.comm = p->comm.get();
  X.st = p->st;
  X.cst = p->cst;
  X.tx = &p->tx;
  X.rx = &p->rx;
  X.ev_fork = p->ev_fork;
  X.ev_join = p->ev_join;
  X.loop = p->loopback;
  X.pin = opts && opts->pin_nccl_algo;
  return X;
}

static std::unique_ptr<Stage> make_stage(const MultiCtx::Impl* p, const Exec& X, int first_gpu, int l0, int l1,
                                         int tp, bool first, bool last, int t5_role = 0, bool enc_last = true) {
  auto s = std::make_unique<Stage>();
  s->l0 = l0;
  s->l1 = l1;
  s->tp = tp;
  s->first_gpu = first_gpu;
  s->first = first;
  s->last = last;
  s->eng.resize(tp);
  for (int r = 0; r < tp; ++r) {
    if (!X.mine(first_gpu + r)) continue;
    EngineShard sh;
    sh.l0 = l0;
    sh.l1 = l1;
    sh.tp = tp;
    sh.tp_rank = r;
    sh.embed = first;
    sh.head = last && r == 0;
    sh.t5_role = t5_role;
    sh.enc_last = enc_last;
    s->eng[r] = std::make_unique<Engine>(p->spec, p->device, sh, p->st);
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
  int G = 0;
  for (int i = 0; i < s.n_stages; ++i) {
    if (s.stage_first_gpu[i] != G) throw std::invalid_argument("schedule stages must occupy consecutive GPUs");
    if (s.stage_n_gpus[i] < 1 || s.stage_n_gpus[i] > 8) throw std::invalid_argument("bad stage GPU count");
    G += s.stage_n_gpus[i];
    (s.strategy != EXG_RRA && s.stage_first_gpu[i] < s.n_enc_gpus ? enc_idx : dec_idx).push_back(i);
  }
  if (p->world > G) throw std::invalid_argument("more ranks than GPUs in the schedule's layout");
  lay->G = G;
  auto check_cover = [&](const std::vector<int>& idx) {
    int next = 0;
    for (int i : idx) {
      if (s.stage_layer_begin[i] != next || s.stage_layer_end[i] <= next)
        throw std::invalid_argument("schedule stages must cover the layers contiguously");
      next = s.stage_layer_end[i];
    }
    if (next != L) throw std::invalid_argument("schedule stages must cover every layer");
  };
  if (s.strategy != EXG_RRA) check_cover(enc_idx);
  check_cover(dec_idx);
  const Exec X = make_exec(p, G);
  const bool t5 = p->spec.arch == EXG_ARCH_T5;
  for (size_t k = 0; k < enc_idx.size(); ++k) {
    const int i = enc_idx[k];
    if (s.stage_n_gpus[i] != 1) throw std::invalid_argument("WAA encoder stages are single-GPU");
    lay->enc.push_back(make_stage(p, X, s.stage_first_gpu[i], s.stage_layer_begin[i], s.stage_layer_end[i], 1,
                                  k == 0, false, t5 ? 1 : 0, k + 1 == enc_idx.size()));
  }
  for (size_t k = 0; k < dec_idx.size(); ++k) {
    const int i = dec_idx[k];
    if (t5 && s.stage_n_gpus[i] != 1) throw std::invalid_argument("T5: tensor-parallel stages are not built yet");
    // T5 under RRA: each stage holds encoder and decoder layers [l0, l1) (role 0)
    const bool rra = s.strategy == EXG_RRA;
    lay->dec.push_back(make_stage(p, X, s.stage_first_gpu[i], s.stage_layer_begin[i], s.stage_layer_end[i],
                                  s.stage_n_gpus[i], k == 0, k + 1 == dec_idx.size(), t5 ? (rra ? 0 : 2) : 0,
                                  k + 1 == dec_idx.size()));
  }
  // TP sub-communicators (collective: every rank builds the same layout at
  // the same point of the run)
  if (p->world > 1 && p->comm) {
    std::vector<std::vector<int>> groups;
    for (auto* side : {&lay->enc, &lay->dec})
      for (auto& st : *side)
        if (st->tp > 1) {
          std::vector<int> g = st->ranks(X);
          if (g.size() > 1) groups.push_back(g);
        }
    p->comm->prepare_groups(groups);
  }
  Layout* out = lay.get();
  p->layouts[key] = std::move(lay);
  return out;
}

// ---------------------------------------------------------------------------
// shared run state: request bookkeeping, device tables, stamps
// ---------------------------------------------------------------------------
namespace {
struct Row {
  int req, slot, pos, emitted;
  int64_t seq = 0;   // admission order (paged KV: the swap-out victim is the latest)
};

struct Tables {
  int32_t* dev = nullptr;
  int32_t* host = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool used = false;
  void ensure(size_t n) {
    if (n <= cap) return;
    if (used) EXG_CUDA(cudaEventSynchronize(ev));
    if (dev) cudaFree(dev);
    if (host) cudaFreeHost(host);
    cap = n;
    used = false;
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

// WAA handoff row tables: a ring of pinned host / device pairs recycled by
// events (no host synchronisation per handoff), plus the loopback transport's
// staging buffer (both halves of a self-message); cached in the context
struct HandoffRing {
  static constexpr int N = 4;
  HandoffRow* d[N] = {};
  HandoffRow* h[N] = {};
  cudaEvent_t ev[N] = {};
  bool used[N] = {};
  int next = 0, cap = 0;
  bf16* stage = nullptr;
  size_t stage_cap = 0;   // elements per half
  void release() {
    for (int i = 0; i < N; ++i) {
      if (ev[i]) cudaEventSynchronize(ev[i]), cudaEventDestroy(ev[i]);
      if (d[i]) cudaFree(d[i]);
      if (h[i]) cudaFreeHost(h[i]);
      d[i] = nullptr, h[i] = nullptr, ev[i] = nullptr, used[i] = false;
    }
    cap = 0;
  }
  ~HandoffRing() {
    release();
    if (stage) cudaFree(stage);
  }
  void ensure(int rows) {
    if (rows <= cap) return;
    release();
    for (int i = 0; i < N; ++i) {
      EXG_CUDA(cudaMalloc(&d[i], sizeof(HandoffRow) * rows));
      EXG_CUDA(cudaMallocHost(&h[i], sizeof(HandoffRow) * rows));
      EXG_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    cap = rows;
  }
};

HandoffRing& handoff_ring(std::shared_ptr<void>& cache, int rows) {
  if (!cache) cache = std::make_shared<HandoffRing>();
  HandoffRing& r = *static_cast<HandoffRing*>(cache.get());
  r.ensure(rows);
  return r;
}

// the executors' table ring, cached in the context across runs
std::vector<Tables>& table_ring(std::shared_ptr<void>& cache) {
  if (!cache) cache = std::make_shared<std::vector<Tables>>(8);
  return *static_cast<std::vector<Tables>*>(cache.get());
}

struct RunState {
  const exg_request* reqs;
  int n;
  std::vector<int64_t> base;
  int64_t total_out = 0;
  int max_in = 1, max_ctx = 1, max_out = 1;
  bool ed = false;   // encoder-decoder token accounting (T6 for T5)
  int32_t* d_out = nullptr;
  uint64_t* d_stamps = nullptr;
  int n_stamps = 0, cap_stamps = 0;
  std::vector<int> admit_ev, done_ev;
  // Table 9 single-stage times: encode batches (start /
  // end stamps) and decode iterations (end stamps, consecutive)
  std::vector<int> enc_start_ev, enc_end_ev, iter_ev;
  std::vector<int64_t> iter_tokens;   // tokens emitted by the iteration ending at iter_ev[k]
  cudaStream_t st;
  int64_t decode_iters = 0, encode_phases = 0, batch_sum = 0;
  // paged decoder KV (WAA; exegpt.h kv_page): page length, page-table row
  // length, pages of each decoder slot
  int P = 0, maxp = 0;
  std::vector<std::vector<int>> slot_pages;
  int64_t preemptions = 0, pages_peak = 0;
  ~RunState() {
    if (st) cudaStreamSynchronize(st);
    if (d_out) cudaFree(d_out);
    if (d_stamps) cudaFree(d_stamps);
  }
  // stamp index k, written (on this rank) only when `mine`
  int record(bool mine) {
    const int k = n_stamps++;
    if (k >= cap_stamps) throw std::logic_error("stamp capacity exceeded");
    if (mine) {
      stamp_kernel<<<1, 1, 0, st>>>(d_stamps + k);
      EXG_CHECK_LAUNCH();
    }
    return k;
  }
};

void validate_requests(RunState& R, int V, int max_pos) {
  R.base.assign(R.n + 1, 0);
  for (int r = 0; r < R.n; ++r) {
    const exg_request& q = R.reqs[r];
    if (q.input_len < 1 || q.output_len < 1 || !q.input_ids) throw std::invalid_argument("request lengths must be >= 1");
    if (R.ed ? std::max(q.input_len, q.output_len) > max_pos : q.input_len + q.output_len > max_pos)
      throw std::invalid_argument(R.ed ? "input_len or output_len > max_pos" : "input_len + output_len > max_pos");
    for (int j = 0; j < q.input_len; ++j)
      if (q.input_ids[j] < 0 || q.input_ids[j] >= V) throw std::invalid_argument("token id out of range");
    R.max_in = std::max(R.max_in, q.input_len);
    R.max_out = std::max(R.max_out, q.output_len);
    R.max_ctx = std::max(R.max_ctx, q.input_len + q.output_len);
    R.base[r + 1] = R.base[r] + q.output_len;
  }
  R.total_out = R.base[R.n];
  const size_t nout = (size_t)std::max<int64_t>(R.total_out, 1);
  EXG_CUDA(cudaMalloc(&R.d_out, sizeof(int32_t) * nout));
  EXG_CUDA(cudaMemsetAsync(R.d_out, 0, sizeof(int32_t) * nout, R.st));
  // one stamp per loop pass (phase start) and per decode iteration, + start;
  // both are bounded by the number of output tokens + requests
  R.cap_stamps = (int)std::min<int64_t>(2 * (R.total_out + R.n) + 16, (int64_t)1 << 30);
  EXG_CUDA(cudaMalloc(&R.d_stamps, sizeof(uint64_t) * R.cap_stamps));
  EXG_CUDA(cudaMemsetAsync(R.d_stamps, 0, sizeof(uint64_t) * R.cap_stamps, R.st));
}

// packed encode tables for requests [r0, r0+k) with the given slots
// paged: the encoding engines page their KV (RRA pipelines; WAA encoders keep
// per-batch slots) -- tokens carry page / offset and requests page tables
EncodeBatch build_encode(const RunState& R, Tables& tb, int r0, int k, const int* slots, cudaStream_t st,
                         std::vector<int32_t>* last_ids, bool paged = false) {
  const int drop = R.ed ? 0 : 1;   // T6: decoder-only encodes positions 0..n-2, T5 all n tokens
  int T = 0, maxlen = 0;
  for (int j = 0; j < k; ++j) T += R.reqs[r0 + j].input_len - drop;
  const size_t pgi = paged ? (size_t)2 * T + (size_t)k * R.maxp : 0;   // paged: page / offset per token, page table
  tb.ensure((size_t)3 * T + 3 * (k + 1) + pgi + 8);
  int32_t* h = tb.begin();
  int32_t *ids = h, *pos = ids + T, *tsl = pos + T, *cu = tsl + T, *rsl = cu + k + 1, *p0 = rsl + k;
  int t = 0;
  cu[0] = 0;
  EncodeBatch eb;
  for (int j = 0; j < k; ++j) {
    const exg_request& q = R.reqs[r0 + j];
    for (int p = 0; p < q.input_len - drop; ++p, ++t) {
      ids[t] = q.input_ids[p];
      pos[t] = p;
      tsl[t] = slots[j];
    }
    cu[j + 1] = t;
    rsl[j] = slots[j];
    p0[j] = 0;
    maxlen = std::max(maxlen, q.input_len - drop);
    const double m = q.input_len - drop;
    eb.attn_pairs += R.ed ? m * m : m * (m + 1) / 2;
    if (last_ids) last_ids->push_back(R.ed ? 0 : q.input_ids[q.input_len - 1]);   // T5: decoder start token
  }
  if (pgi) {
    int32_t *kvb = p0 + k, *kvo = kvb + T, *ptab = kvo + T;
    int t2 = 0;
    for (int j = 0; j < k; ++j) {
      const auto& pg = R.slot_pages[slots[j]];
      if ((int)pg.size() * R.P < R.reqs[r0 + j].input_len - drop || pg.empty())
        throw std::logic_error("paged encode: the request's pages are not allocated");
      for (int p = 0; p < R.reqs[r0 + j].input_len - drop; ++p, ++t2) {
        kvb[t2] = pg[p / R.P];
        kvo[t2] = p % R.P;
      }
      for (int q = 0; q < R.maxp; ++q) ptab[(int64_t)j * R.maxp + q] = pg[q < (int)pg.size() ? q : 0];
    }
  }
  tb.upload((size_t)3 * T + (k + 1) + 2 * k + pgi, st);
  if (pgi) {
    eb.kv_blk = tb.dev + 3 * T + (k + 1) + 2 * k;
    eb.kv_off = eb.kv_blk + T;
    eb.kv = KvMap{eb.kv_off + T, R.maxp};
  }
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
  const size_t pt = R.P > 0 ? (size_t)B * R.maxp : 0;   // paged: page table rows of the batch
  tb.ensure((size_t)5 * B + pt + 8);
  int32_t* h = tb.begin();
  DecodeBatch db;
  for (int i = 0; i < B; ++i) {
    const Row& rw = rows[i0 + i];
    const int n_in = R.reqs[rw.req].input_len;
    h[i] = rw.slot;
    h[B + i] = rw.pos;
    h[2 * B + i] = rw.pos + 1;
    h[3 * B + i] = (int32_t)(R.base[rw.req] + rw.emitted);
    h[4 * B + i] = n_in;
    db.max_keys = std::max(db.max_keys, rw.pos + 1);
    db.sum_keys += rw.pos + 1;
    db.max_xkeys = std::max(db.max_xkeys, n_in);
    db.sum_xkeys += n_in;
    if (pt) {
      const auto& pg = R.slot_pages[rw.slot];
      for (int j = 0; j < R.maxp; ++j) h[5 * B + (int64_t)i * R.maxp + j] = pg[j < (int)pg.size() ? j : 0];
    }
  }
  tb.upload((size_t)5 * B + pt, st);
  if (pt) db.kv = KvMap{tb.dev + 5 * B, R.maxp};
  if (R.ed) db.xkeys = tb.dev + 4 * B;
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

// optional fp32 logits dump (exg_run_opts.logits_out / dump_mask), written
// by the rank holding the LM head
struct Dump {
  const exg_run_opts* opts = nullptr;
  std::vector<int64_t> base;
  bool on() const { return opts && opts->logits_out && opts->dump_mask; }
};

Dump make_dump(const RunState& R, const exg_run_opts* opts) {
  Dump d;
  d.opts = opts;
  d.base.assign(R.n + 1, 0);
  if (d.on())
    for (int r = 0; r < R.n; ++r) d.base[r + 1] = d.base[r] + (opts->dump_mask[r] ? R.reqs[r].output_len : 0);
  return d;
}

// one decode iteration of `rows` through the pipeline in n_mb micro-batches
void decode_pipeline(const Exec& X, RunState& R, std::vector<std::unique_ptr<Stage>>& pipe, std::vector<Tables>& tabs,
                     int& ti, const std::vector<Row>& rows, int n_mb, int d, const Dump& dump) {
  const int B = (int)rows.size();
  for (const auto& mb : chunks(B, n_mb)) {
    Tables& tb = tabs[ti++ % tabs.size()];
    DecodeBatch db = build_decode(R, tb, rows, mb.first, mb.second, R.st);
    for (size_t k = 0; k < pipe.size(); ++k) {
      if (k > 0) hop(X, *pipe[k - 1], *pipe[k], mb.second, d);
      pipe[k]->decode(X, db, d);
    }
    Engine* head = pipe.back()->eng[0].get();
    if (dump.on() && head) {
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

// the last stage's ids become the first stage's next inputs (K15)
void return_tokens(const Exec& X, std::vector<std::unique_ptr<Stage>>& pipe, int slots) {
  Stage& Ls = *pipe.back();
  Stage& Fs = *pipe.front();
  for (int r = 0; r < Fs.tp; ++r)
    X.xfer(Ls.gpu(0), Ls.eng[0] ? Ls.eng[0]->last_tok() : nullptr, Fs.gpu(r),
           Fs.eng[r] ? Fs.eng[r]->last_tok() : nullptr, sizeof(int32_t) * slots);
}

void retire(RunState& R, std::vector<Row>& active, std::vector<int>& free_slots, int ev,
            std::vector<int>* free_pages = nullptr) {
  int w = 0;
  for (size_t i = 0; i < active.size(); ++i) {
    Row rw = active[i];
    rw.emitted += 1;
    rw.pos += 1;
    if (rw.emitted == R.reqs[rw.req].output_len) {
      R.done_ev[rw.req] = ev;
      free_slots.push_back(rw.slot);
      if (free_pages) {
        for (int pg : R.slot_pages[rw.slot]) free_pages->push_back(pg);
        R.slot_pages[rw.slot].clear();
      }
    } else {
      active[w++] = rw;
    }
  }
  active.resize(w);
}

// results to rank 0: the output tokens from the head's rank, the stamps from
// every rank (each stamp is written by exactly one rank, the others hold 0)
void finish(const Exec& X, RunState& R, Stage& head_stage, int32_t* out_tokens, double* out_latency,
            exg_run_stats* stats) {
  const int ho = X.owner(head_stage.gpu(0));
  std::vector<uint64_t> stamps(R.n_stamps, 0);
  auto merge = [&](const uint64_t* dev) {
    std::vector<uint64_t> h(R.n_stamps);
    EXG_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(uint64_t) * R.n_stamps, cudaMemcpyDeviceToHost, R.st));
    EXG_CUDA(cudaStreamSynchronize(R.st));
    for (int k = 0; k < R.n_stamps; ++k) stamps[k] = std::max(stamps[k], h[k]);
  };
  if (X.world > 1) {
    // results to rank 0 over the main communicator, on its stream (cst)
    X.fork();
    if (ho != 0) {
      if (X.me == ho) X.comm->send(R.d_out, sizeof(int32_t) * R.total_out, 0, X.cst);
      if (X.me == 0) X.comm->recv(R.d_out, sizeof(int32_t) * R.total_out, ho, X.cst);
    }
    uint64_t* tmp = nullptr;
    if (X.me == 0) EXG_CUDA(cudaMalloc(&tmp, sizeof(uint64_t) * std::max(1, R.n_stamps)));
    for (int q = 1; q < X.world; ++q) {
      if (X.me == q) X.comm->send(R.d_stamps, sizeof(uint64_t) * R.n_stamps, 0, X.cst);
      if (X.me == 0) {
        X.comm->recv(tmp, sizeof(uint64_t) * R.n_stamps, q, X.cst);
        X.join();
        merge(tmp);
      }
    }
    X.join();
    EXG_CUDA(cudaStreamSynchronize(X.cst));
    if (tmp) {
      EXG_CUDA(cudaStreamSynchronize(R.st));
      cudaFree(tmp);
    }
    X.comm->check_async();
  }
  EXG_CUDA(cudaStreamSynchronize(R.st));
  if (Engine* head = head_stage.eng[0].get()) {
    int32_t err = 0;
    EXG_CUDA(cudaMemcpy(&err, head->err_flag(), sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (err) throw std::runtime_error("NaN logit encountered (T7)");
  }
  if (X.me != 0) {
    if (stats) std::memset(stats, 0, sizeof(*stats));
    return;
  }
  if (out_tokens) EXG_CUDA(cudaMemcpy(out_tokens, R.d_out, sizeof(int32_t) * R.total_out, cudaMemcpyDeviceToHost));
  merge(R.d_stamps);
  const uint64_t t0 = stamps[0];   // run start
  auto sec = [&](int k) { return stamps[k] >= t0 ? (double)(stamps[k] - t0) * 1e-9 : 0.0; };
  std::vector<double> lat(R.n);
  for (int r = 0; r < R.n; ++r) {
    lat[r] = sec(R.done_ev[r]) - sec(R.admit_ev[r]);
    if (out_latency) out_latency[r] = lat[r];
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    double wall = 0;
    for (int k = 0; k < R.n_stamps; ++k) wall = std::max(wall, sec(k));
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
    stats->mean_encode_batch = R.encode_phases ? (double)R.n / R.encode_phases : 0;
    stats->kv_preemptions = R.preemptions;
    stats->kv_pages_peak = R.pages_peak;
    // steady window: admission of request ceil(0.1 n) .. admission of the last
    const int r0 = std::min(R.n - 1, (int)std::ceil(0.1 * R.n));
    const double w0 = sec(R.admit_ev[r0]), w1 = sec(R.admit_ev[R.n - 1]);
    auto spread = [&](const std::vector<double>& v, double* mean, double* p99dev) {
      *mean = *p99dev = 0;
      if (v.empty()) return;
      double m = 0;
      for (double x : v) m += x;
      m /= v.size();
      std::vector<double> dv;
      for (double x : v) dv.push_back(std::fabs(x - m));
      std::sort(dv.begin(), dv.end());
      const double rr = 0.99 * (dv.size() - 1);
      const size_t lo = (size_t)std::floor(rr), hi = (size_t)std::ceil(rr);
      *mean = m;
      *p99dev = dv[lo] + (rr - lo) * (dv[hi] - dv[lo]);
    };
    std::vector<double> te, td;
    for (size_t k = 0; k < R.enc_start_ev.size() && k < R.enc_end_ev.size(); ++k) {
      const double a = sec(R.enc_start_ev[k]), b = sec(R.enc_end_ev[k]);
      if (a >= w0 && b <= w1 && b > a) te.push_back(b - a);
    }
    for (size_t k = 1; k < R.iter_ev.size(); ++k) {
      const double a = sec(R.iter_ev[k - 1]), b = sec(R.iter_ev[k]);
      if (a >= w0 && b <= w1 && b > a) td.push_back(b - a);
    }
    spread(te, &stats->enc_stage_mean_s, &stats->enc_stage_p99dev_s);
    spread(td, &stats->dec_stage_mean_s, &stats->dec_stage_p99dev_s);
    int64_t toks = 0;
    for (size_t k = 0; k < R.iter_ev.size(); ++k) {
      const double t = sec(R.iter_ev[k]);
      if (t > w0 && t <= w1) toks += R.iter_tokens[k];
    }
    stats->tok_s_steady = w1 > w0 ? toks / (w1 - w0) : stats->tok_s;
  }
}
}  // namespace

// ---------------------------------------------------------------------------
// RRA over P pipeline stages with partial TP (S6: encode in
// P micro-batches, decode in P micro-batches)
// ---------------------------------------------------------------------------
// Paged decoder KV of a multi-GPU executor (exegpt.h kv_page):
// every rank runs the same host loop, so the page decisions are identical on
// all ranks and each rank applies them to its own engines.  Pages are
// allocated as rows grow (one page per active row kept in reserve at
// admission); a row that finds no free page swaps the latest-admitted row's
// pages -- the K/V of every layer this rank holds -- to pinned host memory and
// back into new pages once they fit (swap preemption: the K/V return
// unchanged, so paged results are bit-identical to slots).
struct Pager {
  RunState& R;
  std::vector<std::unique_ptr<Stage>>& stages;   // the engines holding the paged KV
  int P = 0, n_pages = 0, dh = 0;
  std::vector<int> free_pages;
  struct Swapped {
    Row row;
    void* host;
    int npg;
  };
  std::vector<Swapped> swapped;   // sorted by request index (arrival order)
  std::vector<void*> host_bufs;   // freed once the stream has drained

  Pager(RunState& R_, std::vector<std::unique_ptr<Stage>>& st, const exg_run_opts* opts, int slot_ctx, int B_D,
        int dh_)
      : R(R_), stages(st), dh(dh_) {
    P = opts ? opts->kv_page : 0;
    if (P <= 0) {
      P = 0;
      return;
    }
    if (R.ed) throw std::invalid_argument("paged KV: decoder-only models");
    if (P % 64 != 0 || 512 % P != 0) throw std::invalid_argument("kv_page must be a multiple of 64 dividing 512");
    if (opts->kv_pages < 0) throw std::invalid_argument("kv_pages < 0");
    R.P = P;
    R.maxp = (slot_ctx + P - 1) / P;
    n_pages = opts->kv_pages > 0 ? opts->kv_pages : B_D * R.maxp;
    if (n_pages < R.maxp + 1) throw std::invalid_argument("kv_pages below one request's pages + 1");
    R.slot_pages.assign(B_D, {});
    for (int i = n_pages - 1; i >= 0; --i) free_pages.push_back(i);
  }
  ~Pager() {
    if (!host_bufs.empty()) cudaStreamSynchronize(R.st);
    for (void* hb : host_bufs)
      if (hb) cudaFreeHost(hb);
  }
  bool on() const { return P > 0; }
  int pages_for(int keys) const { return (keys + P - 1) / P; }
  void note_peak() {
    R.pages_peak = std::max<int64_t>(R.pages_peak, (int64_t)n_pages - (int64_t)free_pages.size());
  }
  void take(int slot, int npg) {
    auto& pg = R.slot_pages[slot];
    for (int j = 0; j < npg; ++j) {
      pg.push_back(free_pages.back());
      free_pages.pop_back();
    }
    note_peak();
  }
  // this rank's K / V blocks of the given pages, in a fixed order (stage, TP
  // rank, layer, K|V, page)
  void for_each_block(const std::vector<int>& pages, const std::function<void(bf16*, size_t)>& fn) {
    for (auto& ds : stages)
      for (auto& e : ds->eng)
        if (e) {
          const size_t blk = (size_t)e->dims().Hl * P * dh;
          for (int l = 0; l < e->n_layers(); ++l)
            for (int kv = 0; kv < 2; ++kv)
              for (int pg : pages) fn((kv ? e->vc(l) : e->kc(l)) + (size_t)pg * blk, blk * sizeof(bf16));
        }
  }
  void swap_out(std::vector<Row>& active, size_t v) {
    const Row vr = active[v];
    auto& pg = R.slot_pages[vr.slot];
    size_t bytes = 0;
    for_each_block(pg, [&](bf16*, size_t b) { bytes += b; });
    void* hb = nullptr;
    if (bytes) EXG_CUDA(cudaMallocHost(&hb, bytes));
    host_bufs.push_back(hb);
    size_t off = 0;
    for_each_block(pg, [&](bf16* dptr, size_t b) {
      EXG_CUDA(cudaMemcpyAsync(static_cast<char*>(hb) + off, dptr, b, cudaMemcpyDeviceToHost, R.st));
      off += b;
    });
    const Swapped sw{vr, hb, (int)pg.size()};
    for (int x : pg) free_pages.push_back(x);   // reused only by later work on this stream
    pg.clear();
    swapped.insert(std::upper_bound(swapped.begin(), swapped.end(), sw,
                                    [](const Swapped& a, const Swapped& b) { return a.row.req < b.row.req; }),
                   sw);
    active.erase(active.begin() + v);   // the row keeps its slot (and last_tok[slot])
    ++R.preemptions;
  }
  // swapped-out rows come back first, each when its pages fit with one page
  // per active row in reserve
  void swap_in_ready(std::vector<Row>& active) {
    while (on() && !swapped.empty() &&
           (int64_t)free_pages.size() - swapped.front().npg >= (int64_t)active.size() + 1) {
      const Swapped sw = swapped.front();
      swapped.erase(swapped.begin());
      take(sw.row.slot, sw.npg);
      size_t off = 0;
      for_each_block(R.slot_pages[sw.row.slot], [&](bf16* dptr, size_t b) {
        EXG_CUDA(cudaMemcpyAsync(dptr, static_cast<char*>(sw.host) + off, b, cudaMemcpyHostToDevice, R.st));
        off += b;
      });
      active.push_back(sw.row);
    }
  }
  // every row writes key `pos` this iteration: a new page when it crosses
  // into one; none free -> swap out the latest-admitted row
  void grow(std::vector<Row>& active) {
    if (!on()) return;
    for (size_t i = 0; i < active.size();) {
      const int slot = active[i].slot, pos = active[i].pos;
      if (pos / P < (int)R.slot_pages[slot].size()) {
        ++i;
        continue;
      }
      if (free_pages.empty()) {
        size_t v = 0;
        for (size_t j = 1; j < active.size(); ++j)
          if (active[j].seq > active[v].seq) v = j;
        swap_out(active, v);
        if (v < i) --i;
        continue;
      }
      take(slot, 1);
      ++i;
    }
  }
};

static void run_rra_multi(MultiCtx::Impl* p, Layout* lay, const exg_schedule& s, const exg_request* reqs, int n,
                          int32_t* out_tokens, double* out_latency, exg_run_stats* stats, const exg_run_opts* opts) {
  auto& pipe = lay->dec;
  const Exec X = make_exec(p, lay->G, opts);
  const int d = p->spec.d_model;
  RunState R;
  R.reqs = reqs;
  R.n = n;
  R.st = p->st;
  R.ed = p->spec.arch == EXG_ARCH_T5;
  validate_requests(R, p->spec.vocab, p->spec.max_pos);
  const int need_ctx = R.ed ? R.max_out : R.max_ctx;
  const int slot_ctx = (opts && opts->slot_ctx > 0) ? opts->slot_ctx : need_ctx;
  if (slot_ctx < need_ctx) throw std::invalid_argument("slot_ctx smaller than a request's input+output length");
  const int B_D = s.b_d, B_E = s.b_e, P = (int)pipe.size();
  if (B_E < 1 || B_D < B_E || s.n_d < 1) throw std::invalid_argument("RRA needs 1 <= B_E <= B_D, N_D >= 1");
  const int drop = R.ed ? 0 : 1;
  // paged KV on every stage (Pager: swap preemption across the pipeline)
  Pager pgr(R, pipe, opts, slot_ctx, B_D, p->spec.d_head);
  for (auto& st : pipe)
    for (auto& e : st->eng)
      if (e) {
        if (pgr.on())
          e->ensure_kv(std::max(pgr.n_pages, B_D), pgr.P, -1, 0);
        else
          e->ensure_kv(B_D, slot_ctx, -1, R.ed ? R.max_in : 0);
        e->ensure_workspace(std::max(1, B_E * (R.max_in - drop)), B_D);
      }
  const bool first_mine = X.mine(pipe.front()->gpu(0)), head_mine = X.mine(pipe.back()->gpu(0));
  std::vector<Tables>& tabs = table_ring(p->tab_cache);
  const Dump dump = make_dump(R, opts);
  std::vector<int> free_slots(B_D);
  for (int i = 0; i < B_D; ++i) free_slots[i] = B_D - 1 - i;
  std::vector<Row> active;
  R.admit_ev.assign(n, -1);
  R.done_ev.assign(n, -1);
  int next_req = 0, ti = 0;
  int64_t admit_seq = 0;
  R.record(first_mine);
  while (next_req < n || !active.empty() || !pgr.swapped.empty()) {
    // paged: swapped-out rows first; new rows only while none is swapped out
    // and their pages fit with one page per active row in reserve
    pgr.swap_in_ready(active);
    int admit = std::min({B_E, B_D - (int)active.size() - (int)pgr.swapped.size(), n - next_req});
    if (pgr.on()) {
      int64_t fr = (int64_t)pgr.free_pages.size();
      int k = 0;
      while (pgr.swapped.empty() && k < admit) {
        const int need = pgr.pages_for(reqs[next_req + k].input_len);   // positions 0 .. n-1
        if (fr - need < (int64_t)active.size() + k + 1) break;
        fr -= need;
        ++k;
      }
      admit = k;
    }
    const int ev_phase = R.record(first_mine);
    if (admit > 0) R.enc_start_ev.push_back(ev_phase);
    if (admit > 0) {
      std::vector<int> slots(admit);
      for (int k = 0; k < admit; ++k) {
        slots[k] = free_slots.back();
        free_slots.pop_back();
        const exg_request& q = reqs[next_req + k];
        if (pgr.on()) pgr.take(slots[k], pgr.pages_for(q.input_len));
        active.push_back(Row{next_req + k, slots[k], R.ed ? 0 : q.input_len - 1, 0, admit_seq++});
        R.admit_ev[next_req + k] = ev_phase;
      }
      for (const auto& mb : chunks(admit, P)) {
        Tables& tb = tabs[ti++ % tabs.size()];
        std::vector<int32_t> last;
        EncodeBatch eb =
            build_encode(R, tb, next_req + mb.first, mb.second, slots.data() + mb.first, R.st, &last, pgr.on());
        // x[n-1] of every admitted request -> last_tok[slot] on the first stage
        Tables& tl = tabs[ti++ % tabs.size()];
        tl.ensure(2 * last.size() + 2);
        int32_t* h = tl.begin();
        for (size_t j = 0; j < last.size(); ++j) {
          h[j] = slots[mb.first + j];
          h[last.size() + j] = last[j];
        }
        tl.upload(2 * last.size(), R.st);
        for (auto& e : pipe.front()->eng)
          if (e) set_last_tokens(e->last_tok(), tl.dev, tl.dev + last.size(), (int)last.size(), R.st);
        for (size_t k = 0; k < pipe.size(); ++k) {
          if (k > 0) hop(X, *pipe[k - 1], *pipe[k], eb.T, d);
          pipe[k]->encode(X, eb, d);
        }
        if (R.ed && P > 1) {
          // T5: the encoder output (bf16 [T][d], last stage) to every other
          // stage, which projects the cross K/V of its own decoder layers
          Stage& Ls = *pipe.back();
          for (int k = 0; k + 1 < P; ++k) {
            Stage& S_k = *pipe[k];
            X.xfer(Ls.gpu(0), Ls.eng[0] ? Ls.eng[0]->h() : nullptr, S_k.gpu(0), S_k.eng[0] ? S_k.eng[0]->h() : nullptr,
                   sizeof(bf16) * (size_t)eb.T * d);
            if (S_k.eng[0]) S_k.eng[0]->cross_kv_all(eb);
          }
        }
      }
      next_req += admit;
      ++R.encode_phases;
      R.enc_end_ev.push_back(R.record(head_mine));
    }
    for (int u = 0; u < s.n_d; ++u) {
      pgr.grow(active);
      if (active.empty()) break;
      decode_pipeline(X, R, pipe, tabs, ti, active, P, d, dump);
      return_tokens(X, pipe, B_D);
      const int ev = R.record(head_mine);
      R.iter_ev.push_back(ev);
      R.iter_tokens.push_back((int64_t)active.size());
      ++R.decode_iters;
      R.batch_sum += (int64_t)active.size();
      retire(R, active, free_slots, ev, pgr.on() ? &pgr.free_pages : nullptr);
    }
  }
  finish(X, R, *pipe.back(), out_tokens, out_latency, stats);
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
  const Exec X = make_exec(p, lay->G, opts);
  const int d = p->spec.d_model, H = p->spec.n_heads, dh = p->spec.d_head;
  RunState R;
  R.reqs = reqs;
  R.n = n;
  R.st = p->st;
  R.ed = p->spec.arch == EXG_ARCH_T5;
  validate_requests(R, p->spec.vocab, p->spec.max_pos);
  // decoder self-attention context: n-1+S keys (decoder-only) or S (T5)
  const int need_ctx = R.ed ? R.max_out : R.max_ctx;
  const int slot_ctx = (opts && opts->slot_ctx > 0) ? opts->slot_ctx : need_ctx;
  if (slot_ctx < need_ctx) throw std::invalid_argument("slot_ctx smaller than a request's input+output length");
  const int B_D = s.b_d, B_E = s.b_e;
  if (B_E < 1 || B_D < B_E) throw std::invalid_argument("WAA needs 1 <= B_E <= B_D");
  const int M = s.b_m > 0 ? std::max(1, (B_D + s.b_m - 1) / s.b_m) : 1;
  // paged decoder KV (exegpt.h kv_page; "the addition of vLLM's
  // paging mechanism can further enhance WAA's performance"): the decoder
  // GPUs page, the encoder side keeps its per-batch slots (Pager)
  Pager pgr(R, dec, opts, slot_ctx, B_D, dh);
  const bool paged = pgr.on();
  const int P = pgr.P;
  const int enc_ctx = std::max(1, R.max_in);
  const int drop = R.ed ? 0 : 1;
  const double dyn = opts ? opts->dyn_threshold : 0.0;
  // encoder capacity: 2 B_E rows under dynamic adjustment, never more tokens
  // than B_E of the longest input
  const int enc_rows = dyn > 0 ? std::min(2 * B_E, B_D) : B_E;
  const int enc_tok_cap = std::max(1, B_E * (R.max_in - drop));
  double mean_enc_tokens = 0, steady_batch_sum = 0;
  int64_t steady_iters = 0;
  for (int r = 0; r < n; ++r) mean_enc_tokens += reqs[r].input_len - drop;
  mean_enc_tokens /= std::max(1, n);
  for (auto& st : enc)
    for (auto& e : st->eng)
      if (e) {
        if (R.ed)
          e->ensure_kv(enc_rows, 1, -1, enc_ctx);   // encoder side: encoder K/V staging + cross K/V of the batch
        else
          e->ensure_kv(enc_rows, enc_ctx);
        e->ensure_workspace(enc_tok_cap, enc_rows);
      }
  for (auto& st : dec)
    for (auto& e : st->eng)
      if (e) {
        if (paged)
          e->ensure_kv(std::max(pgr.n_pages, B_D), P, -1, 0);
        else
          e->ensure_kv(B_D, slot_ctx, -1, R.ed ? R.max_in : 0);
        e->ensure_workspace(1, B_D);
      }
  const bool first_mine = X.mine(enc.front()->gpu(0)), head_mine = X.mine(dec.back()->gpu(0));
  std::vector<Tables>& tabs = table_ring(p->tab_cache);
  const Dump dump = make_dump(R, opts);
  // handoff row tables (cached ring, HandoffRow); packed-message staging for
  // transfers between ranks goes through the exchange rings of Exec
  HandoffRing& hr = handoff_ring(p->hr_cache, enc_rows);
  std::vector<int> free_slots(B_D);
  for (int i = 0; i < B_D; ++i) free_slots[i] = B_D - 1 - i;
  std::vector<Row> active;
  R.admit_ev.assign(n, -1);
  R.done_ev.assign(n, -1);
  int64_t admit_seq = 0;
  int next_req = 0, pend_r0 = -1, pend_k = 0, pend_s0 = 0, pend_ev = -1, ti = 0;
  R.record(first_mine);
  while (next_req < n || pend_k > 0 || !active.empty() || !pgr.swapped.empty()) {
    // encoder: keep one encoded batch ready (encoder slots 0..k-1)
    if (pend_k == 0 && next_req < n) {
      int k = std::min(B_E, n - next_req);
      if (dyn > 0) {
        // dynamic workload adjustment: "a long encoding
        // stage can miss the handover ... uneven decoding batches": the
        // encoder batch's token sum is kept within +-dyn of B_E' x the mean
        // encoded length, B_E' = B_E + round(avg - current decode batch) while
        // the decode batch is outside +-dyn of its running average
        int be = B_E;
        if (steady_iters >= 2 && !active.empty()) {
          const double avg = steady_batch_sum / steady_iters, cur = (double)active.size();
          if (cur < (1 - dyn) * avg || cur > (1 + dyn) * avg) be = B_E + (int)std::lround(avg - cur);
        }
        be = std::max(1, std::min(be, enc_rows));
        const int cap = std::min(enc_rows, n - next_req);
        const double target = be * mean_enc_tokens;
        double tok = 0;
        k = 0;
        while (k < cap) {
          const double t = reqs[next_req + k].input_len - drop;
          if (k >= be && tok >= (1 - dyn) * target) break;
          if (k >= 1 && tok + t > (1 + dyn) * target) break;
          if (k >= 1 && tok + t > enc_tok_cap) break;   // encoder workspace
          tok += t;
          ++k;
        }
      }
      pend_ev = R.record(first_mine);
      R.enc_start_ev.push_back(pend_ev);
      std::vector<int> eslots(k);
      for (int j = 0; j < k; ++j) eslots[j] = j;
      Tables& tb = tabs[ti++ % tabs.size()];
      EncodeBatch eb = build_encode(R, tb, next_req, k, eslots.data(), R.st, nullptr);
      for (size_t q = 0; q < enc.size(); ++q) {
        if (q > 0) hop(X, *enc[q - 1], *enc[q], eb.T, d);
        enc[q]->encode(X, eb, d);
      }
      pend_r0 = next_req;
      pend_k = k;
      pend_s0 = 0;
      next_req += k;
      ++R.encode_phases;
      R.enc_end_ev.push_back(R.record(X.mine(enc.back()->gpu(0))));
    }
    // paged: swapped-out rows come back first, each when its pages fit with
    // one page per active row in reserve
    pgr.swap_in_ready(active);
    // handoff + merge at an iteration boundary when the decoder has room
    // (paged: no row swapped out; the longest prefix of the encoded batch
    // whose pages fit with the reserve -- the rest stays pending)
    int hk = pend_k;
    if (paged && pend_k > 0) {
      hk = 0;
      int64_t fr = (int64_t)pgr.free_pages.size();
      while (pgr.swapped.empty() && hk < pend_k && hk < (int)free_slots.size()) {
        const int need = (reqs[pend_r0 + hk].input_len + P - 1) / P;   // positions 0 .. n-1
        if (fr - need < (int64_t)active.size() + hk + 1) break;
        fr -= need;
        ++hk;
      }
    }
    if (pend_k > 0 && hk > 0 && (int)free_slots.size() >= hk) {
      std::vector<int> dslots(hk);
      int64_t rows_len = 0;
      // a row table slot is rewritten only once its previous upload is done
      const int hs = hr.next;
      hr.next = (hr.next + 1) % HandoffRing::N;
      if (hr.used[hs]) EXG_CUDA(cudaEventSynchronize(hr.ev[hs]));
      HandoffRow* hrow_h = hr.h[hs];
      HandoffRow* hrow_d = hr.d[hs];
      const int32_t* dpt = nullptr;   // paged: destination page table [hk][maxp]
      if (paged) {
        Tables& tp = tabs[ti++ % tabs.size()];
        tp.ensure((size_t)hk * R.maxp + 8);
        int32_t* hp = tp.begin();
        for (int j = 0; j < hk; ++j) {
          const int slot = free_slots[free_slots.size() - 1 - j];
          pgr.take(slot, pgr.pages_for(reqs[pend_r0 + j].input_len));
          const auto& pg = R.slot_pages[slot];
          for (int q = 0; q < R.maxp; ++q) hp[(int64_t)j * R.maxp + q] = pg[q < (int)pg.size() ? q : 0];
        }
        tp.upload((size_t)hk * R.maxp, R.st);
        dpt = tp.dev;
      }
      for (int j = 0; j < hk; ++j) {
        dslots[j] = free_slots.back();
        free_slots.pop_back();
        const exg_request& q = reqs[pend_r0 + j];
        // handed-off K/V rows: positions 0..n-2 (decoder-only) / the n cross K/V rows (T5)
        hrow_h[j] = HandoffRow{pend_s0 + j, dslots[j], q.input_len - drop, rows_len};
        rows_len += q.input_len - drop;
        active.push_back(Row{pend_r0 + j, dslots[j], R.ed ? 0 : q.input_len - 1, 0, admit_seq++});
        R.admit_ev[pend_r0 + j] = pend_ev;
      }
      EXG_CUDA(cudaMemcpyAsync(hrow_d, hrow_h, sizeof(HandoffRow) * hk, cudaMemcpyHostToDevice, R.st));
      EXG_CUDA(cudaEventRecord(hr.ev[hs], R.st));
      hr.used[hs] = true;
      const size_t need = (size_t)rows_len * H * dh;   // largest slice (a TP-1 decoder stage)
      if (X.loop && need > hr.stage_cap) {
        EXG_CUDA(cudaStreamSynchronize(R.st));
        if (hr.stage) cudaFree(hr.stage);
        hr.stage = nullptr;
        hr.stage_cap = 0;
        // loopback: a second half receives the message sent from the first
        EXG_CUDA(cudaMalloc(&hr.stage, sizeof(bf16) * need * 2));
        hr.stage_cap = need;
      }
      bf16* stage_buf = hr.stage;
      const size_t stage_cap = hr.stage_cap;
      // decoder-only: encoder stage es holds the KV of its layers [l0, l1);
      // T5: the last encoder stage holds the cross K/V of every decoder layer
      for (auto& es : enc) {
        if (R.ed && es != enc.back()) continue;
        const int la = R.ed ? 0 : es->l0, lb = R.ed ? p->spec.n_dec_layers : es->l1;
        for (int l = la; l < lb; ++l)
          for (auto& ds : dec) {
            if (l < ds->l0 || l >= ds->l1) continue;
            const int Hd = H / ds->tp;
            for (int r = 0; r < ds->tp; ++r) {
              const int ge = es->gpu(0), gd = ds->gpu(r);
              const bool src_mine = X.mine(ge), dst_mine = X.mine(gd);
              if (!src_mine && !dst_mine) continue;
              Engine* src = es->eng[0].get();
              Engine* dst = ds->eng[r].get();
              const size_t bytes = sizeof(bf16) * (size_t)rows_len * Hd * dh;
              const int ctx_d = R.ed ? R.max_in : (paged ? P : slot_ctx);
              for (int kv = 0; kv < 2; ++kv) {
                const bf16* sp_ = nullptr;
                bf16* dp = nullptr;
                if (src) sp_ = R.ed ? (kv ? src->xvc(l) : src->xkc(l)) : (kv ? src->vc(l - es->l0) : src->kc(l - es->l0));
                if (dst)
                  dp = R.ed ? (kv ? dst->xvc(l - ds->l0) : dst->xkc(l - ds->l0))
                            : (kv ? dst->vc(l - ds->l0) : dst->kc(l - ds->l0));
                if (src_mine && dst_mine && X.loop) {
                  kv_handoff_kernel<<<hk * Hd, 128, 0, R.st>>>(sp_, stage_buf, hrow_d, hk, H, r * Hd, Hd,
                                                               enc_ctx, ctx_d, dh, 1);
                  EXG_CHECK_LAUNCH();
                  p->comm->group_start();
                  p->comm->send(stage_buf, bytes, X.me, R.st);
                  p->comm->recv(stage_buf + stage_cap, bytes, X.me, R.st);
                  p->comm->group_end();
                  kv_handoff_kernel<<<hk * Hd, 128, 0, R.st>>>(stage_buf + stage_cap, dp, hrow_d, hk, H,
                                                               r * Hd, Hd, enc_ctx, ctx_d, dh, 2, dpt, R.maxp);
                  EXG_CHECK_LAUNCH();
                } else if (src_mine && dst_mine) {
                  kv_handoff_kernel<<<hk * Hd, 128, 0, R.st>>>(sp_, dp, hrow_d, hk, H, r * Hd, Hd, enc_ctx,
                                                               ctx_d, dh, 0, dpt, R.maxp);
                  EXG_CHECK_LAUNCH();
                } else if (src_mine) {
                  // pack into a send staging buffer (compute stream), send on the
                  // comm stream: the encoder rank goes on with the next batch
                  const int sl = X.tx->acquire(bytes);
                  if (X.tx->used[sl]) EXG_CUDA(cudaStreamWaitEvent(R.st, X.tx->done[sl], 0));
                  kv_handoff_kernel<<<hk * Hd, 128, 0, R.st>>>(sp_, static_cast<bf16*>(X.tx->buf[sl]), hrow_d,
                                                               hk, H, r * Hd, Hd, enc_ctx, ctx_d, dh, 1);
                  EXG_CHECK_LAUNCH();
                  EXG_CUDA(cudaEventRecord(X.tx->ready[sl], R.st));
                  EXG_CUDA(cudaStreamWaitEvent(X.cst, X.tx->ready[sl], 0));
                  p->comm->send(X.tx->buf[sl], bytes, X.owner(gd), X.cst);
                  EXG_CUDA(cudaEventRecord(X.tx->done[sl], X.cst));
                  X.tx->used[sl] = true;
                } else {
                  // receive on the comm stream (overlapping the decoder's running
                  // iteration), unpack on the compute stream
                  const int sl = X.rx->acquire(bytes);
                  if (X.rx->used[sl]) EXG_CUDA(cudaStreamWaitEvent(X.cst, X.rx->done[sl], 0));
                  p->comm->recv(X.rx->buf[sl], bytes, X.owner(ge), X.cst);
                  EXG_CUDA(cudaEventRecord(X.rx->ready[sl], X.cst));
                  EXG_CUDA(cudaStreamWaitEvent(R.st, X.rx->ready[sl], 0));
                  kv_handoff_kernel<<<hk * Hd, 128, 0, R.st>>>(static_cast<const bf16*>(X.rx->buf[sl]), dp,
                                                               hrow_d, hk, H, r * Hd, Hd, enc_ctx, ctx_d, dh,
                                                               2, dpt, R.maxp);
                  EXG_CHECK_LAUNCH();
                  EXG_CUDA(cudaEventRecord(X.rx->done[sl], R.st));
                  X.rx->used[sl] = true;
                }
              }
            }
          }
      }
      // x[n-1] of the merged requests -> last_tok[slot] on the decoder's first stage
      Tables& tl = tabs[ti++ % tabs.size()];
      tl.ensure(2 * hk + 2);
      int32_t* h = tl.begin();
      for (int j = 0; j < hk; ++j) {
        const exg_request& q = reqs[pend_r0 + j];
        h[j] = dslots[j];
        h[hk + j] = R.ed ? 0 : q.input_ids[q.input_len - 1];   // T5: decoder start token 0
      }
      tl.upload(2 * hk, R.st);
      for (auto& e : dec.front()->eng)
        if (e) set_last_tokens(e->last_tok(), tl.dev, tl.dev + hk, hk, R.st);
      pend_r0 += hk;
      pend_s0 += hk;
      pend_k -= hk;
    }
    pgr.grow(active);
    if (active.empty()) continue;
    decode_pipeline(X, R, dec, tabs, ti, active, M, d, dump);
    return_tokens(X, dec, B_D);
    const int ev = R.record(head_mine);
    R.iter_ev.push_back(ev);
    R.iter_tokens.push_back((int64_t)active.size());
    ++R.decode_iters;
    R.batch_sum += (int64_t)active.size();
    if (next_req < n) {   // decode batch average while requests keep arriving
      steady_batch_sum += (double)active.size();
      ++steady_iters;
    }
    retire(R, active, free_slots, ev, paged ? &pgr.free_pages : nullptr);
  }
  finish(X, R, *dec.back(), out_tokens, out_latency, stats);
  EXG_CUDA(cudaStreamSynchronize(R.st));
}

void MultiCtx::profile_comm(const std::vector<int>& tps, int reps,
                            std::map<int, std::pair<std::vector<double>, std::vector<double>>>* tp,
                            std::vector<double>* pp_x, std::vector<double>* pp_t) {
  Impl* p = p_;
  if (!p->comm || p->world < 2) throw std::invalid_argument("profile_comm needs a multi-rank context (world > 1)");
  EXG_CUDA(cudaSetDevice(p->device));
  const int me = p->rank, world = p->world;
  reps = std::max(1, reps);
  std::vector<double> bytes;
  for (double b = 1024.0; b <= (double)(1u << 30); b *= 4.0) bytes.push_back(b);
  const size_t cap = (size_t)bytes.back();
  void* buf = nullptr;
  void* buf2 = nullptr;
  EXG_CUDA(cudaMalloc(&buf, cap));
  EXG_CUDA(cudaMalloc(&buf2, cap));
  EXG_CUDA(cudaMemset(buf, 0, cap));
  cudaEvent_t a, b;
  EXG_CUDA(cudaEventCreate(&a));
  EXG_CUDA(cudaEventCreate(&b));
  auto median_of = [&](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  cudaStream_t st = p->cst;   // the main communicator's stream
  try {
    // TP all-reduce tables: every t <= world, ranks [0, t)
    std::vector<std::vector<int>> groups;
    for (int t : tps)
      if (t > 1 && t <= world) {
        std::vector<int> g;
        for (int r = 0; r < t; ++r) g.push_back(r);
        groups.push_back(g);
      }
    p->comm->prepare_groups(groups);   // collective over all ranks
    for (const auto& g : groups) {
      const int t = (int)g.size();
      const bool member = me < t;
      std::vector<double> ts;
      for (double nb : bytes) {
        const size_t n = (size_t)nb / sizeof(float);
        std::vector<double> v;
        for (int r = 0; r <= reps; ++r) {   // r = 0: warm-up
          if (!member) continue;
          EXG_CUDA(cudaEventRecord(a, p->st));
          if (p->comm->has_allreduce()) {
            p->comm->allreduce_sum(static_cast<float*>(buf), n, g, p->st);
          } else {   // exchange of the partials (the transport's TP reduction)
            p->comm->group_start();
            for (int q : g)
              if (q != me) p->comm->send(buf, n * sizeof(float), q, st);
            for (int q : g)
              if (q != me) p->comm->recv(buf2, n * sizeof(float), q, st);
            p->comm->group_end();
            EXG_CUDA(cudaEventRecord(p->ev_join, st));
            EXG_CUDA(cudaStreamWaitEvent(p->st, p->ev_join, 0));
          }
          EXG_CUDA(cudaEventRecord(b, p->st));
          EXG_CUDA(cudaEventSynchronize(b));
          float ms = 0;
          EXG_CUDA(cudaEventElapsedTime(&ms, a, b));
          if (r > 0) v.push_back(ms * 1e-3);
        }
        ts.push_back(member ? median_of(v) : 0.0);
      }
      (*tp)[t] = {bytes, ts};
    }
    // pipeline hop: ping-pong rank 0 <-> rank 1, half the round trip
    pp_x->assign(bytes.begin(), bytes.end());
    pp_t->clear();
    for (double nb : bytes) {
      const size_t n = (size_t)nb;
      std::vector<double> v;
      for (int r = 0; r <= reps; ++r) {
        if (me > 1) continue;
        // handshake first (rank 1 -> rank 0, 4 bytes, both streams drained)
        // so the timed round trip does not include the host skew between
        // the two ranks' enqueues
        if (me == 0)
          p->comm->recv(buf2, 4, 1, st);
        else
          p->comm->send(buf, 4, 0, st);
        EXG_CUDA(cudaStreamSynchronize(st));
        EXG_CUDA(cudaEventRecord(a, st));
        if (me == 0) {
          p->comm->send(buf, n, 1, st);
          p->comm->recv(buf2, n, 1, st);
        } else {
          p->comm->recv(buf2, n, 0, st);
          p->comm->send(buf2, n, 0, st);
        }
        EXG_CUDA(cudaEventRecord(b, st));
        EXG_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        EXG_CUDA(cudaEventElapsedTime(&ms, a, b));
        if (r > 0) v.push_back(ms * 1e-3 / 2);
      }
      pp_t->push_back(me <= 1 ? median_of(v) : 0.0);
    }
    p->comm->check_async();
  } catch (...) {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    cudaFree(buf2);
    throw;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(buf2);
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
