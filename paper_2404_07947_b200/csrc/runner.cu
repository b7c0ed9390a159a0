// XRunner schedule executor (RRA PAPER.md:216-220).
//
// RRA cycle on one GPU: an encode phase admitting
//   min(B_E, B_D - active, remaining)
// requests FIFO, then N_D decode iterations over the active
// rows; rows leave the batch the iteration they emit their last token (early
// termination + compaction).  KV stays in its slot (slot
// indirection), so compaction is a host row-table edit: the next iteration's
// row table simply omits the finished rows.  When no requests remain the
// decode phases drain without encoding.
//
// FasterTransformer-style static batch (EXG_STATIC, the in-runner baseline
// of SURVEY.md §8(f) NEXT-4): b_e requests are admitted only
// when the previous batch has finished, encoded together, and decoded with a
// fixed batch -- completed queries are not early-terminated, they keep being
// computed (the "white boxes" of PAPER.md:112) until the batch's longest
// output is done; the batch's results return together at that iteration
// (latency of every request = batch start .. batch end).
//
// The host never waits on the GPU inside the loop: row tables go through a
// ring of pinned staging buffers recycled by events, tokens are written by
// the argmax kernel straight into a device output array, and times come from
// events recorded at phase / iteration boundaries (one device clock).
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "engine.cuh"
#include "runner.h"

namespace exg {

namespace {
struct Staging {
  struct Slot {
    int32_t* host = nullptr;
    cudaEvent_t ev = nullptr;
    bool used = false;
  };
  std::vector<Slot> slots;
  size_t cap_ints = 0;
  int next = 0;
  Staging(int n, size_t cap) : slots(n), cap_ints(cap) {
    for (auto& s : slots) {
      EXG_CUDA(cudaMallocHost(&s.host, cap * sizeof(int32_t)));
      EXG_CUDA(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (auto& s : slots) {
      if (s.ev) cudaEventSynchronize(s.ev), cudaEventDestroy(s.ev);
      if (s.host) cudaFreeHost(s.host);
    }
  }
  Slot& acquire() {
    Slot& s = slots[next];
    next = (next + 1) % (int)slots.size();
    if (s.used) EXG_CUDA(cudaEventSynchronize(s.ev));
    s.used = true;
    return s;
  }
};

struct Row {
  int req, slot, pos, emitted;
  bool live = true;   // false: finished, still computed by the static batch
  int64_t seq = 0;    // admission order (paged KV: the preemption victim is the latest)
};

struct EventPool {
  std::vector<cudaEvent_t> evs;
  int used = 0;
  cudaEvent_t get() {
    if (used == (int)evs.size()) {
      cudaEvent_t e;
      EXG_CUDA(cudaEventCreate(&e));
      evs.push_back(e);
    }
    return evs[used++];
  }
  ~EventPool() {
    for (auto e : evs) cudaEventDestroy(e);
  }
};

// host-side state of the runner kept in the Engine across runs (pinned
// staging ring, events, device table buffers), grown when a run needs more
struct RunCache {
  std::unique_ptr<Staging> stage;
  EventPool evp;
  int32_t* d_out = nullptr;
  int32_t* d_tab = nullptr;
  size_t out_cap = 0, tab_cap = 0;
  ~RunCache() {
    if (d_out) cudaFree(d_out);
    if (d_tab) cudaFree(d_tab);
  }
  int32_t* ensure(int32_t*& p, size_t& cap, size_t n) {
    if (n > cap) {
      if (p) EXG_CUDA(cudaFree(p));
      p = nullptr;
      cap = 0;
      EXG_CUDA(cudaMalloc(&p, sizeof(int32_t) * n));
      cap = n;
    }
    return p;
  }
};

double pct(std::vector<double> v, double q) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double r = q * (v.size() - 1);
  const size_t lo = (size_t)std::floor(r), hi = (size_t)std::ceil(r);
  return v[lo] + (r - lo) * (v[hi] - v[lo]);
}
}  // namespace

void run_rra(Engine& E, const exg_schedule& s, const exg_request* reqs, int n, int32_t* out_tokens,
             double* out_latency, exg_run_stats* stats, const exg_run_opts* opts) {
  const Dims& D = E.dims();
  const bool ft = s.strategy == EXG_STATIC;
  if (s.strategy != EXG_RRA && !ft) throw std::invalid_argument("run_rra: strategy is not RRA or STATIC");
  if (ft ? s.b_e < 1 : (s.b_e < 1 || s.b_d < s.b_e || s.n_d < 1))
    throw std::invalid_argument(ft ? "static batch needs b_e >= 1" : "RRA needs 1 <= B_E <= B_D, N_D >= 1");
  // token accounting: decoder-only encode = positions
  // 0..n-2, decode u consumes x[n-1] / y[u-1] at position n-1+u-1;
  // encoder-decoder encode = all n tokens, decode u consumes the start token
  // 0 / y[u-1] at decoder position u-1 and cross-attends to the n encoder keys
  const bool ed = E.encdec();
  int max_in = 1, max_ctx = 1, max_out = 1;
  int64_t total_out = 0;
  std::vector<int64_t> base(n + 1, 0);
  for (int r = 0; r < n; ++r) {
    const exg_request& q = reqs[r];
    if (q.input_len < 1 || q.output_len < 1 || !q.input_ids) throw std::invalid_argument("request lengths must be >= 1");
    if (ed ? std::max(q.input_len, q.output_len) > D.max_pos : q.input_len + q.output_len > D.max_pos)
      throw std::invalid_argument(ed ? "input_len or output_len > max_pos" : "input_len + output_len > max_pos");
    max_out = std::max(max_out, q.output_len);
    for (int j = 0; j < q.input_len; ++j)
      if (q.input_ids[j] < 0 || q.input_ids[j] >= D.V) throw std::invalid_argument("token id out of range");
    max_in = std::max(max_in, q.input_len);
    max_ctx = std::max(max_ctx, q.input_len + q.output_len);
    base[r + 1] = base[r] + q.output_len;
  }
  total_out = base[n];
  const int need_ctx = ed ? max_out : max_ctx;
  const int slot_ctx = (opts && opts->slot_ctx > 0) ? opts->slot_ctx : need_ctx;
  if (slot_ctx < need_ctx) throw std::invalid_argument("slot_ctx smaller than a request's input+output length");
  const int B_D = ft ? s.b_e : s.b_d, B_E = s.b_e;
  const int enc_drop = ed ? 0 : 1;   // input tokens the encode phase does not process
  const double dyn = (opts && !ft) ? opts->dyn_threshold : 0.0;
  // paged KV (exegpt.h kv_page): pages
  // of P positions from a pool of n_pages, a page table row of maxp entries
  // per batch row
  const int P = opts ? opts->kv_page : 0;
  const bool paged = P > 0;
  int maxp = 0, n_pages = 0;
  if (paged) {
    if (ft || ed || D.f32) throw std::invalid_argument("paged KV: decoder-only bf16 models under RRA");
    if (P % 64 != 0 || 512 % P != 0) throw std::invalid_argument("kv_page must be a multiple of 64 dividing 512");
    if (opts->kv_pages < 0) throw std::invalid_argument("kv_pages < 0");
    maxp = (slot_ctx + P - 1) / P;
    n_pages = opts->kv_pages > 0 ? opts->kv_pages : B_D * maxp;
    if (n_pages < maxp + 1) throw std::invalid_argument("kv_pages below one request's pages + 1");
  }
  // encode-phase capacity: B_E rows of at most max_in - enc_drop tokens.  The
  // dynamic adjustment may admit up to B_D rows, but never more tokens than
  // this (its token target is clamped to enc_tok_cap below).  A preempted
  // row re-encodes up to max_ctx - 1 tokens.
  const int enc_tok_cap = std::max({1, B_E * (max_in - enc_drop), paged ? max_ctx - 1 : 1});
  const int enc_row_cap = dyn > 0 ? B_D : B_E;
  if (paged)
    E.ensure_kv(std::max(n_pages, B_D), P, -1, 0);
  else
    E.ensure_kv(B_D, slot_ctx, -1, ed ? max_in : 0);
  E.ensure_workspace(enc_tok_cap, B_D);
  cudaStream_t st = E.stream();

  // device arrays: output tokens, encode tables, decode tables, and the
  // pinned staging ring -- all kept in the engine's run cache across runs
  auto& rc_any = E.run_cache();
  if (!rc_any) rc_any = std::make_shared<RunCache>();
  RunCache& rc = *static_cast<RunCache*>(rc_any.get());
  const size_t enc_ints = (size_t)3 * enc_tok_cap + 3 * ((size_t)enc_row_cap + 1) + 2 * (size_t)enc_row_cap +
                          (paged ? (size_t)2 * enc_tok_cap + (size_t)enc_row_cap * maxp : 0);
  const size_t dec_ints = (size_t)5 * B_D + (paged ? (size_t)B_D * maxp : 0);
  const size_t tab_ints = std::max(enc_ints, dec_ints);
  // + B_D scratch entries: the tokens of finished rows a static batch still computes
  int32_t* d_out = rc.ensure(rc.d_out, rc.out_cap, (size_t)total_out + B_D);
  int32_t* d_enc = rc.ensure(rc.d_tab, rc.tab_cap, enc_ints + dec_ints);
  int32_t* d_dec = d_enc + enc_ints;
  if (!rc.stage || rc.stage->cap_ints < tab_ints) {
    rc.stage.reset();
    rc.stage = std::make_unique<Staging>(64, tab_ints);
  }
  Staging& stage = *rc.stage;
  EventPool& evp = rc.evp;
  evp.used = 0;   // events of an earlier run are re-recorded
  std::vector<float> dump_host;
  const bool dumping = opts && opts->logits_out && opts->dump_mask;
  std::vector<int64_t> dump_base(n + 1, 0);
  if (dumping)
    for (int r = 0; r < n; ++r) dump_base[r + 1] = dump_base[r] + (opts->dump_mask[r] ? reqs[r].output_len : 0);

  std::vector<int> free_slots(B_D);
  for (int i = 0; i < B_D; ++i) free_slots[i] = B_D - 1 - i;
  // paged KV state: free page stack, pages of each slot, preempted requests
  // waiting for re-admission (sorted by request index = arrival order)
  std::vector<int> free_pages;
  for (int i = n_pages - 1; i >= 0; --i) free_pages.push_back(i);
  std::vector<std::vector<int>> slot_pages(paged ? B_D : 0);
  struct Resume {
    int req, emitted;
  };
  std::vector<Resume> resume;
  int64_t pages_peak = 0, preemptions = 0, admit_seq = 0;
  auto release_pages = [&](int slot) {
    if (!paged) return;
    for (int pg : slot_pages[slot]) free_pages.push_back(pg);
    slot_pages[slot].clear();
  };
  auto note_peak = [&] { pages_peak = std::max<int64_t>(pages_peak, n_pages - (int64_t)free_pages.size()); };
  std::vector<Row> active;
  active.reserve(B_D);
  std::vector<int> order;   // decode-table row -> active row
  std::vector<int> admit_ev(n, -1), done_ev(n, -1);
  std::vector<cudaEvent_t> evs;
  std::vector<int> ev_kind;        // 0 = phase start, 1 = encode end, 2 = iteration end
  std::vector<int> ev_tokens;      // tokens emitted by the iteration ending at this event
  std::vector<int> ev_rows;        // trace: decode batch of the iteration ending here
  std::vector<double> ev_work;     // trace: encoded tokens / attention keys of the stage ending here
  auto record = [&](int kind, int toks) {
    cudaEvent_t e = evp.get();
    EXG_CUDA(cudaEventRecord(e, st));
    evs.push_back(e);
    ev_kind.push_back(kind);
    ev_tokens.push_back(toks);
    ev_rows.push_back(0);
    ev_work.push_back(0.0);
    return (int)evs.size() - 1;
  };
  int enc_T = 0;

  int next_req = 0;
  double mean_enc_tokens = 0, steady_batch_sum = 0;
  int64_t steady_iters = 0, admitted_phases = 0;
  for (int r = 0; r < n; ++r) mean_enc_tokens += reqs[r].input_len - enc_drop;
  mean_enc_tokens /= n;
  int64_t decode_iters = 0, encode_phases = 0, batch_sum = 0;
  const long long launches0 = launch_counter().load();
  E.set_kernel_timing(opts && opts->kernel_timing);
  EXG_CUDA(cudaMemsetAsync(E.err_flag(), 0, sizeof(int32_t), st));
  record(0, 0);
  // admission candidates: preempted requests first (their generated tokens
  // appended to the input), then new requests in arrival order
  auto cand_req = [&](int k) { return k < (int)resume.size() ? resume[k].req : next_req + (k - (int)resume.size()); };
  auto cand_emit = [&](int k) { return k < (int)resume.size() ? resume[k].emitted : 0; };
  auto cand_len = [&](int k) { return reqs[cand_req(k)].input_len + cand_emit(k); };
  while (next_req < n || !active.empty() || !resume.empty()) {
    // ---------------- encode phase ----------------
    const int waiting = (int)resume.size() + (n - next_req);
    int admit = std::min({B_E, B_D - (int)active.size(), waiting});
    if (ft && !active.empty()) admit = 0;   // static batch: no admission until it has drained
    if (dyn > 0 && admit > 0) {
      // dynamic workload adjustment: decoder batch below /
      // above +-dyn of its running average -> admit that many rows more / fewer
      int be = B_E;
      if (steady_iters >= 2 * s.n_d && !active.empty()) {
        const double avg = steady_batch_sum / steady_iters, cur = (double)active.size();
        if (cur < (1 - dyn) * avg || cur > (1 + dyn) * avg) be = B_E + (int)std::lround(avg - cur);
      }
      be = std::max(1, std::min(be, B_D));
      // encoder workload (token sum) within +-dyn of be x the mean encoded length
      const int cap = std::min(B_D - (int)active.size(), waiting);
      const double target = be * mean_enc_tokens;
      double tok = 0;
      int k = 0;
      while (k < cap) {
        const double t = cand_len(k) - enc_drop;
        if (k >= be && tok >= (1 - dyn) * target) break;
        if (k >= 1 && tok + t > (1 + dyn) * target) break;
        if (k >= 1 && tok + t > enc_tok_cap) break;   // workspace / staging capacity
        tok += t;
        ++k;
      }
      admit = k;
    }
    if (paged && admit > 0) {
      // pages for positions 0 .. n'-1 of each admitted row (its encoded
      // tokens and its first decode position), one free page per active row
      // kept in reserve; the encode workspace bounds the token sum
      int64_t fr = (int64_t)free_pages.size();
      int k = 0, tok = 0;
      while (k < admit) {
        const int need = (cand_len(k) + P - 1) / P;
        if (fr - need < (int64_t)active.size() + k + 1) break;
        if (k >= 1 && tok + cand_len(k) - enc_drop > enc_tok_cap) break;
        fr -= need;
        tok += cand_len(k) - enc_drop;
        ++k;
      }
      admit = k;
    }
    const int ev_phase = record(0, 0);
    if (admit > 0) {
      Staging::Slot& sl = stage.acquire();
      int32_t* h = sl.host;
      int T = 0, maxlen = 0;
      for (int k = 0; k < admit; ++k) T += cand_len(k) - enc_drop;
      int32_t* ids = h;
      int32_t* pos = ids + T;
      int32_t* tsl = pos + T;
      int32_t* cu = tsl + T;
      int32_t* rsl = cu + admit + 1;
      int32_t* p0 = rsl + admit;
      int32_t* last = p0 + admit;
      int32_t* kvb = last + admit;            // paged: page / offset per token, page table per request
      int32_t* kvo = kvb + (paged ? T : 0);
      int32_t* ptab = kvo + (paged ? T : 0);
      // tokens a preempted row generated live on the device (d_out): copied
      // into the uploaded table after the upload (dst offset, src offset, count)
      std::vector<std::array<int64_t, 3>> gen_copies;
      int t = 0;
      cu[0] = 0;
      for (int k = 0; k < admit; ++k) {
        const int r = cand_req(k), e = cand_emit(k);
        const exg_request& q = reqs[r];
        const int n1 = q.input_len + e;   // prompt + generated tokens (a preempted row)
        const int slot = free_slots.back();
        free_slots.pop_back();
        const int ne = n1 - enc_drop;
        if (paged) {
          auto& pg = slot_pages[slot];
          for (int j = 0; j < (n1 + P - 1) / P; ++j) {
            pg.push_back(free_pages.back());
            free_pages.pop_back();
          }
          for (int j = 0; j < maxp; ++j) ptab[(int64_t)k * maxp + j] = pg[j < (int)pg.size() ? j : 0];
        }
        const int t_start = t;
        for (int j = 0; j < ne; ++j, ++t) {
          ids[t] = j < q.input_len ? q.input_ids[j] : 0;
          pos[t] = j;
          tsl[t] = slot;
          if (paged) {
            kvb[t] = slot_pages[slot][j / P];
            kvo[t] = j % P;
          }
        }
        if (ne > q.input_len) gen_copies.push_back({t_start + q.input_len, base[r], ne - q.input_len});
        cu[k + 1] = t;
        rsl[k] = slot;
        p0[k] = 0;
        if (ed) {
          last[k] = 0;
        } else if (n1 - 1 < q.input_len) {
          last[k] = q.input_ids[n1 - 1];
        } else {
          last[k] = 0;
          gen_copies.push_back({-1 - (int64_t)k, base[r] + e - 1, 1});   // the last generated token
        }
        maxlen = std::max(maxlen, ne);
        active.push_back(Row{r, slot, ed ? 0 : n1 - 1, e, true, admit_seq++});
        if (admit_ev[r] < 0) admit_ev[r] = ev_phase;
      }
      note_peak();
      const size_t nints = (size_t)3 * T + (admit + 1) + 3 * admit + (paged ? (size_t)2 * T + (size_t)admit * maxp : 0);
      EXG_CUDA(cudaMemcpyAsync(d_enc, h, nints * sizeof(int32_t), cudaMemcpyHostToDevice, st));
      EXG_CUDA(cudaEventRecord(sl.ev, st));
      int32_t* d_last = d_enc + 3 * T + (admit + 1) + 2 * admit;
      for (const auto& c : gen_copies) {
        int32_t* dst = c[0] >= 0 ? d_enc + c[0] : d_last + (-1 - c[0]);
        EXG_CUDA(cudaMemcpyAsync(dst, d_out + c[1], sizeof(int32_t) * c[2], cudaMemcpyDeviceToDevice, st));
      }
      // last_tok[slot] = x[n-1] for the admitted rows
      set_last_tokens(E.last_tok(), d_enc + 3 * T + (admit + 1), d_last, admit, st);
      EncodeBatch eb;
      eb.T = T;
      eb.R = admit;
      eb.max_len = maxlen;
      for (int k = 0; k < admit; ++k) {
        const double m = cand_len(k) - enc_drop;
        eb.attn_pairs += ed ? m * m : m * (m + 1) / 2;
      }
      eb.ids = d_enc;
      eb.pos = d_enc + T;
      eb.tslot = d_enc + 2 * T;
      eb.cu = d_enc + 3 * T;
      eb.rslot = eb.cu + admit + 1;
      eb.pos0 = eb.rslot + admit;
      if (paged) {
        eb.kv_blk = d_last + admit;
        eb.kv_off = eb.kv_blk + T;
        eb.kv = KvMap{eb.kv_off + T, maxp};
      }
      E.encode(eb);
      enc_T = T;
      const int from_resume = std::min(admit, (int)resume.size());
      resume.erase(resume.begin(), resume.begin() + from_resume);
      next_req += admit - from_resume;
      ++encode_phases;
      ++admitted_phases;
    }
    {
      const int k_end = record(1, admit);   // tokens field of an encode-end event: requests admitted
      ev_rows[k_end] = admit;
      ev_work[k_end] = admit > 0 ? enc_T : 0;
    }
    // ---------------- N_D decode iterations ----------------
    for (int u = 0; (ft || u < s.n_d) && !active.empty(); ++u) {
      if (paged) {
        // every row writes key `pos` this iteration: give it the page when
        // pos crosses into a new one; with none free, preempt the most
        // recently admitted row (freeing its pages; re-admitted later with
        // its generated tokens appended -- recompute preemption)
        for (size_t i = 0; i < active.size();) {
          const Row& rw = active[i];
          auto& pg = slot_pages[rw.slot];
          if (rw.pos / P < (int)pg.size()) {
            ++i;
            continue;
          }
          if (free_pages.empty()) {
            size_t v = 0;
            for (size_t j = 1; j < active.size(); ++j)
              if (active[j].seq > active[v].seq) v = j;
            const Row vr = active[v];
            release_pages(vr.slot);
            free_slots.push_back(vr.slot);
            const Resume rs{vr.req, vr.emitted};
            resume.insert(std::upper_bound(resume.begin(), resume.end(), rs,
                                           [](const Resume& a, const Resume& b) { return a.req < b.req; }),
                          rs);
            active.erase(active.begin() + v);
            ++preemptions;
            if (v < i) --i;
            continue;   // retry row i (or the row that moved into its place)
          }
          pg.push_back(free_pages.back());
          free_pages.pop_back();
          ++i;
        }
        note_peak();
        if (active.empty()) break;
      }
      const int B = (int)active.size();
      Staging::Slot& sl = stage.acquire();
      int32_t* h = sl.host;
      int max_keys = 0, max_xkeys = 0;
      double sum_keys = 0, sum_xkeys = 0;
      int live = 0;
      // rows in decreasing attention length: the decode-attention grid is
      // dispatched in row order, so the longest rows start first and the
      // launch's tail is made of short rows (per-row results do not depend on
      // the row order, T13)
      auto row_pos = [&](const Row& rw) {
        // a finished row of a static batch keeps decoding past its length:
        // its position is clamped inside its own slot, its token goes to scratch
        return rw.live ? rw.pos : std::min({rw.pos, slot_ctx - 1, D.max_pos - 1});
      };
      order.resize(B);
      for (int i = 0; i < B; ++i) order[i] = i;
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        const int kx = row_pos(active[x]) + (ed ? reqs[active[x].req].input_len : 0);
        const int ky = row_pos(active[y]) + (ed ? reqs[active[y].req].input_len : 0);
        return kx > ky;
      });
      for (int i = 0; i < B; ++i) {
        const Row& rw = active[order[i]];
        const int pos = row_pos(rw);
        live += rw.live;
        h[i] = rw.slot;
        h[B + i] = pos;
        h[2 * B + i] = pos + 1;
        h[3 * B + i] = rw.live ? (int32_t)(base[rw.req] + rw.emitted) : (int32_t)(total_out + i);
        h[4 * B + i] = reqs[rw.req].input_len;
        if (paged) {
          const auto& pg = slot_pages[rw.slot];
          for (int j = 0; j < maxp; ++j) h[5 * B + (int64_t)i * maxp + j] = pg[j < (int)pg.size() ? j : 0];
        }
        max_keys = std::max(max_keys, pos + 1);
        sum_keys += pos + 1;
        max_xkeys = std::max(max_xkeys, reqs[rw.req].input_len);
        sum_xkeys += reqs[rw.req].input_len;
      }
      EXG_CUDA(cudaMemcpyAsync(d_dec, h, ((size_t)5 * B + (paged ? (size_t)B * maxp : 0)) * sizeof(int32_t),
                               cudaMemcpyHostToDevice, st));
      EXG_CUDA(cudaEventRecord(sl.ev, st));
      DecodeBatch db;
      db.B = B;
      db.max_keys = max_keys;
      db.sum_keys = sum_keys;
      db.slot = d_dec;
      db.pos = d_dec + B;
      db.nkeys = d_dec + 2 * B;
      db.out_off = d_dec + 3 * B;
      if (ed) {
        db.xkeys = d_dec + 4 * B;
        db.max_xkeys = max_xkeys;
        db.sum_xkeys = sum_xkeys;
      }
      db.out_tokens = d_out;
      if (paged) db.kv = KvMap{d_dec + 5 * B, maxp};
      E.decode(db);
      if (dumping) {
        for (int i = 0; i < B; ++i) {
          const Row& rw = active[order[i]];
          if (!rw.live || !opts->dump_mask[rw.req]) continue;
          float* dst = opts->logits_out + (dump_base[rw.req] + rw.emitted) * (int64_t)D.V;
          EXG_CUDA(cudaMemcpyAsync(dst, E.logits() + (int64_t)i * D.V, sizeof(float) * D.V, cudaMemcpyDeviceToHost, st));
        }
      }
      const int ev_it = record(2, live);
      ev_rows[ev_it] = B;
      ev_work[ev_it] = sum_keys + (ed ? sum_xkeys : 0.0);   // T5: self + cross-attention keys
      ++decode_iters;
      batch_sum += B;
      if (next_req < n) {   // decode batch average while requests keep arriving (not the drain)
        steady_batch_sum += B;
        ++steady_iters;
      }
      // early termination + stable compaction of the row table
      int w = 0;
      if (ft) {
        int alive = 0;
        for (Row& rw : active) {
          rw.pos += 1;
          if (rw.live && ++rw.emitted == reqs[rw.req].output_len) rw.live = false;
          alive += rw.live;
        }
        if (alive == 0) {   // the batch is done: every result returns at this iteration
          for (const Row& rw : active) {
            done_ev[rw.req] = ev_it;
            free_slots.push_back(rw.slot);
          }
          active.clear();
        }
        continue;
      }
      for (int i = 0; i < B; ++i) {
        Row rw = active[i];
        rw.emitted += 1;
        rw.pos += 1;
        if (rw.emitted == reqs[rw.req].output_len) {
          done_ev[rw.req] = ev_it;
          free_slots.push_back(rw.slot);
          release_pages(rw.slot);
        } else {
          active[w++] = rw;
        }
      }
      active.resize(w);
    }
  }
  EXG_CUDA(cudaStreamSynchronize(st));
  int32_t err = 0;
  EXG_CUDA(cudaMemcpy(&err, E.err_flag(), sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (out_tokens) EXG_CUDA(cudaMemcpy(out_tokens, d_out, sizeof(int32_t) * total_out, cudaMemcpyDeviceToHost));
  if (err) throw std::runtime_error("NaN logit encountered (T7)");

  // ---------------- timing ----------------
  const int nev = (int)evs.size();
  std::vector<double> t(nev, 0.0);
  for (int k = 1; k < nev; ++k) {
    float ms = 0.f;
    EXG_CUDA(cudaEventElapsedTime(&ms, evs[0], evs[k]));
    t[k] = ms * 1e-3;
  }
  std::vector<double> lat(n);
  for (int r = 0; r < n; ++r) {
    lat[r] = t[done_ev[r]] - t[admit_ev[r]];
    if (out_latency) out_latency[r] = lat[r];
  }
  const long long launches = launch_counter().load() - launches0;
  double kt[EXG_K_CLASSES] = {0}, kw[EXG_K_CLASSES] = {0};
  int64_t kn[EXG_K_CLASSES] = {0};
  E.collect_kernel_timing(kt, kw, kn);
  E.set_kernel_timing(false);
  int64_t n_trace = 0;
  if (opts && opts->trace_out && opts->trace_cap > 0) {
    for (int k = 1; k < nev && n_trace < opts->trace_cap; ++k) {
      const bool enc = ev_kind[k] == 1 && ev_rows[k] > 0, dec = ev_kind[k] == 2;
      if (!enc && !dec) continue;
      double* rec = opts->trace_out + 5 * n_trace++;
      rec[0] = enc ? 1 : 2;
      rec[1] = t[k - 1];
      rec[2] = t[k] - t[k - 1];
      rec[3] = ev_rows[k];
      rec[4] = ev_work[k];
    }
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->trace_records = n_trace;
    stats->kv_preemptions = preemptions;
    stats->kv_pages_peak = pages_peak;
    stats->kernel_launches = launches;
    for (int c = 0; c < EXG_K_CLASSES; ++c) {
      stats->k_time_s[c] = kt[c];
      stats->k_work[c] = kw[c];
      stats->k_launches[c] = kn[c];
    }
    const double wall = t[nev - 1] - t[0];
    stats->wall_s = wall;
    stats->out_tokens = total_out;
    stats->decode_iters = decode_iters;
    stats->encode_phases = encode_phases;
    stats->tok_s = wall > 0 ? total_out / wall : 0;
    stats->seq_s = wall > 0 ? n / wall : 0;
    stats->lat_p50_s = pct(lat, 0.50);
    stats->lat_p99_s = pct(lat, 0.99);
    stats->lat_max_s = lat.empty() ? 0 : *std::max_element(lat.begin(), lat.end());
    stats->mean_decode_batch = decode_iters ? (double)batch_sum / decode_iters : 0;
    double enc = 0, dec = 0;
    for (int k = 1; k < nev; ++k) {
      if (ev_kind[k] == 1) enc += t[k] - t[k - 1];
      if (ev_kind[k] == 2) dec += t[k] - t[k - 1];
    }
    stats->encode_s = enc;
    stats->decode_s = dec;
    stats->mean_encode_batch = admitted_phases ? (double)n / admitted_phases : 0;
    // Table 9: single-stage times of encode phases and
    // decode iterations inside the steady window, mean and p99 of |t - mean|
    {
      const int r0 = std::min(n - 1, (int)std::ceil(0.1 * n));
      const double w0 = t[admit_ev[r0]], w1 = t[admit_ev[n - 1]];
      std::vector<double> te, td;
      for (int k = 1; k < nev; ++k) {
        if (t[k - 1] < w0 || t[k] > w1) continue;
        if (ev_kind[k] == 1 && t[k] - t[k - 1] > 0 && ev_kind[k - 1] == 0 && ev_tokens[k] > 0) te.push_back(t[k] - t[k - 1]);
        if (ev_kind[k] == 2) td.push_back(t[k] - t[k - 1]);
      }
      auto spread = [](const std::vector<double>& v, double* mean, double* p99dev) {
        *mean = *p99dev = 0;
        if (v.empty()) return;
        double m = 0;
        for (double x : v) m += x;
        m /= v.size();
        std::vector<double> dv;
        for (double x : v) dv.push_back(std::fabs(x - m));
        *mean = m;
        *p99dev = pct(dv, 0.99);
      };
      spread(te, &stats->enc_stage_mean_s, &stats->enc_stage_p99dev_s);
      spread(td, &stats->dec_stage_mean_s, &stats->dec_stage_p99dev_s);
    }
    // steady-state window: admission of request ceil(0.1 n) .. admission of
    // the last request
    const int r0 = std::min(n - 1, (int)std::ceil(0.1 * n));
    const double w0 = t[admit_ev[r0]], w1 = t[admit_ev[n - 1]];
    if (w1 > w0) {
      int64_t toks = 0;
      for (int k = 0; k < nev; ++k)
        if (ev_kind[k] == 2 && t[k] > w0 && t[k] <= w1) toks += ev_tokens[k];
      stats->tok_s_steady = toks / (w1 - w0);
    } else {
      stats->tok_s_steady = stats->tok_s;
    }
  }
}

}  // namespace exg
