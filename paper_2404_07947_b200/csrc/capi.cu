// extern "C" boundary of libexegpt.so (include/exegpt.h, include/exegpt_ops.h).
// Every entry point catches all exceptions and maps them to an exg_status
// with a thread-local message; nothing throws across the ABI.
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <new>
#include <sstream>
#include <string>

#include "../../include/exegpt.h"
#include "../../include/exegpt_ops.h"
#include "engine.cuh"
#include "comm.h"
#include "multi.h"
#include "planner.h"
#include "profiler.h"
#include "runner.h"

struct exg_ctx {
  std::unique_ptr<exg::Engine> engine;      // single-GPU context
  std::unique_ptr<exg::MultiCtx> multi;     // n_gpus > 1 emulated on one device
  exg_model_spec spec;
  exg_cluster_spec cluster;
  int rank = 0, world = 1, device = 0;
};

struct exg_profile {
  exg::plan::Profile p;
};

namespace {
thread_local std::string g_err;

exg_status fail(exg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

template <class F>
exg_status guarded(F&& f) {
  try {
    g_err.clear();
    return f();
  } catch (const exg::CudaError& e) {
    const std::string m = e.what();
    if (m.find("out of memory") != std::string::npos) return fail(EXG_E_OOM, m);
    return fail(EXG_E_CUDA, m);
  } catch (const std::bad_alloc&) {
    return fail(EXG_E_OOM, "out of memory");
  } catch (const std::invalid_argument& e) {
    return fail(EXG_E_INPUT, e.what());
  } catch (const exg::plan::OutOfHull&) {
    return fail(EXG_E_INFEASIBLE, "query outside the profiled hull");
  } catch (const std::exception& e) {
    return fail(EXG_E_INTERNAL, e.what());
  } catch (...) {
    return fail(EXG_E_INTERNAL, "unknown error");
  }
}

std::vector<double> pmf_vec(const exg_pmf* p) {
  if (!p || p->max_len < 1 || !p->prob) throw std::invalid_argument("bad pmf");
  std::vector<double> v(p->prob, p->prob + p->max_len);
  for (double x : v)
    if (!(x >= 0.0)) throw std::invalid_argument("pmf has a negative or NaN entry");
  return v;
}

void check_spec(const exg_model_spec* s) {
  if (!s) throw std::invalid_argument("null model spec");
  if (s->n_dec_layers < 1 || s->d_model < 1 || s->n_heads < 1 || s->d_head < 1 || s->d_ff < 1 || s->vocab < 2 ||
      s->max_pos < 2)
    throw std::invalid_argument("invalid model spec");
  if (s->dtype != EXG_BF16 && s->dtype != EXG_FP32) throw std::invalid_argument("unknown dtype");
}

// the fp32 parity path covers decoder-only models on a
// single-GPU context
void check_fp32_scope(const exg_model_spec* s, const exg_cluster_spec* cluster, int world) {
  if (s->dtype != EXG_FP32) return;
  if (s->arch == EXG_ARCH_T5) throw std::invalid_argument("EXG_FP32: encoder-decoder models run bf16 only");
  if (world > 1 || (cluster && cluster->n_gpus > 1))
    throw std::invalid_argument("EXG_FP32: single-GPU contexts only (cluster.n_gpus = 1, world = 1)");
}

void to_c(const exg::plan::Sched& s, exg_schedule* o) {
  std::memset(o, 0, sizeof(*o));
  o->strategy = (exg_strategy)s.strategy;
  o->b_e = s.b_e;
  o->b_d = s.b_d;
  o->b_m = s.b_m;
  o->n_d = s.n_d;
  o->tp_degree = s.tp_degree;
  o->tp_gpus = s.tp_gpus;
  o->n_enc_gpus = s.n_enc_gpus;
  o->n_stages = (int32_t)s.stages.size();
  for (size_t k = 0; k < s.stages.size() && k < EXG_MAX_STAGES; ++k) {
    o->stage_first_gpu[k] = s.stages[k].first_gpu;
    o->stage_n_gpus[k] = s.stages[k].n_gpus;
    o->stage_layer_begin[k] = s.stages[k].layer_begin;
    o->stage_layer_end[k] = s.stages[k].layer_end;
  }
}

exg::plan::Sched from_c(const exg_schedule* o) {
  exg::plan::Sched s;
  s.strategy = o->strategy;
  s.b_e = o->b_e;
  s.b_d = o->b_d;
  s.b_m = o->b_m;
  s.n_d = o->n_d;
  s.tp_degree = o->tp_degree;
  s.tp_gpus = o->tp_gpus;
  s.n_enc_gpus = o->n_enc_gpus;
  if (o->n_stages < 1 || o->n_stages > EXG_MAX_STAGES) throw std::invalid_argument("schedule has no stages");
  for (int k = 0; k < o->n_stages; ++k)
    s.stages.push_back({o->stage_first_gpu[k], o->stage_n_gpus[k], o->stage_layer_begin[k], o->stage_layer_end[k]});
  return s;
}
}  // namespace

extern "C" {

int32_t exg_abi_version(void) { return EXG_ABI_VERSION; }
const char* exg_last_error(void) { return g_err.c_str(); }

exg_status exg_get_unique_id(uint8_t uid[128]) {
  return guarded([&] {
    if (!uid) throw std::invalid_argument("null uid");
    try {
      exg::nccl_unique_id(uid);
    } catch (const std::exception& e) {
      return fail(EXG_E_NCCL, e.what());
    }
    return EXG_OK;
  });
}

exg_status exg_create(const exg_model_spec* spec, const exg_cluster_spec* cluster, int32_t device, int32_t rank,
                      int32_t world, const uint8_t* uid, exg_ctx** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("null out");
    *out = nullptr;
    check_spec(spec);
    check_fp32_scope(spec, cluster, world);
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world");
    if (world > 1 && !uid) throw std::invalid_argument("multi-rank context needs the rank-0 unique id");
    if (world > 1 && (!cluster || cluster->n_gpus < world)) throw std::invalid_argument("cluster has fewer GPUs than ranks");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(EXG_E_CUDA, "no CUDA device");
    if (device < 0 || device >= ndev) throw std::invalid_argument("bad device index");
    auto c = std::make_unique<exg_ctx>();
    c->spec = *spec;
    if (cluster) c->cluster = *cluster;
    c->rank = rank;
    c->world = world;
    c->device = device;
    if (world > 1) {
      std::unique_ptr<exg::Comm> comm;
      EXG_CUDA(cudaSetDevice(device));
      try {
        comm = exg::make_nccl_comm(uid, rank, world);
      } catch (const std::exception& e) {
        return fail(EXG_E_NCCL, e.what());
      }
      c->multi = std::make_unique<exg::MultiCtx>(*spec, device, std::move(comm));
    } else if (cluster && cluster->n_gpus > 1) {
      c->multi = std::make_unique<exg::MultiCtx>(*spec, device);  // every GPU of a layout emulated on `device`
    } else {
      c->engine = std::make_unique<exg::Engine>(*spec, device);
    }
    *out = c.release();
    return EXG_OK;
  });
}

exg_status exg_create_nccl_loopback(const exg_model_spec* spec, const exg_cluster_spec* cluster, int32_t device,
                                    exg_ctx** out) {
  return guarded([&] {
    if (!out || !cluster) throw std::invalid_argument("null argument");
    *out = nullptr;
    check_spec(spec);
    check_fp32_scope(spec, cluster, 2);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(EXG_E_CUDA, "no CUDA device");
    if (device < 0 || device >= ndev) throw std::invalid_argument("bad device index");
    EXG_CUDA(cudaSetDevice(device));
    std::unique_ptr<exg::Comm> comm;
    try {
      uint8_t uid[128];
      exg::nccl_unique_id(uid);
      comm = exg::make_nccl_comm(uid, 0, 1);
    } catch (const std::exception& e) {
      return fail(EXG_E_NCCL, e.what());
    }
    auto c = std::make_unique<exg_ctx>();
    c->spec = *spec;
    c->cluster = *cluster;
    c->device = device;
    c->multi = std::make_unique<exg::MultiCtx>(*spec, device, std::move(comm));
    *out = c.release();
    return EXG_OK;
  });
}

exg_status exg_create_local_group(const exg_model_spec* spec, const exg_cluster_spec* cluster, int32_t device,
                                  int32_t world, exg_ctx** out) {
  return guarded([&] {
    if (!out || !cluster) throw std::invalid_argument("null argument");
    check_spec(spec);
    check_fp32_scope(spec, cluster, world);
    if (world < 2 || world > cluster->n_gpus) throw std::invalid_argument("world must be in [2, cluster.n_gpus]");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(EXG_E_CUDA, "no CUDA device");
    if (device < 0 || device >= ndev) throw std::invalid_argument("bad device index");
    auto hub = exg::make_local_hub(world);
    std::vector<std::unique_ptr<exg_ctx>> cs;
    for (int r = 0; r < world; ++r) {
      auto c = std::make_unique<exg_ctx>();
      c->spec = *spec;
      c->cluster = *cluster;
      c->rank = r;
      c->world = world;
      c->device = device;
      c->multi = std::make_unique<exg::MultiCtx>(*spec, device, exg::make_local_comm(hub, r));
      cs.push_back(std::move(c));
    }
    for (int r = 0; r < world; ++r) out[r] = cs[r].release();
    return EXG_OK;
  });
}

void exg_destroy(exg_ctx* ctx) {
  try {
    delete ctx;
  } catch (...) {
  }
}

exg_status exg_profile_run(exg_ctx* ctx, const exg_profile_grid* grid, exg_profile** out) {
  return guarded([&] {
    if (!ctx || !grid || !out) throw std::invalid_argument("null argument");
    auto p = std::make_unique<exg_profile>();
    if (ctx->multi && ctx->world > 1) {
      // multi-rank context: the interconnect tables, collective
      std::vector<int> tps;
      for (int i = 0; i < grid->n_tp; ++i) tps.push_back(grid->tp[i]);
      std::map<int, std::pair<std::vector<double>, std::vector<double>>> tp;
      std::vector<double> px, pt;
      ctx->multi->profile_comm(tps, grid->reps, &tp, &px, &pt);
      p->p.tps.push_back(1);
      for (auto& kv : tp) {
        p->p.tps.push_back(kv.first);
        exg::plan::Table1D tb;
        tb.x = kv.second.first;
        tb.t = kv.second.second;
        p->p.tp_sync[kv.first] = tb;
      }
      p->p.pp_sync.x = px;
      p->p.pp_sync.t = pt;
      p->p.has_pp = true;
      *out = p.release();
      return EXG_OK;
    }
    if (!ctx->engine) throw std::invalid_argument("layer profile on a single-GPU context (cluster.n_gpus = 1)");
    if (ctx->spec.dtype != EXG_BF16) throw std::invalid_argument("the profiler times the bf16 path");
    exg::profile_layers(*ctx->engine, ctx->spec, *grid, &p->p);
    *out = p.release();
    return EXG_OK;
  });
}

exg_status exg_profile_save(const exg_profile* p, const char* path) {
  return guarded([&] {
    if (!p || !path) throw std::invalid_argument("null argument");
    std::ofstream f(path);
    if (!f) throw std::invalid_argument(std::string("cannot open ") + path);
    f << p->p.dumps();
    return EXG_OK;
  });
}

exg_status exg_profile_comm_model(exg_profile* p, double alpha_s, double bw_bytes_per_s) {
  return guarded([&] {
    if (!p) throw std::invalid_argument("null profile");
    if (!(alpha_s >= 0) || !(bw_bytes_per_s > 0)) throw std::invalid_argument("bad alpha / bandwidth");
    exg::plan::Table1D pp;
    for (double b = 1024.0; b <= 64.0 * (1ull << 30); b *= 4.0) {
      pp.x.push_back(b);
      pp.t.push_back(alpha_s + b / bw_bytes_per_s);
    }
    p->p.pp_sync = pp;
    p->p.has_pp = true;
    p->p.tp_sync.clear();
    for (int t : p->p.tps) {
      if (t <= 1) continue;
      exg::plan::Table1D tb;
      for (double b : pp.x) {
        tb.x.push_back(b);
        tb.t.push_back(alpha_s + (t - 1) * b / bw_bytes_per_s);
      }
      p->p.tp_sync[t] = tb;
    }
    return EXG_OK;
  });
}

exg_status exg_profile_copy_comm(exg_profile* dst, const exg_profile* src) {
  return guarded([&] {
    if (!dst || !src) throw std::invalid_argument("null profile");
    if (!src->p.has_pp && src->p.tp_sync.empty()) throw std::invalid_argument("source profile has no interconnect tables");
    dst->p.tp_sync = src->p.tp_sync;
    dst->p.pp_sync = src->p.pp_sync;
    dst->p.has_pp = src->p.has_pp;
    return EXG_OK;
  });
}

exg_status exg_profile_load(const char* path, exg_profile** out) {
  return guarded([&] {
    if (!path || !out) throw std::invalid_argument("null argument");
    std::ifstream f(path);
    if (!f) throw std::invalid_argument(std::string("cannot open ") + path);
    std::stringstream ss;
    ss << f.rdbuf();
    auto p = std::make_unique<exg_profile>();
    p->p = exg::plan::Profile::loads(ss.str());
    *out = p.release();
    return EXG_OK;
  });
}

void exg_profile_free(exg_profile* p) { delete p; }

exg_status exg_simulate(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                        const exg_pmf* in, const exg_pmf* out_len, int32_t target_len, const exg_schedule* sched,
                        exg_estimate* est) {
  return guarded([&] {
    if (!p || !cluster || !sched || !est) throw std::invalid_argument("null argument");
    check_spec(spec);
    exg::plan::Simulator S(p->p, *spec, *cluster, pmf_vec(in), pmf_vec(out_len), target_len, false);
    if (sched->strategy == EXG_STATIC && sched->b_e < 1) throw std::invalid_argument("static batch b_e < 1");
    exg::plan::Est e = sched->strategy == EXG_STATIC ? S.simulate_static(sched->b_e) : S.simulate(from_c(sched));
    est->thrput_seq_s = e.thr;
    est->thrput_tok_s = e.tok;
    est->latency_s = e.lat;
    est->perf_evals = 1;
    est->feasible = e.feasible;
    return EXG_OK;
  });
}

exg_status exg_profile_stage_time(const exg_profile* p, int32_t phase, int32_t tp_degree, int32_t n_layers,
                                  double rows, double work, double* seconds) {
  return guarded([&] {
    if (!p || !seconds) throw std::invalid_argument("null argument");
    if (phase != 0 && phase != 1) throw std::invalid_argument("phase must be 0 (encode) or 1 (decode)");
    if (!(rows > 0) || !(work > 0) || n_layers < 1) throw std::invalid_argument("rows, work, n_layers must be > 0");
    const std::string ph = phase ? "dec" : "enc";
    auto ia = p->p.attn.find({ph, tp_degree});
    auto ir = p->p.rest.find({ph, tp_degree});
    if (ia == p->p.attn.end() || ir == p->p.rest.end()) throw std::invalid_argument("profile has no such table");
    const double a = exg::plan::interp2(ia->second, rows, work / rows);
    const double r = exg::plan::interp1(ir->second.x, ir->second.t, phase ? rows : work);
    double t = n_layers * (a + r);
    if (phase && p->p.has_head) t += exg::plan::interp1(p->p.head.x, p->p.head.t, rows);
    *seconds = t;
    return EXG_OK;
  });
}

exg_status exg_schedule_memory(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                               const exg_pmf* in, const exg_pmf* out_len, const exg_schedule* sched,
                               double* weight_bytes, double* kv_bytes) {
  return guarded([&] {
    if (!p || !cluster || !sched || !weight_bytes || !kv_bytes) throw std::invalid_argument("null argument");
    check_spec(spec);
    exg::plan::Simulator S(p->p, *spec, *cluster, pmf_vec(in), pmf_vec(out_len), 1, false);
    exg::plan::Sched s;
    if (sched->strategy == EXG_STATIC) {
      if (sched->b_e < 1) throw std::invalid_argument("static batch b_e < 1");
      s.strategy = EXG_STATIC;
      s.b_e = sched->b_e;
    } else {
      s = from_c(sched);
    }
    std::vector<double> w, kv;
    S.memory(s, w, kv);
    for (int g = 0; g < cluster->n_gpus; ++g) {
      weight_bytes[g] = w[g];
      kv_bytes[g] = kv[g];
    }
    return EXG_OK;
  });
}

exg_status exg_schedule_resolve(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                                const exg_pmf* in, const exg_pmf* out_len, int32_t m_count, exg_schedule* sched) {
  return guarded([&] {
    if (!p || !cluster || !sched) throw std::invalid_argument("null argument");
    check_spec(spec);
    exg::plan::Simulator S(p->p, *spec, *cluster, pmf_vec(in), pmf_vec(out_len), 1, false);
    exg::plan::Sched s;
    if (sched->strategy == EXG_RRA) {
      if (sched->b_e < 1 || sched->n_d < 1) throw std::invalid_argument("RRA needs b_e >= 1, n_d >= 1");
      s = S.rra_schedule(sched->b_e, sched->n_d, std::max(1, sched->tp_degree), sched->tp_gpus);
    } else if (sched->strategy == EXG_WAA_C || sched->strategy == EXG_WAA_M) {
      s = S.waa_schedule(sched->b_e, std::max(1, m_count), std::max(1, sched->tp_degree), sched->tp_gpus,
                         sched->strategy);
      if (!s.valid) return fail(EXG_E_INFEASIBLE, "WAA needs >= 2 GPUs and tp_gpus <= decoder GPUs");
    } else {
      throw std::invalid_argument("unknown strategy");
    }
    to_c(s, sched);
    return EXG_OK;
  });
}

exg_status exg_schedule_find(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                             const exg_pmf* in, const exg_pmf* out_len, int32_t target_len, double latency_bound_s,
                             uint32_t strategy_mask, const exg_search_opts* opts, exg_schedule* out,
                             exg_estimate* est) {
  return guarded([&] {
    if (!p || !cluster || !out) throw std::invalid_argument("null argument");
    check_spec(spec);
    if (!(strategy_mask & (EXG_RRA | EXG_WAA_C | EXG_WAA_M))) throw std::invalid_argument("unknown strategy");
    if (target_len < 1) throw std::invalid_argument("target_len < 1");
    exg_search_opts o{0.02, 0.02, 256, 0, 8, 0, 0};
    if (opts) o = *opts;
    exg::plan::Simulator S(p->p, *spec, *cluster, pmf_vec(in), pmf_vec(out_len), target_len,
                           o.use_little_fraction != 0);
    exg::plan::Found f;
    if (!exg::plan::schedule_find(S, latency_bound_s, strategy_mask, o, &f))
      return fail(EXG_E_INFEASIBLE, "no schedule satisfies the latency bound");
    to_c(f.sched, out);
    if (est) {
      est->thrput_seq_s = f.est.thr;
      est->thrput_tok_s = f.est.tok;
      est->latency_s = f.est.lat;
      est->perf_evals = f.evals;
      est->feasible = f.est.feasible;
    }
    return EXG_OK;
  });
}

exg_status exg_run(exg_ctx* ctx, const exg_schedule* sched, const exg_request* reqs, int32_t n, int32_t* out_tokens,
                   double* out_latency_s, exg_run_stats* stats, const exg_run_opts* opts) {
  return guarded([&] {
    if (!ctx || !sched || (!reqs && n > 0)) throw std::invalid_argument("null argument");
    if (n < 1) throw std::invalid_argument("empty request batch");
    EXG_CUDA(cudaSetDevice(ctx->device));
    if (ctx->multi) {
      int gpus = 0;
      for (int k = 0; k < sched->n_stages && k < EXG_MAX_STAGES; ++k) gpus += sched->stage_n_gpus[k];
      if (gpus > ctx->cluster.n_gpus) return fail(EXG_E_INFEASIBLE, "schedule needs more GPUs than the cluster has");
      ctx->multi->run(*sched, reqs, n, out_tokens, out_latency_s, stats, opts);
      return EXG_OK;
    }
    if (sched->strategy != EXG_RRA && sched->strategy != EXG_STATIC)
      return fail(EXG_E_INFEASIBLE, "WAA needs >= 2 GPUs (SPEC.md:233); this context has 1");
    if (sched->tp_degree > 1 || sched->n_stages > 1)
      return fail(EXG_E_INFEASIBLE, "schedule needs more GPUs than this context has");
    exg::run_rra(*ctx->engine, *sched, reqs, n, out_tokens, out_latency_s, stats, opts);
    return EXG_OK;
  });
}

// ----------------------------------------------------------------- ops ----
exg_status exg_op_weightgen(void* dst, int64_t rows, int64_t cols, int64_t ld, uint64_t seed, uint64_t tensor_id,
                            int32_t gain, int32_t transposed, int64_t canon_cols, int64_t row_off, int64_t col_off,
                            int32_t blocked, void* stream) {
  return guarded([&] {
    exg::GenParams g{seed,    tensor_id, gain,    (float)(2.0 * std::sqrt(3.0) * 0.02), 0.2f, transposed, canon_cols,
                     row_off, col_off,   blocked, 0};
    exg::weightgen((exg::bf16*)dst, rows, cols, ld, g, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_pack_weight(void* dst, const void* src, int64_t rows, int64_t K, int64_t ld, void* stream) {
  return guarded([&] {
    exg::pack_blocked((exg::bf16*)dst, (const exg::bf16*)src, rows, K, ld, (cudaStream_t)stream);
    return EXG_OK;
  });
}

int64_t exg_op_blocked_elems(int64_t rows, int64_t K) { return exg::blocked_elems(rows, K); }

exg_status exg_op_linear(const void* X, int64_t ldx, const void* Wb, int32_t tokens, int32_t features, int32_t K,
                         int32_t mode, int32_t act, const void* bias, void* out, int64_t ldo, float* resid,
                         int64_t ldr, int32_t decode, float* ws, int64_t ws_floats, void* stream) {
  return guarded([&] {
    if (K % 8) throw std::invalid_argument("K must be a multiple of 8");
    exg::LinearArgs a;
    a.X = (const exg::bf16*)X;
    a.ldx = ldx;
    a.Wb = (const exg::bf16*)Wb;
    a.K = K;
    a.ep.mode = mode;
    a.ep.act = act;
    a.ep.bias = (const exg::bf16*)bias;
    a.ep.out_bf16 = (exg::bf16*)out;
    a.ep.out_f32 = (float*)out;
    a.ep.ldo = ldo;
    a.ep.resid = resid;
    a.ep.ldr = ldr;
    a.ep.tokens = tokens;
    a.ep.features = features;
    a.decode = decode != 0;
    a.ws = ws;
    a.ws_floats = ws_floats > 0 ? (size_t)ws_floats : 0;
    exg::linear(a, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_layernorm(void* y, int64_t ldy, const float* x, int64_t ldx, const void* g, const void* b, int32_t T,
                            int32_t d, float eps, void* stream) {
  return guarded([&] {
    exg::layernorm((exg::bf16*)y, ldy, x, ldx, (const exg::bf16*)g, (const exg::bf16*)b, T, d, eps,
                   (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_rmsnorm(void* y, int64_t ldy, const float* x, int64_t ldx, const void* g, int32_t T, int32_t d,
                          float eps, float out_scale, void* stream) {
  return guarded([&] {
    exg::rmsnorm((exg::bf16*)y, ldy, x, ldx, (const exg::bf16*)g, T, d, eps, out_scale, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_embed(float* x, const int32_t* ids, const int32_t* pos, const void* tok_emb, const void* pos_emb,
                        int32_t T, int32_t d, void* stream) {
  return guarded([&] {
    exg::embed(x, ids, pos, (const exg::bf16*)tok_emb, (const exg::bf16*)pos_emb, T, d, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_kv_scatter(void* kc, void* vc, const void* qkv, const int32_t* slot, const int32_t* pos, int32_t T,
                             int32_t H, int32_t dh, int32_t max_ctx, void* stream) {
  return guarded([&] {
    exg::kv_scatter((exg::bf16*)kc, (exg::bf16*)vc, (const exg::bf16*)qkv, slot, pos, T, H, dh, max_ctx,
                    (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_decode_attention(const void* q, int64_t ldq, const void* kc, const void* vc, const int32_t* slot,
                                   const int32_t* n_keys, void* out, int64_t ldo, int32_t B, int32_t H, int32_t dh,
                                   int32_t max_ctx, float scale, int32_t split_len, int32_t max_splits, float* partial,
                                   const float* bias, int32_t bias_ld, int32_t bias_off, void* stream) {
  return guarded([&] {
    if (max_splits > 1 && !partial) throw std::invalid_argument("max_splits > 1 needs a partial buffer");
    exg::DecodeAttnArgs a;
    a.q = (const exg::bf16*)q;
    a.ldq = ldq;
    a.kc = (const exg::bf16*)kc;
    a.vc = (const exg::bf16*)vc;
    a.slot = slot;
    a.n_keys = n_keys;
    a.out = (exg::bf16*)out;
    a.ldo = ldo;
    a.B = B;
    a.H = H;
    a.dh = dh;
    a.max_ctx = max_ctx;
    a.scale = scale;
    a.split_len = split_len;
    a.max_splits = max_splits;
    a.partial = partial;
    a.bias = bias;
    a.bias_ld = bias_ld;
    a.bias_off = bias_off;
    exg::decode_attention(a, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_prefill_attention(const void* q, int64_t ldq, const void* kc, const void* vc,
                                    const int32_t* cu_seqlens, const int32_t* slot, const int32_t* pos0, int32_t R,
                                    int32_t max_len, void* out, int64_t ldo, int32_t H, int32_t dh, int32_t max_ctx,
                                    int32_t n_slots, int32_t T, float scale, int32_t causal, const float* bias,
                                    int32_t bias_ld, int32_t bias_off, void* stream) {
  return guarded([&] {
    exg::PrefillAttnArgs a{(const exg::bf16*)q, ldq, (const exg::bf16*)kc, (const exg::bf16*)vc, cu_seqlens, slot,
                           pos0, R, max_len, (exg::bf16*)out, ldo, H, dh, max_ctx, scale, (int64_t)T,
                           (int64_t)n_slots * H * max_ctx, causal, bias, bias_ld, bias_off};
    exg::prefill_attention(a, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_decode_attention_paged(const void* q, int64_t ldq, const void* kc, const void* vc, const int32_t* slot,
                                   const int32_t* n_keys, void* out, int64_t ldo, int32_t B, int32_t H, int32_t dh,
                                   int32_t max_ctx, float scale, int32_t split_len, int32_t max_splits, float* partial,
                                   const float* bias, int32_t bias_ld, int32_t bias_off,
                                         const int32_t* page_table, int32_t maxp, void* stream) {
  return guarded([&] {
    if (max_splits > 1 && !partial) throw std::invalid_argument("max_splits > 1 needs a partial buffer");
    exg::DecodeAttnArgs a;
    a.q = (const exg::bf16*)q;
    a.ldq = ldq;
    a.kc = (const exg::bf16*)kc;
    a.vc = (const exg::bf16*)vc;
    a.slot = slot;
    a.n_keys = n_keys;
    a.out = (exg::bf16*)out;
    a.ldo = ldo;
    a.B = B;
    a.H = H;
    a.dh = dh;
    a.max_ctx = max_ctx;
    a.scale = scale;
    a.split_len = split_len;
    a.max_splits = max_splits;
    a.partial = partial;
    a.bias = bias;
    a.bias_ld = bias_ld;
    a.bias_off = bias_off;
    if (!page_table || maxp < 1) throw std::invalid_argument("paged: page_table / maxp");
    if (max_ctx < 64 || max_ctx % 64 != 0 || split_len % max_ctx != 0)
      throw std::invalid_argument("paged: the page length must be a multiple of 64 dividing split_len");
    a.kv = exg::KvMap{page_table, maxp};
    exg::decode_attention(a, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_prefill_attention_paged(const void* q, int64_t ldq, const void* kc, const void* vc,
                                    const int32_t* cu_seqlens, const int32_t* slot, const int32_t* pos0, int32_t R,
                                    int32_t max_len, void* out, int64_t ldo, int32_t H, int32_t dh, int32_t max_ctx,
                                    int32_t n_slots, int32_t T, float scale, int32_t causal, const float* bias,
                                    int32_t bias_ld, int32_t bias_off, const int32_t* page_table, int32_t maxp,
                                          void* stream) {
  return guarded([&] {
    exg::PrefillAttnArgs a{(const exg::bf16*)q, ldq, (const exg::bf16*)kc, (const exg::bf16*)vc, cu_seqlens, slot,
                           pos0, R, max_len, (exg::bf16*)out, ldo, H, dh, max_ctx, scale, (int64_t)T,
                           (int64_t)n_slots * H * max_ctx, causal, bias, bias_ld, bias_off};
    if (!page_table || maxp < 1) throw std::invalid_argument("paged: page_table / maxp");
    if (max_ctx < 64 || max_ctx % 64 != 0) throw std::invalid_argument("paged: the page length must be a multiple of 64");
    a.kv = exg::KvMap{page_table, maxp};
    exg::prefill_attention(a, (cudaStream_t)stream);
    return EXG_OK;
  });
}

exg_status exg_op_argmax(int32_t* out, const float* logits, int64_t ld, int32_t B, int32_t V, int32_t* err_flag,
                         void* stream) {
  return guarded([&] {
    exg::argmax_rows(out, logits, ld, B, V, err_flag, (cudaStream_t)stream);
    return EXG_OK;
  });
}

int64_t exg_op_decode_workspace(int32_t features, int32_t K, int32_t tokens) {
  try {
    return (int64_t)exg::decode_ws_floats(features, K, tokens);
  } catch (...) {
    return -1;
  }
}

}  // extern "C"
