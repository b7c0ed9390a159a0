// Host planner implementation (see planner.h).  Operation order mirrors the
// readings written out in DESIGN.md; compile with -ffp-contract=off.
#include "planner.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>
#include <queue>
#include <sstream>
#include <stdexcept>

namespace exg {
namespace plan {

static const double INF = std::numeric_limits<double>::infinity();

static constexpr double Z99 = 2.3263478740408408;   // standard normal 0.99 quantile (RRA latency buffer)

// ---------------------------------------------------------------- profile --
static std::string g17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

std::string Profile::dumps() const {
  std::ostringstream o;
  o << "profile-v1\n" << "tp " << tps.size();
  for (int t : tps) o << " " << t;
  o << "\n";
  for (const auto& kv : attn) {
    const Table2D& tb = kv.second;
    o << "attn " << kv.first.first << " " << kv.first.second << " " << tb.b.size() << " " << tb.c.size() << "\n";
    for (size_t i = 0; i < tb.b.size(); ++i) o << (i ? " " : "") << g17(tb.b[i]);
    o << "\n";
    for (size_t i = 0; i < tb.c.size(); ++i) o << (i ? " " : "") << g17(tb.c[i]);
    o << "\n";
    bool first = true;
    for (const auto& row : tb.t)
      for (double v : row) {
        o << (first ? "" : " ") << g17(v);
        first = false;
      }
    o << "\n";
  }
  for (const auto& kv : rest) {
    const Table1D& tb = kv.second;
    o << "rest " << kv.first.first << " " << kv.first.second << " " << tb.x.size() << "\n";
    for (size_t i = 0; i < tb.x.size(); ++i) o << (i ? " " : "") << g17(tb.x[i]);
    o << "\n";
    for (size_t i = 0; i < tb.t.size(); ++i) o << (i ? " " : "") << g17(tb.t[i]);
    o << "\n";
  }
  for (const auto& kv : tp_sync) {
    o << "tp_sync " << kv.first << " " << kv.second.x.size() << "\n";
    for (size_t i = 0; i < kv.second.x.size(); ++i) o << (i ? " " : "") << g17(kv.second.x[i]);
    o << "\n";
    for (size_t i = 0; i < kv.second.t.size(); ++i) o << (i ? " " : "") << g17(kv.second.t[i]);
    o << "\n";
  }
  if (has_pp) {
    o << "pp_sync " << pp_sync.x.size() << "\n";
    for (size_t i = 0; i < pp_sync.x.size(); ++i) o << (i ? " " : "") << g17(pp_sync.x[i]);
    o << "\n";
    for (size_t i = 0; i < pp_sync.t.size(); ++i) o << (i ? " " : "") << g17(pp_sync.t[i]);
    o << "\n";
  }
  if (has_head) {
    o << "head " << head.x.size() << "\n";
    for (size_t i = 0; i < head.x.size(); ++i) o << (i ? " " : "") << g17(head.x[i]);
    o << "\n";
    for (size_t i = 0; i < head.t.size(); ++i) o << (i ? " " : "") << g17(head.t[i]);
    o << "\n";
  }
  if (has_sw) {
    o << "switch " << sw.b.size() << " " << sw.c.size() << "\n";
    for (size_t i = 0; i < sw.b.size(); ++i) o << (i ? " " : "") << g17(sw.b[i]);
    o << "\n";
    for (size_t i = 0; i < sw.c.size(); ++i) o << (i ? " " : "") << g17(sw.c[i]);
    o << "\n";
    bool first = true;
    for (const auto& row : sw.t)
      for (double v : row) {
        o << (first ? "" : " ") << g17(v);
        first = false;
      }
    o << "\n";
  }
  o << "end\n";
  return o.str();
}

Profile Profile::loads(const std::string& text) {
  std::istringstream in(text);
  std::string tok;
  auto nxt = [&]() {
    if (!(in >> tok)) throw std::invalid_argument("profile-v1: unexpected end of file");
    return tok;
  };
  auto num = [&]() {
    std::string s = nxt();
    char* end = nullptr;
    double v = std::strtod(s.c_str(), &end);
    if (end == s.c_str() || *end) throw std::invalid_argument("profile-v1: bad number '" + s + "'");
    return v;
  };
  auto integer = [&]() { return (int)std::strtol(nxt().c_str(), nullptr, 10); };
  if (nxt() != "profile-v1") throw std::invalid_argument("not a profile-v1 file");
  if (nxt() != "tp") throw std::invalid_argument("profile-v1: expected 'tp'");
  Profile p;
  int n = integer();
  for (int i = 0; i < n; ++i) p.tps.push_back(integer());
  while (true) {
    std::string kw = nxt();
    if (kw == "end") break;
    if (kw == "attn") {
      std::string ph = nxt();
      int tp = integer(), nb = integer(), nc = integer();
      Table2D tb;
      for (int i = 0; i < nb; ++i) tb.b.push_back(num());
      for (int i = 0; i < nc; ++i) tb.c.push_back(num());
      tb.t.assign(nb, std::vector<double>(nc));
      for (int i = 0; i < nb; ++i)
        for (int j = 0; j < nc; ++j) tb.t[i][j] = num();
      p.attn[{ph, tp}] = tb;
    } else if (kw == "rest") {
      std::string ph = nxt();
      int tp = integer(), m = integer();
      Table1D tb;
      for (int i = 0; i < m; ++i) tb.x.push_back(num());
      for (int i = 0; i < m; ++i) tb.t.push_back(num());
      p.rest[{ph, tp}] = tb;
    } else if (kw == "tp_sync") {
      int tp = integer(), m = integer();
      Table1D tb;
      for (int i = 0; i < m; ++i) tb.x.push_back(num());
      for (int i = 0; i < m; ++i) tb.t.push_back(num());
      p.tp_sync[tp] = tb;
    } else if (kw == "pp_sync") {
      int m = integer();
      for (int i = 0; i < m; ++i) p.pp_sync.x.push_back(num());
      for (int i = 0; i < m; ++i) p.pp_sync.t.push_back(num());
      p.has_pp = true;
    } else if (kw == "head") {
      int m = integer();
      for (int i = 0; i < m; ++i) p.head.x.push_back(num());
      for (int i = 0; i < m; ++i) p.head.t.push_back(num());
      p.has_head = true;
    } else if (kw == "switch") {
      int nb = integer(), nk = integer();
      for (int i = 0; i < nb; ++i) p.sw.b.push_back(num());
      for (int i = 0; i < nk; ++i) p.sw.c.push_back(num());
      p.sw.t.assign(nb, std::vector<double>(nk));
      for (int i = 0; i < nb; ++i)
        for (int j = 0; j < nk; ++j) p.sw.t[i][j] = num();
      p.has_sw = true;
    } else {
      throw std::invalid_argument("profile-v1: bad keyword '" + kw + "'");
    }
  }
  return p;
}

// ------------------------------------------------------------ interpolation --
double interp1(const std::vector<double>& xs, const std::vector<double>& ts, double x) {
  const size_t n = xs.size();
  if (x <= xs[0]) return ts[0];
  for (size_t i = 1; i < n; ++i) {
    if (x == xs[i]) return ts[i];
    if (x < xs[i]) {
      const double x0 = xs[i - 1], x1 = xs[i], t0 = ts[i - 1], t1 = ts[i];
      return t0 + (x - x0) * (t1 - t0) / (x1 - x0);
    }
  }
  throw OutOfHull{};
}

double interp2(const Table2D& tb, double b, double c) {
  const std::vector<double>& bs = tb.b;
  if (b <= bs[0]) return interp1(tb.c, tb.t[0], c);
  for (size_t i = 1; i < bs.size(); ++i) {
    if (b == bs[i]) return interp1(tb.c, tb.t[i], c);
    if (b < bs[i]) {
      const double f0 = interp1(tb.c, tb.t[i - 1], c);
      const double f1 = interp1(tb.c, tb.t[i], c);
      return f0 + (b - bs[i - 1]) * (f1 - f0) / (bs[i] - bs[i - 1]);
    }
  }
  throw OutOfHull{};
}

// ------------------------------------------------------------- pipelines --
std::vector<Stage> stage_layout(int n_gpus, int t, int c, int n_layers, int first_gpu) {
  std::vector<int> g;
  int rest = n_gpus;
  if (t > 1) {
    for (int k = 0; k < c / t; ++k) g.push_back(t);
    rest = n_gpus - c;
  }
  for (int k = 0; k < rest; ++k) g.push_back(1);
  std::vector<int> base;
  int sum = 0;
  for (int gk : g) {
    base.push_back(n_layers * gk / n_gpus);
    sum += base.back();
  }
  const int rem = n_layers - sum;
  for (int k = 0; k < rem; ++k) base[k] += 1;
  std::vector<Stage> st;
  int gpu = first_gpu, layer = 0;
  for (size_t k = 0; k < g.size(); ++k) {
    st.push_back(Stage{gpu, g[k], layer, layer + base[k]});
    gpu += g[k];
    layer += base[k];
  }
  return st;
}

double fill(const std::vector<double>& ts, int M) {
  double s = 0.0, m = 0.0;
  for (double v : ts) {
    s += v;
    m = std::max(m, v);
  }
  return s + (M - 1) * m;
}

double period(const std::vector<double>& ts, int M) {
  double s = 0.0, m = 0.0;
  for (double v : ts) {
    s += v;
    m = std::max(m, v);
  }
  return std::max(s, M * m);
}

// --------------------------------------------------------------- seqdist --
std::vector<double> completion_distribution(const std::vector<double>& pmf_out, int n_d) {
  std::vector<double> pu(n_d, 0.0);
  for (int k = 1; k <= (int)pmf_out.size(); ++k) {
    const double p = pmf_out[k - 1];
    if (k <= n_d) {
      pu[k - 1] += p;
    } else {
      const int q = (k + n_d - 1) / n_d;
      pu[(k - 1) % n_d] += p * (1.0 / q);
    }
  }
  return pu;
}

double completion_fraction(const std::vector<double>& pu) {
  double f = 0.0;
  for (double p : pu) f += p;
  return f;
}

double little_fraction(const std::vector<double>& pmf_out, int n_d) {
  double e = 0.0;
  for (int k = 1; k <= (int)pmf_out.size(); ++k) e += pmf_out[k - 1] * (double)((k + n_d - 1) / n_d);
  return 1.0 / e;
}

int rra_b_d(int b_e, double f) { return std::max(b_e, (int)std::floor(b_e / f + 0.5)); }
int waa_b_d(int b_e, double s_d_mean) { return b_e * (int)std::floor(s_d_mean + 0.5); }

std::vector<double> rra_iteration_batches(int b_d, const std::vector<double>& pu) {
  std::vector<double> out;
  double acc = 0.0;
  for (size_t u = 0; u < pu.size(); ++u) {
    out.push_back(b_d * (1.0 - acc));
    acc += pu[u];
  }
  return out;
}

double pmf_mean(const std::vector<double>& pmf) {
  double m = 0.0;
  for (int k = 1; k <= (int)pmf.size(); ++k) m += k * pmf[k - 1];
  return m;
}

// ------------------------------------------------------------- simulator --
Simulator::Simulator(const Profile& p_, const exg_model_spec& m_, const exg_cluster_spec& cl_,
                     std::vector<double> pin, std::vector<double> pout, int target, bool little)
    : p(p_), m(m_), cl(cl_), pmf_in(std::move(pin)), pmf_out(std::move(pout)), target_len(target),
      use_little(little) {
  s_e = pmf_mean(pmf_in);
  s_d = pmf_mean(pmf_out);
  max_in = (int)pmf_in.size();
  max_out = (int)pmf_out.size();
  // decode-attention context: the row-iteration mean age E[S(S+1)] / (2 E[S])
  // on top of the input (oracle/simulator.py ctx_mean)
  {
    double m2o = 0.0;
    for (size_t k = 1; k <= pmf_out.size(); ++k) m2o += (double)k * (double)k * pmf_out[k - 1];
    age_mean = (m2o + s_d) / (2.0 * s_d);
  }
  ctx_mean = s_e + age_mean - (m.arch == EXG_ARCH_T5 ? 0.0 : 1.0);
  // RMS input length: the encode-attention lookup length (its per-request
  // cost grows as n^2, so b requests of this length cost sum_i n_i^2)
  {
    double m2 = 0.0;
    for (size_t k = 1; k <= pmf_in.size(); ++k) m2 += (double)k * (double)k * pmf_in[k - 1];
    s_e_rms = std::sqrt(m2);
    const double var = m2 - s_e * s_e;   // input-length variance
    s_e_sd = std::sqrt(var > 0.0 ? var : 0.0);
  }
  n_layers = m.n_dec_layers;
  k_dec = m.arch == EXG_ARCH_T5 ? 3 : 2;
  // decoder KV context per row (oracle/simulator.py kv_ctx_dec): slots of
  // max_in + max_out, or with paged KV the row-iteration average of the live
  // positions S_E - 1 + E[S(S+1)] / (2 E[S]) plus 3P/2
  kv_ctx_dec = (double)(max_in + max_out);
  if (cl.kv_page > 0 && m.arch != EXG_ARCH_T5) {
    const double live = s_e - 1.0 + age_mean;
    kv_ctx_dec = std::min(live + 1.5 * (double)cl.kv_page, (double)(max_in + max_out));
  }
}

double Simulator::tp_sync(int t, double bytes) {
  if (t <= 1) return 0.0;
  auto it = p.tp_sync.find(t);
  if (it == p.tp_sync.end()) throw OutOfHull{};
  return interp1(it->second.x, it->second.t, bytes);
}

double Simulator::pp_sync(double bytes) {
  if (!p.has_pp) throw OutOfHull{};
  return interp1(p.pp_sync.x, p.pp_sync.t, bytes);
}

double Simulator::layer_enc(int t, double b) {
  const double toks = b * s_e;
  auto ia = p.attn.find({"enc", t});
  auto ir = p.rest.find({"enc", t});
  if (ia == p.attn.end() || ir == p.rest.end()) throw OutOfHull{};
  const double a = interp2(ia->second, b, s_e_rms);
  const double r = interp1(ir->second.x, ir->second.t, toks);
  return a + r + 2 * tp_sync(t, toks * m.d_model * 4.0);
}

double Simulator::layer_dec(int t, double b) {
  auto ia = p.attn.find({"dec", t});
  auto ir = p.rest.find({"dec", t});
  if (ia == p.attn.end() || ir == p.rest.end()) throw OutOfHull{};
  const double a = interp2(ia->second, b, ctx_mean);
  const double r = interp1(ir->second.x, ir->second.t, b);
  return a + r + k_dec * tp_sync(t, b * m.d_model * 4.0);
}

std::vector<double> Simulator::stage_times(const std::vector<Stage>& st, bool enc, double b) {
  std::vector<double> out;
  const int P = (int)st.size();
  for (int k = 0; k < P; ++k) {
    const Stage& s = st[k];
    const double per = enc ? layer_enc(s.n_gpus, b) : layer_dec(s.n_gpus, b);
    double v = (s.layer_end - s.layer_begin) * per;
    if (k < P - 1) {
      const double toks = enc ? b * s_e : b;
      v += pp_sync(toks * m.d_model * 2.0);
    }
    // the decode head runs once per iteration on the last stage
    if (!enc && k == P - 1 && p.has_head) v += interp1(p.head.x, p.head.t, b);
    out.push_back(v);
  }
  return out;
}

const std::pair<std::vector<double>, double>& Simulator::pu(int n_d) {
  auto it = pu_cache_.find(n_d);
  if (it != pu_cache_.end()) return it->second;
  std::vector<double> d = completion_distribution(pmf_out, n_d);
  const double f = use_little ? little_fraction(pmf_out, n_d) : completion_fraction(d);
  return pu_cache_[n_d] = {d, f};
}

double Simulator::layer_bytes() const {
  const int64_t d = m.d_model, inner = (int64_t)m.n_heads * m.d_head, ff = m.d_ff;
  const int64_t params = d * 3 * inner + 3 * inner + inner * d + d + d * ff + ff + ff * d + d + 4 * d;
  return params * 2.0;
}
double Simulator::emb_bytes() const {
  return ((int64_t)m.vocab * m.d_model + (int64_t)m.max_pos * m.d_model + 2 * (int64_t)m.d_model) * 2.0;
}
double Simulator::kv_bytes_per_token_layer() const { return 2.0 * ((int64_t)m.n_heads * m.d_head) * 2.0; }

bool Simulator::mem_ok(const std::vector<Stage>& st, int64_t kv_rows, double ctx) {
  const int P = (int)st.size();
  for (int k = 0; k < P; ++k) {
    const Stage& s = st[k];
    const int64_t nl = s.layer_end - s.layer_begin;
    double b = nl * layer_bytes() / s.n_gpus;
    if (k == 0 || k == P - 1) b += emb_bytes();
    b += (double)kv_rows * ctx * (double)nl * kv_bytes_per_token_layer() / s.n_gpus;
    b += (double)cl.workspace_bytes;
    if (b > (double)cl.mem_per_gpu_bytes) return false;
  }
  return true;
}

// Memory-overhead accounting: the weight shard (+ the
// embeddings on the first / last stage of each side) and the KV slots
// (kv_rows x ctx for the stage's layers) each GPU holds -- mem_ok's model,
// summed per GPU.  RRA / STATIC: B_D (B) rows of max_in + max_out; WAA:
// encoder stages B_E rows of max_in, decoder stages B_D rows of max_in +
// max_out.
void Simulator::memory(const Sched& s, std::vector<double>& w, std::vector<double>& kv) {
  w.assign(cl.n_gpus, 0.0);
  kv.assign(cl.n_gpus, 0.0);
  auto account = [&](const std::vector<Stage>& st, int64_t rows, double ctx) {
    const int P = (int)st.size();
    for (int k = 0; k < P; ++k) {
      const Stage& g = st[k];
      const int64_t nl = g.layer_end - g.layer_begin;
      double b = nl * layer_bytes() / g.n_gpus;
      if (k == 0 || k == P - 1) b += emb_bytes();
      const double c = (double)rows * ctx * (double)nl * kv_bytes_per_token_layer() / g.n_gpus;
      for (int i = g.first_gpu; i < std::min(g.first_gpu + g.n_gpus, cl.n_gpus); ++i) {
        w[i] += b;
        kv[i] += c;
      }
    }
  };
  if (s.strategy == EXG_STATIC) {
    account(stage_layout(cl.n_gpus, 1, 0, n_layers, 0), s.b_e, (int64_t)max_in + max_out);
  } else if (s.strategy == EXG_RRA) {
    account(s.stages, s.b_d, kv_ctx_dec);
  } else {
    std::vector<Stage> enc, dec;
    for (const Stage& st : s.stages) (st.first_gpu < s.n_enc_gpus ? enc : dec).push_back(st);
    account(enc, s.b_e, max_in);
    account(dec, s.b_d, kv_ctx_dec);
  }
}

Sched Simulator::rra_schedule(int b_e, int n_d, int t, int c) {
  Sched s;
  s.strategy = EXG_RRA;
  s.b_e = b_e;
  s.n_d = n_d;
  s.b_d = rra_b_d(b_e, pu(n_d).second);
  s.tp_degree = t;
  s.tp_gpus = c;
  s.stages = stage_layout(cl.n_gpus, t, c, n_layers, 0);
  return s;
}

// WAA-C: compute-proportional; WAA-M: equal per-GPU memory
// (mirror of oracle/simulator.py waa_split, same expression order)
int Simulator::waa_split(int b_e, int b_d, int strat) {
  const int N = cl.n_gpus;
  int n_enc;
  if (strat == EXG_WAA_M) {
    const double kv = kv_bytes_per_token_layer();
    const double W = n_layers * layer_bytes() + emb_bytes();
    const double mem_e = W + (double)((int64_t)b_e * max_in * n_layers) * kv;
    const double mem_d = W + ((double)b_d * kv_ctx_dec * (double)n_layers) * kv;
    n_enc = (int)std::floor(N * mem_e / (mem_e + mem_d) + 0.5);
  } else {
    const double C_E = n_layers * layer_enc(1, b_e);
    const double C_D = n_layers * layer_dec(1, b_d);
    n_enc = (int)std::floor(N * C_E / (C_E + C_D) + 0.5);
  }
  return std::min(std::max(n_enc, 1), N - 1);
}

Sched Simulator::waa_schedule(int b_e, int M, int t, int c, int strat) {
  Sched s;
  s.valid = false;
  if (cl.n_gpus < 2) return s;
  const int b_d = waa_b_d(b_e, s_d);
  M = std::min(M, b_d);
  const int b_m = (b_d + M - 1) / M;
  int n_enc;
  try {
    n_enc = waa_split(b_e, b_d, strat);
  } catch (const OutOfHull&) {
    return s;
  }
  const int n_dec = cl.n_gpus - n_enc;
  if (c > n_dec) return s;
  s.valid = true;
  s.strategy = strat;
  s.b_e = b_e;
  s.b_d = b_d;
  s.b_m = b_m;
  s.tp_degree = t;
  s.tp_gpus = c;
  s.n_enc_gpus = n_enc;
  s.stages = stage_layout(n_enc, 1, 0, n_layers, 0);
  std::vector<Stage> dec = stage_layout(n_dec, t, c, n_layers, n_enc);
  s.stages.insert(s.stages.end(), dec.begin(), dec.end());
  return s;
}

Est Simulator::simulate_rra(const Sched& s) {
  Est bad{0.0, 0.0, INF, false};
  if (!mem_ok(s.stages, s.b_d, kv_ctx_dec)) return bad;
  const auto& pf = pu(s.n_d);
  const int P = (int)s.stages.size();
  double T_encph;
  std::vector<double> Pi, Fu;
  try {
    std::vector<double> t_enc = stage_times(s.stages, true, (double)s.b_e / P);
    T_encph = fill(t_enc, P);
    std::vector<double> bu = rra_iteration_batches(s.b_d, pf.first);
    for (int u = 0; u < s.n_d; ++u) {
      std::vector<double> tu = stage_times(s.stages, false, bu[u] / P);
      if (u == 0 && p.has_sw) {
        // the phase's decode iterations follow an encode phase: the clock
        // recovers from the power cap over the first few of them; their
        // cumulative extra time (profile table `switch` at k = min(N_D, k_max))
        // is charged to the first iteration, each stage its layer share
        const double w = interp2(p.sw, bu[0] / P, std::min((double)s.n_d, p.sw.c.back()));
        for (int k = 0; k < P; ++k)
          tu[k] = tu[k] + w * (double)(s.stages[k].layer_end - s.stages[k].layer_begin) / n_layers;
      }
      Pi.push_back(period(tu, P));
      Fu.push_back(fill(tu, P));
    }
  } catch (const OutOfHull&) {
    return bad;
  }
  double T_decph = 0.0;
  for (int u = 0; u < s.n_d - 1; ++u) T_decph += Pi[u];
  T_decph += Fu[s.n_d - 1];
  const double T_cyc = T_encph + T_decph;
  const double thr = s.b_e / T_cyc;
  const int S = target_len;
  const int q = (S + s.n_d - 1) / s.n_d;
  const int r = 1 + (S - 1) % s.n_d;
  double lat = (q - 1) * T_cyc + T_encph;
  for (int u = 0; u < r - 1; ++u) lat += Pi[u];
  lat += Fu[r - 1];
  // buffer time: the 99th-percentile excess of the encoder
  // workload over the query's q encode phases, z99 sqrt(q B_E) sigma_in
  // tokens spread over the q phases, at the profile's encode cost
  if (s_e_sd > 0.0) {
    const double db = Z99 * s_e_sd * std::sqrt((double)(q * s.b_e)) / (q * s_e);
    double T_buf;
    try {
      T_buf = fill(stage_times(s.stages, true, (s.b_e + db) / P), P);
    } catch (const OutOfHull&) {
      return bad;
    }
    lat += q * (T_buf - T_encph);
  }
  return Est{thr, thr * s_d, lat, true};
}

Est Simulator::simulate_waa(const Sched& s) {
  Est bad{0.0, 0.0, INF, false};
  std::vector<Stage> enc, dec;
  for (const Stage& st : s.stages) (st.first_gpu < s.n_enc_gpus ? enc : dec).push_back(st);
  if (!(mem_ok(enc, s.b_e, max_in) && mem_ok(dec, s.b_d, kv_ctx_dec))) return bad;
  const int M = (s.b_d + s.b_m - 1) / s.b_m;
  std::vector<double> te, td;
  double handoff;
  try {
    te = stage_times(enc, true, (double)s.b_e);
    td = stage_times(dec, false, (double)s.b_m);
    handoff = pp_sync(s.b_e * s_e * n_layers * kv_bytes_per_token_layer());
  } catch (const OutOfHull&) {
    return bad;
  }
  double T_E = 0.0, T_trav = 0.0;
  for (double v : te) {
    T_E = std::max(T_E, v);
    T_trav += v;
  }
  const double T_D = period(td, M);
  const double thr = s.b_e / std::max(T_E, T_D);
  const double lat = T_trav + handoff + T_E + (target_len - 1) * T_D + fill(td, M);
  return Est{thr, thr * s_d, lat, true};
}

Est Simulator::simulate_static(int B) {
  Est bad{0.0, 0.0, INF, false};
  const std::vector<Stage> st = stage_layout(cl.n_gpus, 1, 0, n_layers, 0);
  if (!mem_ok(st, B, (int64_t)max_in + max_out)) return bad;
  double lat;
  try {
    const std::vector<double> t_enc = stage_times(st, true, (double)B);
    const std::vector<double> t_dec = stage_times(st, false, (double)B);
    lat = fill(t_enc, 1) + max_out * fill(t_dec, 1);
    if (p.has_sw) lat += interp2(p.sw, (double)B, std::min((double)max_out, p.sw.c.back()));
  } catch (const OutOfHull&) {
    return bad;
  }
  const double thr = B / lat;
  return Est{thr, thr * s_d, lat, true};
}

Est Simulator::simulate(const Sched& s) {
  if (!s.valid) return Est{0.0, 0.0, INF, false};
  if (s.strategy == EXG_STATIC) return simulate_static(s.b_e);
  return s.strategy == EXG_RRA ? simulate_rra(s) : simulate_waa(s);
}

// ------------------------------------------------------------ Algorithm 1 --
namespace {
struct Block {
  int a1, a2, b1, b2;
  Perf lowr, upp;
};
struct HeapItem {
  double key;  // lowr.thrput
  int64_t seq;
  Block blk;
};
struct HeapCmp {
  bool operator()(const HeapItem& x, const HeapItem& y) const {
    // max-heap on key; ties -> earliest insertion first
    if (x.key != y.key) return x.key < y.key;
    return x.seq > y.seq;
  }
};
}  // namespace

template <class F>
BnBResult branch_and_bound(int a1, int b1, int a2, int b2, F&& perf_fn, double L_b, double eps_t_frac,
                           double eps_l_frac) {
  std::map<std::pair<int, int>, Perf> memo;
  auto perf = [&](int x1, int x2) -> Perf {
    auto it = memo.find({x1, x2});
    if (it != memo.end()) return it->second;
    Perf p = perf_fn(x1, x2);
    memo[{x1, x2}] = p;
    return p;
  };
  BnBResult res;
  const double eps_l = (L_b != INF) ? eps_l_frac * L_b : INF;
  const Perf lowr = perf(a1, a2);
  if (!(lowr.latency < L_b)) {
    res.evals = (int64_t)memo.size();
    return res;
  }
  const Perf upp = perf(b1, b2);
  if (upp.latency < L_b) {
    res.found = true;
    res.x1 = b1;
    res.x2 = b2;
    res.perf = upp;
    res.evals = (int64_t)memo.size();
    return res;
  }
  double T_star = lowr.thrput;
  int cx1 = a1, cx2 = a2;
  std::vector<HeapItem> heap;
  HeapCmp cmp;
  int64_t seq = 0;
  heap.push_back(HeapItem{lowr.thrput, seq, Block{a1, a2, b1, b2, lowr, upp}});
  std::push_heap(heap.begin(), heap.end(), cmp);
  while (!heap.empty()) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    const Block B = heap.back().blk;
    heap.pop_back();
    if (B.a1 == B.b1 && B.a2 == B.b2) continue;
    int axis;
    if (B.a1 == B.b1) {
      axis = 2;
    } else if (B.a2 == B.b2) {
      axis = 1;
    } else {
      const Perf p_tl = perf(B.a1, B.b2);
      const Perf p_br = perf(B.b1, B.a2);
      const bool tl_ok = p_tl.latency < L_b, br_ok = p_br.latency < L_b;
      if (tl_ok && (!br_ok || p_tl.thrput >= p_br.thrput))
        axis = 1;
      else if (br_ok)
        axis = 2;
      else
        axis = (B.b1 - B.a1) >= (B.b2 - B.a2) ? 1 : 2;
    }
    int kids[2][4];
    if (axis == 1) {
      const int mid = (int)std::floor((B.a1 + B.b1) / 2.0);
      int k0[4] = {B.a1, B.a2, mid, B.b2}, k1[4] = {mid + 1, B.a2, B.b1, B.b2};
      std::copy(k0, k0 + 4, kids[0]);
      std::copy(k1, k1 + 4, kids[1]);
    } else {
      const int mid = (int)std::floor((B.a2 + B.b2) / 2.0);
      int k0[4] = {B.a1, B.a2, B.b1, mid}, k1[4] = {B.a1, mid + 1, B.b1, B.b2};
      std::copy(k0, k0 + 4, kids[0]);
      std::copy(k1, k1 + 4, kids[1]);
    }
    bool have_best = false;
    Perf best{0, 0};
    int bx1 = 0, bx2 = 0;
    for (int k = 0; k < 2; ++k) {
      const int ka1 = kids[k][0], ka2 = kids[k][1], kb1 = kids[k][2], kb2 = kids[k][3];
      const Perf kupp = perf(kb1, kb2);
      const Perf klowr = perf(ka1, ka2);
      if (kupp.latency < L_b) {
        if (!have_best || kupp.thrput > best.thrput) {
          have_best = true;
          best = kupp;
          bx1 = kb1;
          bx2 = kb2;
        }
      } else if (klowr.latency < L_b + eps_l) {
        ++seq;
        heap.push_back(HeapItem{klowr.thrput, seq, Block{ka1, ka2, kb1, kb2, klowr, kupp}});
        std::push_heap(heap.begin(), heap.end(), cmp);
      }
    }
    if (have_best && best.thrput > T_star) {
      T_star = best.thrput;
      cx1 = bx1;
      cx2 = bx2;
      const double eps_t = eps_t_frac * T_star;
      std::vector<HeapItem> kept;
      for (const HeapItem& h : heap)
        if (!(h.blk.upp.thrput + eps_t < T_star)) kept.push_back(h);
      heap.swap(kept);
      std::make_heap(heap.begin(), heap.end(), cmp);
    }
  }
  res.found = true;
  res.x1 = cx1;
  res.x2 = cx2;
  res.perf = perf(cx1, cx2);
  res.evals = (int64_t)memo.size();
  return res;
}

static Perf perf_of(const Est& e) {
  if (!e.feasible) return Perf{INF, INF};
  return Perf{e.lat, e.thr};
}

bool schedule_find(Simulator& S, double L_b, uint32_t mask, const exg_search_opts& o, Found* out) {
  const int N = S.cl.n_gpus, H = S.m.n_heads;
  const int n_d_max = o.n_d_max > 0 ? o.n_d_max : S.max_out;
  bool have = false;
  // key: (-thr, lat, strat, t, c, x1, x2)
  double k_thr = 0, k_lat = 0;
  int k_rest[5] = {0, 0, 0, 0, 0};
  int64_t total_evals = 0;
  const int strats[3] = {EXG_RRA, EXG_WAA_C, EXG_WAA_M};
  for (int strat : strats) {
    if (!(mask & (uint32_t)strat)) continue;
    if (strat != EXG_RRA && N < 2) continue;
    for (int t : {1, 2, 4, 8}) {
      if (t > N || H % t != 0) continue;
      if (o.tp_degree_only > 0 && t != o.tp_degree_only) continue;
      std::vector<int> cs;
      if (t == 1)
        cs.push_back(0);
      else
        for (int c = t; c <= N; c += t) cs.push_back(c);
      for (int c : cs) {
        auto mk = [&](int x1, int x2) {
          return strat == EXG_RRA ? S.rra_schedule(x1, n_d_max + 1 - x2, t, c)
                                  : S.waa_schedule(x1, o.m_max + 1 - x2, t, c, strat);
        };
        // x2 ranges: RRA searches N_D inside Algorithm 1; for WAA the
        // micro-batch count is an outer variable like the TP degree
        // -- it is not monotone (DESIGN.md reading)
        std::vector<std::pair<int, int>> x2r;
        if (strat == EXG_RRA)
          x2r.push_back({1, n_d_max});
        else
          for (int x2 = 1; x2 <= o.m_max; ++x2) x2r.push_back({x2, x2});
        auto perf_fn = [&](int x1, int x2) -> Perf {
          Sched s = mk(x1, x2);
          if (!s.valid) return Perf{INF, INF};
          return perf_of(S.simulate(s));
        };
        for (const auto& ab2 : x2r) {
          const int a2 = ab2.first, b2 = ab2.second;
          int b1 = 0;
          for (int be = 1; be <= o.b_e_max; ++be) {
            if (std::isfinite(perf_fn(be, a2).latency))
              b1 = be;
            else
              break;
          }
          if (b1 == 0) continue;
          BnBResult r = branch_and_bound(1, b1, a2, b2, perf_fn, L_b, o.eps_t_frac, o.eps_l_frac);
          total_evals += r.evals + b1;
          if (!r.found) continue;
          Sched sch = mk(r.x1, r.x2);
          Est est = S.simulate(sch);
          const double nthr = -est.thr;
          const int rest[5] = {strat, t, c, r.x1, r.x2};
          bool better = !have;
          if (have) {
            if (nthr != k_thr)
              better = nthr < k_thr;
            else if (est.lat != k_lat)
              better = est.lat < k_lat;
            else
              better = std::lexicographical_compare(rest, rest + 5, k_rest, k_rest + 5);
          }
          if (better) {
            have = true;
            k_thr = nthr;
            k_lat = est.lat;
            std::copy(rest, rest + 5, k_rest);
            out->sched = sch;
            out->est = est;
          }
        }
      }
    }
  }
  out->evals = total_evals;
  return have;
}

}  // namespace plan
}  // namespace exg
