// Host planner: profile-v1 tables, XSimulator (§6) and
// XScheduler (Algorithm 1, with the outer loops of
// PAPER.md:312, 348).  Pure double-precision host code compiled with
// -ffp-contract=off; every expression follows the operation order of the
// written-out readings in DESIGN.md so that results
// are bit-identical on every rank and reproducible from the text.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/exegpt.h"

namespace exg {
namespace plan {

struct Table1D {
  std::vector<double> x, t;
};
struct Table2D {
  std::vector<double> b, c;
  std::vector<std::vector<double>> t;  // t[ib][ic]
};

struct Profile {
  std::vector<int> tps;
  std::map<std::pair<std::string, int>, Table2D> attn;
  std::map<std::pair<std::string, int>, Table1D> rest;
  std::map<int, Table1D> tp_sync;
  Table1D pp_sync;
  bool has_pp = false;
  Table1D head;            // decode head (final norm + LM head + argmax) vs batch
  bool has_head = false;
  Table2D sw;              // encode -> decode switch: cumulative extra time of the first k
  bool has_sw = false;     // decode iterations after an encode phase, [batch][k]
  std::string dumps() const;
  static Profile loads(const std::string& text);
};

struct OutOfHull {};

double interp1(const std::vector<double>& xs, const std::vector<double>& ts, double x);
double interp2(const Table2D& tb, double b, double c);

struct Stage {
  int first_gpu, n_gpus, layer_begin, layer_end;
};
std::vector<Stage> stage_layout(int n_gpus, int t, int c, int n_layers, int first_gpu);
double fill(const std::vector<double>& ts, int M);
double period(const std::vector<double>& ts, int M);

// seqdist
std::vector<double> completion_distribution(const std::vector<double>& pmf_out, int n_d);
double completion_fraction(const std::vector<double>& pu);
double little_fraction(const std::vector<double>& pmf_out, int n_d);
int rra_b_d(int b_e, double f);
int waa_b_d(int b_e, double s_d_mean);
std::vector<double> rra_iteration_batches(int b_d, const std::vector<double>& pu);
double pmf_mean(const std::vector<double>& pmf);

struct Sched {
  int strategy = EXG_RRA;
  int b_e = 0, b_d = 0, b_m = 0, n_d = 0, tp_degree = 1, tp_gpus = 0, n_enc_gpus = 0;
  std::vector<Stage> stages;
  bool valid = true;
};

struct Est {
  double thr = 0, tok = 0, lat = 0;
  bool feasible = true;
};

class Simulator {
 public:
  Simulator(const Profile& p, const exg_model_spec& m, const exg_cluster_spec& cl, std::vector<double> pmf_in,
            std::vector<double> pmf_out, int target_len, bool use_little);
  Sched rra_schedule(int b_e, int n_d, int t, int c);
  Sched waa_schedule(int b_e, int M, int t, int c, int strat = EXG_WAA_C);
  Est simulate(const Sched& s);
  Est simulate_static(int B);
  double layer_enc(int t, double b);
  double layer_dec(int t, double b);
  std::vector<double> stage_times(const std::vector<Stage>& st, bool enc, double b);
  bool mem_ok(const std::vector<Stage>& st, int64_t kv_rows, double ctx);
  // per-GPU model / KV-cache bytes of a schedule (mem_ok's memory model)
  void memory(const Sched& s, std::vector<double>& w, std::vector<double>& kv);

  const Profile& p;
  exg_model_spec m;
  exg_cluster_spec cl;
  std::vector<double> pmf_in, pmf_out;
  int target_len;
  double s_e, s_d, ctx_mean, s_e_rms, s_e_sd, age_mean;
  double kv_ctx_dec;   // decoder KV positions charged per row (slots, or the paged live average)
  int max_in, max_out, n_layers, k_dec;
  bool use_little;

 private:
  std::map<int, std::pair<std::vector<double>, double>> pu_cache_;
  const std::pair<std::vector<double>, double>& pu(int n_d);
  double tp_sync(int t, double bytes);
  double pp_sync(double bytes);
  double layer_bytes() const;
  double emb_bytes() const;
  double kv_bytes_per_token_layer() const;
  int waa_split(int b_e, int b_d, int strat = EXG_WAA_C);
  Est simulate_rra(const Sched& s);
  Est simulate_waa(const Sched& s);
};

struct Perf {
  double latency, thrput;
};
struct BnBResult {
  bool found = false;
  int x1 = 0, x2 = 0;
  Perf perf{0, 0};
  int64_t evals = 0;
};
template <class F>
BnBResult branch_and_bound(int a1, int b1, int a2, int b2, F&& perf_fn, double L_b, double eps_t_frac,
                           double eps_l_frac);

struct Found {
  Sched sched;
  Est est;
  int64_t evals = 0;
};
bool schedule_find(Simulator& S, double L_b, uint32_t mask, const exg_search_opts& o, Found* out);

}  // namespace plan
}  // namespace exg
