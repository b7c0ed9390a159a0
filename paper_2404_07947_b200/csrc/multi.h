// Multi-stage schedule execution (see multi.cu).
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <utility>
#include <vector>

#include "../../include/exegpt.h"

namespace exg {

class Engine;
struct Comm;

// Sum the TP partial buffers of a group of engines in rank order and write
// the sum back to every rank.
void sum_tp_parts(const std::vector<Engine*>& ranks, int64_t n, cudaStream_t st);

// Runs multi-GPU layouts (PP, partial TP, WAA).  One MultiCtx per rank; the
// layout's GPUs are split over the ranks of `comm` (see multi.cu).  comm ==
// nullptr: a single rank runs every GPU of the layout on `device`.
class MultiCtx {
 public:
  MultiCtx(const exg_model_spec& spec, int device, std::unique_ptr<Comm> comm = nullptr);
  ~MultiCtx();
  int rank() const;
  int world() const;
  void run(const exg_schedule& s, const exg_request* reqs, int n, int32_t* out_tokens, double* out_latency,
           exg_run_stats* stats, const exg_run_opts* opts);
  // XProfiler's interconnect tables, collective over the
  // ranks: tp_sync[t] = fp32 all-reduce of `bytes` over ranks [0, t) (the
  // transport's TP reduction), pp_sync = one pipeline hop of `bytes` rank 0 ->
  // rank 1 (ping-pong / 2).  Byte grid 1 KB .. 1 GB (x4); median of `reps`.
  // Fills tp_sync / pp_sync (rank 0's measurements are authoritative).
  void profile_comm(const std::vector<int>& tps, int reps, std::map<int, std::pair<std::vector<double>, std::vector<double>>>* tp,
                    std::vector<double>* pp_x, std::vector<double>* pp_t);
  struct Impl;

 private:
  Impl* p_;
};

}  // namespace exg
