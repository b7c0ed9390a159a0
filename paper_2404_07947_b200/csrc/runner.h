// XRunner entry points (see runner.cu).
#pragma once
#include "../../include/exegpt.h"
#include "engine.cuh"

namespace exg {
// RRA schedule on one GPU.
void run_rra(Engine& E, const exg_schedule& s, const exg_request* reqs, int n, int32_t* out_tokens,
             double* out_latency, exg_run_stats* stats, const exg_run_opts* opts);
// last_tok[rslot[k]] = tok[k], k < n (device arrays)
void set_last_tokens(int32_t* last_tok, const int32_t* rslot, const int32_t* tok, int n, cudaStream_t st);
}  // namespace exg
