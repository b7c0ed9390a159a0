/*
 * exegpt.h -- C-ABI of libexegpt.so, a B200-native (sm_100a) runner for the
 * decoupled-inference computation that ExeGPT (arXiv 2404.07947) schedules.
 *
 * The calls follow the paper's problem statement (§5):
 * profile the cost model (XProfiler), pick the max-
 * throughput schedule under a latency bound for the given input/output
 * length distributions (XSimulator + XScheduler, §5-§6,
 * host code), and run that schedule on a request batch (XRunner,
 * PAPER.md:171-176) returning greedy tokens and per-request latencies.
 *
 * Conventions
 *  - Plain C types only; no torch/CUDA types cross this boundary.
 *  - Every function returns an exg_status and never throws or exits; on an
 *    error exg_last_error() (thread-local) holds a message and output
 *    buffers are unspecified.
 *  - The caller owns every input array and every output buffer; the library
 *    copies inputs before returning.  Opaque objects are library-owned and
 *    released with their *_free / exg_destroy.
 *  - Host pointers unless stated otherwise.
 */
#ifndef EXEGPT_H
#define EXEGPT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EXG_ABI_VERSION 5

typedef enum {
  EXG_OK = 0,
  EXG_E_INPUT = 1,       /* invalid argument (SPEC.md:562 exit code 1)            */
  EXG_E_INFEASIBLE = 2,  /* no schedule meets L_B / memory / WAA on < 2 GPUs (2)  */
  EXG_E_CUDA = 3,
  EXG_E_NCCL = 4,
  EXG_E_OOM = 5,
  EXG_E_INTERNAL = 6     /* e.g. a NaN logit                  */
} exg_status;

typedef enum { EXG_ARCH_OPT = 0, EXG_ARCH_GPT3 = 1, EXG_ARCH_T5 = 2 } exg_arch; /* tiny = GPT3-style */
typedef enum { EXG_BF16 = 0, EXG_FP32 = 1 } exg_dtype;
/* bitmask of scheduling policies.  EXG_STATIC is the
 * FasterTransformer-style static batch (fixed batch, no early
 * termination): exg_simulate estimates it to derive latency bounds by the
 * paper's recipe, and exg_run executes it on one GPU as the
 * in-runner baseline; b_e = the static batch size.
 * It is never chosen by exg_schedule_find. */
typedef enum { EXG_RRA = 1, EXG_WAA_C = 2, EXG_WAA_M = 4, EXG_STATIC = 8 } exg_strategy;

/* Model shape (Table 1) plus the weight seed of the
 * counter-hash generator.  n_enc_layers = 0 for
 * decoder-only models. */
typedef struct {
  exg_arch arch;
  int32_t n_enc_layers, n_dec_layers, d_model, n_heads, d_head, d_ff, vocab, max_pos;
  exg_dtype dtype;
  uint64_t weight_seed;
} exg_model_spec;

/* Cluster: GPUs used and usable bytes per GPU (memory check);
 * workspace_bytes is reserved per GPU for activations / scratch.  kv_page > 0:
 * the runner pages the decoder KV cache (exg_run_opts.kv_page) and the
 * simulator charges each decoder row the row-iteration average of its live
 * positions, S_E - 1 + E[S(S+1)] / (2 E[S]) + 3 kv_page / 2, instead of
 * max_in + max_out (decoder-only models; reading of PAPER.md:545). */
typedef struct {
  int32_t n_gpus;
  int64_t mem_per_gpu_bytes;
  int64_t workspace_bytes;
  int32_t kv_page;
} exg_cluster_spec;

/* A length distribution P(len = k) = prob[k-1], k = 1..max_len. */
typedef struct {
  int32_t max_len;
  const double* prob;
} exg_pmf;

/* Control variables: B_E, B_D, B_m, T_P (degree and
 * applied GPU count), F_E = 1/N_D, strategy S; plus the resolved layout:
 * stage k covers GPUs [stage_first_gpu[k], +stage_n_gpus[k]) and layers
 * [stage_layer_begin[k], stage_layer_end[k]).  For WAA the n_enc_gpus
 * encoder stages come first, then the decoder stages. */
#define EXG_MAX_STAGES 8
typedef struct {
  exg_strategy strategy;
  int32_t b_e, b_d, b_m, n_d;
  int32_t tp_degree, tp_gpus;
  int32_t n_enc_gpus;
  int32_t n_stages;
  int32_t stage_first_gpu[EXG_MAX_STAGES], stage_n_gpus[EXG_MAX_STAGES];
  int32_t stage_layer_begin[EXG_MAX_STAGES], stage_layer_end[EXG_MAX_STAGES];
} exg_schedule;

/* Simulator estimate: steady-state throughput and the
 * latency of a target_len-long query. */
typedef struct {
  double thrput_seq_s, thrput_tok_s, latency_s;
  int64_t perf_evals;
  int32_t feasible;
} exg_estimate;

/* Algorithm 1 options: tolerances as fractions of T* / L_B,
 * search ranges, and the Little's-law completion fraction option
 * (SURVEY.md §8(c) S3). */
typedef struct {
  double eps_t_frac, eps_l_frac;
  int32_t b_e_max, n_d_max, m_max;
  int32_t use_little_fraction;
  int32_t tp_degree_only;     /* > 0: search only this TP degree (a forced partial-TP
                                 plan, e.g. config 4's WAA with t = 2); 0 = all   */
} exg_search_opts;

/* XProfiler sweep axes. */
typedef struct {
  int32_t n_batch;  const int32_t* batch;   /* attention: batch sweep              */
  int32_t n_ctx;    const int32_t* ctx;     /* attention: context sweep per batch  */
  int32_t n_tokens; const int32_t* tokens;  /* rest of the layer: input-size sweep */
  int32_t n_tp;     const int32_t* tp;      /* TP degrees                          */
  int32_t reps;                             /* timed repetitions per point         */
} exg_profile_grid;

/* One request: input ids (length input_len >= 1) and the forced output
 * length (no EOS). */
typedef struct {
  const int32_t* input_ids;
  int32_t input_len, output_len;
} exg_request;

typedef struct {
  float* logits_out;          /* optional fp32 [sum dumped output_len][vocab]   */
  const uint8_t* dump_mask;   /* optional [n]: 1 = dump this request's logits   */
  int32_t slot_ctx;           /* KV slot length; 0 -> max(input_len+output_len) */
  int32_t pin_nccl_algo;      /* 1: TP partial sums exchanged and summed in member
                                 order on every rank (bitwise the one-rank sum,
                                 batch invariant, T13) instead of the NCCL
                                 all-reduce on the TP sub-communicator        */
  int32_t kernel_timing;      /* 1: CUDA events around every launch of the
                                 kernel classes below (roofline evidence)       */
  double dyn_threshold;       /* > 0: dynamic workload adjustment (
                                 RRA on one GPU and WAA layouts):
                                 while the decode batch sits outside
                                 +-threshold of its running average, the next
                                 encode batch targets B_E' = B_E + round(avg -
                                 current) rows (clamped to [1, B_D]); its token
                                 sum is kept within +-threshold of B_E' x the
                                 mean encoded length and never above B_E x the
                                 longest input (the encode workspace); 0 = off */
  /* optional per-stage trace (single-GPU runs; simulator-fidelity and Table 9
   * analyses): one record of 5 doubles per encode phase that admitted
   * requests and per decode iteration, in time order --
   *   {kind (1 encode, 2 decode), start [s from the run's first event],
   *    duration [s], rows (admitted requests | decode batch),
   *    work (encoded tokens | sum of attention keys; encoder-decoder
   *    models: self + cross-attention keys)};
   * at most trace_cap records are written (their count is
   * exg_run_stats.trace_records). */
  double* trace_out;
  int32_t trace_cap;
  /* Paged KV cache ("the addition of
   * vLLM's paging mechanism can further enhance WAA's performance"):
   * kv_page > 0 stores K/V in pages of kv_page positions (a multiple of 64
   * dividing 512) allocated as a row grows, instead of one slot of slot_ctx
   * positions per row; kv_pages = pages in the pool (0: B_D x
   * ceil(slot_ctx / kv_page), the slots' memory).  A row gets the pages of
   * its encoded positions at admission and one more each time its next
   * position crosses a page boundary; admission keeps one free page per
   * active row in reserve.  When a row needs a page and none is free, the
   * most recently admitted active row is preempted.  RRA on one GPU:
   * recompute -- its pages are freed and it is re-admitted (before any new
   * request) with its generated tokens appended to its input, re-encoded, and
   * continues.  Multi-GPU layouts (RRA pipelines / TP groups: every stage
   * pages with the same page ids; WAA: the decoder GPUs page, the encoder side
   * keeps its per-batch slots): swap -- every rank copies the row's pages of
   * the layers it holds to pinned host memory and back into new pages once
   * they fit (before any new admission / handoff), so results are
   * bit-identical to the slot cache; a WAA handoff merges the longest prefix
   * of the encoded batch whose pages fit.  Decoder-only bf16 models; other
   * scopes (T5, fp32, EXG_STATIC) return EXG_E_INPUT.  0 = slots. */
  int32_t kv_page;
  int32_t kv_pages;
} exg_run_opts;

/* Kernel classes timed when exg_run_opts.kernel_timing = 1.  Work is the
 * algorithmic amount: FLOPs for the tensor-core kernels,
 * HBM bytes for the bandwidth kernels. */
enum {
  EXG_K_PREFILL_GEMM = 0,  /* 2*T*F*K flops                                          */
  EXG_K_DECODE_GEMM = 1,   /* weight + activation + output bytes                     */
  EXG_K_DECODE_ATTN = 2,   /* sum_i c_i*2*H*dh*2 (K,V read) + B*H*dh*2*2 (q in, o out) */
  EXG_K_PREFILL_ATTN = 3,  /* 4*H*dh*sum_i n_i(n_i+1)/2 flops                        */
  EXG_K_CLASSES = 4
};

/* Measured run statistics.  Times come from device
 * events on one clock. */
typedef struct {
  double tok_s, tok_s_steady, seq_s;
  double lat_p50_s, lat_p99_s, lat_max_s;
  double wall_s;                       /* first encode start -> last iteration end */
  int64_t out_tokens, decode_iters, encode_phases;
  double mean_decode_batch;            /* measured, vs the simulated B_D           */
  double encode_s, decode_s;           /* device time spent per phase kind         */
  int64_t kernel_launches;             /* library kernels launched by this run     */
  double k_time_s[EXG_K_CLASSES];      /* summed launch durations per class        */
  double k_work[EXG_K_CLASSES];        /* summed algorithmic work per class        */
  int64_t k_launches[EXG_K_CLASSES];
  /* workload variance (Table 9): mean single-stage time and
   * the 99th percentile of |t - mean| of encode phases and decode iterations */
  double enc_stage_mean_s, enc_stage_p99dev_s, dec_stage_mean_s, dec_stage_p99dev_s;
  double mean_encode_batch;            /* requests per encode phase (admissions)  */
  int64_t trace_records;               /* records written to exg_run_opts.trace_out */
  int64_t kv_preemptions;              /* paged KV: rows preempted (recompute / swap) */
  int64_t kv_pages_peak;               /* paged KV: most pages in use at once      */
} exg_run_stats;

typedef struct exg_ctx exg_ctx;           /* one per rank: device state + comms */
typedef struct exg_profile exg_profile;   /* profile-v1 table     */

/* ---- lifecycle ---------------------------------------------------------- */
/* Library ABI version (EXG_ABI_VERSION). */
int32_t exg_abi_version(void);
/* Thread-local message of the last failing call on this thread. */
const char* exg_last_error(void);

/* NCCL unique id for a multi-rank context (call on rank 0, broadcast the
 * 128 bytes).  Single-GPU runs may pass NULL uid to exg_create. */
exg_status exg_get_unique_id(uint8_t uid[128]);

/* Create a rank's context on `device`: allocates and generates this rank's
 * weights on the GPU from spec->weight_seed (K14).  Collective over `world`
 * ranks when world > 1 (one process per GPU, NCCL over NVLink; uid from
 * exg_get_unique_id on rank 0): GPU g of a schedule's layout (G GPUs) belongs
 * to rank g*world/G, every rank calls exg_run with identical arguments and the
 * outputs are written on rank 0.  world = 1 with cluster->n_gpus > 1 runs every
 * GPU of a layout in this one process on `device` (single-device emulation).
 * *out is owned by the library (exg_destroy). */
exg_status exg_create(const exg_model_spec* spec, const exg_cluster_spec* cluster, int32_t device, int32_t rank,
                      int32_t world, const uint8_t* uid, exg_ctx** out);
/* One rank owning every GPU of a layout on `device`, with a one-rank NCCL
 * communicator through which every exchange of the layout (pipeline hops,
 * token return, packed WAA handoff messages) is sent to itself -- runs the
 * NCCL transport on a single GPU (transport test). */
exg_status exg_create_nccl_loopback(const exg_model_spec* spec, const exg_cluster_spec* cluster, int32_t device,
                                    exg_ctx** out);
/* `world` rank contexts of one process on one `device`, connected by a
 * device-copy transport instead of NCCL (each rank's exg_run must be called
 * from its own thread).  For testing the multi-rank executor on one GPU;
 * out[0..world) are destroyed individually with exg_destroy. */
exg_status exg_create_local_group(const exg_model_spec* spec, const exg_cluster_spec* cluster, int32_t device,
                                  int32_t world, exg_ctx** out);
void exg_destroy(exg_ctx* ctx);

/* ---- XProfiler --------------------------------------- */
/* Single-GPU context: times one encoder layer and one decoder layer on the
 * real kernels -- attention over (batch x ctx) and the rest of the layer over
 * tokens per TP degree (a TP-rank-0 shard for t > 1), the decode head
 * (final norm + LM head + argmax) and the encode->decode switch per batch.
 * Multi-rank context (world > 1, collective, every rank calls it): the
 * interconnect tables PAPER.md:154 names -- tp_sync[t] = fp32 all-reduce
 * over ranks [0, t) for each grid TP degree t <= world, pp_sync = one hop rank
 * 0 -> rank 1 (ping-pong / 2), 1 KB .. 1 GB; rank 0's tables are
 * authoritative.  Merge them into a layer profile with exg_profile_copy_comm. */
exg_status exg_profile_run(exg_ctx* ctx, const exg_profile_grid* grid, exg_profile** out);
/* Replace dst's tp_sync / pp_sync tables with src's (a multi-rank profile). */
exg_status exg_profile_copy_comm(exg_profile* dst, const exg_profile* src);
/* profile-v1 text file ("%.17g" numbers, lossless). */
exg_status exg_profile_save(const exg_profile* p, const char* path);
/* Fill the communication tables from an alpha-beta model of the
 * interconnect, for profiles taken on a single-GPU context (a reading,
 * DESIGN.md §3): pp_sync(bytes) = alpha + bytes/bw; for every TP degree t > 1
 * of the profile, tp_sync[t](bytes) = alpha + (t-1)*bytes/bw (each rank
 * sends its fp32 partial to t-1 peers over its own link).  Byte grid 1 KB ..
 * 64 GB, factor 4.  Replaces existing tables. */
exg_status exg_profile_comm_model(exg_profile* p, double alpha_s, double bw_bytes_per_s);
exg_status exg_profile_load(const char* path, exg_profile** out);
void exg_profile_free(exg_profile* p);

/* ---- XSimulator / XScheduler (pure host, deterministic) ----------------- */
/* Estimate of one schedule.  sched must be a resolved
 * schedule (as returned by exg_schedule_find / exg_schedule_resolve). */
exg_status exg_simulate(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                        const exg_pmf* in, const exg_pmf* out_len, int32_t target_len, const exg_schedule* sched,
                        exg_estimate* est);
/* The profile's time of one single-GPU stage holding `n_layers` layers
 * (PAPER.md:150-154 tables): phase 0 = an encode phase of `rows` requests and
 * `work` encoded tokens, n_layers x (attn(rows, work/rows) + rest(work));
 * phase 1 = a decode iteration of `rows` rows attending to `work` keys in
 * total, n_layers x (attn(rows, work/rows) + rest(rows)) + head(rows).
 * Used to separate the workload-driven part of measured stage times from
 * the rest (Table 9 analysis).  Pure host. */
exg_status exg_profile_stage_time(const exg_profile* p, int32_t phase, int32_t tp_degree, int32_t n_layers,
                                  double rows, double work, double* seconds);

/* Memory-overhead accounting: the model bytes and KV-cache
 * bytes each GPU of the schedule's layout holds under the simulator's memory
 * model (weight shard + embeddings on the first / last stage of each side;
 * KV slots sized at max_in + max_out rows per decode row -- B_D for RRA / WAA
 * decoder stages, B for EXG_STATIC -- and max_in per encode row on WAA
 * encoder stages; with cluster->kv_page > 0 a decode row of RRA / WAA is
 * charged the paged live average instead, see exg_cluster_spec).  weight_bytes / kv_bytes: caller-owned double
 * [cluster->n_gpus]; GPUs outside the layout get 0.  Pure host. */
exg_status exg_schedule_memory(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                               const exg_pmf* in, const exg_pmf* out_len, const exg_schedule* sched,
                               double* weight_bytes, double* kv_bytes);
/* Resolve derived fields (B_D, B_m, stage layout) of a schedule given by its
 * control variables (strategy, b_e, n_d | b_m-count, tp_degree, tp_gpus). */
exg_status exg_schedule_resolve(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                                const exg_pmf* in, const exg_pmf* out_len, int32_t m_count, exg_schedule* sched);
/* argmax Throughput s.t. Latency < latency_bound_s by
 * Algorithm 1 inside the strategy x TP-degree x
 * applied-GPU loops.  latency_bound_s may be +inf.
 * Returns EXG_E_INFEASIBLE if no configuration meets the bound. */
exg_status exg_schedule_find(const exg_profile* p, const exg_model_spec* spec, const exg_cluster_spec* cluster,
                             const exg_pmf* in, const exg_pmf* out_len, int32_t target_len, double latency_bound_s,
                             uint32_t strategy_mask, const exg_search_opts* opts, exg_schedule* out,
                             exg_estimate* est);

/* ---- XRunner ------------------------------------------ */
/* Run `sched` on the closed request batch reqs[0..n) (all available at t=0).
 * out_tokens: int32 [sum output_len] in request order (prefix-sum offsets);
 * out_latency_s: [n], from the start of the encode phase that admitted the
 * request to the end of the iteration that emitted its last token.
 * Greedy decoding, token accounting SURVEY.md §8(c) T6.  Collective.
 * sched->strategy == EXG_STATIC (one GPU): batches of b_e requests admitted
 * only when the previous batch has drained; finished rows keep being
 * computed until the batch's longest output is done and every
 * request of the batch completes at that iteration (its latency ends there).
 * Tokens are identical to RRA's (greedy, per-request; T13). */
exg_status exg_run(exg_ctx* ctx, const exg_schedule* sched, const exg_request* reqs, int32_t n, int32_t* out_tokens,
                   double* out_latency_s, exg_run_stats* stats, const exg_run_opts* opts);

#ifdef __cplusplus
}
#endif
#endif /* EXEGPT_H */
