/*
 * rs.h — C-ABI of the B200-native planning core (librs_b200.so).
 *
 * This is the drop-in boundary for the data-parallel hot path of the
 * RLHFless `rollsim` library (reference: /root/reference/proj). Every entry
 * point below replaces one reference function; the cited file:line is the
 * interface it stands in for. Signatures use plain pointers and sizes only.
 *
 * Conventions
 *  - Every function returns an rs_status. On failure a message is available
 *    from rs_last_error() (thread-local). RS_E_VALIDATION / RS_E_CONFIG map
 *    1:1 onto rollsim::ValidationError / rollsim::ConfigError
 *    (proj/include/rollsim/errors.hpp:17-32) and are raised in the same
 *    order as the reference raises them.
 *  - Host-pointer entry points are synchronous: inputs are copied to HBM,
 *    the kernels run on the context stream, results are copied back and the
 *    stream is synchronised before return. `*_device` entry points take
 *    device pointers and are asynchronous on the context stream.
 *  - Caller owns every buffer it passes. Opaque handles are freed with the
 *    matching *_free / *_destroy call. Index and trace handles may outlive
 *    the context that built them.
 *  - Every entry point taking a context runs on the context's device and
 *    restores the caller's current device before returning, so contexts of
 *    several GPUs can be driven from one host thread.
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point fails with RS_E_CUDA.
 */
#ifndef RS_H_
#define RS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1

typedef enum rs_status {
  RS_OK = 0,
  RS_E_VALIDATION = 1, /* rollsim::ValidationError */
  RS_E_CONFIG = 2,     /* rollsim::ConfigError */
  RS_E_CUDA = 3,       /* CUDA runtime / launch failure, or no device */
  RS_E_NOMEM = 4,      /* device or pinned allocation failed */
  RS_E_ARG = 5,        /* NULL handle / pointer misuse (programming error) */
  RS_E_PLACEMENT = 6,  /* rollsim::PlacementError (cluster cannot host the plan) */
  RS_E_PARSE = 7       /* rollsim::ParseError (malformed trace text) */
} rs_status;

const char* rs_last_error(void);
int rs_abi_version(void);

/* ------------------------------------------------------------------ */
/* Context: one per device (and per host thread that drives it).       */
/* Owns the stream, a grow-only scratch arena and per-profile tables.  */
/* ------------------------------------------------------------------ */
typedef struct rs_ctx rs_ctx;

int rs_ctx_create(int device, rs_ctx** out);
int rs_ctx_destroy(rs_ctx* ctx);
/* Use a caller stream (e.g. torch.cuda.current_stream().cuda_stream). NULL
 * restores the context's own stream. Work queued on the previous stream is
 * waited for first (it may still use the context's scratch). */
int rs_ctx_set_stream(rs_ctx* ctx, void* cuda_stream);
int rs_ctx_synchronize(rs_ctx* ctx);
/* Number of kernels this context has launched since creation. */
int rs_ctx_kernel_launches(const rs_ctx* ctx, uint64_t* count);
/* Per-kernel timing: when enabled, every launch of a named kernel is
 * bracketed by CUDA events on the launching stream; rs_ctx_kernel_time
 * returns the summed milliseconds and launch count since the last reset. */
int rs_ctx_enable_kernel_timing(rs_ctx* ctx, int enable);
int rs_ctx_reset_kernel_timing(rs_ctx* ctx);
int rs_ctx_kernel_time(rs_ctx* ctx, const char* kernel_name, double* total_ms,
                       uint64_t* launches);

/* ------------------------------------------------------------------ */
/* Latency profile (proj/include/rollsim/profile.hpp:17-35).          */
/* ------------------------------------------------------------------ */
typedef struct rs_profile {
  const double* batch_knots;   /* nb, strictly increasing */
  int32_t nb;
  const double* context_knots; /* nc, strictly increasing */
  int32_t nc;
  const double* tpot_grid;     /* nb*nc row-major: [batch][context] */
  double rho;                  /* dollars per GPU-second */
} rs_profile;

/* LatencyProfile::tpot_seconds (proj/src/profile.cpp:43-59) evaluated on
 * the device for n (batch, context) points. Bit-identical to the reference. */
int rs_tpot_seconds(rs_ctx* ctx, const rs_profile* profile, const double* batch,
                    const double* context, int64_t n, double* out);

/* ------------------------------------------------------------------ */
/* (1) Shared-prefix dedup (proj/include/rollsim/dedup.hpp:20-78).     */
/* Prompts are CSR: tokens[offsets[i] .. offsets[i+1]) is prompt i.    */
/* ------------------------------------------------------------------ */
typedef struct rs_prefix_index rs_prefix_index;

/* PrefixIndex::build (proj/include/rollsim/dedup.hpp:22,
 * proj/src/dedup.cpp:30-100). Host CSR in, index handle out. */
int rs_prefix_index_build(rs_ctx* ctx, const int32_t* tokens,
                          const int64_t* offsets, int32_t batch,
                          rs_prefix_index** out);
/* Same with the CSR already resident in HBM (device pointers). */
int rs_prefix_index_build_device(rs_ctx* ctx, const int32_t* d_tokens,
                                 const int64_t* d_offsets, int32_t batch,
                                 rs_prefix_index** out);
/* Device-resident outputs for benchmarking: no host copies of the CSR or the
 * tables (the build still synchronises once, at its end, for the stats). The five
 * tables land in d_tables (5 consecutive int64 arrays of max_len_cap+2
 * entries: nodes_at_depth, short_count_below, short_tokens_below,
 * longer_count_from, longer_tokens_from) and d_info receives
 * {batch, min_len, max_len, total_tokens, 0}. max_len_cap must be >=
 * the longest prompt. Validation errors (an empty prompt) are returned by the
 * call itself (RS_E_VALIDATION) after its synchronisation; d_info[4] is
 * always written as 0 and kept only for layout compatibility. */
int rs_prefix_index_build_device_async(rs_ctx* ctx, const int32_t* d_tokens,
                                       const int64_t* d_offsets, int32_t batch,
                                       int32_t max_len_cap, int64_t* d_tables,
                                       int64_t* d_info);
/* An index built on the device keeps its tables in a pinned host block the
 * tables kernel wrote (no copy after the build's sync); the block belongs
 * to a pool shared with the context, so an index may outlive its context.
 * Freeing the index returns the block. */
void rs_prefix_index_free(rs_prefix_index* idx);
/* Rebuild a handle from its five tables (sizes as rs_prefix_index_tables),
 * so a caller that keeps only the tables (the C++ drop-in's PrefixIndex)
 * can still query rs_select_prefix_length / rs_dedup_savings. */
int rs_prefix_index_from_tables(int32_t batch_size, int32_t min_len, int32_t max_len,
                                int64_t total_tokens, const int64_t* nodes_at_depth,
                                const int64_t* short_count_below,
                                const int64_t* short_tokens_below,
                                const int64_t* longer_count_from,
                                const int64_t* longer_tokens_from,
                                rs_prefix_index** out);

/* Accessors (proj/include/rollsim/dedup.hpp:25-34, dedup.cpp:102-122). */
int rs_prefix_index_info(const rs_prefix_index* idx, int32_t* batch_size,
                         int32_t* min_len, int32_t* max_len,
                         int64_t* total_tokens);
int rs_unique_prefix_count(const rs_prefix_index* idx, int32_t prefix_len,
                           int64_t* out);
int rs_unique_prefix_tokens(const rs_prefix_index* idx, int32_t prefix_len,
                            int64_t* out);
int rs_remainder_tokens(const rs_prefix_index* idx, int32_t prefix_len,
                        int64_t* out);
/* Raw tables (the private members of PrefixIndex, dedup.hpp:43-47):
 * nodes_at_depth has max_len+1 entries, the other four max_len+2. */
int rs_prefix_index_tables(const rs_prefix_index* idx, int64_t* nodes_at_depth,
                           int64_t* short_count_below,
                           int64_t* short_tokens_below,
                           int64_t* longer_count_from,
                           int64_t* longer_tokens_from);

/* select_prefix_length (dedup.hpp:63-65, dedup.cpp:124-144). */
int rs_select_prefix_length(const rs_prefix_index* idx,
                            int32_t max_unique_prefixes, int32_t gpu_count,
                            int32_t l_min, int32_t l_max, int32_t* prefix_len,
                            int32_t* capacity_exceeded);
/* dedup_savings (dedup.hpp:73-74, dedup.cpp:146-161). */
int rs_dedup_savings(const rs_prefix_index* idx, int32_t l_star,
                     int32_t responses_per_prompt, int64_t* raw_prefill_tokens,
                     int64_t* dedup_prefill_tokens, double* saved_fraction);
/* unique_prefix_count_among (dedup.hpp:77-78, dedup.cpp:163-183). */
int rs_unique_prefix_count_among(rs_ctx* ctx, const int32_t* tokens,
                                 const int64_t* offsets, int32_t count,
                                 int32_t prefix_len, int64_t* out);
/* Dedup map (extension): labels[i] = smallest batch index j
 * whose length-L prefix (full sequence if shorter) equals prompt i's. */
int rs_dedup_map(rs_ctx* ctx, const int32_t* tokens, const int64_t* offsets,
                 int32_t count, int32_t prefix_len, int32_t* labels);
/* Chained block hashes (extension). For prompt i with
 * n_i = ceil(len_i / block_tokens) blocks, hashes[hash_offset(i) + j] is the
 * chained hash of tokens [0, min(len_i, (j+1)*block_tokens)), where
 * hash_offset(i) = sum_{k<i} n_k. Definition in DESIGN.md §3.4. */
int rs_block_hashes(rs_ctx* ctx, const int32_t* tokens, const int64_t* offsets,
                    int32_t count, int32_t block_tokens, uint64_t* hashes);

/* ------------------------------------------------------------------ */
/* (2) Length-aware assignment (proj/include/rollsim/planner.hpp).     */
/* Prompts are SoA: pred (predicted_len), prompt_len, id_rank (rank of */
/* the prompt id under std::string ordering; ties in predicted length  */
/* are broken by it).                                                  */
/* ------------------------------------------------------------------ */

/* Rank of each string under std::string ordering (unsigned bytewise, a
 * proper prefix first): the id tie-break of assign (planner.cpp:25-31).
 * String i is bytes[offsets[i] .. offsets[i+1]); equal strings keep input
 * order. Used by the C++ drop-in to turn PredictedPrompt ids into id_rank. */
int rs_rank_strings(rs_ctx* ctx, const char* bytes, const int64_t* offsets,
                    int32_t count, int32_t* rank);

/* assign (planner.hpp:33-34, planner.cpp:16-51): order[r] = input index of
 * the prompt at rank r (pred desc, id asc); group g is
 * order[group_offsets[g] .. group_offsets[g+1]). */
int rs_assign(rs_ctx* ctx, const double* pred, const int32_t* id_rank,
              int32_t count, int32_t n_actors, int32_t* order,
              int32_t* group_offsets);

/* integrate_decode_seconds (planner.hpp:47-48, planner.cpp:88-130). */
int rs_integrate_decode_seconds(rs_ctx* ctx, const int32_t* prompt_len,
                                const double* target_len, int64_t count,
                                const rs_profile* profile, double* out);

/* estimate_actor_time (planner.hpp:52-54, planner.cpp:132-146) for one
 * group given as SoA. */
int rs_estimate_actor_time(rs_ctx* ctx, const int32_t* prompt_len,
                           const double* pred, int32_t count,
                           const rs_profile* profile,
                           int32_t responses_per_prompt, double* out);

/* estimate_cost (planner.hpp:57-58, planner.cpp:148-157): groups are
 * consecutive slices [group_offsets[g], group_offsets[g+1]) of the SoA;
 * times (nullable) receives each group's estimate_actor_time. */
int rs_estimate_cost(rs_ctx* ctx, const int32_t* prompt_len, const double* pred,
                     const int32_t* group_offsets, const int32_t* gpu_count,
                     int32_t n_groups, const rs_profile* profile,
                     int32_t responses_per_prompt, double* cost, double* times);

/* ------------------------------------------------------------------ */
/* (3) Cost-aware actor scaling (planner.hpp:60-91, planner.cpp:159-218) */
/* ------------------------------------------------------------------ */
typedef struct rs_scale_out {
  /* Arrays of C = n_max - n_min + 1 entries, ascending N; any may be NULL. */
  int32_t n_star;
  double* t_total;
  double* t_penalty;
  double* cost;
  double* t_norm;
  double* c_norm;
  double* score;
  int64_t* idle_slot_ticks; /* sum over groups of G*(max ceil - ceil_i) */
  /* count entries: input index at each rank (shared by every candidate). */
  int32_t* order;
  /* n_star entries: estimate per actor for the chosen N. */
  double* actor_times;
  /* sum_{N=n_min}^{n_max} N entries: every group time of every candidate,
   * candidate-major (for host TimePenaltyFn callbacks). */
  double* group_times;
  /* LPT extension, C entries each, nullable: the same
   * predictions as G responses of ceil(pred) tokens, greedy LPT onto N actors
   * (as rs_lpt): token makespan and intra-function idle N*makespan - sum. */
  int64_t* lpt_makespan;
  int64_t* lpt_idle;
} rs_scale_out;

/* scale(): t_penalty (nullable, C entries) is added to each candidate's
 * t_total before normalisation, like TimePenaltyFn (planner.hpp:80-82). */
int rs_scale(rs_ctx* ctx, const double* pred, const int32_t* prompt_len,
             const int32_t* id_rank, int32_t count, const rs_profile* profile,
             int32_t responses_per_prompt, int32_t n_min, int32_t n_max,
             double lambda, int32_t gpus_per_actor, const double* t_penalty,
             rs_scale_out* out);

/* ------------------------------------------------------------------ */
/* (3b) scale() with the placement penalty on the device               */
/* ------------------------------------------------------------------ */
/* ClusterTopology (placement.hpp:14-38). bw_matrix, when non-NULL, is
 * n_nodes x n_nodes row-major and wins over the two-tier bandwidths. */
typedef struct rs_topology {
  int32_t n_nodes;
  const int32_t* node_gpus;     /* GPUs per node */
  double intra_node_bw, inter_node_bw; /* bytes/s */
  const double* bw_matrix;
  int32_t learner_node;
  int32_t n_learner_gpus;
  const int32_t* learner_gpus;  /* local GPU indices on learner_node */
} rs_topology;

/* The TimePenaltyFn plan_rlhfless installs (training.cpp:150-164): place the
 * candidate (placement.cpp:177-291: heaviest actor on the learner node, the
 * rest by descending estimated time onto the highest-bandwidth node with room),
 * then charge max(0, max_i -slack_i) with slack_i = (l_prefill + T_heaviest)
 * - (model_bytes/bw_i + kv_bytes_i/bw_i + T_i) (placement.cpp:339-363), where
 * kv_bytes_i = kv_bytes_per_token * sum of the group's prompt lengths
 * (transfers_for, training.cpp:68-80). */
typedef struct rs_placement_penalty {
  const rs_topology* topology;
  double model_bytes;
  double kv_bytes_per_token;
  double l_prefill_seconds;
} rs_placement_penalty;

/* scale() with that penalty computed on the device for every candidate.
 * Errors in the reference's order: scale's own argument checks, then
 * ClusterTopology::validate / transfer checks (RS_E_CONFIG), then
 * RS_E_PLACEMENT when a candidate's actors do not fit the cluster.
 * out->t_penalty receives the per-candidate penalties. */
int rs_scale_placed(rs_ctx* ctx, const double* pred, const int32_t* prompt_len,
                    const int32_t* id_rank, int32_t count, const rs_profile* profile,
                    int32_t responses_per_prompt, int32_t n_min, int32_t n_max,
                    double lambda, int32_t gpus_per_actor,
                    const rs_placement_penalty* penalty, rs_scale_out* out);

/* The normalise + argmin tail of scale() (planner.cpp:196-217) on
 * caller-provided per-candidate totals; used after host penalty callbacks. */
int rs_scale_select(rs_ctx* ctx, const double* t_total, const double* t_penalty,
                    const double* cost, int32_t n_candidates, int32_t n_min,
                    double lambda, double* t_norm, double* c_norm,
                    double* score, int32_t* n_star);

/* ------------------------------------------------------------------ */
/* (3c) Prediction snapshot                             */
/* ------------------------------------------------------------------ */
/* NoiseModel (predictor.hpp:18-27). kind 0 = identity, 1 = bucket. */
typedef struct rs_noise_model {
  int32_t kind;
  double bucket_accuracy;
  int32_t bucket_width;
  uint64_t seed;
} rs_noise_model;

/* LengthHistory::predict / predict_noisy (predictor.cpp:52-98) for a batch of
 * prompts, i.e. snapshot_predictions (training.cpp:53-66):
 *   obs[i * window + k], k < depth[i]: prompt i's retained per-step means,
 *   oldest first (depth 0 = never observed: ground_truth_len[i] is used);
 *   noise NULL or kind 0 = predict(); kind 1 needs the prompt ids as CSR
 *   bytes (id_bytes, id_offsets[count+1]) for its fnv1a-keyed stream.
 * device_ptrs != 0: every array, out included, is device memory (the result
 * can feed rs_sweep_arrays directly). out[i] = the prediction. */
int rs_predict_lengths(rs_ctx* ctx, const double* obs, const int32_t* depth,
                       const int32_t* ground_truth_len, int32_t count, int32_t window,
                       double alpha, int32_t max_response_len, const rs_noise_model* noise,
                       const char* id_bytes, const int64_t* id_offsets, int device_ptrs,
                       double* out);

/* ------------------------------------------------------------------ */
/* (1b) Trace prompt table -> device CSR                */
/* ------------------------------------------------------------------ */
/* A CSV trace (csv_from_string, workload.cpp:169-263): the '# prompt <id>
 * <ground_truth> <tok>...' metadata and the step rows, parsed on the device from the file bytes (host, or device memory
 * when device_ptr != 0) into an id-sorted token CSR in HBM that
 * rs_prefix_index_build_device takes directly. Errors in the reference's
 * order: RS_E_PARSE (malformed metadata or step rows, missing or misplaced
 * column header, first offending line), then RS_E_VALIDATION
 * (WorkloadTrace::validate's prompt rules, then its step rules). */
typedef struct rs_trace_csr rs_trace_csr;
int rs_trace_csr_parse(rs_ctx* ctx, const char* text, int64_t n_bytes, int device_ptr,
                       rs_trace_csr** out);
/* The JSONL form (jsonl_from_string, workload.cpp:294-352: a header object
 * {"type":"header","g",..,"prompts":[{"id","ground_truth_len","token_ids"}]}
 * then one {"step","scheduled","lengths"} object per line, each read by
 * nlohmann::json) into the same handle. RS_E_PARSE at the first malformed
 * line (JSON syntax or the schema's types), then RS_E_VALIDATION. Not read
 * (RS_E_PARSE "not support"): nesting deeper than 256, floats converted to
 * int within 1e-6 below an integer or with an exponent beyond +-60. */
int rs_trace_csr_parse_jsonl(rs_ctx* ctx, const char* text, int64_t n_bytes, int device_ptr,
                             rs_trace_csr** out);
int rs_trace_csr_info(const rs_trace_csr* trace, int32_t* count, int64_t* n_tokens,
                      int64_t* id_bytes, int32_t* g, int32_t* max_prompt_len,
                      int32_t* max_response_len);
/* Device views, valid until rs_trace_csr_free: tokens[n_tokens] (int32),
 * offsets[count + 1] (int64), prompts in id order. */
int rs_trace_csr_device(const rs_trace_csr* trace, const int32_t** d_tokens,
                        const int64_t** d_offsets);
/* Host copies (any pointer may be NULL): tokens[n_tokens], offsets[count+1],
 * id_bytes[id_bytes], id_offsets[count+1], ground_truth[count]. */
int rs_trace_csr_copy(rs_ctx* ctx, const rs_trace_csr* trace, int32_t* tokens, int64_t* offsets,
                      char* id_bytes, int64_t* id_offsets, int32_t* ground_truth);
/* The step rows (StepRecord, workload.hpp:29-33) as a step table, built on
 * the device: n_steps steps, n_entries scheduled (step, prompt) entries.
 * step_idx[n_steps]; entry_off[n_steps + 1] (entries of step s are
 * [entry_off[s], entry_off[s+1]), in scheduled_prompts order);
 * entry_prompt[n_entries] indexes the id-sorted prompt table;
 * lengths[n_entries * g] holds each entry's actual_lengths in response
 * order. Device views (valid until rs_trace_csr_free; NULL when there are
 * no rows) and host copies (any pointer may be NULL). */
int rs_trace_csr_steps_info(const rs_trace_csr* trace, int32_t* n_steps, int64_t* n_entries);
int rs_trace_csr_steps_device(const rs_trace_csr* trace, const int32_t** step_idx,
                              const int32_t** entry_off, const int32_t** entry_prompt,
                              const int32_t** lengths);
int rs_trace_csr_steps_copy(rs_ctx* ctx, const rs_trace_csr* trace, int32_t* step_idx,
                            int32_t* entry_off, int32_t* entry_prompt, int32_t* lengths);
void rs_trace_csr_free(rs_trace_csr* trace);

/* ------------------------------------------------------------------ */
/* Monte-Carlo scaling sweep: scale() for every        */
/* scenario x candidate, scenarios generated on the device.            */
/* ------------------------------------------------------------------ */
typedef struct rs_scenario_spec {
  uint64_t base_seed;     /* scenario s uses Rng(hash_combine(base_seed, s)) */
  int64_t first_scenario; /* global index of the first scenario (sharding) */
  int32_t n_scenarios;
  int32_t count;          /* prompts per scenario */
  double plen_mean, plen_sigma;
  int32_t plen_min, plen_max;
  double pred_scale, pred_min, pred_max;
} rs_scenario_spec;

/* Materialise scenarios (pred, prompt_len: n_scenarios*count each).
 * device_ptrs != 0: outputs are device pointers and the call is async. */
int rs_generate_scenarios(rs_ctx* ctx, const rs_scenario_spec* spec,
                          double* pred, int32_t* prompt_len, int device_ptrs);

typedef struct rs_sweep_out {
  /* Per scenario x candidate (scenario-major, S*C); nullable. */
  double* t_total;
  double* cost;
  int64_t* idle_slot_ticks;
  /* Per scenario (S); nullable. */
  int32_t* n_star;
  /* Per candidate (C) aggregates over this call's scenarios; nullable. */
  int32_t* nstar_hist;
  double* sum_t;
  double* sum_c;
} rs_sweep_out;

/* Sweep over generated scenarios. device_ptrs != 0: every out pointer is a
 * device pointer. Both forms return once every result is written (the call
 * reads the device status once at the end: a scenario the bucketed fast path
 * cannot take reruns the sweep on the generic path). Host outputs may be
 * pageable (staged through pinned bounce buffers) or pinned (written
 * directly, overlapping the next batch's kernels). */
int rs_sweep(rs_ctx* ctx, const rs_scenario_spec* spec,
             const rs_profile* profile, int32_t responses_per_prompt,
             int32_t n_min, int32_t n_max, double lambda,
             int32_t gpus_per_actor, rs_sweep_out* out, int device_ptrs);

/* Sweep over caller scenarios (pred/prompt_len: S*count, id_rank = index).
 * Host inputs stream in batch by batch on a separate copy stream while the
 * previous batch computes (pinned inputs copy fully asynchronously). */
int rs_sweep_arrays(rs_ctx* ctx, const double* pred, const int32_t* prompt_len,
                    int32_t n_scenarios, int32_t count,
                    const rs_profile* profile, int32_t responses_per_prompt,
                    int32_t n_min, int32_t n_max, double lambda,
                    int32_t gpus_per_actor, rs_sweep_out* out, int device_ptrs);

/* Aggregate pick over the whole sweep from per-candidate sums (after the
 * cross-rank allreduce): mean t and mean c are min-max normalised like
 * scale() and the first strict minimum wins. Host-side O(C). */
int rs_sweep_select(const double* sum_t, const double* sum_c,
                    int64_t n_scenarios, int32_t n_candidates, int32_t n_min,
                    double lambda, int32_t* n_star);

/* ------------------------------------------------------------------ */
/* Multi-GPU sweep. Scenarios shard in contiguous blocks    */
/* ([S*r/W, S*(r+1)/W) on rank r) with no data-path exchange; the one    */
/* collective is a single NCCL all-reduce of the packed per-candidate    */
/* aggregates (3 x C doubles), after which every rank computes the       */
/* aggregate pick (as rs_sweep_select). NCCL is loaded at run time       */
/* (libnccl.so.2); without it these calls fail with RS_E_CUDA and the    */
/* single-GPU API is unaffected. The unit being sharded is scale()       */
/* (proj/src/planner.cpp:159-218).                                        */
/* ------------------------------------------------------------------ */
#define RS_COMM_ID_BYTES 128
typedef struct rs_comm rs_comm;
/* One process per GPU: rank 0 makes the id, the caller ships it to every
 * rank out of band (e.g. over its launcher's store), each rank joins. */
int rs_comm_unique_id(uint8_t* id /* RS_COMM_ID_BYTES */);
int rs_comm_init(rs_ctx* ctx, const uint8_t* id, int32_t n_ranks, int32_t rank, rs_comm** out);
int rs_comm_destroy(rs_comm* comm);
/* spec describes the WHOLE sweep; this rank evaluates its block. The
 * per-scenario outputs of `out` hold this rank's block (scenario-major from
 * its first scenario); sum_t / sum_c / nstar_hist receive the all-reduced
 * aggregates over every rank; *n_star_all (nullable) the aggregate pick.
 * Synchronous, like rs_sweep. */
int rs_sweep_sharded(rs_ctx* ctx, rs_comm* comm, const rs_scenario_spec* spec,
                     const rs_profile* profile, int32_t responses_per_prompt, int32_t n_min,
                     int32_t n_max, double lambda, int32_t gpus_per_actor, rs_sweep_out* out,
                     int device_ptrs, int32_t* n_star_all);

/* One process driving several GPUs (one host thread each): the handle owns
 * a context per device and an NCCL clique over them. */
typedef struct rs_multi rs_multi;
int rs_multi_create(const int32_t* devices, int32_t n_devices, rs_multi** out);
int rs_multi_size(const rs_multi* m, int32_t* n_devices);
int rs_multi_context(rs_multi* m, int32_t index, rs_ctx** out);
int rs_multi_destroy(rs_multi* m);
/* The whole sweep over the handle's devices; `out` holds HOST arrays for
 * every scenario (as rs_sweep with device_ptrs = 0). */
int rs_multi_sweep(rs_multi* m, const rs_scenario_spec* spec, const rs_profile* profile,
                   int32_t responses_per_prompt, int32_t n_min, int32_t n_max, double lambda,
                   int32_t gpus_per_actor, rs_sweep_out* out, int32_t* n_star_all);

/* ------------------------------------------------------------------ */
/* LPT extension: responses (prompt i, r<G) of length  */
/* ceil(pred_i) sorted (len desc, id_rank asc, r asc) are placed one by */
/* one on the least-loaded actor (ties -> lowest index).               */
/* ------------------------------------------------------------------ */
int rs_lpt(rs_ctx* ctx, const double* pred, const int32_t* id_rank,
           int32_t count, int32_t responses_per_prompt, int32_t n_min,
           int32_t n_max, int64_t* makespan, int64_t* idle_tokens);

#ifdef __cplusplus
}
#endif
#endif /* RS_H_ */
