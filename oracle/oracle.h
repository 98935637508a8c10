/*
 * oracle.h — TEST INFRASTRUCTURE ONLY. Never linked into the product.
 *
 * Two CPU checkers expose the same plain-C surface:
 *   ref_*  — the UNMODIFIED reference library (/root/reference/proj/src,
 *            compiled by oracle/Makefile into oracle/_ref/) behind a thin
 *            C wrapper (oracle/ref_capi.cpp).
 *   orc_*  — a plain-C restatement of the reference algorithms
 *            (oracle/rs_oracle.c), each function citing the reference
 *            file:line it follows, plus builder-defined oracles for the
 *            extensions the reference does not have (block hashes, dedup
 *            map, LPT, scenario generator).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these libraries.
 *
 * Status codes match include/rs.h: 0 ok, 1 ValidationError, 2 ConfigError,
 * 5 other error, 6 PlacementError, 7 ParseError.
 */
#ifndef RS_ORACLE_H_
#define RS_ORACLE_H_

#include <stdint.h>

#include "../include/rs.h"

#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_API(prefix)                                                     \
  const char* prefix##last_error(void);                                        \
  int prefix##tpot_seconds(const rs_profile* p, const double* b,               \
                           const double* c, int64_t n, double* out);           \
  /* info = {batch, min_len, max_len, total_tokens}; curves for L=1..n_l */     \
  int prefix##prefix_curves(const int32_t* tok, const int64_t* off,            \
                            int32_t batch, int32_t n_l, int64_t* info,         \
                            int64_t* ucount, int64_t* utokens, int64_t* rem);  \
  int prefix##select_prefix_length(const int32_t* tok, const int64_t* off,     \
                                   int32_t batch, int32_t cap, int32_t gpus,   \
                                   int32_t l_min, int32_t l_max,               \
                                   int32_t* len, int32_t* exceeded);           \
  int prefix##dedup_savings(const int32_t* tok, const int64_t* off,            \
                            int32_t batch, int32_t l_star, int32_t g,          \
                            int64_t* raw, int64_t* dedup, double* frac);       \
  int prefix##unique_prefix_count_among(const int32_t* tok,                    \
                                        const int64_t* off, int32_t count,     \
                                        int32_t len, int64_t* out);            \
  int prefix##assign(const double* pred, const int32_t* id_rank,               \
                     int32_t count, int32_t n_actors, int32_t* order,          \
                     int32_t* group_offsets);                                  \
  int prefix##integrate_decode_seconds(const int32_t* plen,                    \
                                       const double* target, int64_t count,    \
                                       const rs_profile* p, double* out);      \
  int prefix##estimate_actor_time(const int32_t* plen, const double* pred,     \
                                  int32_t count, const rs_profile* p,          \
                                  int32_t g, double* out);                     \
  int prefix##estimate_cost(const int32_t* plen, const double* pred,           \
                            const int32_t* group_offsets,                      \
                            const int32_t* gpu_count, int32_t n_groups,        \
                            const rs_profile* p, int32_t g, double* cost,      \
                            double* times);                                    \
  int prefix##scale(const double* pred, const int32_t* plen,                   \
                    const int32_t* id_rank, int32_t count,                     \
                    const rs_profile* p, int32_t g, int32_t n_min,             \
                    int32_t n_max, double lambda, int32_t gpus,                \
                    const double* t_penalty, int32_t* n_star,                  \
                    double* t_total, double* t_pen_out, double* cost,          \
                    double* t_norm, double* c_norm, double* score,             \
                    int32_t* order, double* actor_times);                      \
  int prefix##sweep_arrays(const double* pred, const int32_t* plen,            \
                           int32_t n_scenarios, int32_t count,                 \
                           const rs_profile* p, int32_t g, int32_t n_min,      \
                           int32_t n_max, double lambda, int32_t gpus,         \
                           int32_t n_threads, double* t_total, double* cost,   \
                           int32_t* n_star);                            \
  /* scale() with plan_rlhfless's placement penalty (training.cpp:150-164) */  \
  int prefix##scale_placed(const double* pred, const int32_t* plen,            \
                           const int32_t* id_rank, int32_t count,              \
                           const rs_profile* p, int32_t g, int32_t n_min,      \
                           int32_t n_max, double lambda, int32_t gpus,         \
                           const rs_placement_penalty* pen, int32_t* n_star,   \
                           double* t_total, double* t_pen_out, double* cost,   \
                           double* t_norm, double* c_norm, double* score,      \
                           int32_t* order, double* actor_times);         \
  /* LengthHistory::predict / predict_noisy per prompt (predictor.cpp:52-98) */\
  int prefix##predict_lengths(const double* obs, const int32_t* depth,         \
                              const int32_t* gt, int32_t count,                \
                              int32_t window, double alpha, int32_t max_len,   \
                              const rs_noise_model* noise,                     \
                              const char* id_bytes, const int64_t* id_offsets, \
                              double* out);

ORACLE_API(ref_)
ORACLE_API(orc_)

/* Reference-only: the prompt table of a CSV trace via trace_from_string. */
void ref_trace_set_format(int fmt);
int ref_trace_convert(const char* text, int64_t n_bytes, int fmt_in, int fmt_out, char* out,
                      int64_t cap, int64_t* out_len);
int ref_trace_prompts(const char* text, int64_t n_bytes, int64_t* info, int32_t* tokens,
                      int64_t* offsets, char* ids, int64_t* id_offsets, int32_t* gt);
int ref_trace_steps(const char* text, int64_t n_bytes, int64_t* info, int32_t* step_idx,
                    int32_t* entry_off, int32_t* entry_prompt, int32_t* lengths);

/* Builder-defined oracles (port only). */
int orc_generate_scenarios(const rs_scenario_spec* spec, double* pred,
                           int32_t* plen);
int orc_scale_idle(const double* pred, const int32_t* id_rank, int32_t count,
                   int32_t g, int32_t n_min, int32_t n_max, int64_t* idle);
int orc_dedup_map(const int32_t* tok, const int64_t* off, int32_t count,
                  int32_t len, int32_t* labels);
int orc_block_hashes(const int32_t* tok, const int64_t* off, int32_t count,
                     int32_t block_tokens, uint64_t* hashes);
int orc_lpt(const double* pred, const int32_t* id_rank, int32_t count,
            int32_t g, int32_t n_min, int32_t n_max, int64_t* makespan,
            int64_t* idle);
int orc_prefix_tables(const int32_t* tok, const int64_t* off, int32_t batch,
                      int64_t* info, int64_t* nodes, int64_t* scb,
                      int64_t* stb, int64_t* lcf, int64_t* ltf);
int orc_sweep_select(const double* sum_t, const double* sum_c,
                     int64_t n_scenarios, int32_t n_candidates, int32_t n_min,
                     double lambda, int32_t* n_star);

/* Reference-only: the reference sweep leg for bench.py --impl reference,
 * with a std::thread pool over scenarios generated by orc_generate_scenarios
 * semantics (the caller passes the arrays). Same as ref_sweep_arrays. */

#ifdef __cplusplus
}
#endif
#endif /* RS_ORACLE_H_ */
