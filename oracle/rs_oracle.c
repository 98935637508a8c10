/*
 * rs_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU "port" checker).
 *
 * A plain-C restatement of the reference rollsim algorithms on the hot path,
 * each function citing the reference file:line it follows
 * (/root/reference/proj). It is pinned against the reference itself
 * (oracle/_ref, tests/test_oracle.py) and against the golden vectors under
 * tests/golden/. Only tests/, __graft_entry__.smoke() and bench.py's CPU
 * legs may load it; the product (librs_b200.so) never does.
 *
 * Compiled with -O2 -ffp-contract=off and no -march flags so that every
 * double operation is a single IEEE operation in source order, exactly like
 * the reference's Release build (proj/CMakeLists.txt:8-12).
 *
 * Builder-defined oracles for extensions with no reference equivalent are
 * at the end (scenario generator, block hashes, dedup map, LPT, idle).
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"
#include "../include/rs_scenario_tables.h"

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ */
/* profile.cpp                                                          */
/* ------------------------------------------------------------------ */

/* interval_of — proj/src/profile.cpp:21-26 (upper_bound - 1, clamped). */
static int32_t interval_of(const double* k, int32_t n, double v) {
  if (v <= k[0]) return 0;
  if (v >= k[n - 1]) return n - 2;
  int32_t lo = 0, hi = n; /* first index with k[i] > v */
  while (lo < hi) {
    int32_t mid = (lo + hi) / 2;
    if (k[mid] > v) hi = mid; else lo = mid + 1;
  }
  return lo - 1;
}

/* clamp_to — proj/src/profile.cpp:28-30. */
static double clamp_to(const double* k, int32_t n, double v) {
  double lo = v > k[0] ? v : k[0];          /* std::max(front, v) */
  return k[n - 1] < lo ? k[n - 1] : lo;      /* std::min(back, .)  */
}

/* LatencyProfile::tpot_seconds — proj/src/profile.cpp:43-59. */
static double tpot(const rs_profile* p, double batch, double ctx) {
  double b = clamp_to(p->batch_knots, p->nb, batch);
  double c = clamp_to(p->context_knots, p->nc, ctx);
  int32_t bi = interval_of(p->batch_knots, p->nb, b);
  int32_t ci = interval_of(p->context_knots, p->nc, c);
  const double* bk = p->batch_knots;
  const double* ck = p->context_knots;
  double tb = (b - bk[bi]) / (bk[bi + 1] - bk[bi]);
  double tc = (c - ck[ci]) / (ck[ci + 1] - ck[ci]);
  const double* g = p->tpot_grid;
  int32_t nc = p->nc;
  double v00 = g[bi * nc + ci], v01 = g[bi * nc + ci + 1];
  double v10 = g[(bi + 1) * nc + ci], v11 = g[(bi + 1) * nc + ci + 1];
  double lo = v00 + (v01 - v00) * tc;
  double hi = v10 + (v11 - v10) * tc;
  return lo + (hi - lo) * tb;
}

int orc_tpot_seconds(const rs_profile* p, const double* b, const double* c,
                     int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = tpot(p, b[i], c[i]);
  return 0;
}

/* ------------------------------------------------------------------ */
/* planner.cpp                                                          */
/* ------------------------------------------------------------------ */

/* tpot_context_run_sum — proj/src/planner.cpp:61-84. */
static double run_sum(const rs_profile* p, double batch, double c_lo,
                      double c_hi) {
  const double* k = p->context_knots;
  int32_t n = p->nc;
  double total = 0;
  double c = c_lo;
  while (c <= c_hi) {
    double piece_end;
    if (c < k[0]) {
      double e = ceil(k[0]) - 1.0;
      piece_end = c_hi < e ? c_hi : e;
    } else if (c >= k[n - 1]) {
      piece_end = c_hi;
    } else {
      int32_t lo = 0, hi = n; /* std::upper_bound */
      while (lo < hi) {
        int32_t mid = (lo + hi) / 2;
        if (k[mid] > c) hi = mid; else lo = mid + 1;
      }
      double e = floor(k[lo]);
      piece_end = c_hi < e ? c_hi : e;
    }
    double count = piece_end - c + 1.0;
    total += count * (tpot(p, batch, c) + tpot(p, batch, piece_end)) / 2.0;
    c = piece_end + 1.0;
  }
  return total;
}

typedef struct { int64_t fin; int32_t plen; } resp_t;

static int cmp_resp(const void* a, const void* b) {
  int64_t x = ((const resp_t*)a)->fin, y = ((const resp_t*)b)->fin;
  return (x > y) - (x < y);
}

/* Integral over responses already sorted by ascending finish tick; the
 * body of integrate_decode_seconds — proj/src/planner.cpp:100-129. */
static double integrate_sorted(const resp_t* r, int64_t n, const rs_profile* p,
                               int32_t* suf /* n+1 scratch */) {
  suf[n] = 0;
  for (int64_t i = n; i-- > 0;) suf[i] = suf[i + 1] > r[i].plen ? suf[i + 1] : r[i].plen;
  double total = 0;
  int64_t done = 0, t = 1;
  const int64_t last = r[n - 1].fin;
  while (t <= last) {
    while (done < n && r[done].fin < t) ++done;
    int64_t run_end = r[done].fin;
    double batch = (double)(n - done);
    double base = (double)suf[done];
    total += run_sum(p, batch, base + (double)(t - 1), base + (double)(run_end - 1));
    t = run_end + 1;
  }
  return total;
}

/* integrate_decode_seconds — proj/src/planner.cpp:88-130. */
int orc_integrate_decode_seconds(const int32_t* plen, const double* target,
                                 int64_t count, const rs_profile* p,
                                 double* out) {
  if (count <= 0) { *out = 0; return 0; }                        /* :90 */
  for (int64_t i = 0; i < count; ++i)                            /* :91-94 */
    if (target[i] < 1)
      return fail(1, "integrate_decode_seconds: target length < 1");
  resp_t* r = malloc(sizeof(resp_t) * count);
  int32_t* suf = malloc(sizeof(int32_t) * (count + 1));
  for (int64_t i = 0; i < count; ++i) { r[i].fin = (int64_t)ceil(target[i]); r[i].plen = plen[i]; }
  qsort(r, count, sizeof(resp_t), cmp_resp);                     /* :97-101 */
  *out = integrate_sorted(r, count, p, suf);
  free(r); free(suf);
  return 0;
}

/* estimate_actor_time — proj/src/planner.cpp:132-146: G copies of every
 * prompt, reverse order, then the integral. */
int orc_estimate_actor_time(const int32_t* plen, const double* pred,
                            int32_t count, const rs_profile* p, int32_t g,
                            double* out) {
  if (g < 1) return fail(1, "estimate_actor_time: responses_per_prompt >= 1");
  int64_t n = (int64_t)count * g;
  if (n == 0) { *out = 0; return 0; }
  int32_t* pl = malloc(sizeof(int32_t) * n);
  double* tg = malloc(sizeof(double) * n);
  int64_t k = 0;
  for (int32_t i = count; i-- > 0;)
    for (int32_t r = 0; r < g; ++r) { pl[k] = plen[i]; tg[k] = pred[i]; ++k; }
  int st = orc_integrate_decode_seconds(pl, tg, n, p, out);
  free(pl); free(tg);
  return st;
}

/* estimate_cost — proj/src/planner.cpp:148-157 (sequential in group order). */
int orc_estimate_cost(const int32_t* plen, const double* pred,
                      const int32_t* off, const int32_t* gpu_count,
                      int32_t n_groups, const rs_profile* p, int32_t g,
                      double* cost, double* times) {
  double dollars = 0;
  for (int32_t k = 0; k < n_groups; ++k) {
    double t;
    int st = orc_estimate_actor_time(plen + off[k], pred + off[k],
                                     off[k + 1] - off[k], p, g, &t);
    if (st) return st;
    if (times) times[k] = t;
    dollars += p->rho * t * gpu_count[k];
  }
  *cost = dollars;
  return 0;
}

/* assign ordering — proj/src/planner.cpp:25-31: predicted desc, id asc. */
typedef struct { double pred; int32_t id; int32_t idx; } rank_t;

static int cmp_rank(const void* a, const void* b) {
  const rank_t* x = a; const rank_t* y = b;
  if (x->pred != y->pred) return x->pred > y->pred ? -1 : 1;
  return (x->id > y->id) - (x->id < y->id);
}

static rank_t* rank_prompts(const double* pred, const int32_t* id_rank,
                            int32_t count) {
  rank_t* v = malloc(sizeof(rank_t) * (count > 0 ? count : 1));
  for (int32_t i = 0; i < count; ++i) {
    v[i].pred = pred[i]; v[i].id = id_rank ? id_rank[i] : i; v[i].idx = i;
  }
  qsort(v, count, sizeof(rank_t), cmp_rank);
  return v;
}

/* assign — proj/src/planner.cpp:16-51. */
int orc_assign(const double* pred, const int32_t* id_rank, int32_t count,
               int32_t n_actors, int32_t* order, int32_t* off) {
  if (count <= 0) return fail(1, "assign: empty batch");
  if (n_actors < 1) return fail(1, "assign: n_actors must be >= 1");
  if (n_actors > count) return fail(1, "assign: more actors than prompts");
  rank_t* v = rank_prompts(pred, id_rank, count);
  for (int32_t i = 0; i < count; ++i) order[i] = v[i].idx;
  int32_t q = count / n_actors, r = count % n_actors, pos = 0;
  for (int32_t a = 0; a < n_actors; ++a) { off[a] = pos; pos += q + (a < r ? 1 : 0); }
  off[n_actors] = pos;
  free(v);
  return 0;
}

/* Group time at prompt granularity on a rank-ordered slice (descending
 * prediction): identical runs to estimate_actor_time's G-fold expansion,
 * since each prompt contributes G responses with the same finish tick
 * (batch = G * live prompts). planner.cpp:132-146 + :88-130. */
static double group_time(const rank_t* v, const int32_t* plen, int32_t a,
                         int32_t b, int32_t g, const rs_profile* p,
                         resp_t* scratch, int32_t* suf) {
  int32_t n = b - a;
  for (int32_t i = 0; i < n; ++i) {             /* reversed: ascending */
    const rank_t* e = &v[b - 1 - i];
    scratch[i].fin = (int64_t)ceil(e->pred);
    scratch[i].plen = plen[e->idx];
  }
  suf[n] = 0;
  for (int32_t i = n; i-- > 0;) suf[i] = suf[i + 1] > scratch[i].plen ? suf[i + 1] : scratch[i].plen;
  double total = 0;
  int64_t done = 0, t = 1;
  const int64_t last = scratch[n - 1].fin;
  while (t <= last) {
    while (done < n && scratch[done].fin < t) ++done;
    int64_t run_end = scratch[done].fin;
    double batch = (double)((int64_t)g * (n - done));
    double base = (double)suf[done];
    total += run_sum(p, batch, base + (double)(t - 1), base + (double)(run_end - 1));
    t = run_end + 1;
  }
  return total;
}

/* Normalise + argmin tail of scale — proj/src/planner.cpp:196-217. */
static int32_t select_best(const double* t_tot, const double* t_pen,
                           const double* cost, int32_t nc, double lambda,
                           double* t_norm, double* c_norm, double* score) {
  double t_min = t_tot[0] + (t_pen ? t_pen[0] : 0.0);
  double t_max = t_min, c_min = cost[0], c_max = c_min;
  for (int32_t i = 0; i < nc; ++i) {
    double t = t_tot[i] + (t_pen ? t_pen[i] : 0.0);
    t_min = t < t_min ? t : t_min;              /* std::min(a, b): b < a ? b : a */
    t_max = t_max < t ? t : t_max;              /* std::max(a, b): a < b ? b : a */
    c_min = cost[i] < c_min ? cost[i] : c_min;
    c_max = c_max < cost[i] ? cost[i] : c_max;
  }
  int32_t best = 0;
  double best_score = 0;
  for (int32_t i = 0; i < nc; ++i) {
    double t = t_tot[i] + (t_pen ? t_pen[i] : 0.0);
    double tn = t_max > t_min ? (t - t_min) / (t_max - t_min) : 0.0;
    double cn = c_max > c_min ? (cost[i] - c_min) / (c_max - c_min) : 0.0;
    double sc = lambda * tn + (1.0 - lambda) * cn;
    if (t_norm) t_norm[i] = tn;
    if (c_norm) c_norm[i] = cn;
    if (score) score[i] = sc;
    if (i == 0) best_score = sc;
    if (sc < best_score) { best = i; best_score = sc; }
  }
  return best;
}

/* scale — proj/src/planner.cpp:159-218, restated: the (pred desc, id asc)
 * order is the same for every candidate, so it is computed once. */
int orc_scale(const double* pred, const int32_t* plen, const int32_t* id_rank,
              int32_t count, const rs_profile* p, int32_t g, int32_t n_min,
              int32_t n_max, double lambda, int32_t gpus,
              const double* t_penalty, int32_t* n_star, double* t_total,
              double* t_pen_out, double* cost, double* t_norm, double* c_norm,
              double* score, int32_t* order, double* actor_times) {
  if (n_min < 1 || n_min > n_max) return fail(1, "scale: need 1 <= n_min <= n_max");
  if (n_max > count) return fail(1, "scale: n_max exceeds prompt count");
  if (lambda < 0 || lambda > 1) return fail(2, "scale: lambda must be in [0, 1]");
  if (g < 1) return fail(1, "estimate_actor_time: responses_per_prompt >= 1");
  for (int32_t i = 0; i < count; ++i)
    if (pred[i] < 1) return fail(1, "integrate_decode_seconds: target length < 1");
  int32_t nc = n_max - n_min + 1;
  rank_t* v = rank_prompts(pred, id_rank, count);
  resp_t* scratch = malloc(sizeof(resp_t) * count);
  int32_t* suf = malloc(sizeof(int32_t) * (count + 1));
  double* tt = malloc(sizeof(double) * nc);
  double* cc = malloc(sizeof(double) * nc);
  for (int32_t n = n_min; n <= n_max; ++n) {
    int32_t q = count / n, r = count % n, pos = 0;
    double t_tot = 0, dollars = 0;
    for (int32_t a = 0; a < n; ++a) {
      int32_t size = q + (a < r ? 1 : 0);
      double t = group_time(v, plen, pos, pos + size, g, p, scratch, suf);
      t_tot = t_tot < t ? t : t_tot;                         /* :184 */
      dollars += p->rho * t * gpus;                          /* :185 */
      pos += size;
    }
    tt[n - n_min] = t_tot;
    cc[n - n_min] = dollars;
  }
  int32_t best = select_best(tt, t_penalty, cc, nc, lambda, t_norm, c_norm, score);
  *n_star = n_min + best;
  for (int32_t i = 0; i < nc; ++i) {
    if (t_total) t_total[i] = tt[i];
    if (cost) cost[i] = cc[i];
    if (t_pen_out) t_pen_out[i] = t_penalty ? t_penalty[i] : 0.0;
  }
  if (order) for (int32_t i = 0; i < count; ++i) order[i] = v[i].idx;
  if (actor_times) {
    int32_t n = *n_star, q = count / n, r = count % n, pos = 0;
    for (int32_t a = 0; a < n; ++a) {
      int32_t size = q + (a < r ? 1 : 0);
      actor_times[a] = group_time(v, plen, pos, pos + size, g, p, scratch, suf);
      pos += size;
    }
  }
  free(v); free(scratch); free(suf); free(tt); free(cc);
  return 0;
}

/* ---- placement penalty: plan_rlhfless's TimePenaltyFn
 * (training.cpp:150-164) = place() (placement.cpp:177-291) + check_overlap()
 * (placement.cpp:339-363) with transfers_for (training.cpp:68-80). Restated
 * actor by actor, as the reference does it. */
static double topo_bw(const rs_topology* t, int a, int b) {
  if (t->bw_matrix) return t->bw_matrix[(size_t)a * t->n_nodes + b];
  return a == b ? t->intra_node_bw : t->inter_node_bw;
}

static int topo_validate(const rs_topology* t) {                 /* placement.cpp:28-62 */
  if (t->n_nodes < 1) return fail(2, "topology needs at least one node");
  for (int i = 0; i < t->n_nodes; ++i)
    if (t->node_gpus[i] < 1) return fail(2, "every node needs at least one GPU");
  if (!t->bw_matrix) {
    if (!(t->intra_node_bw > 0) || !(t->inter_node_bw > 0)) return fail(2, "bandwidths must be positive");
    if (t->intra_node_bw < t->inter_node_bw) return fail(2, "intra-node bandwidth below inter-node bandwidth");
  } else {
    for (int i = 0; i < t->n_nodes; ++i)
      for (int j = 0; j < t->n_nodes; ++j) {
        double v = t->bw_matrix[(size_t)i * t->n_nodes + j];
        if (!(v > 0)) return fail(2, "bandwidth matrix entries must be positive");
        if (v != t->bw_matrix[(size_t)j * t->n_nodes + i]) return fail(2, "bandwidth matrix must be symmetric");
      }
  }
  if (t->learner_node < 0 || t->learner_node >= t->n_nodes) return fail(2, "learner_node out of range");
  if (t->n_learner_gpus < 1) return fail(2, "learner needs at least one GPU");
  for (int k = 0; k < t->n_learner_gpus; ++k)
    if (t->learner_gpus[k] < 0 || t->learner_gpus[k] >= t->node_gpus[t->learner_node])
      return fail(2, "learner GPU index out of range");
  return 0;
}

static int placement_penalty(const rs_placement_penalty* pen, int32_t n, const double* times,
                             const int64_t* tokens, int32_t gpus, double* out) {
  const rs_topology* t = pen->topology;
  int rc = topo_validate(t);
  if (rc) return rc;
  if (!(pen->model_bytes >= 0) || !isfinite(pen->model_bytes))    /* placement.cpp:151-152 */
    return fail(2, "model_bytes must be finite and >= 0");
  double* kv = malloc(sizeof(double) * n);
  double* lm = calloc(n, sizeof(double));
  double* lkv = calloc(n, sizeof(double));
  int32_t* order = malloc(sizeof(int32_t) * n);
  int32_t* rank = malloc(sizeof(int32_t) * t->n_nodes);
  int32_t* freeg = malloc(sizeof(int32_t) * t->n_nodes);
  rc = 0;
  for (int32_t i = 0; i < n; ++i) {
    kv[i] = (double)tokens[i] * pen->kv_bytes_per_token;           /* training.cpp:76-77 */
    if (!(kv[i] >= 0) || !isfinite(kv[i])) rc = fail(2, "kv bytes must be finite and >= 0");
  }
  if (!rc) {
    int32_t heaviest = 0;                                           /* placement.cpp:193-197 */
    for (int32_t i = 1; i < n; ++i) if (times[i] > times[heaviest]) heaviest = i;
    int32_t m = 0;
    order[m++] = heaviest;
    for (int32_t i = 0; i < n; ++i) if (i != heaviest) order[m++] = i;
    for (int32_t i = 2; i < n; ++i) {                               /* :201-205 stable by (t desc, idx asc) */
      int32_t x = order[i], j = i - 1;
      while (j >= 1 && (times[order[j]] < times[x] ||
                        (times[order[j]] == times[x] && order[j] > x))) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = x;
    }
    for (int k = 0; k < t->n_nodes; ++k) { rank[k] = k; freeg[k] = t->node_gpus[k]; }
    for (int k = 1; k < t->n_nodes; ++k) {                          /* :209-215 */
      int32_t x = rank[k], j = k - 1;
      double bx = topo_bw(t, x, t->learner_node);
      while (j >= 0) {
        double bj = topo_bw(t, rank[j], t->learner_node);
        if (bj < bx || (bj == bx && rank[j] > x)) { rank[j + 1] = rank[j]; --j; } else break;
      }
      rank[j + 1] = x;
    }
    int32_t coloc = -1;
    for (int32_t oi = 0; oi < n && !rc; ++oi) {                     /* :233-270 */
      int32_t actor = order[oi], placed = 0;
      if (oi == 0 && freeg[t->learner_node] >= gpus) {
        freeg[t->learner_node] -= gpus;
        coloc = actor;
        placed = 1;
      }
      for (int k = 0; k < t->n_nodes && !placed; ++k) {
        int nd = rank[k];
        if (freeg[nd] < gpus) continue;
        freeg[nd] -= gpus;
        double bw = topo_bw(t, nd, t->learner_node);
        lm[actor] = pen->model_bytes / bw;
        lkv[actor] = kv[actor] / bw;
        placed = 1;
      }
      if (!placed) rc = fail(6, "cannot place actor");
    }
    if (!rc) {
      int32_t ref = coloc;                                          /* :342-347 */
      if (ref < 0) { ref = 0; for (int32_t i = 1; i < n; ++i) if (times[i] > times[ref]) ref = i; }
      double d1 = times[ref], exposed = 0;
      for (int32_t i = 0; i < n; ++i) {
        if (i == ref) continue;
        double slack = (pen->l_prefill_seconds + d1) - (lm[i] + lkv[i] + times[i]);
        exposed = exposed < -slack ? -slack : exposed;              /* training.cpp:161-162 */
      }
      *out = exposed;
    }
  }
  free(kv); free(lm); free(lkv); free(order); free(rank); free(freeg);
  return rc;
}

int orc_scale_placed(const double* pred, const int32_t* plen, const int32_t* id_rank,
                     int32_t count, const rs_profile* p, int32_t g, int32_t n_min,
                     int32_t n_max, double lambda, int32_t gpus,
                     const rs_placement_penalty* pen, int32_t* n_star, double* t_total,
                     double* t_pen_out, double* cost, double* t_norm, double* c_norm,
                     double* score, int32_t* order, double* actor_times) {
  /* scale()'s own checks first (the penalty runs inside its loop) */
  int rc = orc_scale(pred, plen, id_rank, count, p, g, n_min, n_max, lambda, gpus, NULL, n_star,
                     NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL);
  if (rc) return rc;
  int32_t nc = n_max - n_min + 1;
  rank_t* v = rank_prompts(pred, id_rank, count);
  resp_t* scratch = malloc(sizeof(resp_t) * count);
  int32_t* suf = malloc(sizeof(int32_t) * (count + 1));
  double* tp = malloc(sizeof(double) * nc);
  double* times = malloc(sizeof(double) * n_max);
  int64_t* tokens = malloc(sizeof(int64_t) * n_max);
  for (int32_t n = n_min; n <= n_max && !rc; ++n) {
    int32_t q = count / n, r = count % n, pos = 0;
    for (int32_t a = 0; a < n; ++a) {
      int32_t size = q + (a < r ? 1 : 0);
      times[a] = group_time(v, plen, pos, pos + size, g, p, scratch, suf);
      tokens[a] = 0;
      for (int32_t k = pos; k < pos + size; ++k) tokens[a] += plen[v[k].idx];
      pos += size;
    }
    rc = placement_penalty(pen, n, times, tokens, gpus, &tp[n - n_min]);
  }
  if (!rc)
    rc = orc_scale(pred, plen, id_rank, count, p, g, n_min, n_max, lambda, gpus, tp, n_star,
                   t_total, t_pen_out, cost, t_norm, c_norm, score, order, actor_times);
  free(v); free(scratch); free(suf); free(tp); free(times); free(tokens);
  return rc;
}

/* ---- prediction snapshot: LengthHistory::predict / predict_noisy
 * (predictor.cpp:52-98), splitmix Rng (rng.hpp:14-49), fnv1a (rng.hpp:64-71). */
static uint64_t ors_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t ors_hash(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
static uint64_t ors_combine(uint64_t a, uint64_t b) {
  return ors_hash(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}
static uint64_t ors_next(uint64_t* st) { *st += 0x9e3779b97f4a7c15ULL; return ors_mix(*st); }
static double ors_uniform(uint64_t* st) { return (double)(ors_next(st) >> 11) * 0x1.0p-53; }
static double clamp_len(double est, double mlen) {                 /* predictor.cpp:64 */
  double lo = 1.0 < est ? est : 1.0;
  return lo < mlen ? lo : mlen;
}

int orc_predict_lengths(const double* obs, const int32_t* depth, const int32_t* gt,
                        int32_t count, int32_t window, double alpha, int32_t max_len,
                        const rs_noise_model* noise, const char* id_bytes,
                        const int64_t* id_offsets, double* out) {
  if (window < 1) return fail(2, "predictor window must be >= 1");  /* :24-31 */
  if (!(alpha > 0) || alpha > 1) return fail(2, "predictor alpha must be in (0, 1]");
  if (max_len < 1) return fail(2, "predictor max_response_len must be >= 1");
  int noisy = noise && noise->kind != 0;
  if (noisy) {                                                      /* :17-22 */
    if (noise->bucket_accuracy < 0 || noise->bucket_accuracy > 1)
      return fail(2, "noise bucket_accuracy must be in [0, 1]");
    if (noise->bucket_width < 1 || noise->bucket_width > max_len)
      return fail(2, "noise bucket_width must be in [1, max_response_len]");
  }
  double mlen = (double)max_len;
  for (int32_t i = 0; i < count; ++i) {
    double est;
    if (depth[i] == 0) {
      est = (double)gt[i];
    } else {                                                        /* :58-62 */
      const double* q = obs + (size_t)i * window;
      est = q[0];
      for (int32_t k = 1; k < depth[i]; ++k) est = alpha * q[k] + (1.0 - alpha) * est;
    }
    double base = clamp_len(est, mlen);
    out[i] = base;
    if (!noisy) continue;
    int32_t bc = (max_len + noise->bucket_width - 1) / noise->bucket_width;   /* :73-75 */
    if (bc <= 1) continue;
    uint64_t h = 0xcbf29ce484222325ULL, bits;
    for (int64_t b = id_offsets[i]; b < id_offsets[i + 1]; ++b) {
      h ^= (unsigned char)id_bytes[b];
      h *= 0x100000001b3ULL;
    }
    memcpy(&bits, &base, sizeof bits);
    uint64_t key = ors_combine(noise->seed, h);                     /* :79-84 */
    key = ors_combine(key, (uint64_t)depth[i]);
    key = ors_combine(key, bits);
    uint64_t st = key;
    if (ors_uniform(&st) < noise->bucket_accuracy) continue;        /* :86 */
    int32_t tb = (int32_t)((base - 1.0) / noise->bucket_width);
    if (tb > bc - 1) tb = bc - 1;
    int32_t wrong = (int32_t)(ors_next(&st) % (uint64_t)(bc - 1));  /* uniform_int(0, bc-2) */
    if (wrong >= tb) ++wrong;
    double lo = wrong * noise->bucket_width + 1.0;
    double hb = (double)((wrong + 1) * noise->bucket_width);
    double hi = mlen < hb ? mlen : hb;
    double v = lo + (hi - lo) * ors_uniform(&st);
    out[i] = clamp_len(v, mlen);
  }
  return 0;
}

typedef struct {
  const double* pred; const int32_t* plen; int32_t s0, s1, count;
  const rs_profile* p; int32_t g, n_min, n_max; double lambda; int32_t gpus;
  double* t_total; double* cost; int32_t* n_star; int status; char err[256];
} sweep_job_t;

static void* sweep_worker(void* arg) {
  sweep_job_t* j = arg;
  int32_t nc = j->n_max - j->n_min + 1;
  for (int32_t s = j->s0; s < j->s1 && !j->status; ++s) {
    j->status = orc_scale(j->pred + (size_t)s * j->count, j->plen + (size_t)s * j->count,
                          NULL, j->count, j->p, j->g, j->n_min, j->n_max, j->lambda,
                          j->gpus, NULL, &j->n_star[s], j->t_total + (size_t)s * nc, NULL,
                          j->cost + (size_t)s * nc, NULL, NULL, NULL, NULL, NULL);
    if (j->status) snprintf(j->err, sizeof(j->err), "%s", g_err);
  }
  return NULL;
}

/* The scenario sweep: scale() per scenario. */
int orc_sweep_arrays(const double* pred, const int32_t* plen,
                     int32_t n_scenarios, int32_t count, const rs_profile* p,
                     int32_t g, int32_t n_min, int32_t n_max, double lambda,
                     int32_t gpus, int32_t n_threads, double* t_total,
                     double* cost, int32_t* n_star) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > n_scenarios) n_threads = n_scenarios > 0 ? n_scenarios : 1;
  sweep_job_t* jobs = calloc(n_threads, sizeof(sweep_job_t));
  pthread_t* th = calloc(n_threads, sizeof(pthread_t));
  for (int32_t t = 0; t < n_threads; ++t) {
    sweep_job_t* j = &jobs[t];
    j->pred = pred; j->plen = plen; j->count = count; j->p = p; j->g = g;
    j->n_min = n_min; j->n_max = n_max; j->lambda = lambda; j->gpus = gpus;
    j->t_total = t_total; j->cost = cost; j->n_star = n_star;
    j->s0 = (int32_t)((int64_t)n_scenarios * t / n_threads);
    j->s1 = (int32_t)((int64_t)n_scenarios * (t + 1) / n_threads);
    if (t) pthread_create(&th[t], NULL, sweep_worker, j);
  }
  sweep_worker(&jobs[0]);
  for (int32_t t = 1; t < n_threads; ++t) pthread_join(th[t], NULL);
  int st = 0;
  for (int32_t t = 0; t < n_threads && !st; ++t)
    if (jobs[t].status) { st = jobs[t].status; snprintf(g_err, sizeof(g_err), "%s", jobs[t].err); }
  free(jobs); free(th);
  return st;
}

/* ------------------------------------------------------------------ */
/* dedup.cpp                                                            */
/* ------------------------------------------------------------------ */

typedef struct { const int32_t* tok; const int64_t* off; int32_t cap; } lex_ctx_t;
static __thread lex_ctx_t g_lex;

static int32_t plen_of(int32_t i) { return (int32_t)(g_lex.off[i + 1] - g_lex.off[i]); }

/* token_less — proj/src/dedup.cpp:14-19 (std::lexicographical_compare);
 * g_lex.cap > 0 truncates both sides like trunc_less (dedup.cpp:167-174). */
static int cmp_lex(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  int32_t nx = plen_of(x), ny = plen_of(y);
  if (g_lex.cap > 0) { if (nx > g_lex.cap) nx = g_lex.cap; if (ny > g_lex.cap) ny = g_lex.cap; }
  const int32_t* px = g_lex.tok + g_lex.off[x];
  const int32_t* py = g_lex.tok + g_lex.off[y];
  int32_t n = nx < ny ? nx : ny;
  for (int32_t i = 0; i < n; ++i)
    if (px[i] != py[i]) return px[i] < py[i] ? -1 : 1;
  if (nx != ny) return nx < ny ? -1 : 1;
  return (x > y) - (x < y); /* deterministic among equals (no effect on counts) */
}

typedef struct {
  int32_t batch, min_len, max_len; int64_t total;
  int64_t *nodes, *scb, *stb, *lcf, *ltf;
} pindex_t;

static void pindex_free(pindex_t* x) { free(x->nodes); free(x->scb); free(x->stb); free(x->lcf); free(x->ltf); }

/* PrefixIndex::build — proj/src/dedup.cpp:30-100. */
static int pindex_build(const int32_t* tok, const int64_t* off, int32_t batch, pindex_t* ix) {
  memset(ix, 0, sizeof(*ix));
  if (batch <= 0) return fail(1, "prefix index needs a non-empty batch");   /* :31 */
  for (int32_t i = 0; i < batch; ++i)                                        /* :32-35 */
    if (off[i + 1] - off[i] < 1) return fail(1, "prefix index: empty prompt in batch");
  ix->batch = batch;
  int32_t* s = malloc(sizeof(int32_t) * batch);
  for (int32_t i = 0; i < batch; ++i) s[i] = i;
  g_lex.tok = tok; g_lex.off = off; g_lex.cap = 0;
  qsort(s, batch, sizeof(int32_t), cmp_lex);                                 /* :39-40 */
  ix->min_len = plen_of(s[0]); ix->max_len = 0;
  for (int32_t i = 0; i < batch; ++i) {                                      /* :42-47 */
    int32_t l = plen_of(s[i]);
    if (l < ix->min_len) ix->min_len = l;
    if (l > ix->max_len) ix->max_len = l;
    ix->total += l;
  }
  int32_t maxd = ix->max_len;
  int64_t* node_diff = calloc(maxd + 2, sizeof(int64_t));
  int64_t* end_count = calloc(maxd + 1, sizeof(int64_t));
  int64_t* len_count = calloc(maxd + 1, sizeof(int64_t));
  int32_t prev = -1;
  for (int32_t k = 0; k < batch; ++k) {                                      /* :57-71 */
    int32_t p = s[k], lp = plen_of(p);
    len_count[lp] += 1;
    if (prev >= 0) {
      int32_t lq = plen_of(prev), n = lp < lq ? lp : lq, lcp = 0;
      const int32_t* a = tok + off[prev];
      const int32_t* b = tok + off[p];
      while (lcp < n && a[lcp] == b[lcp]) ++lcp;                             /* :21-26 */
      if (lcp == lq && lcp == lp) continue;
      node_diff[lcp + 1] += 1;
      node_diff[lp + 1] -= 1;
    } else {
      node_diff[1] += 1;
      node_diff[lp + 1] -= 1;
    }
    end_count[lp] += 1;
    prev = p;
  }
  ix->nodes = calloc(maxd + 1, sizeof(int64_t));                             /* :73-78 */
  int64_t run = 0;
  for (int32_t d = 1; d <= maxd; ++d) { run += node_diff[d]; ix->nodes[d] = run; }
  ix->scb = calloc(maxd + 2, sizeof(int64_t));                               /* :80-87 */
  ix->stb = calloc(maxd + 2, sizeof(int64_t));
  for (int32_t d = 1; d <= maxd + 1; ++d) {
    ix->scb[d] = ix->scb[d - 1] + (d - 1 >= 1 ? end_count[d - 1] : 0);
    ix->stb[d] = ix->stb[d - 1] + (d - 1 >= 1 ? end_count[d - 1] * (d - 1) : 0);
  }
  ix->lcf = calloc(maxd + 2, sizeof(int64_t));                               /* :89-97 */
  ix->ltf = calloc(maxd + 2, sizeof(int64_t));
  for (int32_t d = maxd; d >= 0; --d) {
    ix->lcf[d] = ix->lcf[d + 1] + (d + 1 <= maxd ? len_count[d + 1] : 0);
    ix->ltf[d] = ix->ltf[d + 1] + (d + 1 <= maxd ? len_count[d + 1] * (d + 1) : 0);
  }
  free(s); free(node_diff); free(end_count); free(len_count);
  return 0;
}

/* unique_prefix_count / _tokens / remainder_tokens — dedup.cpp:102-122. */
static int64_t px_count(const pindex_t* ix, int32_t l) {
  int32_t m = l < ix->max_len ? l : ix->max_len;
  return ix->nodes[m] + ix->scb[m];
}
static int64_t px_tokens(const pindex_t* ix, int32_t l) {
  int32_t m = l < ix->max_len ? l : ix->max_len;
  return ix->nodes[m] * m + ix->stb[m];
}
static int64_t px_rem(const pindex_t* ix, int32_t l) {
  if (l >= ix->max_len) return 0;
  return ix->ltf[l] - ix->lcf[l] * l;
}

int orc_prefix_tables(const int32_t* tok, const int64_t* off, int32_t batch,
                      int64_t* info, int64_t* nodes, int64_t* scb,
                      int64_t* stb, int64_t* lcf, int64_t* ltf) {
  pindex_t ix;
  int st = pindex_build(tok, off, batch, &ix);
  if (st) return st;
  info[0] = ix.batch; info[1] = ix.min_len; info[2] = ix.max_len; info[3] = ix.total;
  int32_t m = ix.max_len;
  if (nodes) memcpy(nodes, ix.nodes, sizeof(int64_t) * (m + 1));
  if (scb) memcpy(scb, ix.scb, sizeof(int64_t) * (m + 2));
  if (stb) memcpy(stb, ix.stb, sizeof(int64_t) * (m + 2));
  if (lcf) memcpy(lcf, ix.lcf, sizeof(int64_t) * (m + 2));
  if (ltf) memcpy(ltf, ix.ltf, sizeof(int64_t) * (m + 2));
  pindex_free(&ix);
  return 0;
}

int orc_prefix_curves(const int32_t* tok, const int64_t* off, int32_t batch,
                      int32_t n_l, int64_t* info, int64_t* ucount,
                      int64_t* utokens, int64_t* rem) {
  pindex_t ix;
  int st = pindex_build(tok, off, batch, &ix);
  if (st) return st;
  info[0] = ix.batch; info[1] = ix.min_len; info[2] = ix.max_len; info[3] = ix.total;
  for (int32_t l = 1; l <= n_l; ++l) {
    ucount[l - 1] = px_count(&ix, l);
    utokens[l - 1] = px_tokens(&ix, l);
    rem[l - 1] = px_rem(&ix, l);
  }
  pindex_free(&ix);
  return 0;
}

/* select_prefix_length — proj/src/dedup.cpp:124-144. */
int orc_select_prefix_length(const int32_t* tok, const int64_t* off,
                             int32_t batch, int32_t cap, int32_t gpus,
                             int32_t l_min, int32_t l_max, int32_t* len,
                             int32_t* exceeded) {
  (void)gpus;
  pindex_t ix;
  int st = pindex_build(tok, off, batch, &ix);
  if (st) return st;
  if (l_min < 1 || l_min > l_max) { pindex_free(&ix); return fail(1, "select_prefix_length: need 1 <= l_min <= l_max"); }
  if (cap < 1) { pindex_free(&ix); return fail(2, "prefill capacity must allow at least one prefix"); }
  if (px_count(&ix, l_min) > cap) { *len = l_min; *exceeded = 1; pindex_free(&ix); return 0; }
  int32_t lo = l_min, hi = l_max;
  while (lo < hi) {
    int32_t mid = lo + (hi - lo + 1) / 2;
    if (px_count(&ix, mid) <= cap) lo = mid; else hi = mid - 1;
  }
  *len = lo; *exceeded = 0;
  pindex_free(&ix);
  return 0;
}

/* dedup_savings — proj/src/dedup.cpp:146-161. */
int orc_dedup_savings(const int32_t* tok, const int64_t* off, int32_t batch,
                      int32_t l_star, int32_t g, int64_t* raw, int64_t* dedup,
                      double* frac) {
  pindex_t ix;
  int st = pindex_build(tok, off, batch, &ix);
  if (st) return st;
  if (g < 1) { pindex_free(&ix); return fail(1, "dedup_savings: responses_per_prompt must be >= 1"); }
  if (l_star < 1) { pindex_free(&ix); return fail(1, "unique_prefix_tokens: prefix_len must be >= 1"); }
  *raw = ix.total * (int64_t)g;
  *dedup = px_tokens(&ix, l_star) + px_rem(&ix, l_star);
  *frac = *raw == 0 ? 0.0 : (double)(*raw - *dedup) / (double)(*raw);
  pindex_free(&ix);
  return 0;
}

/* unique_prefix_count_among — proj/src/dedup.cpp:163-183. */
int orc_unique_prefix_count_among(const int32_t* tok, const int64_t* off,
                                  int32_t count, int32_t len, int64_t* out) {
  if (len < 1) return fail(1, "unique_prefix_count_among: prefix_len must be >= 1");
  if (count <= 0) { *out = 0; return 0; }
  int32_t* s = malloc(sizeof(int32_t) * count);
  for (int32_t i = 0; i < count; ++i) s[i] = i;
  g_lex.tok = tok; g_lex.off = off; g_lex.cap = len;
  qsort(s, count, sizeof(int32_t), cmp_lex);
  int64_t distinct = 1;
  for (int32_t i = 1; i < count; ++i) {
    /* trunc_less(prev, cur): compare truncated sequences only (no index tie) */
    int32_t x = s[i - 1], y = s[i];
    int32_t nx = plen_of(x), ny = plen_of(y);
    if (nx > len) nx = len;
    if (ny > len) ny = len;
    int32_t n = nx < ny ? nx : ny, k = 0;
    const int32_t* px = tok + off[x];
    const int32_t* py = tok + off[y];
    while (k < n && px[k] == py[k]) ++k;
    if (k < n || nx != ny) ++distinct;
  }
  free(s);
  *out = distinct;
  g_lex.cap = 0;
  return 0;
}

/* ------------------------------------------------------------------ */
/* Builder-defined oracles (no reference equivalent). */
/* ------------------------------------------------------------------ */

/* rng.hpp:14-71 primitives. */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t hash_u64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}
static uint64_t hash_combine(uint64_t a, uint64_t b) {
  return hash_u64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}
/* k-th next_u64() (k >= 1) of Rng(seed): splitmix64's state advances by a
 * constant, so any draw is addressable. rng.hpp:20-25. */
static uint64_t draw_at(uint64_t seed, uint64_t k) {
  return mix64(seed + k * 0x9e3779b97f4a7c15ULL);
}

/* Quantile interpolation of the generator tables. */
static double qinterp(const double* t, uint64_t u) {
  uint64_t j = u >> 52;
  double f = (double)((u >> 11) & ((1ULL << 41) - 1)) * 0x1.0p-41;
  return t[j] + (t[j + 1] - t[j]) * f;
}

int orc_generate_scenarios(const rs_scenario_spec* sp, double* pred, int32_t* plen) {
  for (int32_t s = 0; s < sp->n_scenarios; ++s) {
    uint64_t seed = hash_combine(sp->base_seed, (uint64_t)(sp->first_scenario + s));
    for (int32_t i = 0; i < sp->count; ++i) {
      uint64_t u1 = draw_at(seed, 2 * (uint64_t)i + 1);
      uint64_t u2 = draw_at(seed, 2 * (uint64_t)i + 2);
      double z = qinterp(RS_NZ, u1);
      double pl = round(sp->plen_mean + sp->plen_sigma * z);
      if (pl < sp->plen_min) pl = sp->plen_min;
      if (pl > sp->plen_max) pl = sp->plen_max;
      double pr = sp->pred_scale * qinterp(RS_LNZ, u2);
      if (pr < sp->pred_min) pr = sp->pred_min;
      if (pr > sp->pred_max) pr = sp->pred_max;
      plen[(size_t)s * sp->count + i] = (int32_t)pl;
      pred[(size_t)s * sp->count + i] = pr;
    }
  }
  return 0;
}

/* Reference-model idle slot-ticks per candidate: for the contiguous split of
 * scale(), sum over groups and responses of (group max ceil - own ceil). */
int orc_scale_idle(const double* pred, const int32_t* id_rank, int32_t count,
                   int32_t g, int32_t n_min, int32_t n_max, int64_t* idle) {
  rank_t* v = rank_prompts(pred, id_rank, count);
  for (int32_t n = n_min; n <= n_max; ++n) {
    int32_t q = count / n, r = count % n, pos = 0;
    int64_t tot = 0;
    for (int32_t a = 0; a < n; ++a) {
      int32_t size = q + (a < r ? 1 : 0);
      int64_t mx = (int64_t)ceil(v[pos].pred);
      for (int32_t i = pos; i < pos + size; ++i) tot += (int64_t)g * (mx - (int64_t)ceil(v[i].pred));
      pos += size;
    }
    idle[n - n_min] = tot;
  }
  free(v);
  return 0;
}

/* Dedup map: labels[i] = smallest index whose truncated-to-len sequence
 * equals prompt i's (trunc as in dedup.cpp:167-174). */
int orc_dedup_map(const int32_t* tok, const int64_t* off, int32_t count,
                  int32_t len, int32_t* labels) {
  if (len < 1) return fail(1, "dedup_map: prefix_len must be >= 1");
  if (count <= 0) return 0;
  int32_t* s = malloc(sizeof(int32_t) * count);
  for (int32_t i = 0; i < count; ++i) s[i] = i;
  g_lex.tok = tok; g_lex.off = off; g_lex.cap = len;
  qsort(s, count, sizeof(int32_t), cmp_lex);  /* index breaks ties: class head = min */
  int32_t head = s[0];
  labels[s[0]] = head;
  for (int32_t i = 1; i < count; ++i) {
    int32_t x = s[i - 1], y = s[i];
    int32_t nx = plen_of(x), ny = plen_of(y);
    if (nx > len) nx = len;
    if (ny > len) ny = len;
    int same = nx == ny && memcmp(tok + off[x], tok + off[y], sizeof(int32_t) * nx) == 0;
    if (!same) head = y;
    labels[y] = head;
  }
  g_lex.cap = 0;
  free(s);
  return 0;
}

/* Chained block hash. */
#define RS_HASH_MUL 0x9e3779b97f4a7c15ULL
#define RS_HASH_SEED 0x243f6a8885a308d3ULL
int orc_block_hashes(const int32_t* tok, const int64_t* off, int32_t count,
                     int32_t block_tokens, uint64_t* hashes) {
  if (block_tokens < 1) return fail(1, "block_hashes: block_tokens must be >= 1");
  int64_t w = 0;
  for (int32_t i = 0; i < count; ++i) {
    int64_t len = off[i + 1] - off[i];
    const int32_t* t = tok + off[i];
    uint64_t h = RS_HASH_SEED;
    for (int64_t b0 = 0; b0 < len; b0 += block_tokens) {
      int64_t m = len - b0 < block_tokens ? len - b0 : block_tokens;
      uint64_t poly = 0;
      for (int64_t k = 0; k < m; ++k) poly = poly * RS_HASH_MUL + ((uint64_t)(uint32_t)t[b0 + k] + 1);
      h = hash_combine(h, hash_u64(poly ^ ((uint64_t)m << 56)));
      hashes[w++] = h;
    }
  }
  return 0;
}

/* LPT bin-pack. */
typedef struct { int64_t len; int32_t id; int32_t r; } lpt_item_t;
static int cmp_lpt(const void* a, const void* b) {
  const lpt_item_t* x = a; const lpt_item_t* y = b;
  if (x->len != y->len) return x->len > y->len ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return (x->r > y->r) - (x->r < y->r);
}
int orc_lpt(const double* pred, const int32_t* id_rank, int32_t count,
            int32_t g, int32_t n_min, int32_t n_max, int64_t* makespan,
            int64_t* idle) {
  int64_t n_items = (int64_t)count * g;
  lpt_item_t* it = malloc(sizeof(lpt_item_t) * (n_items > 0 ? n_items : 1));
  for (int32_t i = 0; i < count; ++i)
    for (int32_t r = 0; r < g; ++r) {
      lpt_item_t* e = &it[(int64_t)i * g + r];
      e->len = (int64_t)ceil(pred[i]); e->id = id_rank ? id_rank[i] : i; e->r = r;
    }
  qsort(it, n_items, sizeof(lpt_item_t), cmp_lpt);
  int64_t* load = malloc(sizeof(int64_t) * n_max);
  for (int32_t n = n_min; n <= n_max; ++n) {
    memset(load, 0, sizeof(int64_t) * n);
    for (int64_t k = 0; k < n_items; ++k) {
      int32_t best = 0;
      for (int32_t a = 1; a < n; ++a) if (load[a] < load[best]) best = a;
      load[best] += it[k].len;
    }
    int64_t mk = 0, tot = 0;
    for (int32_t a = 0; a < n; ++a) { if (load[a] > mk) mk = load[a]; tot += load[a]; }
    makespan[n - n_min] = mk;
    idle[n - n_min] = mk * n - tot;
  }
  free(it); free(load);
  return 0;
}

/* Aggregate pick over a sweep: normalise mean t / mean c like scale(). */
int orc_sweep_select(const double* sum_t, const double* sum_c,
                     int64_t n_scenarios, int32_t n_candidates, int32_t n_min,
                     double lambda, int32_t* n_star) {
  double* mt = malloc(sizeof(double) * n_candidates);
  double* mc = malloc(sizeof(double) * n_candidates);
  for (int32_t i = 0; i < n_candidates; ++i) {
    mt[i] = sum_t[i] / (double)n_scenarios;
    mc[i] = sum_c[i] / (double)n_scenarios;
  }
  *n_star = n_min + select_best(mt, NULL, mc, n_candidates, lambda, NULL, NULL, NULL);
  free(mt); free(mc);
  return 0;
}
