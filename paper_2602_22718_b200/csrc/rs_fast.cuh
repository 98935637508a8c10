// rs_fast.cuh — the fast scaling-sweep path (bucketed finish ticks).
#pragma once
#include "rs_internal.cuh"

namespace rs {

// Packed, rank-ordered scenario structure of the fast path. Scenario s owns
// items [item_off[s], item_off[s+1]) and segment slots starting at
// item_off[s] + s (D_s + 1 slots).
//   seg[k]   = {F_k | MX_k << 16, E_k}: finish tick, max prompt_len and end
//              rank of run-segment k (segments in descending finish order)
//   segCF[k] = sum_{k' < k} count_k' * F_k'   (segCF[D] = total)
//   rinfo[r] = {seg_of(r), smx(r) | pmx(r) << 16} with smx / pmx the max
//              prompt_len from r to the end / from the start of r's segment
struct FastSS {
  const int* flags;  // the context's status word: kFastBad set -> structure unusable
  const int64_t* item_off;
  int2* seg;
  int64_t* segCF;
  int32_t* nseg;
  int2* rinfo;
  int32_t* plen_r;
  int32_t* order_r;
  int4* rec;  // scratch: scattered {pred lo, pred hi, idx, plen}
  // Range-max helpers over the per-segment max prompt_len (16-segment blocks):
  uint32_t* pmsm;  // per segment slot: in-block prefix max | in-block suffix max << 16
  uint16_t* st;    // per scenario: sparse table over block maxima, [kStLevels][kStBlocks]
  uint16_t* bq;    // per 16-segment block: max MX over [i, j], in-block i <= j (kBlkPairs u16,
                   // upper triangle row-major); block jb of scenario s at slot (so >> 4) + s + jb
};

constexpr int kFastFmax = 16384;   // finish ticks of the fast path
constexpr int kFastPlenMax = 65535;
constexpr int kBlk = 16;           // segment block of the lane evaluator
constexpr int kBlkPairs = kBlk * (kBlk + 1) / 2;  // 136 in-block ranges
static_assert(kBlkPairs % 4 == 0, "bq rows are written as 64-bit words");
__host__ __device__ constexpr int blk_pair(int i, int j) { return i * (2 * kBlk + 1 - i) / 2 + (j - i); }
constexpr int kMaxSeg = kFastFmax; // D <= Fmax
constexpr int kTopCap = 4096;      // smem tpot row entries
constexpr int kStBlocks = kMaxSeg / kBlk;  // 1024
constexpr int kStLevels = 11;              // floor(log2(1024)) + 1
constexpr int kStStride = kStBlocks * kStLevels;

size_t fast_ss_bytes(int64_t items, int S);
FastSS fast_ss_alloc(rs_ctx* ctx, const int64_t* d_off, int64_t items, int S);

struct GenSpec {
  uint64_t base_seed;
  int64_t first;
  int count;
  double plen_mean, plen_sigma;
  int plen_min, plen_max;
  double pred_scale, pred_min, pred_max;
};

// kShared: t is a shared-memory copy of the table (generic loads).
template <bool kShared = false>
__device__ __forceinline__ double fast_qinterp(const double* t, uint64_t u) {
  uint64_t j = u >> 52;
  double f = dmul((double)((u >> 11) & ((1ULL << 41) - 1)), 0x1.0p-41);
  double a = kShared ? t[j] : __ldg(t + j), b = kShared ? t[j + 1] : __ldg(t + j + 1);
  return dadd(a, dmul(dsub(b, a), f));
}

// The predicted length of scenario item i (its second draw).
template <bool kShared = false>
__device__ __forceinline__ double fast_gen_pred(const GenSpec& g, const double* lnz, uint64_t seed,
                                                int i) {
  uint64_t u2 = draw_at(seed, 2 * (uint64_t)i + 2);
  double pr = dmul(g.pred_scale, fast_qinterp<kShared>(lnz, u2));
  pr = pr < g.pred_min ? g.pred_min : pr;
  pr = pr > g.pred_max ? g.pred_max : pr;
  return pr;
}

// Scenario item i of one Monte-Carlo scenario (oracle:
// orc_generate_scenarios): two splitmix64 draws -> quantile interpolation.
template <bool kShared = false>
__device__ __forceinline__ void fast_gen(const GenSpec& g, const double* nz, const double* lnz,
                                         uint64_t seed, int i, double* pred, int32_t* plen) {
  uint64_t u1 = draw_at(seed, 2 * (uint64_t)i + 1);
  double z = fast_qinterp<kShared>(nz, u1);
  double pl = round(dadd(g.plen_mean, dmul(g.plen_sigma, z)));
  pl = pl < (double)g.plen_min ? (double)g.plen_min : pl;
  pl = pl > (double)g.plen_max ? (double)g.plen_max : pl;
  *pred = fast_gen_pred<kShared>(g, lnz, seed, i);
  *plen = (int32_t)pl;
}

// Build the fast structure for S scenarios (one CTA each). When gen is
// non-null the scenarios are generated on the device (written to pred/plen
// only when keep_inputs; the sweep does not need them); otherwise pred/plen
// are read. Sets kFlagBucketOverflow in ctx->d_flags if an input is outside
// the fast path's range.
int fast_build(rs_ctx* ctx, int S, const int64_t* d_off, double* pred, int32_t* plen,
               FastSS ss, const GenSpec* gen, const double* nz, const double* lnz,
               bool keep_inputs = true, bool need_order = true);

struct CandRange {
  int n_min, n_max;
  int64_t T;  // groups per scenario over [n_min, n_max]
  int G;
};

// Evaluate every group of every candidate for S scenarios: gt[s*T + flat].
// units_per_scenario splits a scenario's candidates over several CTAs.
int fast_eval(rs_ctx* ctx, int S, const FastSS& ss, const DevProfile& prof, CandRange cr,
              int units_per_scenario, double* gt);

// The fast evaluator needs exact memo tables small enough for its row cache.
bool fast_profile_ok(const DevProfile& prof, int G);
size_t fast_eval_bytes(const DevProfile& prof, int G);

// Candidate-lockstep evaluator (large S): lanes are candidates walking
// the scenario's segments k = D-1 .. 0 together.
// Optional fused tail for the lockstep evaluator: per (scenario, candidate)
// t_total / cost / idle (like fast_reduce) and, when the candidate range fits
// one CTA (lockstep_fuses_select), n_star (like select_kernel).
struct LsFuse {
  double* tt;
  double* cc;
  int64_t* idle;
  int32_t* n_star;
  double rho;
  double lambda;
  int gpus;
};
// ctas_per_sm > 0: persistent grid of that many CTAs per SM (each loops over
// scenarios); 0: as many as fit.
int lockstep_eval(rs_ctx* ctx, int S, const FastSS& ss, const DevProfile& prof, CandRange cr,
                  double* gt, const LsFuse* fuse = nullptr, int ctas_per_sm = 0);
bool lockstep_fuses_select(CandRange cr);
// The lockstep evaluator's profile limits (context memo, shared memory).
bool lockstep_ok(const DevProfile& prof, int G);
// CTA slots of the lockstep evaluator on this device (one scenario each).
int lockstep_slots(rs_ctx* ctx, const DevProfile& prof, int G);

// Per (scenario, candidate): t_total, cost, idle slot-ticks.
int fast_reduce(rs_ctx* ctx, int S, const FastSS& ss, CandRange cr, double rho, int gpus,
                const double* gt, double* t_total, double* cost, int64_t* idle);

}  // namespace rs
