// rs_planner.cu — length-aware assignment (2) and cost-aware actor scaling
// (3) of the RLHFless planning core on sm_100a.
//
// Reference semantics (proj/src/planner.cpp):
//   assign            :16-51   sort (pred desc, id asc) + contiguous split
//   run sum           :61-84   per knot piece count*(tpot(lo)+tpot(hi))/2
//   integrate         :88-130  runs of equal ceil(target), ascending, summed
//                              sequentially; batch = live responses, context
//                              = max live prompt_len + tick - 1
//   estimate_actor_time :132-146 (G copies per prompt), estimate_cost :148-157
//   scale             :159-218 per-candidate max/sum, min-max normalise,
//                              first strict argmin
//
// Device pipeline: every "scenario" (one predicted-length
// vector) is turned into a rank-ordered scenario structure (SS):
//   plen_r[r], order_r[r], seg_of[r]          r = rank (pred desc, id asc)
//   segF[k], segS[k], segMX[k], segCF[k]      k = run of equal ceil(pred)
// built either by a per-scenario bucket sort in shared memory (finish ticks
// <= 16384, the Monte-Carlo path) or by the generic radix sort. Then one warp
// evaluates one (scenario, candidate N, group g): the group is the contiguous
// rank range [a, b); its runs are the segments it spans, taken in ascending
// finish order; each lane evaluates one run (prefix-max base via a warp
// scan + carry), and the lanes' run sums are added in lane order so the FP64
// sum is the reference's sequential sum bit for bit.
#include <algorithm>
#include <numeric>
#include <cmath>
#include <cstring>
#include <vector>

#include "rs_scenario_tables.h"
#include "rs_fast.cuh"
#include "rs_placement.cuh"
#include "rs_sort.cuh"

namespace rs {

// ---------------------------------------------------------------- views --
struct SSView {
  int S;
  const int64_t* item_off;  // S+1
  const int32_t* plen_r;
  const int32_t* order_r;
  const int32_t* seg_of;
  const int64_t* segF;   // segment arrays of scenario s start at item_off[s]+s
  const int32_t* segS;   // k in [0, D]; segS[D] = P_s
  const int32_t* segMX;
  const int64_t* segCF;  // exclusive prefix of count*F, segCF[D] = total
  const int32_t* nseg;
};

struct SSBuffers {
  int32_t* plen_r;
  int32_t* order_r;
  int32_t* seg_of;
  int64_t* segF;
  int32_t* segS;
  int32_t* segMX;
  int64_t* segCF;
  int32_t* nseg;
  int32_t* tmp_idx;
};

static size_t ss_bytes(int64_t items, int S) {
  int64_t segs = items + S;
  return abytes(items, 4) * 4 + abytes(segs, 8) * 2 + abytes(segs, 4) * 2 +
         abytes(S, 4);
}

static SSBuffers ss_alloc(rs_ctx* ctx, int64_t items, int S) {
  int64_t segs = items + S;
  SSBuffers b;
  b.plen_r = arena_alloc<int32_t>(ctx, items);
  b.order_r = arena_alloc<int32_t>(ctx, items);
  b.seg_of = arena_alloc<int32_t>(ctx, items);
  b.tmp_idx = arena_alloc<int32_t>(ctx, items);
  b.segF = arena_alloc<int64_t>(ctx, segs);
  b.segCF = arena_alloc<int64_t>(ctx, segs);
  b.segS = arena_alloc<int32_t>(ctx, segs);
  b.segMX = arena_alloc<int32_t>(ctx, segs);
  b.nseg = arena_alloc<int32_t>(ctx, S);
  return b;
}

static SSView ss_view(const SSBuffers& b, const int64_t* item_off, int S) {
  return SSView{S, item_off, b.plen_r, b.order_r, b.seg_of, b.segF,
                b.segS, b.segMX, b.segCF, b.nseg};
}

// --------------------------------------------------- scenario generation --
__global__ void gen_scenarios_kernel(GenSpec g, const double* nz,
                                     const double* lnz, int S, double* pred,
                                     int32_t* plen) {
  int64_t total = (int64_t)S * g.count;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int s = (int)(t / g.count), i = (int)(t % g.count);
    uint64_t seed = hash_combine(g.base_seed, (uint64_t)(g.first + s));
    fast_gen(g, nz, lnz, seed, i, pred + t, plen + t);
  }
}

constexpr int kBuildThreads = 1024;

// --------------------------------------------- generic structure builder --
// Input: rank-ordered pred_r / plen_r (after the radix sort). One CTA per
// scenario: segment flags, block scan, segment arrays.
__global__ void __launch_bounds__(kBuildThreads)
build_structure_kernel(const double* pred_r, const int64_t* item_off,
                       SSBuffers ss) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry_s;
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t i0 = item_off[s];
  const int P = (int)(item_off[s + 1] - i0);
  const int64_t so = i0 + s;
  if (tid == 0) carry_s = -1;
  __syncthreads();
  for (int t0 = 0; t0 < P; t0 += kBuildThreads) {
    int r = t0 + tid;
    bool valid = r < P;
    int64_t fin = valid ? (int64_t)ceil(pred_r[i0 + r]) : 0;
    int64_t prev = (valid && r > 0) ? (int64_t)ceil(pred_r[i0 + r - 1]) : -1;
    int flag = valid && (r == 0 || fin != prev) ? 1 : 0;
    int incl = warp_incl_sum(flag);
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int x = wsum[lane];
      wsum[lane] = warp_incl_sum(x) - x;
    }
    __syncthreads();
    int carry = carry_s;
    int seg = carry + wsum[wid] + incl;
    if (valid) {
      ss.seg_of[i0 + r] = seg;
      if (flag) {
        ss.segF[so + seg] = fin;
        ss.segS[so + seg] = r;
      }
    }
    __syncthreads();
    if (tid == kBuildThreads - 1) carry_s = seg;
    __syncthreads();
  }
  const int D = carry_s + 1;
  if (tid == 0) {
    ss.nseg[s] = D;
    ss.segS[so + D] = P;
  }
  __syncthreads();
  // Segment maxima: one warp per segment.
  for (int k = wid; k < D; k += kBuildThreads / 32) {
    int lo = ss.segS[so + k], hi = ss.segS[so + k + 1];
    int mx = INT32_MIN;
    for (int r = lo + lane; r < hi; r += 32) mx = max(mx, ss.plen_r[i0 + r]);
    mx = warp_max(mx);
    if (lane == 0) ss.segMX[so + k] = mx;
  }
  // segCF: exclusive prefix of count*F (one warp, sequential chunks).
  if (wid == 0) {
    int64_t run = 0;
    for (int k0 = 0; k0 < D; k0 += 32) {
      int k = k0 + lane;
      int64_t v = k < D ? (int64_t)(ss.segS[so + k + 1] - ss.segS[so + k]) * ss.segF[so + k] : 0;
      int64_t incl = warp_incl_sum(v);
      if (k < D) ss.segCF[so + k] = run + incl - v;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) ss.segCF[so + D] = run;
  }
}

// ---------------------------------------------------- group evaluation --
struct CandSpec {
  int n_min, n_max;
  int64_t T;  // groups per scenario = sum_{N=n_min}^{n_max} N
  int G;
};

__device__ __forceinline__ int64_t tri(int64_t n) { return n * (n - 1) / 2; }

// flat index within a scenario -> (N, g)
__device__ __forceinline__ void flat_to_ng(int64_t flat, int n_min, int* N, int* g) {
  int64_t x = flat + tri(n_min);
  int64_t n = (int64_t)floor((1.0 + sqrt(1.0 + 8.0 * (double)x)) * 0.5);
  while (n > 1 && tri(n) > x) --n;
  while (tri(n + 1) <= x) ++n;
  *N = (int)n;
  *g = (int)(x - tri(n));
}

constexpr int kEvalThreads = 256;
constexpr int kEvalWarps = kEvalThreads / 32;
constexpr int kCarry = 128;  // chunks of 32 runs per carry window

// Time of one group [a, b) of scenario s (all lanes return the same value).
__device__ double group_time_warp(const SSView& ss, const DevProfile& prof,
                                  int s, int a, int b, int G, int* carry_buf) {
  const int lane = lane_id();
  const int64_t i0 = ss.item_off[s];
  const int64_t so = i0 + s;
  const int32_t* plen = ss.plen_r + i0;
  const int32_t* sof = ss.seg_of + i0;
  const int64_t* F = ss.segF + so;
  const int32_t* Sg = ss.segS + so;
  const int32_t* MX = ss.segMX + so;
  if (b <= a) return 0.0;
  const int ka = __ldg(sof + a), kb = __ldg(sof + b - 1);
  if (ka == kb) {
    int m = INT32_MIN;
    for (int i = a + lane; i < b; i += 32) m = max(m, __ldg(plen + i));
    m = warp_max(m);
    int64_t f = __ldg(F + ka);
    double rs = run_sum_int(prof, (int64_t)G * (b - a), m, (int64_t)m + f - 1);
    return dadd(0.0, rs);
  }
  // Partial maxima of the two boundary segments.
  int va = INT32_MIN, vb = INT32_MIN;
  {
    int ea = __ldg(Sg + ka + 1);
    for (int i = a + lane; i < ea; i += 32) va = max(va, __ldg(plen + i));
    int sb = __ldg(Sg + kb);
    for (int i = sb + lane; i < b; i += 32) vb = max(vb, __ldg(plen + i));
    va = warp_max(va);
    vb = warp_max(vb);
  }
  auto vk_of = [&](int k) -> int {
    return k == ka ? va : (k == kb ? vb : __ldg(MX + k));
  };
  const int nk = kb - ka + 1;
  const int J = (nk + 31) >> 5;
  double total = 0.0;
  int64_t prevF = 0;
  for (int j0 = 0; j0 < J; j0 += kCarry) {
    const int j1 = min(J, j0 + kCarry);
    // max of v over all chunks below the window (lower k)
    int lm = INT32_MIN;
    for (int j = j1; j < J; ++j) {
      int k = kb - 32 * j - lane;
      if (k >= ka) lm = max(lm, vk_of(k));
    }
    int run = warp_max(lm);
    for (int j = j1 - 1; j >= j0; --j) {
      if (lane == 0) carry_buf[j - j0] = run;
      int k = kb - 32 * j - lane;
      int m = k >= ka ? vk_of(k) : INT32_MIN;
      run = max(run, warp_max(m));
    }
    __syncwarp();
    for (int j = j0; j < j1; ++j) {
      const int k = kb - 32 * j - lane;
      const bool act = k >= ka;
      int64_t Fk = act ? __ldg(F + k) : 0;
      int vk = act ? vk_of(k) : INT32_MIN;
      int xk = act ? (k == kb ? b : __ldg(Sg + k + 1)) : 0;
      int m = vk;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int u = __shfl_down_sync(0xffffffffu, m, o);
        if (lane + o < 32) m = max(m, u);
      }
      int base = max(m, carry_buf[j - j0]);
      int64_t Fup = __shfl_up_sync(0xffffffffu, Fk, 1);
      if (lane == 0) Fup = prevF;
      double rs = 0.0;
      if (act) {
        int64_t tstart = (k == kb) ? 1 : Fup + 1;
        int64_t live = xk - a;
        rs = run_sum_int(prof, (int64_t)G * live, (int64_t)base + tstart - 1,
                         (int64_t)base + Fk - 1);
      }
      const int nact = min(32, kb - 32 * j - ka + 1);
      for (int l = 0; l < nact; ++l) total = dadd(total, __shfl_sync(0xffffffffu, rs, l));
      prevF = __shfl_sync(0xffffffffu, Fk, 31);
    }
    __syncwarp();
  }
  return total;
}

__global__ void __launch_bounds__(kEvalThreads)
group_eval_kernel(SSView ss, DevProfile prof, CandSpec cs, double* gt) {
  __shared__ int carry[kEvalWarps][kCarry];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t W = (int64_t)gridDim.x * kEvalWarps;
  const int64_t total = (int64_t)ss.S * cs.T;
  for (int64_t item = (int64_t)blockIdx.x * kEvalWarps + wid; item < total; item += W) {
    int s = (int)(item / cs.T);
    int64_t flat = item - (int64_t)s * cs.T;
    int N, g;
    flat_to_ng(flat, cs.n_min, &N, &g);
    int P = (int)(ss.item_off[s + 1] - ss.item_off[s]);
    int q = P / N, r = P % N;
    int a = g * q + min(g, r);
    int b = a + q + (g < r ? 1 : 0);
    double t = group_time_warp(ss, prof, s, a, b, cs.G, carry[wid]);
    if (lane == 0) gt[item] = t;
  }
}

// Per (scenario, candidate): t_total = max, cost = sequential sum in group
// order (planner.cpp:181-186), reference-model idle slot-ticks.
__global__ void candidate_reduce_kernel(SSView ss, CandSpec cs, double rho,
                                        int gpus, const double* gt,
                                        double* t_total, double* cost,
                                        int64_t* idle) {
  const int C = cs.n_max - cs.n_min + 1;
  const int64_t total = (int64_t)ss.S * C;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int s = (int)(t / C), ci = (int)(t % C);
    int N = cs.n_min + ci;
    const double* g = gt + (int64_t)s * cs.T + (tri(N) - tri(cs.n_min));
    double tt = 0.0, dollars = 0.0;
    const double gd = (double)gpus;
    for (int k = 0; k < N; ++k) {
      double v = g[k];
      tt = tt < v ? v : tt;                          // std::max(t_total, t)
      dollars = dadd(dollars, dmul(dmul(rho, v), gd));  // rho * t * gpu_count
    }
    t_total[t] = tt;
    cost[t] = dollars;
    if (idle) {
      const int64_t i0 = ss.item_off[s];
      const int64_t so = i0 + s;
      const int P = (int)(ss.item_off[s + 1] - i0);
      const int D = ss.nseg[s];
      auto cfpos = [&](int p) -> int64_t {
        if (p >= P) return ss.segCF[so + D];
        int k = ss.seg_of[i0 + p];
        return ss.segCF[so + k] + (int64_t)(p - ss.segS[so + k]) * ss.segF[so + k];
      };
      int q = P / N, r = P % N;
      int64_t acc = 0;
      for (int k = 0; k < N; ++k) {
        int a = k * q + min(k, r), b = a + q + (k < r ? 1 : 0);
        if (b <= a) continue;
        int64_t fa = ss.segF[so + ss.seg_of[i0 + a]];
        acc += (int64_t)(b - a) * fa - (cfpos(b) - cfpos(a));
      }
      idle[t] = acc * cs.G;
    }
  }
}

// Normalise + first strict argmin (planner.cpp:196-217), one thread per
// scenario, sequential exactly like the reference.
// One warp per scenario: the minima and maxima of t (t_total + penalty) and
// cost are order-free over finite values; the first strict minimum of the
// score (planner.cpp:210-214) is the lexicographic (score, index) minimum.
__global__ void select_kernel(int S, int C, int n_min, double lambda,
                              const double* t_total, const double* t_pen,
                              const double* cost, double* t_norm,
                              double* c_norm, double* score, int32_t* n_star) {
  const int lane = threadIdx.x & 31;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < S;
       s += (gridDim.x * blockDim.x) >> 5) {
    const double* tt = t_total + (int64_t)s * C;
    const double* cc = cost + (int64_t)s * C;
    const double* tp = t_pen ? t_pen + (int64_t)s * C : nullptr;
    double t_min = dadd(tt[0], tp ? tp[0] : 0.0);  // planner.cpp:196-205
    double t_max = t_min, c_min = cc[0], c_max = c_min;
    for (int i = lane; i < C; i += 32) {
      const double t = dadd(tt[i], tp ? tp[i] : 0.0);
      t_min = t < t_min ? t : t_min;
      t_max = t_max < t ? t : t_max;
      c_min = cc[i] < c_min ? cc[i] : c_min;
      c_max = c_max < cc[i] ? cc[i] : c_max;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double a = __shfl_xor_sync(0xffffffffu, t_min, o), b = __shfl_xor_sync(0xffffffffu, t_max, o);
      const double c = __shfl_xor_sync(0xffffffffu, c_min, o), d = __shfl_xor_sync(0xffffffffu, c_max, o);
      t_min = a < t_min ? a : t_min;
      t_max = t_max < b ? b : t_max;
      c_min = c < c_min ? c : c_min;
      c_max = c_max < d ? d : c_max;
    }
    int best = INT32_MAX;
    double best_score = 0.0;
    for (int i = lane; i < C; i += 32) {
      const double t = dadd(tt[i], tp ? tp[i] : 0.0);
      const double tn = t_max > t_min ? ddiv(dsub(t, t_min), dsub(t_max, t_min)) : 0.0;
      const double cn = c_max > c_min ? ddiv(dsub(cc[i], c_min), dsub(c_max, c_min)) : 0.0;
      const double sc = dadd(dmul(lambda, tn), dmul(dsub(1.0, lambda), cn));
      if (t_norm) t_norm[(int64_t)s * C + i] = tn;
      if (c_norm) c_norm[(int64_t)s * C + i] = cn;
      if (score) score[(int64_t)s * C + i] = sc;
      if (best == INT32_MAX || sc < best_score) {  // ascending i per lane: first strict minimum
        best = i;
        best_score = sc;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, best_score, o);
      const int wi = __shfl_xor_sync(0xffffffffu, best, o);
      if (wi != INT32_MAX && (best == INT32_MAX || w < best_score || (!(best_score < w) && wi < best))) {
        best_score = w;
        best = wi;
      }
    }
    if (lane == 0) n_star[s] = n_min + best;
  }
}

// Sweep aggregate over this batch's scenarios: one warp per candidate, lane l
// sums scenarios l, l+32, ... in order, then a fixed shuffle tree
// (deterministic; the per-candidate sums are aggregates, compared at 1e-12).
__global__ void aggregate_kernel(int S, int C, int n_min, const double* t_total,
                                 const double* cost, const int32_t* n_star,
                                 double* sum_t, double* sum_c, int32_t* hist) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < C;
       i += (gridDim.x * blockDim.x) >> 5) {
    double st = 0.0, sc = 0.0;
    int h = 0;
    for (int s = lane; s < S; s += 32) {
      st = dadd(st, t_total[(int64_t)s * C + i]);
      sc = dadd(sc, cost[(int64_t)s * C + i]);
      h += n_star[s] == n_min + i ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      st = dadd(st, __shfl_xor_sync(0xffffffffu, st, o));
      sc = dadd(sc, __shfl_xor_sync(0xffffffffu, sc, o));
      h += __shfl_xor_sync(0xffffffffu, h, o);
    }
    if (lane == 0) {
      sum_t[i] = dadd(sum_t[i], st);
      sum_c[i] = dadd(sum_c[i], sc);
      hist[i] += h;
    }
  }
}

// {sum_t, sum_c, (double) hist} packed for the one cross-rank all-reduce
// (rs_comm.cu; counts are exact in FP64).
__global__ void pack_aggregates_kernel(int C, const double* sum_t, const double* sum_c,
                                       const int32_t* hist, double* pack) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < C; i += gridDim.x * blockDim.x) {
    pack[i] = sum_t[i];
    pack[C + i] = sum_c[i];
    pack[2 * C + i] = (double)hist[i];
  }
}

// ------------------------------------------------------ input shaping --
// Scatter caller SoA into id order (id_rank[i] = rank of prompt i's id) and
// validate. The bucketed / generic builders then treat the position as the
// tie-break index.
__global__ void to_id_order_kernel(const double* pred, const int32_t* plen,
                                   const int32_t* id_rank, int64_t n,
                                   double* pred_o, int32_t* plen_o,
                                   int32_t* orig, int32_t* seen, int* flags,
                                   int require_ge1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p = pred[i];
    int64_t j = id_rank ? id_rank[i] : i;
    if (j < 0 || j >= n) {
      atomicOr(flags, kFlagBadPerm);
      continue;
    }
    if (seen && atomicAdd(seen + j, 1) != 0) atomicOr(flags, kFlagBadPerm);
    if (!isfinite(p)) atomicOr(flags, kFlagNotFinite);
    else if (require_ge1 && p < 1.0) atomicOr(flags, kFlagTargetBelowOne);
    pred_o[j] = p == 0.0 ? 0.0 : p;  // -0.0 == +0.0 in the reference order
    if (plen_o) plen_o[j] = plen ? plen[i] : 0;
    if (orig) orig[j] = (int32_t)i;
  }
}

// Order-preserving u64 key of a double, descending (negated total order).
__device__ __forceinline__ uint64_t desc_key(double p) {
  uint64_t b = (uint64_t)__double_as_longlong(p);
  uint64_t asc = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
  return ~asc;
}

__global__ void make_keys_kernel(const double* pred, int64_t n, uint64_t* keys,
                                 uint32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = desc_key(pred[i]);
    vals[i] = (uint32_t)i;
  }
}

__global__ void scenario_keys_kernel(const int64_t* item_off, int S,
                                     const uint32_t* vals, int64_t n,
                                     uint64_t* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = vals[i];
    int lo = 0, hi = S;  // scenario containing item v
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (item_off[mid] <= v) lo = mid; else hi = mid;
    }
    keys[i] = (uint64_t)lo;
  }
}

__global__ void gather_ranked_kernel(const int64_t* item_off, int S,
                                     const uint32_t* vals, int64_t n,
                                     const double* pred, const int32_t* plen,
                                     double* pred_r, SSBuffers ss) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t v = vals[j];
    int lo = 0, hi = S;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (item_off[mid] <= v) lo = mid; else hi = mid;
    }
    pred_r[j] = pred[v];
    ss.plen_r[j] = plen ? plen[v] : 0;
    ss.order_r[j] = (int32_t)(v - item_off[lo]);
  }
}

// ----------------------------------------------------- host orchestration --
static int grid_for(rs_ctx* ctx, int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads,
                                                     (int64_t)ctx->num_sms * 8));
}

// Generic path: radix sort by (scenario, pred desc, index asc).
static int build_generic(rs_ctx* ctx, int S, const int64_t* d_off, int64_t n,
                         const double* pred, const int32_t* plen, SSBuffers ss,
                         char* scratch) {
  char* q = scratch;
  uint64_t* keys = (uint64_t*)q; q += abytes(n, 8);
  uint32_t* vals = (uint32_t*)q; q += abytes(n, 4);
  double* pred_r = (double*)q; q += abytes(n, 8);
  char* sort_scratch = q;
  int blocks = grid_for(ctx, n, 256);
  RS_LAUNCH(ctx, "make_keys", make_keys_kernel, blocks, 256, 0, pred, n, keys, vals);
  uint64_t* ko;
  uint32_t* vo;
  RS_TRY(radix_sort_pairs(ctx, keys, vals, n, sort_scratch, &ko, &vo));
  if (S > 1) {
    // Second stable pass by scenario id -> order (scenario, pred desc, idx).
    // The sorted pred keys are no longer needed, so `keys` holds the new
    // keys; the values must not live in the sort scratch (ping-pong target).
    if (vo != vals)
      RS_CUDA_TRY(cudaMemcpyAsync(vals, vo, 4 * n, cudaMemcpyDeviceToDevice, ctx->stream));
    RS_LAUNCH(ctx, "scenario_keys", scenario_keys_kernel, blocks, 256, 0, d_off, S, vals, n, keys);
    RS_TRY(radix_sort_pairs(ctx, keys, vals, n, sort_scratch, &ko, &vo));
  }
  RS_LAUNCH(ctx, "gather_ranked", gather_ranked_kernel, blocks, 256, 0, d_off, S, vo, n,
            pred, plen, pred_r, ss);
  RS_LAUNCH(ctx, "build_structure", build_structure_kernel, S, kBuildThreads, 0,
            pred_r, d_off, ss);
  return RS_OK;
}

static size_t generic_scratch_bytes(int64_t n) {
  return abytes(n, 8) * 2 + abytes(n, 4) + radix_sort_scratch_bytes64(n);
}

static int read_flags(rs_ctx* ctx, int* flags) {
  RS_CUDA_TRY(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *flags = *ctx->h_flags;
  if (*flags) {  // consumed here: the next call starts from a clean status
    *ctx->h_flags = 0;
    RS_TRY(clear_flags(ctx));
  }
  return RS_OK;
}

static int64_t groups_per_scenario(int n_min, int n_max) {
  return (int64_t)n_max * (n_max + 1) / 2 - (int64_t)(n_min - 1) * n_min / 2;
}

static int eval_grid(rs_ctx* ctx, int64_t items) {
  int64_t want = (items + kEvalWarps - 1) / kEvalWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->num_sms * 8));
}

// scale()'s argument checks, in the reference order (planner.cpp:164-168),
// then the ones the reference raises from inside its loop.
static int check_scale_args(int32_t count, int32_t G, int32_t n_min,
                            int32_t n_max, double lambda) {
  if (n_min < 1 || n_min > n_max)
    return fail(RS_E_VALIDATION, "scale: need 1 <= n_min <= n_max");
  if (n_max > count) return fail(RS_E_VALIDATION, "scale: n_max exceeds prompt count");
  if (lambda < 0 || lambda > 1) return fail(RS_E_CONFIG, "scale: lambda must be in [0, 1]");
  if (G < 1) return fail(RS_E_VALIDATION, "estimate_actor_time: responses_per_prompt >= 1");
  return RS_OK;
}

static int gen_tables(rs_ctx* ctx, double** nz, double** lnz) {
  const size_t nt = RS_QTABLE_N + 1;
  double* t = arena_alloc<double>(ctx, 2 * nt);
  if (!t) return fail(RS_E_NOMEM, "arena exhausted (tables)");
  RS_TRY(h2d(ctx, t, RS_NZ, 8 * nt));
  RS_TRY(h2d(ctx, t + nt, RS_LNZ, 8 * nt));
  *nz = t;
  *lnz = t + nt;
  return RS_OK;
}

static GenSpec to_gen(const rs_scenario_spec* sp, int64_t first) {
  return GenSpec{sp->base_seed, first, sp->count, sp->plen_mean, sp->plen_sigma,
                 sp->plen_min, sp->plen_max, sp->pred_scale, sp->pred_min, sp->pred_max};
}

static int check_spec(const rs_scenario_spec* sp) {
  if (!sp) return fail(RS_E_ARG, "spec is NULL");
  if (sp->n_scenarios < 0 || sp->count < 1)
    return fail(RS_E_VALIDATION, "scenario spec needs count >= 1 and n_scenarios >= 0");
  if (!(sp->pred_min >= 1.0) || !(sp->pred_max >= sp->pred_min))
    return fail(RS_E_VALIDATION, "scenario spec needs 1 <= pred_min <= pred_max");
  if (sp->plen_min > sp->plen_max) return fail(RS_E_VALIDATION, "scenario spec plen range");
  return RS_OK;
}


// A built batch of scenario structures: the fast packed layout (bucketed
// finish ticks, rs_fast.cu) or the generic one (radix sort).
struct Built {
  bool fast = false;
  FastSS fss{};
  SSBuffers gss{};
  SSView gview{};
  const int32_t* order_r() const { return fast ? fss.order_r : gss.order_r; }
  const int32_t* plen_r() const { return fast ? fss.plen_r : gss.plen_r; }
};

static size_t built_bytes(int64_t n, int S, bool with_generic) {
  return fast_ss_bytes(n, S) + (with_generic ? ss_bytes(n, S) + generic_scratch_bytes(n) : 0) +
         (1 << 16);
}


// pred / plen: id-ordered device arrays (written by the generator when gen).
// defer: the fast build's status is not read here — the kernels that read the
// structure skip themselves on kFastBad and the sweep driver checks the flags
// (and reruns on the generic path) once per sweep; otherwise the flags are
// read at once and an inapplicable fast build falls back to the generic one.
static int build_batch(rs_ctx* ctx, int S, const int64_t* d_off, int64_t n, double* pred,
                       int32_t* plen, const GenSpec* gen, const double* nz, const double* lnz,
                       bool allow_fast, Built* out, bool keep_inputs = true,
                       bool need_order = true, bool defer = false) {
  if (allow_fast) {
    out->fss = fast_ss_alloc(ctx, d_off, n, S);
    if (!out->fss.rec) return fail(RS_E_NOMEM, "arena exhausted (fast structure)");
    if (!defer) RS_TRY(clear_flags(ctx));
    RS_TRY(fast_build(ctx, S, d_off, pred, plen, out->fss, gen, nz, lnz, keep_inputs, need_order));
    if (defer) {
      out->fast = true;
      return RS_OK;
    }
    int fl;
    RS_TRY(read_flags(ctx, &fl));
    if (fl & kFlagNotFinite) return flags_to_status(fl);
    if (!(fl & (kFlagBucketOverflow | kFlagBucketTooWide))) {
      out->fast = true;
      return RS_OK;
    }
    RS_TRY(clear_flags(ctx));
  }
  out->fast = false;
  out->gss = ss_alloc(ctx, n, S);
  char* scratch = arena_alloc<char>(ctx, generic_scratch_bytes(n));
  if (!scratch) return fail(RS_E_NOMEM, "arena exhausted (generic structure)");
  RS_TRY(build_generic(ctx, S, d_off, n, pred, plen, out->gss, scratch));
  out->gview = ss_view(out->gss, d_off, S);
  return RS_OK;
}

// Batches of fewer scenarios evaluate one group per lane / warp
// (fast_eval): with its per-batch warp-cooperative threshold it beats the
// lockstep walk (+ group table) up to ~50 C4-shaped scenarios (32: 1.55 vs
// 1.93 ms, 48: 1.89 vs 2.02, 64: 2.24 vs 2.11, kernels of one batch).
constexpr int kLockstepMinScenarios = 56;

static int units_for(rs_ctx* ctx, int S, int C) {
  int want = (2 * ctx->num_sms + S - 1) / S;
  return std::max(1, std::min(want, C));
}

// fuse (nullable): when the lockstep evaluator runs it also produces the
// reduce (and, if *fused_select, select) outputs; *fused is set accordingly.
static int eval_batch(rs_ctx* ctx, const Built& b, int S, const DevProfile& dp, int n_min,
                      int n_max, int G, double* gt, const LsFuse* fuse = nullptr,
                      bool* fused = nullptr, bool* fused_select = nullptr, int ctas_per_sm = 0) {
  if (fused) *fused = false;
  if (fused_select) *fused_select = false;
  const int64_t T = groups_per_scenario(n_min, n_max);
  if (b.fast) {
    CandRange cr{n_min, n_max, T, G};
    // Many scenarios: candidates in lockstep (one lane per candidate).
    // Few scenarios: one group per lane, candidates split over CTAs.
    // the lockstep evaluator runs one CTA per scenario: even a partial wave
    // (a sweep's last batch) beats splitting candidates over CTAs from about
    // 56 scenarios on (kLockstepMinScenarios)
    if (S >= kLockstepMinScenarios && lockstep_ok(dp, G)) {
      const bool f = fuse && fused && lockstep_fuses_select(cr);
      if (f) {
        *fused = true;
        if (fused_select) *fused_select = fuse->n_star != nullptr;
      }
      return lockstep_eval(ctx, S, b.fss, dp, cr, gt, f ? fuse : nullptr, ctas_per_sm);
    }
    return fast_eval(ctx, S, b.fss, dp, cr, units_for(ctx, S, n_max - n_min + 1), gt);
  }
  CandSpec cs{n_min, n_max, T, G};
  RS_LAUNCH(ctx, "group_eval", group_eval_kernel, eval_grid(ctx, (int64_t)S * T), kEvalThreads,
            0, b.gview, dp, cs, gt);
  return RS_OK;
}

static int reduce_batch(rs_ctx* ctx, const Built& b, int S, int n_min, int n_max, int G,
                        double rho, int gpus, const double* gt, double* tt, double* cc,
                        int64_t* idle) {
  const int64_t T = groups_per_scenario(n_min, n_max);
  if (b.fast) {
    CandRange cr{n_min, n_max, T, G};
    return fast_reduce(ctx, S, b.fss, cr, rho, gpus, gt, tt, cc, idle);
  }
  CandSpec cs{n_min, n_max, T, G};
  RS_LAUNCH(ctx, "candidate_reduce", candidate_reduce_kernel,
            grid_for(ctx, (int64_t)S * (n_max - n_min + 1), 128), 128, 0, b.gview, cs, rho, gpus,
            gt, tt, cc, idle);
  return RS_OK;
}

static bool fast_spec_ok(const rs_scenario_spec* sp) {
  return std::ceil(sp->pred_max) <= (double)kFastFmax && sp->pred_min >= 1.0 &&
         sp->plen_min >= 0 && sp->plen_max <= kFastPlenMax;
}

// Relative round time of the lockstep evaluator (lockstep2_kernel) at c
// resident CTAs per SM, measured on B200 with the C4 workload (one round of
// c x 148 scenarios, tools/round_costs.py): 2.05 / 2.19 / 2.43 / 2.80 ms for
// c = 1..4 (a lone CTA's walk is latency-bound, four share the issue
// slots). E.g. a rank's 1,250 scenarios at 8 GPUs run as three rounds of 444
// (three deep) rather than 592 + 592 + a lone 66.
static double lockstep_round_cost(int c) {
  static const double rel[5] = {0.0, 1.00, 1.07, 1.19, 1.37};
  return c <= 4 ? rel[c] : rel[4] * c / 4.0;
}

// Modelled time of one lockstep batch of U scenarios and the CTAs per SM
// that achieve it (rounds x round cost, minimised over 1..cmax).
static double lockstep_batch_cost(int U, int cmax, int nsm, int* best_c) {
  double best = 1e300;
  *best_c = cmax;
  for (int c = 1; c <= cmax; ++c) {
    const int64_t rounds = (U + (int64_t)c * nsm - 1) / ((int64_t)c * nsm);
    const double t = rounds * lockstep_round_cost(c);
    if (t < best - 1e-12) {
      best = t;
      *best_c = c;
    }
  }
  return best;
}

// Batch sizes for S scenarios under a budget of Bmem per batch: full batches
// of whole waves, with the remainder alone or merged into the last one —
// whichever the round model prefers — and each batch's CTAs per SM.
static void plan_batches(int S, int Bmem, int cmax, int nsm, std::vector<int>* sizes,
                         std::vector<int>* cps) {
  cmax = std::max(1, cmax);
  std::vector<std::vector<int>> plans;
  for (int cw = 1; cw <= cmax; ++cw) {  // full batches in whole waves of cw CTAs per SM
    const int slots = cw * nsm;
    const int F = Bmem >= slots ? Bmem / slots * slots : Bmem;
    std::vector<int> a;
    for (int s0 = 0; s0 < S; s0 += F) a.push_back(std::min(F, S - s0));
    plans.push_back(a);
    if (a.size() >= 2 && a[a.size() - 2] + a.back() <= Bmem) {
      std::vector<int> m(a.begin(), a.end() - 1);
      m.back() += a.back();
      plans.push_back(m);
    }
  }
  double best = 1e300;
  for (const auto& pl : plans) {
    double t = 0;
    std::vector<int> c(pl.size());
    for (size_t i = 0; i < pl.size(); ++i) t += lockstep_batch_cost(pl[i], cmax, nsm, &c[i]);
    if (t < best - 1e-12) {
      best = t;
      *sizes = pl;
      *cps = c;
    }
  }
}

// True when p is page-locked (cudaMallocHost / cudaHostRegister) host memory:
// device-to-host copies into it are asynchronous; pageable memory goes
// through the context's pinned bounce buffers instead.
static bool host_pinned(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

static int bounce_reserve(rs_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->bounce_cap) return RS_OK;
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->copy_stream));
  if (ctx->bounce) cudaFreeHost(ctx->bounce);
  ctx->bounce = nullptr;
  ctx->bounce_cap = 0;
  if (cudaMallocHost(&ctx->bounce, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(RS_E_NOMEM, "pinned bounce allocation failed");
  }
  ctx->bounce_cap = bytes;
  return RS_OK;
}

// One pass of the sweep. allow_fast_in = false forces the generic structure
// (radix sort) for every batch. *redo is set when a fast structure turned out
// not to apply (a finish tick outside [1, 16384], a prompt_len outside
// [0, 65535] or a finish bucket wider than the in-CTA sort): the caller then
// reruns the whole sweep on the generic path. The status flags are read after
// the first batch (so such a rerun wastes one batch at most) and at the end;
// in between, the kernels that read a fast structure skip themselves when
// the flags say it is unusable (kFastBad), so stale scratch is never indexed.
static int sweep_pass(rs_ctx* ctx, const rs_scenario_spec* spec, const double* h_pred,
                      const int32_t* h_plen, int S, int P, const DevProfile& dp, int G,
                      int n_min, int n_max, double lambda, int gpus, rs_sweep_out* out,
                      int device_ptrs, bool allow_fast_in, bool* redo, double* agg_pack) {
  *redo = false;
  const int C = n_max - n_min + 1;
  const int64_t T = groups_per_scenario(n_min, n_max);
  const bool generated = spec != nullptr;
  const bool allow_fast = allow_fast_in && fast_profile_ok(dp, G);
  const bool gen_fast = generated && allow_fast && fast_spec_ok(spec);
  const bool with_generic = !allow_fast;
  const bool host_in = !generated && !device_ptrs;  // caller arrays in host memory
  const size_t in_bytes = abytes(P, 8) + abytes(P, 4);
  const size_t per_scen = in_bytes * (host_in ? 2 : 1) + built_bytes(P, 1, with_generic) +
                          abytes(T, 8) * 2 + abytes(T, 16) + abytes(T, 2) + abytes(C, 8) * 3 +
                          abytes(1, 4) + 2048;
  // Batches: what an 8 GiB scratch budget holds (<= 2048 scenarios), planned
  // as whole waves of the lockstep evaluator (S = 10,000 on 148 SMs x 4:
  // batches of 1,184) with the remainder merged into the last batch when it
  // fits, each batch run at the CTAs per SM that minimise its rounds x round
  // cost (plan_batches); e.g. a rank's 1,250 scenarios at 8 GPUs run as 740
  // five deep + 510 four deep (two rounds) instead of 1,184 + a lone 66.
  const int Bmem = (int)std::max<size_t>(
      1, std::min<size_t>({(size_t)S, (size_t)(8ull << 30) / per_scen, (size_t)2048}));
  std::vector<int> sizes, cps;  // scenarios and lockstep CTAs per SM, per batch
  if (allow_fast && lockstep_ok(dp, G)) {
    plan_batches(S, Bmem, lockstep_slots(ctx, dp, G) / ctx->num_sms, ctx->num_sms, &sizes, &cps);
  } else {
    for (int s0 = 0; s0 < S; s0 += Bmem) {
      sizes.push_back(std::min(Bmem, S - s0));
      cps.push_back(0);
    }
  }
  const int nb = (int)sizes.size();
  const int B = *std::max_element(sizes.begin(), sizes.end());
  // a second set of per-batch result buffers when host copies overlap
  const size_t out_set = abytes((size_t)B * C, 8) * 3 + abytes(B, 4);
  size_t need = (size_t)B * per_scen + out_set + fast_eval_bytes(dp, G) + abytes(B + 1, 8) +
                abytes(2 * (RS_QTABLE_N + 1), 8) +
                abytes(C, 8) * 2 + abytes(C, 4) + abytes(dp.c_hi - dp.c_lo + 1, 4) + (4 << 20);
  RS_TRY(arena_reserve(ctx, need));
  double* nz = nullptr;
  double* lnz = nullptr;
  RS_TRY(gen_tables(ctx, &nz, &lnz));
  int64_t* d_off = arena_alloc<int64_t>(ctx, B + 1);
  // input sets: two when host inputs stream in on in_stream ahead of compute
  const int nin = host_in && nb > 1 ? 2 : 1;
  double* pred[2] = {nullptr, nullptr};
  int32_t* plen[2] = {nullptr, nullptr};
  for (int k = 0; k < nin; ++k) {
    pred[k] = arena_alloc<double>(ctx, (size_t)B * P);
    plen[k] = arena_alloc<int32_t>(ctx, (size_t)B * P);
  }
  double* gt = arena_alloc<double>(ctx, (size_t)B * T);
  double* agg_t = arena_alloc<double>(ctx, C);
  double* agg_c = arena_alloc<double>(ctx, C);
  int32_t* agg_h = arena_alloc<int32_t>(ctx, C);
  // Host outputs of several batches: two buffer sets, each batch's results
  // copied out on the context's copy stream while the next batch computes;
  // pinned caller buffers receive them directly, pageable ones through the
  // pinned bounce buffers (drained on the host once the copy's event is done).
  const bool overlap_out = !device_ptrs && nb > 1;
  const int nsets = overlap_out ? 2 : 1;
  double* b_tt[2] = {nullptr, nullptr};
  double* b_cc[2] = {nullptr, nullptr};
  int64_t* b_idle[2] = {nullptr, nullptr};
  int32_t* b_ns[2] = {nullptr, nullptr};
  for (int k = 0; k < nsets; ++k) {
    b_tt[k] = arena_alloc<double>(ctx, (size_t)B * C);
    b_cc[k] = arena_alloc<double>(ctx, (size_t)B * C);
    b_idle[k] = arena_alloc<int64_t>(ctx, (size_t)B * C);
    b_ns[k] = arena_alloc<int32_t>(ctx, B);
    if (!b_ns[k]) return fail(RS_E_NOMEM, "arena exhausted (sweep)");
  }
  struct HostOut {
    char* dst;        // caller array
    size_t elem;      // bytes per scenario
    bool direct;      // pinned: copy straight into dst
    char* bounce[2];  // per buffer set otherwise
  };
  HostOut ho[4] = {{(char*)out->t_total, 8ull * C, false, {}}, {(char*)out->cost, 8ull * C, false, {}},
                   {(char*)out->idle_slot_ticks, 8ull * C, false, {}}, {(char*)out->n_star, 4, false, {}}};
  if (!device_ptrs) {
    size_t bb = 0;
    for (auto& h : ho)
      if (h.dst && !(h.direct = host_pinned(h.dst))) bb += abytes(B * h.elem, 1) * nsets;
    RS_TRY(bounce_reserve(ctx, bb));
    char* q = ctx->bounce;
    for (auto& h : ho)
      if (h.dst && !h.direct)
        for (int k = 0; k < nsets; ++k, q += abytes(B * h.elem, 1)) h.bounce[k] = q;
  }
  // pending bounce drains per buffer set: (first scenario, scenarios)
  int pend_s0[2] = {-1, -1}, pend_n[2] = {0, 0};
  auto drain = [&](int set) -> int {
    if (pend_s0[set] < 0) return RS_OK;
    RS_CUDA_TRY(cudaEventSynchronize(ctx->ev_copied[set]));
    for (auto& h : ho)
      if (h.dst && !h.direct)
        std::memcpy(h.dst + (size_t)pend_s0[set] * h.elem, h.bounce[set], (size_t)pend_n[set] * h.elem);
    pend_s0[set] = -1;
    return RS_OK;
  };
  // every return below first waits for the copies (their buffers are the caller's)
  struct CopyDrain {
    cudaStream_t a, b;
    ~CopyDrain() {
      if (a) cudaStreamSynchronize(a);
      if (b) cudaStreamSynchronize(b);
    }
  } guard{overlap_out ? ctx->copy_stream : nullptr, nin > 1 ? ctx->in_stream : nullptr};
  const size_t mark = ctx->arena_used;  // per-batch structures live above
  {
    std::vector<int64_t> off(B + 1);
    for (int i = 0; i <= B; ++i) off[i] = (int64_t)i * P;
    RS_TRY(h2d(ctx, d_off, off.data(), 8 * (B + 1)));
  }
  RS_CUDA_TRY(cudaMemsetAsync(agg_t, 0, 8 * C, ctx->stream));
  RS_CUDA_TRY(cudaMemsetAsync(agg_c, 0, 8 * C, ctx->stream));
  RS_CUDA_TRY(cudaMemsetAsync(agg_h, 0, 4 * C, ctx->stream));
  RS_TRY(clear_flags(ctx));
  std::vector<int> first(nb);
  for (int bi = 0, s0 = 0; bi < nb; s0 += sizes[bi], ++bi) first[bi] = s0;
  // host inputs of batch bi into input set bi % nin, on in_stream once the
  // set's previous batch has been consumed by its build
  auto stage_in = [&](int bi) -> int {
    const int k = bi % nin;
    const int64_t n = (int64_t)sizes[bi] * P;
    const size_t o = (size_t)first[bi] * P;
    if (nin == 1) {
      RS_TRY(h2d(ctx, pred[0], h_pred + o, 8ull * n));
      RS_TRY(h2d(ctx, plen[0], h_plen + o, 4ull * n));
      return RS_OK;
    }
    if (bi >= 2) RS_CUDA_TRY(cudaStreamWaitEvent(ctx->in_stream, ctx->ev_inused[k], 0));
    RS_CUDA_TRY(cudaMemcpyAsync(pred[k], h_pred + o, 8ull * n, cudaMemcpyHostToDevice, ctx->in_stream));
    RS_CUDA_TRY(cudaMemcpyAsync(plen[k], h_plen + o, 4ull * n, cudaMemcpyHostToDevice, ctx->in_stream));
    RS_CUDA_TRY(cudaEventRecord(ctx->ev_in[k], ctx->in_stream));
    return RS_OK;
  };
  if (host_in) RS_TRY(stage_in(0));
  for (int bi = 0; bi < nb; ++bi) {
    const int Sb = sizes[bi], s0 = first[bi];
    const int64_t n = (int64_t)Sb * P;
    const int k_in = bi % nin;
    ctx->arena_used = mark;
    Built built;
    if (generated) {
      GenSpec g = to_gen(spec, spec->first_scenario + s0);
      if (gen_fast) {
        // the generated scenarios only feed the structure: not stored
        RS_TRY(build_batch(ctx, Sb, d_off, n, pred[0], plen[0], &g, nz, lnz, true, &built, false,
                           false, true));
      } else {
        RS_LAUNCH(ctx, "gen_scenarios", gen_scenarios_kernel, grid_for(ctx, n, 256), 256, 0, g,
                  nz, lnz, Sb, pred[0], plen[0]);
        RS_TRY(build_batch(ctx, Sb, d_off, n, pred[0], plen[0], nullptr, nullptr, nullptr,
                           allow_fast, &built, true, false, true));
      }
    } else {
      if (device_ptrs) {
        const size_t o = (size_t)s0 * P;
        RS_CUDA_TRY(cudaMemcpyAsync(pred[0], h_pred + o, 8ull * n, cudaMemcpyDeviceToDevice, ctx->stream));
        RS_CUDA_TRY(cudaMemcpyAsync(plen[0], h_plen + o, 4ull * n, cudaMemcpyDeviceToDevice, ctx->stream));
      } else if (nin > 1) {
        RS_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_in[k_in], 0));
      }
      RS_LAUNCH(ctx, "validate_inputs", to_id_order_kernel, grid_for(ctx, n, 256), 256, 0,
                pred[k_in], (const int32_t*)nullptr, (const int32_t*)nullptr, n, pred[k_in],
                (int32_t*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr, ctx->d_flags, 1);
      RS_TRY(build_batch(ctx, Sb, d_off, n, pred[k_in], plen[k_in], nullptr, nullptr, nullptr,
                         allow_fast, &built, true, false, true));
      if (nin > 1) RS_CUDA_TRY(cudaEventRecord(ctx->ev_inused[k_in], ctx->stream));
    }
    const int set = overlap_out ? (bi & 1) : 0;
    // the copies out of this buffer set two batches ago must be done
    if (overlap_out && bi >= 2) {
      RS_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[set], 0));
      RS_TRY(drain(set));
    }
    double* o_tt = (device_ptrs && out->t_total) ? out->t_total + (size_t)s0 * C : b_tt[set];
    double* o_cc = (device_ptrs && out->cost) ? out->cost + (size_t)s0 * C : b_cc[set];
    int64_t* o_idle = (device_ptrs && out->idle_slot_ticks) ? out->idle_slot_ticks + (size_t)s0 * C
                                                            : b_idle[set];
    int32_t* o_ns = (device_ptrs && out->n_star) ? out->n_star + s0 : b_ns[set];
    LsFuse fuse{o_tt, o_cc, out->idle_slot_ticks ? o_idle : (int64_t*)nullptr, o_ns, dp.rho,
                lambda, gpus};
    bool fused = false, fused_select = false;
    RS_TRY(eval_batch(ctx, built, Sb, dp, n_min, n_max, G, gt, &fuse, &fused,
                      &fused_select, cps[bi]));
    if (!fused)
      RS_TRY(reduce_batch(ctx, built, Sb, n_min, n_max, G, dp.rho, gpus, gt, o_tt, o_cc,
                          out->idle_slot_ticks ? o_idle : (int64_t*)nullptr));
    if (!fused_select)
      RS_LAUNCH(ctx, "select", select_kernel, grid_for(ctx, (int64_t)Sb * 32, 128), 128, 0, Sb, C, n_min,
                lambda, o_tt, (const double*)nullptr, o_cc, (double*)nullptr, (double*)nullptr,
                (double*)nullptr, o_ns);
    RS_LAUNCH(ctx, "aggregate", aggregate_kernel, grid_for(ctx, (int64_t)C * 32, 256), 256, 0, Sb, C, n_min,
              o_tt, o_cc, o_ns, agg_t, agg_c, agg_h);
    if (!device_ptrs) {
      // on the copy stream (overlapping the next batch), else in stream order
      cudaStream_t cs = ctx->stream;
      if (overlap_out) {
        RS_CUDA_TRY(cudaEventRecord(ctx->ev_done[set], ctx->stream));
        RS_CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_done[set], 0));
        cs = ctx->copy_stream;
      }
      const void* src[4] = {o_tt, o_cc, o_idle, o_ns};
      for (int j = 0; j < 4; ++j) {
        HostOut& h = ho[j];
        if (!h.dst) continue;
        void* dst = h.direct ? h.dst + (size_t)s0 * h.elem : h.bounce[set];
        RS_CUDA_TRY(cudaMemcpyAsync(dst, src[j], (size_t)Sb * h.elem, cudaMemcpyDeviceToHost, cs));
      }
      if (overlap_out) RS_CUDA_TRY(cudaEventRecord(ctx->ev_copied[set], ctx->copy_stream));
      pend_s0[set] = s0;
      pend_n[set] = Sb;
      if (!overlap_out) RS_CUDA_TRY(cudaEventRecord(ctx->ev_copied[set], ctx->stream));
    }
    // the next batch's host inputs stream in while this batch computes
    if (host_in && bi + 1 < nb) RS_TRY(stage_in(bi + 1));
    if (bi == 0 && nb > 1 && allow_fast) {
      // one early look at the status: an inapplicable fast structure costs
      // one batch, not a whole sweep
      int fl;
      RS_TRY(read_flags(ctx, &fl));
      if (fl & ~(kFlagBucketOverflow | kFlagBucketTooWide)) return flags_to_status(fl);
      if (fl) {
        *redo = true;
        return RS_OK;
      }
    }
  }
  if (!device_ptrs) {
    if (overlap_out)  // the final sync on the context stream covers every copy
      for (int k = 0; k < 2; ++k) RS_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ctx->ev_copied[k], 0));
    if (out->sum_t) RS_TRY(d2h(ctx, out->sum_t, agg_t, 8 * C));
    if (out->sum_c) RS_TRY(d2h(ctx, out->sum_c, agg_c, 8 * C));
    if (out->nstar_hist) RS_TRY(d2h(ctx, out->nstar_hist, agg_h, 4 * C));
  } else {
    if (out->sum_t)
      RS_CUDA_TRY(cudaMemcpyAsync(out->sum_t, agg_t, 8 * C, cudaMemcpyDeviceToDevice, ctx->stream));
    if (out->sum_c)
      RS_CUDA_TRY(cudaMemcpyAsync(out->sum_c, agg_c, 8 * C, cudaMemcpyDeviceToDevice, ctx->stream));
    if (out->nstar_hist)
      RS_CUDA_TRY(cudaMemcpyAsync(out->nstar_hist, agg_h, 4 * C, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (agg_pack)
    RS_LAUNCH(ctx, "pack_aggregates", pack_aggregates_kernel, (C + 255) / 256, 256, 0, C, agg_t,
              agg_c, agg_h, agg_pack);
  int fl;
  RS_TRY(read_flags(ctx, &fl));  // synchronises the context stream
  if (ctx->timing) RS_TRY(collect_timers(ctx));
  if (fl & ~(kFlagBucketOverflow | kFlagBucketTooWide)) return flags_to_status(fl);
  if (fl) {
    *redo = true;
    return RS_OK;
  }
  for (int k = 0; k < 2; ++k) RS_TRY(drain(k));
  return RS_OK;
}

// Argument checks of a sweep, in scale()'s order (planner.cpp:164-168) —
// also run by every rank of a sharded sweep before its collective, so a
// rank with no scenarios fails exactly like the others.
int sweep_validate(const rs_scenario_spec* spec, const rs_profile* profile, int P, int G,
                   int n_min, int n_max, double lambda) {
  if (spec) RS_TRY(check_spec(spec));
  RS_TRY(check_scale_args(P, G, n_min, n_max, lambda));
  return validate_profile_shape(profile);
}

// Shared sweep driver: scenarios either generated (spec) or from arrays.
// Synchronous: it returns once every result (device or host) is written.
// agg_pack (device, nullable): also receives the packed aggregates.
int sweep_impl_packed(rs_ctx* ctx, const rs_scenario_spec* spec, const double* h_pred,
                      const int32_t* h_plen, int S, int P, const rs_profile* profile, int G,
                      int n_min, int n_max, double lambda, int gpus, rs_sweep_out* out,
                      int device_ptrs, double* agg_pack) {
  RS_TRY(check_scale_args(P, G, n_min, n_max, lambda));
  DevProfile dp;
  RS_TRY(get_profile(ctx, profile, &dp));
  bool redo = false;
  RS_TRY(sweep_pass(ctx, spec, h_pred, h_plen, S, P, dp, G, n_min, n_max, lambda, gpus, out,
                    device_ptrs, true, &redo, agg_pack));
  if (redo)
    RS_TRY(sweep_pass(ctx, spec, h_pred, h_plen, S, P, dp, G, n_min, n_max, lambda, gpus, out,
                      device_ptrs, false, &redo, agg_pack));
  return redo ? fail(RS_E_CUDA, "internal: generic sweep pass flagged the fast path") : RS_OK;
}

static int sweep_impl(rs_ctx* ctx, const rs_scenario_spec* spec, const double* h_pred,
                      const int32_t* h_plen, int S, int P, const rs_profile* profile, int G,
                      int n_min, int n_max, double lambda, int gpus, rs_sweep_out* out,
                      int device_ptrs) {
  return sweep_impl_packed(ctx, spec, h_pred, h_plen, S, P, profile, G, n_min, n_max, lambda,
                           gpus, out, device_ptrs, nullptr);
}

// Aggregate pick over a whole sweep (host, O(C)): mean t and mean c, min-max
// normalised like scale() (planner.cpp:196-209), first strict minimum.
int sweep_select_host(const double* sum_t, const double* sum_c, int64_t n_scenarios, int C,
                      int n_min, double lambda, int32_t* n_star) {
  if (!sum_t || !sum_c || !n_star || C < 1 || n_scenarios < 1)
    return fail(RS_E_ARG, "bad arguments");
  if (lambda < 0 || lambda > 1) return fail(RS_E_CONFIG, "lambda must be in [0, 1]");
  std::vector<double> mt(C), mc(C);
  for (int i = 0; i < C; ++i) {
    mt[i] = sum_t[i] / (double)n_scenarios;
    mc[i] = sum_c[i] / (double)n_scenarios;
  }
  double t_min = mt[0], t_max = mt[0], c_min = mc[0], c_max = mc[0];
  for (int i = 0; i < C; ++i) {
    t_min = mt[i] < t_min ? mt[i] : t_min;
    t_max = t_max < mt[i] ? mt[i] : t_max;
    c_min = mc[i] < c_min ? mc[i] : c_min;
    c_max = c_max < mc[i] ? mc[i] : c_max;
  }
  int best = 0;
  double bs = 0;
  for (int i = 0; i < C; ++i) {
    double tn = t_max > t_min ? (mt[i] - t_min) / (t_max - t_min) : 0.0;
    double cn = c_max > c_min ? (mc[i] - c_min) / (c_max - c_min) : 0.0;
    double sc = lambda * tn + (1.0 - lambda) * cn;
    if (i == 0) bs = sc;
    if (sc < bs) {
      best = i;
      bs = sc;
    }
  }
  *n_star = n_min + best;
  return RS_OK;
}

// S caller item sets (host SoA), each its own scenario, in id order.
struct SetRun {
  int S;
  int64_t n;
  int64_t* d_off;
  double* pred;
  int32_t* plen;
  int32_t* orig;
  Built built;
};

static int prepare_sets(rs_ctx* ctx, const double* h_pred, const int32_t* h_plen,
                        const int32_t* h_id_rank, const std::vector<int64_t>& off,
                        int require_ge1, const DevProfile* dp, int G, size_t extra_bytes,
                        SetRun* run) {
  const int S = (int)off.size() - 1;
  const int64_t n = off.back();
  size_t need = abytes(S + 1, 8) + abytes(n, 8) * 2 + abytes(n, 4) * 4 +
                built_bytes(n, S, true) + extra_bytes + (1 << 20);
  if (dp) need += fast_eval_bytes(*dp, G);
  RS_TRY(arena_reserve(ctx, need));
  run->S = S;
  run->n = n;
  run->d_off = arena_alloc<int64_t>(ctx, S + 1);
  double* raw_pred = arena_alloc<double>(ctx, n);
  int32_t* raw_plen = arena_alloc<int32_t>(ctx, n);
  int32_t* raw_rank = arena_alloc<int32_t>(ctx, n);
  int32_t* seen = arena_alloc<int32_t>(ctx, n);
  run->pred = arena_alloc<double>(ctx, n);
  run->plen = arena_alloc<int32_t>(ctx, n);
  run->orig = arena_alloc<int32_t>(ctx, n);
  if (!run->orig) return fail(RS_E_NOMEM, "arena exhausted (sets)");
  RS_TRY(h2d(ctx, run->d_off, off.data(), 8 * (S + 1)));
  RS_TRY(clear_flags(ctx));
  if (n > 0) {
    RS_TRY(h2d(ctx, raw_pred, h_pred, 8 * n));
    if (h_plen) RS_TRY(h2d(ctx, raw_plen, h_plen, 4 * n));
    if (h_id_rank) {
      RS_TRY(h2d(ctx, raw_rank, h_id_rank, 4 * n));
      RS_CUDA_TRY(cudaMemsetAsync(seen, 0, 4 * n, ctx->stream));
    }
    RS_LAUNCH(ctx, "to_id_order", to_id_order_kernel, grid_for(ctx, n, 256), 256, 0, raw_pred,
              h_plen ? raw_plen : (const int32_t*)nullptr,
              h_id_rank ? raw_rank : (const int32_t*)nullptr, n, run->pred, run->plen, run->orig,
              h_id_rank ? seen : (int32_t*)nullptr, ctx->d_flags, require_ge1);
    int fl;
    RS_TRY(read_flags(ctx, &fl));
    if (fl & (kFlagBadPerm))
      return fail(RS_E_ARG, "id_rank is not a permutation of [0, count)");
    if (fl) return flags_to_status(fl);
    const bool allow_fast = dp == nullptr || fast_profile_ok(*dp, G);
    RS_TRY(build_batch(ctx, S, run->d_off, n, run->pred, run->plen, nullptr, nullptr, nullptr,
                       allow_fast, &run->built));
  }
  return RS_OK;
}

__global__ void map_order_kernel(const int32_t* order_r, const int32_t* orig,
                                 int64_t n, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = orig[order_r[i]];
}

__global__ void chunk_offsets_kernel(int P, int N, int32_t* off) {
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a <= N; a += gridDim.x * blockDim.x) {
    int q = P / N, r = P % N;
    off[a] = a * q + min(a, r);
  }
}

// Sequential dollars over groups with per-group GPU counts (planner.cpp:148-157).
__global__ void cost_sum_kernel(const double* times, const int32_t* gpu_count,
                                int n, double rho, double* cost) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double d = 0.0;
    for (int k = 0; k < n; ++k) d = dadd(d, dmul(dmul(rho, times[k]), (double)gpu_count[k]));
    *cost = d;
  }
}

// --------------------------------------------------------------- LPT --
// Warp per candidate N <= 32*R: loads live in registers, each response goes
// to the least-loaded actor (ties -> lowest index) via a packed u64 warp
// argmin (load << 11 | actor).
template <int R>
__global__ void lpt_kernel(const int64_t* len_r, int64_t count, int G, int n_min,
                           int n_max, int64_t* makespan, int64_t* idle) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int N = n_min + w;
  if (N > n_max) return;
  uint64_t load[R];
#pragma unroll
  for (int j = 0; j < R; ++j) load[j] = 0;
  for (int64_t i0 = 0; i0 < count; i0 += 32) {
    int64_t my = i0 + lane < count ? len_r[i0 + lane] : 0;
    int nn = (int)(count - i0 < 32 ? count - i0 : 32);
    for (int e = 0; e < nn; ++e) {
      uint64_t len = (uint64_t)__shfl_sync(0xffffffffu, my, e);
      for (int r = 0; r < G; ++r) {
        uint64_t best = ~0ULL;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          int a = j * 32 + lane;
          uint64_t key = a < N ? (load[j] << 11) | (uint64_t)a : ~0ULL;
          best = key < best ? key : best;
        }
        best = warp_min(best);
        int a = (int)(best & 2047);
        if ((a & 31) == lane) {
#pragma unroll
          for (int j = 0; j < R; ++j)
            if (j == (a >> 5)) load[j] += len;
        }
      }
    }
  }
  uint64_t mx = 0, sum = 0;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    int a = j * 32 + lane;
    if (a < N) {
      mx = load[j] > mx ? load[j] : mx;
      sum += load[j];
    }
  }
  mx = warp_max(mx);
  sum = warp_sum(sum);
  if (lane == 0) {
    makespan[N - n_min] = (int64_t)mx;
    idle[N - n_min] = (int64_t)(mx * (uint64_t)N - sum);
  }
}

__global__ void lpt_keys_kernel(const double* pred_id, int64_t n, uint64_t* keys,
                                uint32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = ~(uint64_t)(int64_t)ceil(pred_id[i]);  // finish desc
    vals[i] = (uint32_t)i;                           // id order is stable
  }
}

__global__ void lpt_gather_kernel(const double* pred_id, const uint32_t* vals,
                                  int64_t n, int64_t* len_r) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    len_r[i] = (int64_t)ceil(pred_id[vals[i]]);
}

}  // namespace rs

using namespace rs;

__global__ void gather_keys_kernel(const uint64_t* src, const uint32_t* perm, int64_t n,
                                   uint64_t* keys, uint32_t* vals) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x) {
    keys[j] = src[perm[j]];
    vals[j] = perm[j];
  }
}

__global__ void rank_scatter_kernel(const uint32_t* perm, int64_t n, int32_t* rank) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    rank[perm[j]] = (int32_t)j;
}

__global__ void iota_kernel(uint32_t* v, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
       j += (int64_t)gridDim.x * blockDim.x)
    v[j] = (uint32_t)j;
}

// LSD radix over (length, then 8-byte big-endian words from the last to the
// first): lexicographic unsigned-byte order with a proper prefix first.
// Big-endian 8-byte words of each string (zero padded); plane 0 = length.
__global__ void string_words_kernel(const char* bytes, const int64_t* off, int64_t n, int64_t W,
                                    uint64_t* words) {
  const int64_t total = (W + 1) * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t plane = t / n, i = t - plane * n;
    const int64_t a = off[i], len = off[i + 1] - a;
    uint64_t w = 0;
    if (plane == 0) {
      w = (uint64_t)len;
    } else {
      const int64_t b0 = (plane - 1) * 8;
      for (int b = 0; b < 8 && b0 + b < len; ++b)
        w |= (uint64_t)(unsigned char)bytes[a + b0 + b] << (56 - 8 * b);
    }
    words[t] = w;
  }
}

namespace rs {

size_t rank_strings_device_bytes(int64_t n, int64_t maxlen) {
  const int64_t W = (maxlen + 7) / 8;
  return abytes((W + 1) * n, 8) + abytes(n, 8) + abytes(n, 4) + radix_sort_scratch_bytes64(n) + 1024;
}

// d_perm[r] = index of the string of rank r in std::string order: LSD radix
// passes over the length plane, then the word planes last to first (a
// shorter string that is a prefix of a longer one sorts first, as its zero
// padding ties and the length decides). Allocates from the arena (the caller
// reserves rank_strings_device_bytes).
int rank_strings_device(rs_ctx* ctx, const char* d_bytes, const int64_t* d_off, int64_t n,
                        int64_t maxlen, uint32_t* d_perm) {
  if (n <= 0) return RS_OK;
  const int64_t W = (maxlen + 7) / 8;
  uint64_t* d_words = arena_alloc<uint64_t>(ctx, (W + 1) * n);
  uint64_t* keys = arena_alloc<uint64_t>(ctx, n);
  uint32_t* vals = arena_alloc<uint32_t>(ctx, n);
  char* scratch = arena_alloc<char>(ctx, radix_sort_scratch_bytes64(n));
  if (!scratch) return fail(RS_E_NOMEM, "arena exhausted (rank_strings)");
  RS_LAUNCH(ctx, "string_words", string_words_kernel, grid_for(ctx, (W + 1) * n, 256), 256, 0,
            d_bytes, d_off, n, W, d_words);
  const int blocks = grid_for(ctx, n, 256);
  RS_LAUNCH(ctx, "iota", iota_kernel, blocks, 256, 0, d_perm, n);
  for (int64_t plane = 0; plane <= W; ++plane) {
    const int64_t w = plane == 0 ? 0 : W + 1 - plane;  // length first, then last word .. first
    RS_LAUNCH(ctx, "gather_keys", gather_keys_kernel, blocks, 256, 0, d_words + w * n, d_perm, n,
              keys, vals);
    uint64_t* ko;
    uint32_t* vo;
    RS_TRY(radix_sort_pairs(ctx, keys, vals, n, scratch, &ko, &vo));
    RS_CUDA_TRY(cudaMemcpyAsync(d_perm, vo, 4 * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  return RS_OK;
}

}  // namespace rs

extern "C" {

int rs_generate_scenarios(rs_ctx* ctx, const rs_scenario_spec* spec, double* pred,
                          int32_t* plen, int device_ptrs) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "ctx is NULL");
  RS_TRY(check_spec(spec));
  int64_t n = (int64_t)spec->n_scenarios * spec->count;
  if (n == 0) return RS_OK;
  RS_TRY(arena_reserve(ctx, abytes(2 * (RS_QTABLE_N + 1), 8) +
                                (device_ptrs ? 0 : abytes(n, 8) + abytes(n, 4)) + 4096));
  double *nz, *lnz;
  RS_TRY(gen_tables(ctx, &nz, &lnz));
  double* dp = device_ptrs ? pred : arena_alloc<double>(ctx, n);
  int32_t* dl = device_ptrs ? plen : arena_alloc<int32_t>(ctx, n);
  GenSpec g = to_gen(spec, spec->first_scenario);
  RS_LAUNCH(ctx, "gen_scenarios", gen_scenarios_kernel, grid_for(ctx, n, 256), 256, 0, g, nz,
            lnz, spec->n_scenarios, dp, dl);
  if (device_ptrs) return RS_OK;
  RS_TRY(d2h(ctx, pred, dp, 8 * n));
  RS_TRY(d2h(ctx, plen, dl, 4 * n));
  return sync_and_check(ctx);
}

int rs_sweep(rs_ctx* ctx, const rs_scenario_spec* spec, const rs_profile* profile,
             int32_t G, int32_t n_min, int32_t n_max, double lambda, int32_t gpus,
             rs_sweep_out* out, int device_ptrs) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out) return fail(RS_E_ARG, "NULL argument");
  RS_TRY(check_spec(spec));
  if (spec->n_scenarios == 0) return RS_OK;
  return sweep_impl(ctx, spec, nullptr, nullptr, spec->n_scenarios, spec->count, profile, G,
                    n_min, n_max, lambda, gpus, out, device_ptrs);
}

int rs_sweep_arrays(rs_ctx* ctx, const double* pred, const int32_t* plen, int32_t S,
                    int32_t count, const rs_profile* profile, int32_t G, int32_t n_min,
                    int32_t n_max, double lambda, int32_t gpus, rs_sweep_out* out,
                    int device_ptrs) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out || !pred || !plen) return fail(RS_E_ARG, "NULL argument");
  if (S <= 0) return RS_OK;
  return sweep_impl(ctx, nullptr, pred, plen, S, count, profile, G, n_min, n_max, lambda,
                    gpus, out, device_ptrs);
}

int rs_sweep_select(const double* sum_t, const double* sum_c, int64_t n_scenarios,
                    int32_t C, int32_t n_min, double lambda, int32_t* n_star) {
  return sweep_select_host(sum_t, sum_c, n_scenarios, C, n_min, lambda, n_star);
}

// LPT over id-ordered predictions already in HBM (pid): the (len desc, id
// asc, r asc) order by a stable radix sort, then one warp per candidate.
static int lpt_core(rs_ctx* ctx, const double* pid, int64_t count, int G, int n_min, int n_max,
                    uint64_t* keys, uint32_t* vals, int64_t* len_r, char* sscr, int64_t* mk,
                    int64_t* id) {
  const int C = n_max - n_min + 1;
  RS_LAUNCH(ctx, "lpt_keys", lpt_keys_kernel, grid_for(ctx, count, 256), 256, 0, pid,
            count, keys, vals);
  uint64_t* ko;
  uint32_t* vo;
  RS_TRY(radix_sort_pairs(ctx, keys, vals, count, sscr, &ko, &vo));
  RS_LAUNCH(ctx, "lpt_gather", lpt_gather_kernel, grid_for(ctx, count, 256), 256, 0, pid, vo,
            count, len_r);
  int warps_per_block = 4;
  int blocks = (C + warps_per_block - 1) / warps_per_block;
  int R = (n_max + 31) / 32;
#define RS_LPT(RR)                                                                           \
  RS_LAUNCH(ctx, "lpt", lpt_kernel<RR>, blocks, 32 * warps_per_block, 0, len_r, count, \
            G, n_min, n_max, mk, id)
  if (R <= 1) RS_LPT(1);
  else if (R <= 2) RS_LPT(2);
  else if (R <= 4) RS_LPT(4);
  else if (R <= 8) RS_LPT(8);
  else if (R <= 16) RS_LPT(16);
  else RS_LPT(32);
#undef RS_LPT
  return RS_OK;
}

static size_t lpt_bytes(int64_t count, int C) {
  return abytes(count, 8) * 2 + abytes(count, 4) + radix_sort_scratch_bytes64(count) +
         abytes(C, 8) * 2;
}

// scale() with either a caller-provided penalty array (t_penalty) or the
// device placement penalty (pen), or neither.
static int scale_impl(rs_ctx* ctx, const double* pred, const int32_t* plen,
                      const int32_t* id_rank, int32_t count, const rs_profile* profile, int32_t G,
                      int32_t n_min, int32_t n_max, double lambda, int32_t gpus,
                      const double* t_penalty, const rs_placement_penalty* pen,
                      rs_scale_out* out) {
  if (!ctx || !out) return fail(RS_E_ARG, "NULL argument");
  RS_TRY(check_scale_args(count, G, n_min, n_max, lambda));
  if (!pred || !plen) return fail(RS_E_ARG, "NULL argument");
  PlacementSlots slots;
  if (pen) {
    // the penalty runs inside scale's candidate loop: topology / transfer
    // errors first, then the first candidate whose actors do not fit
    RS_TRY(placement_slots(pen, gpus, n_max, &slots));
    if (slots.n_placeable < n_max)
      return fail(RS_E_PLACEMENT,
                  "cannot place actor: candidate N=" + std::to_string(std::max(n_min, slots.n_placeable + 1)) +
                      " needs " + std::to_string(gpus) + " GPUs on one node per actor, the cluster hosts " +
                      std::to_string(slots.n_placeable) + " such actors");
  }
  const bool want_lpt = out->lpt_makespan || out->lpt_idle;
  if (want_lpt) {  // LPT extension on the same predictions
    if (n_max > 1024) return fail(RS_E_CONFIG, "lpt: n_max <= 1024 supported");
    double mx = 0;
    for (int32_t i = 0; i < count; ++i) mx = pred[i] > mx ? pred[i] : mx;
    if (std::ceil(mx) * (double)count * G >= 0x1.0p52)
      return fail(RS_E_CONFIG, "lpt: total response tokens must stay below 2^52");
  }
  DevProfile dp;
  RS_TRY(get_profile(ctx, profile, &dp));
  const int C = n_max - n_min + 1;
  const int64_t T = groups_per_scenario(n_min, n_max);
  std::vector<int64_t> off = {0, count};
  SetRun run;
  size_t extra = abytes(T, 8) + abytes(C, 8) * 7 + abytes(count, 4) + abytes(C, 8) + 4096 +
                 (pen ? placement_bytes(count, n_max) : 0) + (want_lpt ? lpt_bytes(count, C) : 0);
  RS_TRY(prepare_sets(ctx, pred, plen, id_rank, off, 1, &dp, G, extra, &run));
  double* gt = arena_alloc<double>(ctx, T);
  double* tt = arena_alloc<double>(ctx, C);
  double* cc = arena_alloc<double>(ctx, C);
  double* tp = arena_alloc<double>(ctx, C);
  double* tn = arena_alloc<double>(ctx, C);
  double* cn = arena_alloc<double>(ctx, C);
  double* sc = arena_alloc<double>(ctx, C);
  int64_t* idle = arena_alloc<int64_t>(ctx, C);
  int32_t* order = arena_alloc<int32_t>(ctx, count);
  int32_t* ns = arena_alloc<int32_t>(ctx, 1);
  if (!ns) return fail(RS_E_NOMEM, "arena exhausted (scale)");
  if (t_penalty) RS_TRY(h2d(ctx, tp, t_penalty, 8 * C));
  RS_TRY(eval_batch(ctx, run.built, 1, dp, n_min, n_max, G, gt));
  RS_TRY(reduce_batch(ctx, run.built, 1, n_min, n_max, G, dp.rho, gpus, gt, tt, cc, idle));
  if (pen)
    RS_TRY(placement_penalties(ctx, gt, run.built.plen_r(), count, n_min, n_max, slots, pen, tp));
  const bool with_pen = t_penalty || pen;
  RS_LAUNCH(ctx, "select", select_kernel, 1, 32, 0, 1, C, n_min, lambda, tt,
            with_pen ? tp : (const double*)nullptr, cc, tn, cn, sc, ns);
  RS_LAUNCH(ctx, "map_order", map_order_kernel, grid_for(ctx, count, 256), 256, 0,
            run.built.order_r(), run.orig, (int64_t)count, order);
  if (want_lpt) {
    uint64_t* keys = arena_alloc<uint64_t>(ctx, count);
    uint32_t* vals = arena_alloc<uint32_t>(ctx, count);
    int64_t* len_r = arena_alloc<int64_t>(ctx, count);
    char* sscr = arena_alloc<char>(ctx, radix_sort_scratch_bytes64(count));
    int64_t* mk = arena_alloc<int64_t>(ctx, C);
    int64_t* li = arena_alloc<int64_t>(ctx, C);
    if (!li) return fail(RS_E_NOMEM, "arena exhausted (lpt)");
    RS_TRY(lpt_core(ctx, run.pred, count, G, n_min, n_max, keys, vals, len_r, sscr, mk, li));
    if (out->lpt_makespan) RS_TRY(d2h(ctx, out->lpt_makespan, mk, 8 * C));
    if (out->lpt_idle) RS_TRY(d2h(ctx, out->lpt_idle, li, 8 * C));
  }
  RS_TRY(d2h(ctx, &out->n_star, ns, 4));
  if (out->t_total) RS_TRY(d2h(ctx, out->t_total, tt, 8 * C));
  if (out->cost) RS_TRY(d2h(ctx, out->cost, cc, 8 * C));
  if (out->t_norm) RS_TRY(d2h(ctx, out->t_norm, tn, 8 * C));
  if (out->c_norm) RS_TRY(d2h(ctx, out->c_norm, cn, 8 * C));
  if (out->score) RS_TRY(d2h(ctx, out->score, sc, 8 * C));
  if (out->idle_slot_ticks) RS_TRY(d2h(ctx, out->idle_slot_ticks, idle, 8 * C));
  if (out->order) RS_TRY(d2h(ctx, out->order, order, 4 * count));
  if (out->group_times) RS_TRY(d2h(ctx, out->group_times, gt, 8 * T));
  if (out->t_penalty && pen) RS_TRY(d2h(ctx, out->t_penalty, tp, 8 * C));
  RS_TRY(sync_and_check(ctx));
  if (out->t_penalty && !pen)
    for (int i = 0; i < C; ++i) out->t_penalty[i] = t_penalty ? t_penalty[i] : 0.0;
  if (out->actor_times) {
    int n = out->n_star;
    int64_t base = (int64_t)n * (n - 1) / 2 - (int64_t)n_min * (n_min - 1) / 2;
    RS_CUDA_TRY(cudaMemcpy(out->actor_times, gt + base, 8 * n, cudaMemcpyDeviceToHost));
  }
  return RS_OK;
}

int rs_scale(rs_ctx* ctx, const double* pred, const int32_t* plen, const int32_t* id_rank,
             int32_t count, const rs_profile* profile, int32_t G, int32_t n_min,
             int32_t n_max, double lambda, int32_t gpus, const double* t_penalty,
             rs_scale_out* out) {
  RS_DEVICE_GUARD(ctx);
  return scale_impl(ctx, pred, plen, id_rank, count, profile, G, n_min, n_max, lambda, gpus,
                    t_penalty, nullptr, out);
}

int rs_scale_placed(rs_ctx* ctx, const double* pred, const int32_t* plen,
                    const int32_t* id_rank, int32_t count, const rs_profile* profile, int32_t G,
                    int32_t n_min, int32_t n_max, double lambda, int32_t gpus,
                    const rs_placement_penalty* penalty, rs_scale_out* out) {
  RS_DEVICE_GUARD(ctx);
  if (!penalty) return fail(RS_E_ARG, "NULL placement penalty");
  return scale_impl(ctx, pred, plen, id_rank, count, profile, G, n_min, n_max, lambda, gpus,
                    nullptr, penalty, out);
}

int rs_scale_select(rs_ctx* ctx, const double* t_total, const double* t_penalty,
                    const double* cost, int32_t C, int32_t n_min, double lambda,
                    double* t_norm, double* c_norm, double* score, int32_t* n_star) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !t_total || !cost || !n_star || C < 1) return fail(RS_E_ARG, "bad arguments");
  if (lambda < 0 || lambda > 1) return fail(RS_E_CONFIG, "scale: lambda must be in [0, 1]");
  RS_TRY(arena_reserve(ctx, abytes(C, 8) * 6 + 4096));
  double* d[6];
  for (auto& x : d) x = arena_alloc<double>(ctx, C);
  int32_t* ns = arena_alloc<int32_t>(ctx, 1);
  RS_TRY(h2d(ctx, d[0], t_total, 8 * C));
  RS_TRY(h2d(ctx, d[1], cost, 8 * C));
  if (t_penalty) RS_TRY(h2d(ctx, d[2], t_penalty, 8 * C));
  RS_LAUNCH(ctx, "select", select_kernel, 1, 32, 0, 1, C, n_min, lambda, d[0],
            t_penalty ? d[2] : (const double*)nullptr, d[1], d[3], d[4], d[5], ns);
  RS_TRY(d2h(ctx, n_star, ns, 4));
  if (t_norm) RS_TRY(d2h(ctx, t_norm, d[3], 8 * C));
  if (c_norm) RS_TRY(d2h(ctx, c_norm, d[4], 8 * C));
  if (score) RS_TRY(d2h(ctx, score, d[5], 8 * C));
  return sync_and_check(ctx);
}

int rs_rank_strings(rs_ctx* ctx, const char* bytes, const int64_t* offsets, int32_t count,
                    int32_t* rank) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !offsets || !rank) return fail(RS_E_ARG, "NULL argument");
  if (count <= 0) return RS_OK;
  int64_t maxlen = 0;
  for (int32_t i = 0; i < count; ++i) {
    int64_t l = offsets[i + 1] - offsets[i];
    if (l < 0) return fail(RS_E_ARG, "offsets must be non-decreasing");
    maxlen = std::max(maxlen, l);
  }
  const int64_t n = count, nb = offsets[count] - offsets[0];
  RS_TRY(arena_reserve(ctx, abytes(nb + 1, 1) + abytes(n + 1, 8) + abytes(n, 4) * 2 +
                                rank_strings_device_bytes(n, maxlen) + 4096));
  char* d_bytes = arena_alloc<char>(ctx, nb + 1);
  int64_t* d_off = arena_alloc<int64_t>(ctx, n + 1);
  uint32_t* perm = arena_alloc<uint32_t>(ctx, n);
  int32_t* d_rank = arena_alloc<int32_t>(ctx, n);
  if (!d_rank) return fail(RS_E_NOMEM, "arena exhausted (rank_strings)");
  std::vector<int64_t> rel(n + 1);
  for (int64_t i = 0; i <= n; ++i) rel[i] = offsets[i] - offsets[0];
  if (nb) RS_TRY(h2d(ctx, d_bytes, bytes + offsets[0], nb));
  RS_TRY(h2d(ctx, d_off, rel.data(), 8 * (n + 1)));
  RS_TRY(rank_strings_device(ctx, d_bytes, d_off, n, maxlen, perm));
  RS_LAUNCH(ctx, "rank_scatter", rank_scatter_kernel, grid_for(ctx, n, 256), 256, 0, perm, n, d_rank);
  RS_TRY(d2h(ctx, rank, d_rank, 4 * n));
  return sync_and_check(ctx);
}

int rs_assign(rs_ctx* ctx, const double* pred, const int32_t* id_rank, int32_t count,
              int32_t n_actors, int32_t* order, int32_t* group_offsets) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "ctx is NULL");
  if (count <= 0) return fail(RS_E_VALIDATION, "assign: empty batch");
  if (n_actors < 1) return fail(RS_E_VALIDATION, "assign: n_actors must be >= 1");
  if (n_actors > count)
    return fail(RS_E_VALIDATION, "assign: more actors (" + std::to_string(n_actors) +
                                     ") than prompts (" + std::to_string(count) + ")");
  if (!pred || !order || !group_offsets) return fail(RS_E_ARG, "NULL argument");
  std::vector<int64_t> off = {0, count};
  SetRun run;
  RS_TRY(prepare_sets(ctx, pred, nullptr, id_rank, off, 0, nullptr, 1,
                      abytes(count, 4) + abytes(n_actors + 1, 4) + 4096, &run));
  int32_t* d_order = arena_alloc<int32_t>(ctx, count);
  int32_t* d_off = arena_alloc<int32_t>(ctx, n_actors + 1);
  RS_LAUNCH(ctx, "map_order", map_order_kernel, grid_for(ctx, count, 256), 256, 0,
            run.built.order_r(), run.orig, (int64_t)count, d_order);
  RS_LAUNCH(ctx, "chunk_offsets", chunk_offsets_kernel, grid_for(ctx, n_actors + 1, 256), 256, 0,
            count, n_actors, d_off);
  RS_TRY(d2h(ctx, order, d_order, 4 * count));
  RS_TRY(d2h(ctx, group_offsets, d_off, 4 * (n_actors + 1)));
  return sync_and_check(ctx);
}

// Integral of S independent item sets (one group each = whole set).
static int integrate_sets(rs_ctx* ctx, const int32_t* plen, const double* target,
                          const std::vector<int64_t>& off, int G, const rs_profile* profile,
                          double* times_host, const int32_t* gpu_count, double* cost_host) {
  DevProfile dp;
  RS_TRY(get_profile(ctx, profile, &dp));
  const int S = (int)off.size() - 1;
  SetRun run;
  RS_TRY(prepare_sets(ctx, target, plen, nullptr, off, 1, &dp, G,
                      abytes(S, 8) + abytes(S, 4) + abytes(1, 8) + 4096, &run));
  double* gt = arena_alloc<double>(ctx, S);
  int32_t* gc = arena_alloc<int32_t>(ctx, S);
  double* dcost = arena_alloc<double>(ctx, 1);
  RS_TRY(eval_batch(ctx, run.built, S, dp, 1, 1, G, gt));
  if (cost_host) {
    RS_TRY(h2d(ctx, gc, gpu_count, 4 * S));
    RS_LAUNCH(ctx, "cost_sum", cost_sum_kernel, 1, 32, 0, gt, gc, S, dp.rho, dcost);
    RS_TRY(d2h(ctx, cost_host, dcost, 8));
  }
  if (times_host) RS_TRY(d2h(ctx, times_host, gt, 8 * S));
  return sync_and_check(ctx);
}

int rs_integrate_decode_seconds(rs_ctx* ctx, const int32_t* prompt_len,
                                const double* target_len, int64_t count,
                                const rs_profile* profile, double* out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out) return fail(RS_E_ARG, "NULL argument");
  if (count <= 0) {
    *out = 0.0;
    return RS_OK;
  }
  if (count > INT32_MAX) return fail(RS_E_VALIDATION, "too many responses");
  std::vector<int64_t> off = {0, count};
  return integrate_sets(ctx, prompt_len, target_len, off, 1, profile, out, nullptr, nullptr);
}

int rs_estimate_actor_time(rs_ctx* ctx, const int32_t* prompt_len, const double* pred,
                           int32_t count, const rs_profile* profile, int32_t G, double* out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !out) return fail(RS_E_ARG, "NULL argument");
  if (G < 1) return fail(RS_E_VALIDATION, "estimate_actor_time: responses_per_prompt >= 1");
  if (count <= 0) {
    *out = 0.0;
    return RS_OK;
  }
  std::vector<int64_t> off = {0, count};
  return integrate_sets(ctx, prompt_len, pred, off, G, profile, out, nullptr, nullptr);
}

int rs_estimate_cost(rs_ctx* ctx, const int32_t* prompt_len, const double* pred,
                     const int32_t* group_offsets, const int32_t* gpu_count, int32_t n_groups,
                     const rs_profile* profile, int32_t G, double* cost, double* times) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !cost) return fail(RS_E_ARG, "NULL argument");
  if (n_groups <= 0) {
    *cost = 0.0;
    return RS_OK;
  }
  if (G < 1) return fail(RS_E_VALIDATION, "estimate_actor_time: responses_per_prompt >= 1");
  std::vector<int64_t> off(n_groups + 1);
  for (int k = 0; k <= n_groups; ++k) off[k] = group_offsets[k] - group_offsets[0];
  std::vector<double> t(n_groups);
  RS_TRY(integrate_sets(ctx, prompt_len + group_offsets[0], pred + group_offsets[0], off, G,
                        profile, t.data(), gpu_count, cost));
  if (times) std::memcpy(times, t.data(), 8 * n_groups);
  return RS_OK;
}

int rs_lpt(rs_ctx* ctx, const double* pred, const int32_t* id_rank, int32_t count, int32_t G,
           int32_t n_min, int32_t n_max, int64_t* makespan, int64_t* idle) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !pred || !makespan || !idle) return fail(RS_E_ARG, "NULL argument");
  if (count <= 0) return fail(RS_E_VALIDATION, "lpt: empty batch");
  if (n_min < 1 || n_min > n_max) return fail(RS_E_VALIDATION, "lpt: need 1 <= n_min <= n_max");
  if (G < 1) return fail(RS_E_VALIDATION, "lpt: responses_per_prompt >= 1");
  if (n_max > 1024) return fail(RS_E_CONFIG, "lpt: n_max <= 1024 supported");
  {
    double mx = 0;
    for (int32_t i = 0; i < count; ++i) {
      if (!std::isfinite(pred[i])) return fail(RS_E_VALIDATION, "predicted length is not finite");
      mx = pred[i] > mx ? pred[i] : mx;
    }
    if (std::ceil(mx) * (double)count * G >= 0x1.0p52)
      return fail(RS_E_CONFIG, "lpt: total response tokens must stay below 2^52");
  }
  const int C = n_max - n_min + 1;
  size_t need = abytes(count, 8) * 4 + abytes(count, 4) * 6 + radix_sort_scratch_bytes64(count) +
                abytes(C, 8) * 2 + (1 << 20);
  RS_TRY(arena_reserve(ctx, need));
  double* raw = arena_alloc<double>(ctx, count);
  int32_t* rk = arena_alloc<int32_t>(ctx, count);
  int32_t* seen = arena_alloc<int32_t>(ctx, count);
  double* pid = arena_alloc<double>(ctx, count);
  uint64_t* keys = arena_alloc<uint64_t>(ctx, count);
  uint32_t* vals = arena_alloc<uint32_t>(ctx, count);
  int64_t* len_r = arena_alloc<int64_t>(ctx, count);
  int64_t* mk = arena_alloc<int64_t>(ctx, C);
  int64_t* id = arena_alloc<int64_t>(ctx, C);
  char* sscr = arena_alloc<char>(ctx, radix_sort_scratch_bytes64(count));
  if (!sscr) return fail(RS_E_NOMEM, "arena exhausted (lpt)");
  RS_TRY(clear_flags(ctx));
  RS_TRY(h2d(ctx, raw, pred, 8 * count));
  if (id_rank) {
    RS_TRY(h2d(ctx, rk, id_rank, 4 * count));
    RS_CUDA_TRY(cudaMemsetAsync(seen, 0, 4 * count, ctx->stream));
  }
  RS_LAUNCH(ctx, "to_id_order", to_id_order_kernel, grid_for(ctx, count, 256), 256, 0, raw,
            (const int32_t*)nullptr, id_rank ? rk : (const int32_t*)nullptr, (int64_t)count, pid,
            (int32_t*)nullptr, (int32_t*)nullptr, id_rank ? seen : (int32_t*)nullptr,
            ctx->d_flags, 1);
  int fl;
  RS_TRY(read_flags(ctx, &fl));
  if (fl & (kFlagBadPerm)) return fail(RS_E_ARG, "id_rank is not a permutation of [0, count)");
  if (fl) return flags_to_status(fl);
  RS_TRY(lpt_core(ctx, pid, count, G, n_min, n_max, keys, vals, len_r, sscr, mk, id));
  RS_TRY(d2h(ctx, makespan, mk, 8 * C));
  RS_TRY(d2h(ctx, idle, id, 8 * C));
  return sync_and_check(ctx);
}

}  // extern "C"
