// rs_internal.cuh — shared internals of librs_b200.so (sm_100a).
//
// Context / scratch arena / launch accounting, the device copy of a latency
// profile with exact memo tables, and the IEEE-exact FP64 helpers every
// planner kernel uses. The whole library is compiled with --fmad=false and
// the arithmetic that must match the reference bit for bit is spelled with
// explicit __d*_rn intrinsics as well, so no FMA contraction can change a
// result.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "rs.h"

namespace rs {

// ---------------------------------------------------------------- errors --
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define RS_CUDA_TRY(expr)                                                    \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return ::rs::fail(RS_E_CUDA, std::string(#expr ": ") +                 \
                                       cudaGetErrorString(e_));              \
  } while (0)

#define RS_TRY(expr)          \
  do {                        \
    int s_ = (expr);          \
    if (s_ != RS_OK) return s_; \
  } while (0)

// ------------------------------------------------------------ constants --
constexpr int kWarp = 32;
constexpr int kMemoMax = 1 << 22;   // max entries of an exact tpot memo axis
constexpr int kBucketFmax = 16384;  // finish-tick range of the bucketed path

// Device status flags written by kernels (bitmask in a device int).
enum : int {
  kFlagTargetBelowOne = 1,   // integrate_decode_seconds: target length < 1
  kFlagNotFinite = 2,        // NaN/inf prediction (rejected; reference UB)
  kFlagBucketOverflow = 4,   // bucketed path not applicable (finish > Fmax)
  kFlagBucketTooWide = 8,    // a finish bucket too wide for in-warp sort
  kFlagEmptyPrompt = 16,     // prefix index: prompt of length < 1
  kFlagWorkOverflow = 32,    // dedup refinement exceeded its work capacity
  kFlagBadPerm = 64,         // id_rank is not a permutation of [0, count)
};
// Flags after which the fast scenario structure is not usable: every kernel
// that reads it returns at once (the host reruns the batch on the generic path
// or reports the validation error).
constexpr int kFastBad = kFlagBucketOverflow | kFlagBucketTooWide | kFlagNotFinite;

// -------------------------------------------------------------- profile --
// Device view of a LatencyProfile. tpot(b, c) is only ever evaluated at
// integer (b, c) by the planner (batch = G * live prompts, context = integer
// base + tick; proj/src/planner.cpp:122-126, piece ends are floor/ceil of
// knots :69-74), so per-axis tables of the clamp/interval/division results,
// computed with the same operations, are bit-identical to the reference.
struct DevProfile {
  int nb, nc;
  const double* bk;    // batch knots
  const double* ck;    // context knots
  const double* grid;  // nb*nc
  double rho;
  // Batch memo over integers [b_lo, b_hi] (= [floor(front), ceil(back)]).
  int64_t b_lo, b_hi;
  const double* tb;
  const int32_t* bi;
  // Context memo over integers [c_lo, c_hi].
  int64_t c_lo, c_hi;
  const double* tc;
  const int32_t* ci;
  const double* top_row;  // tpot(batch_knots.back(), c) for c in memo range
  const double* kfloor;   // floor(context_knots[i])
  double cfront_m1;       // ceil(front) - 1
  double ck_front, ck_back;  // context_knots.front() / .back(), host copies
  int has_bmemo, has_cmemo;
};

struct ProfileCache {
  std::vector<double> key;  // flattened profile contents
  DevProfile dev{};
  void* mem = nullptr;
};

// ------------------------------------------------------------------ ctx --
struct KernelTimer {
  double total_ms = 0;
  uint64_t launches = 0;
};

// Recycled pinned host blocks. Shared by a context and the objects it
// builds (a prefix index keeps its tables in the block the tables kernel
// wrote), so a block outlives the context and returns here when the index
// is freed.
struct PinnedPool {
  std::mutex m;
  std::vector<std::pair<void*, size_t>> free;
  ~PinnedPool();
  void* take(size_t bytes, size_t* cap);  // nullptr if the allocation fails
  void give(void* p, size_t cap);
};

}  // namespace rs

struct rs_ctx {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  // Grow-only device arena; a bump allocator resets per public call.
  char* arena = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  // Pinned host staging.
  char* pinned = nullptr;
  size_t pinned_cap = 0;
  int* d_flags = nullptr;  // kernel status bits
  int* h_flags = nullptr;  // pinned mirror
  std::shared_ptr<rs::PinnedPool> pin_pool = std::make_shared<rs::PinnedPool>();
  // Second stream for device-to-host result copies that overlap the next
  // batch's kernels (the sweep), with per-buffer-set events.
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
  // Third stream for host-to-device input copies of the next batch (the
  // sweep over caller arrays), with per-input-set events.
  cudaStream_t in_stream = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_inused[2] = {nullptr, nullptr};
  // Pinned bounce buffers for results bound for pageable caller memory.
  char* bounce = nullptr;
  size_t bounce_cap = 0;
  uint64_t launches = 0;
  bool timing = false;
  std::map<std::string, rs::KernelTimer> timers;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<rs::ProfileCache> profiles;
  int num_sms = 148;
  // Kernel attributes / occupancy are per device: cached on the context
  // (one context per device), set under its device guard.
  struct {
    int refine_per_sm = 0, stream_per_sm = 0;
    bool tables_ready = false;
  } dev_cache;
  // Grow-only device copy of host inputs (CSR token batches), kept apart
  // from the arena, which may grow during a call.
  char* in_buf = nullptr;
  size_t in_cap = 0;
};

namespace rs {

// Arena: reserve `bytes` (256-aligned). Grows (after a stream sync) when
// needed; pointers handed out earlier in the same call stay valid because
// growth only happens through arena_reserve() before any allocation.
int arena_reserve(rs_ctx* ctx, size_t bytes);
void arena_reset(rs_ctx* ctx);
template <class T>
T* arena_alloc(rs_ctx* ctx, size_t count) {
  size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
  if (ctx->arena_used + bytes > ctx->arena_cap) return nullptr;
  T* p = reinterpret_cast<T*>(ctx->arena + ctx->arena_used);
  ctx->arena_used += bytes;
  return p;
}
inline size_t abytes(size_t count, size_t elem) {
  return (count * elem + 255) & ~size_t(255);
}
int pinned_reserve(rs_ctx* ctx, size_t bytes);

// Launch accounting + optional per-kernel CUDA-event timing.
void timer_begin(rs_ctx* ctx, const char* name, cudaEvent_t* a);
void timer_end(rs_ctx* ctx, const char* name, cudaEvent_t a);
int collect_timers(rs_ctx* ctx);

#define RS_LAUNCH(ctx, name, kernel, grid, block, smem, ...)               \
  do {                                                                      \
    cudaEvent_t ev_a_ = nullptr;                                            \
    ::rs::timer_begin((ctx), (name), &ev_a_);                               \
    kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);        \
    (ctx)->launches++;                                                      \
    cudaError_t le_ = cudaGetLastError();                                   \
    if (le_ != cudaSuccess)                                                 \
      return ::rs::fail(RS_E_CUDA, std::string("launch ") + (name) + ": " + \
                                       cudaGetErrorString(le_));            \
    ::rs::timer_end((ctx), (name), ev_a_);                                  \
  } while (0)

// Every entry point that takes a context runs on the context's device: the
// guard makes it current and restores the caller's device on return.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const rs_ctx* c) : DeviceGuard(c ? c->device : -1) {}
  explicit DeviceGuard(int device) {
    int cur = -1;
    if (device >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != device &&
        cudaSetDevice(device) == cudaSuccess)
      prev = cur;
    cudaGetLastError();
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#define RS_DEVICE_GUARD(ctx) ::rs::DeviceGuard rs_device_guard_(ctx)

// Synchronise the context stream and translate kernel status flags.
int sync_and_check(rs_ctx* ctx);
int flags_to_status(int flags);
int clear_flags(rs_ctx* ctx);

// Upload (or fetch the cached) device profile.
int get_profile(rs_ctx* ctx, const rs_profile* p, DevProfile* out);
int validate_profile_shape(const rs_profile* p);

// H2D / D2H helpers through the context stream (host pointers may be
// pageable; large copies are staged through pinned memory by the runtime).
int h2d(rs_ctx* ctx, void* dst, const void* src, size_t bytes);
int d2h(rs_ctx* ctx, void* dst, const void* src, size_t bytes);

// ---------------------------------------------------- exact FP64 helpers --
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// std::upper_bound over a small sorted array.
__device__ __forceinline__ int upper_bound_d(const double* k, int n, double v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(k + mid) > v) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// interval_of + clamp_to + the division of one axis
// (proj/src/profile.cpp:21-30, :45-51).
__device__ __forceinline__ void axis_direct(const double* k, int n, double v,
                                            int* idx, double* t) {
  double front = __ldg(k), back = __ldg(k + n - 1);
  double x = v > front ? v : front;  // std::max(front, v)
  x = back < x ? back : x;           // std::min(back, x)
  int i;
  if (x <= front) i = 0;
  else if (x >= back) i = n - 2;
  else i = upper_bound_d(k, n, x) - 1;
  double k0 = __ldg(k + i), k1 = __ldg(k + i + 1);
  *idx = i;
  *t = ddiv(dsub(x, k0), dsub(k1, k0));
}

// Bilinear blend (proj/src/profile.cpp:52-58), fixed operation order.
__device__ __forceinline__ double blend(const double* grid, int nc, int bi,
                                        double tb, int ci, double tc) {
  const double* r0 = grid + (size_t)bi * nc + ci;
  const double* r1 = r0 + nc;
  double v00 = __ldg(r0), v01 = __ldg(r0 + 1);
  double v10 = __ldg(r1), v11 = __ldg(r1 + 1);
  double lo = dadd(v00, dmul(dsub(v01, v00), tc));
  double hi = dadd(v10, dmul(dsub(v11, v10), tc));
  return dadd(lo, dmul(dsub(hi, lo), tb));
}

// LatencyProfile::tpot_seconds at arbitrary doubles (no memo).
__device__ __forceinline__ double tpot_direct(const DevProfile& p, double b,
                                              double c) {
  int bi, ci;
  double tb, tc;
  axis_direct(p.bk, p.nb, b, &bi, &tb);
  axis_direct(p.ck, p.nc, c, &ci, &tc);
  return blend(p.grid, p.nc, bi, tb, ci, tc);
}

__device__ __forceinline__ int64_t clamp64(int64_t v, int64_t lo, int64_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

// tpot at integer (batch, context) — memo tables when available.
__device__ __forceinline__ double tpot_int(const DevProfile& p, int64_t b,
                                           int64_t c) {
  if (p.has_cmemo) {
    int64_t jc = clamp64(c, p.c_lo, p.c_hi) - p.c_lo;
    if (b >= p.b_hi) return __ldg(p.top_row + jc);  // b clamps to back
    int ci = __ldg(p.ci + jc);
    double tc = __ldg(p.tc + jc);
    int bi;
    double tb;
    if (p.has_bmemo) {
      int64_t jb = clamp64(b, p.b_lo, p.b_hi) - p.b_lo;
      bi = __ldg(p.bi + jb);
      tb = __ldg(p.tb + jb);
    } else {
      axis_direct(p.bk, p.nb, (double)b, &bi, &tb);
    }
    return blend(p.grid, p.nc, bi, tb, ci, tc);
  }
  return tpot_direct(p, (double)b, (double)c);
}

// tpot_context_run_sum (proj/src/planner.cpp:61-84) over integer contexts
// [c_lo, c_hi] at integer batch b: per knot piece count*(first+last)/2,
// accumulated in piece order.
__device__ __forceinline__ double run_sum_int(const DevProfile& p, int64_t b,
                                              int64_t c_lo, int64_t c_hi) {
  const double front = __ldg(p.ck), back = __ldg(p.ck + p.nc - 1);
  double total = 0.0;
  int64_t c = c_lo;
  while (c <= c_hi) {
    double cd = (double)c;
    int64_t pe;
    if (cd < front) {
      double e = p.cfront_m1;
      pe = (double)c_hi < e ? c_hi : (int64_t)e;
    } else if (cd >= back) {
      pe = c_hi;
    } else {
      int up;
      if (p.has_cmemo) up = __ldg(p.ci + (clamp64(c, p.c_lo, p.c_hi) - p.c_lo)) + 1;
      else up = upper_bound_d(p.ck, p.nc, cd);
      double e = __ldg(p.kfloor + up);
      pe = (double)c_hi < e ? c_hi : (int64_t)e;
    }
    double count = (double)(pe - c + 1);
    double s = dadd(tpot_int(p, b, c), tpot_int(p, b, pe));
    total = dadd(total, dmul(dmul(count, s), 0.5));  // count*(a+b)/2.0
    c = pe + 1;
  }
  return total;
}

// ----------------------------------------------------------- rng (rng.hpp) --
__device__ __host__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
__device__ __host__ __forceinline__ uint64_t hash_u64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}
__device__ __host__ __forceinline__ uint64_t hash_combine(uint64_t a, uint64_t b) {
  return hash_u64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}
// k-th next_u64() (k >= 1) of Rng(seed) (proj/include/rollsim/rng.hpp:20-25).
__device__ __host__ __forceinline__ uint64_t draw_at(uint64_t seed, uint64_t k) {
  return mix64(seed + k * 0x9e3779b97f4a7c15ULL);
}

// ------------------------------------------------------------ warp utils --
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u > v ? u : v;
  }
  return v;
}
template <class T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(0xffffffffu, v, o);
    v = u < v ? u : v;
  }
  return v;
}
template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Inclusive prefix sum over lanes.
template <class T>
__device__ __forceinline__ T warp_incl_sum(T v) {
  int l = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (l >= o) v += u;
  }
  return v;
}

}  // namespace rs
