// rs_predict.cu — the prediction snapshot on the device:
// LengthHistory::predict / predict_noisy (proj/src/predictor.cpp:52-98) for
// every scheduled prompt of a step (snapshot_predictions,
// proj/src/training.cpp:53-66). One thread per prompt; the window is a
// handful of observations, so the work is the per-prompt sequential EWMA
// plus, for the bucket noise model, a keyed splitmix64 stream. The output
// can stay in HBM and feed the scaling sweep (rs_sweep_arrays) directly.
#include <algorithm>
#include <string>

#include "rs_internal.cuh"

namespace rs {

namespace {

// std::max(1.0, est) then std::min(max_len, .) (predictor.cpp:64, 97)
__device__ __forceinline__ double clamp_len(double est, double max_len) {
  const double lo = 1.0 < est ? est : 1.0;
  return lo < max_len ? lo : max_len;
}

// splitmix64 Rng (rng.hpp:14-49)
struct DevRng {
  uint64_t state;
  __device__ uint64_t next_u64() {
    state += 0x9e3779b97f4a7c15ULL;
    return mix64(state);
  }
  __device__ double uniform() { return dmul((double)(next_u64() >> 11), 0x1.0p-53); }
  __device__ double uniform(double lo, double hi) { return dadd(lo, dmul(dsub(hi, lo), uniform())); }
  __device__ int64_t uniform_int(int64_t lo, int64_t hi) {
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    return lo + (int64_t)(next_u64() % span);
  }
};

__global__ void predict_kernel(const double* obs, const int32_t* depth, const int32_t* gt,
                               int32_t count, int32_t window, double alpha, int32_t max_len,
                               int32_t noisy, double accuracy, int32_t bucket_width,
                               uint64_t seed, const char* ids, const int64_t* id_off,
                               double* out) {
  const double mlen = (double)max_len;
  const double one_m_alpha = dsub(1.0, alpha);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = depth[i];
    double est;
    if (d == 0) {
      est = (double)gt[i];
    } else {  // est = o_1; est = alpha * o_k + (1 - alpha) * est (predictor.cpp:58-62)
      const double* q = obs + i * (int64_t)window;
      est = q[0];
      for (int k = 1; k < d; ++k) est = dadd(dmul(alpha, q[k]), dmul(one_m_alpha, est));
    }
    const double base = clamp_len(est, mlen);
    if (!noisy) {
      out[i] = base;
      continue;
    }
    // predict_noisy (predictor.cpp:67-98)
    const int bucket_count = (max_len + bucket_width - 1) / bucket_width;
    if (bucket_count <= 1) {
      out[i] = base;
      continue;
    }
    uint64_t h = 0xcbf29ce484222325ULL;  // fnv1a (rng.hpp:64-71)
    for (int64_t b = id_off[i]; b < id_off[i + 1]; ++b) {
      h ^= (unsigned char)ids[b];
      h *= 0x100000001b3ULL;
    }
    uint64_t key = hash_combine(seed, h);
    key = hash_combine(key, (uint64_t)d);
    key = hash_combine(key, (uint64_t)__double_as_longlong(base));
    DevRng rng{key};
    if (rng.uniform() < accuracy) {
      out[i] = base;
      continue;
    }
    int true_bucket = (int)ddiv(dsub(base, 1.0), (double)bucket_width);
    true_bucket = min(true_bucket, bucket_count - 1);
    int wrong = (int)rng.uniform_int(0, bucket_count - 2);
    if (wrong >= true_bucket) ++wrong;
    const double lo = dadd((double)(wrong * bucket_width), 1.0);
    const double hb = (double)((wrong + 1) * bucket_width);
    const double hi = mlen < hb ? mlen : hb;  // std::min<double>(hb, max_len)
    out[i] = clamp_len(rng.uniform(lo, hi), mlen);
  }
}

}  // namespace

}  // namespace rs

using namespace rs;

extern "C" int rs_predict_lengths(rs_ctx* ctx, const double* obs, const int32_t* depth,
                                  const int32_t* ground_truth_len, int32_t count, int32_t window,
                                  double alpha, int32_t max_response_len,
                                  const rs_noise_model* noise, const char* id_bytes,
                                  const int64_t* id_offsets, int device_ptrs, double* out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "NULL context");
  // LengthHistory's constructor checks (predictor.cpp:24-31)
  if (window < 1) return fail(RS_E_CONFIG, "predictor window must be >= 1");
  if (!(alpha > 0) || alpha > 1) return fail(RS_E_CONFIG, "predictor alpha must be in (0, 1]");
  if (max_response_len < 1) return fail(RS_E_CONFIG, "predictor max_response_len must be >= 1");
  if (count < 0) return fail(RS_E_VALIDATION, "predict: negative prompt count");
  const bool noisy = noise && noise->kind != 0;
  if (noisy) {  // NoiseModel::validate (predictor.cpp:17-22)
    if (noise->kind != 1) return fail(RS_E_CONFIG, "unknown noise model kind");
    if (noise->bucket_accuracy < 0 || noise->bucket_accuracy > 1)
      return fail(RS_E_CONFIG, "noise bucket_accuracy must be in [0, 1]");
    if (noise->bucket_width < 1 || noise->bucket_width > max_response_len)
      return fail(RS_E_CONFIG, "noise bucket_width must be in [1, max_response_len]");
  }
  if (count == 0) return RS_OK;
  if (!depth || !ground_truth_len || !out || (noisy && (!id_bytes || !id_offsets)))
    return fail(RS_E_ARG, "NULL argument");
  try {
    const double* d_obs = obs;
    const int32_t* d_depth = depth;
    const int32_t* d_gt = ground_truth_len;
    const char* d_ids = id_bytes;
    const int64_t* d_off = id_offsets;
    double* d_out = out;
    if (!device_ptrs) {
      int64_t id_bytes_n = 0;
      if (noisy) id_bytes_n = id_offsets[count];
      for (int32_t i = 0; i < count; ++i)
        if (depth[i] < 0 || depth[i] > window)
          return fail(RS_E_VALIDATION, "predict: observation depth outside [0, window]");
      const size_t n_obs = (size_t)count * window;
      RS_TRY(arena_reserve(ctx, abytes(n_obs, 8) + abytes(count, 4) * 2 + abytes(count, 8) +
                                    (noisy ? abytes(id_bytes_n + 1, 1) + abytes(count + 1, 8) : 0) +
                                    4096));
      double* o = arena_alloc<double>(ctx, n_obs);
      int32_t* dp = arena_alloc<int32_t>(ctx, count);
      int32_t* g = arena_alloc<int32_t>(ctx, count);
      d_out = arena_alloc<double>(ctx, count);
      if (obs) RS_TRY(h2d(ctx, o, obs, 8 * n_obs));
      RS_TRY(h2d(ctx, dp, depth, 4 * (size_t)count));
      RS_TRY(h2d(ctx, g, ground_truth_len, 4 * (size_t)count));
      d_obs = o;
      d_depth = dp;
      d_gt = g;
      if (noisy) {
        char* ib = arena_alloc<char>(ctx, id_bytes_n + 1);
        int64_t* io = arena_alloc<int64_t>(ctx, count + 1);
        if (id_bytes_n) RS_TRY(h2d(ctx, ib, id_bytes, id_bytes_n));
        RS_TRY(h2d(ctx, io, id_offsets, 8 * ((size_t)count + 1)));
        d_ids = ib;
        d_off = io;
      }
    }
    const int grid = (int)std::min<int64_t>((count + 255) / 256, 8 * (int64_t)ctx->num_sms);
    RS_LAUNCH(ctx, "predict_lengths", predict_kernel, grid, 256, 0, d_obs,
              d_depth, d_gt, count, window, alpha, max_response_len, noisy ? 1 : 0,
              noisy ? noise->bucket_accuracy : 1.0, noisy ? noise->bucket_width : 1,
              noisy ? noise->seed : 0, d_ids, d_off, d_out);
    if (!device_ptrs) RS_TRY(d2h(ctx, out, d_out, 8 * (size_t)count));
    return sync_and_check(ctx);
  } catch (const std::exception& e) {
    return fail(RS_E_NOMEM, e.what());
  }
}
