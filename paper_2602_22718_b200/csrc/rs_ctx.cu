// rs_ctx.cu — context, scratch arena, error plumbing, launch accounting and
// the device latency-profile tables of librs_b200.so.
#include <cmath>
#include <cstring>
#include <string>

#include "rs_internal.cuh"

namespace rs {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int arena_reserve(rs_ctx* ctx, size_t bytes) {
  arena_reset(ctx);
  if (bytes <= ctx->arena_cap) return RS_OK;
  // Kernels of an earlier asynchronous call may still use the arena.
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (ctx->arena) cudaFree(ctx->arena);
  ctx->arena = nullptr;
  ctx->arena_cap = 0;
  size_t cap = bytes + bytes / 4 + (1 << 20);
  if (cudaMalloc(&ctx->arena, cap) != cudaSuccess) {
    cudaGetLastError();
    return fail(RS_E_NOMEM, "device scratch allocation of " +
                                std::to_string(cap) + " bytes failed");
  }
  ctx->arena_cap = cap;
  return RS_OK;
}

void arena_reset(rs_ctx* ctx) { ctx->arena_used = 0; }

int pinned_reserve(rs_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->pinned_cap) return RS_OK;
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  ctx->pinned = nullptr;
  ctx->pinned_cap = 0;
  size_t cap = bytes + bytes / 4 + (1 << 20);
  if (cudaMallocHost(&ctx->pinned, cap) != cudaSuccess) {
    cudaGetLastError();
    return fail(RS_E_NOMEM, "pinned allocation failed");
  }
  ctx->pinned_cap = cap;
  return RS_OK;
}

PinnedPool::~PinnedPool() {
  for (auto& b : free) cudaFreeHost(b.first);
}

void* PinnedPool::take(size_t bytes, size_t* cap) {
  {
    std::lock_guard<std::mutex> g(m);
    for (size_t i = 0; i < free.size(); ++i)
      if (free[i].second >= bytes) {
        const auto b = free[i];
        free.erase(free.begin() + i);
        *cap = b.second;
        return b.first;
      }
  }
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  *cap = bytes;
  return p;
}

void PinnedPool::give(void* p, size_t cap) {
  std::lock_guard<std::mutex> g(m);
  if (free.size() < 8) {
    free.emplace_back(p, cap);
    return;
  }
  cudaFreeHost(p);
}

void timer_begin(rs_ctx* ctx, const char* name, cudaEvent_t* a) {
  (void)name;
  *a = nullptr;
  if (!ctx->timing) return;
  cudaEvent_t e;
  if (!ctx->event_pool.empty()) {
    e = ctx->event_pool.back();
    ctx->event_pool.pop_back();
  } else if (cudaEventCreate(&e) != cudaSuccess) {
    return;
  }
  cudaEventRecord(e, ctx->stream);
  *a = e;
}

void timer_end(rs_ctx* ctx, const char* name, cudaEvent_t a) {
  if (!ctx->timing || !a) return;
  cudaEvent_t b;
  if (!ctx->event_pool.empty()) {
    b = ctx->event_pool.back();
    ctx->event_pool.pop_back();
  } else if (cudaEventCreate(&b) != cudaSuccess) {
    return;
  }
  cudaEventRecord(b, ctx->stream);
  ctx->pending.push_back({name, a, b});
}

int collect_timers(rs_ctx* ctx) {
  for (auto& pd : ctx->pending) {
    RS_CUDA_TRY(cudaEventSynchronize(pd.b));
    float ms = 0;
    cudaEventElapsedTime(&ms, pd.a, pd.b);
    KernelTimer& t = ctx->timers[pd.name];
    t.total_ms += ms;
    t.launches += 1;
    ctx->event_pool.push_back(pd.a);
    ctx->event_pool.push_back(pd.b);
  }
  ctx->pending.clear();
  return RS_OK;
}

int flags_to_status(int flags) {
  if (flags & kFlagEmptyPrompt)
    return fail(RS_E_VALIDATION, "prefix index: empty prompt in batch");
  if (flags & kFlagNotFinite)
    return fail(RS_E_VALIDATION, "predicted length is not finite");
  if (flags & kFlagTargetBelowOne)
    return fail(RS_E_VALIDATION, "integrate_decode_seconds: target length < 1");
  if (flags & kFlagBadPerm)
    return fail(RS_E_ARG, "id_rank is not a permutation of [0, count)");
  if (flags & kFlagWorkOverflow)
    return fail(RS_E_CUDA, "internal work capacity exceeded");
  if (flags & (kFlagBucketOverflow | kFlagBucketTooWide))
    return fail(RS_E_CUDA, "internal: fast scenario structure not applicable (unhandled fallback)");
  if (flags) return fail(RS_E_CUDA, "internal: unhandled device status flags " + std::to_string(flags));
  return RS_OK;
}

int clear_flags(rs_ctx* ctx) {
  RS_CUDA_TRY(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), ctx->stream));
  return RS_OK;
}

int sync_and_check(rs_ctx* ctx) {
  RS_CUDA_TRY(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(int),
                              cudaMemcpyDeviceToHost, ctx->stream));
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (ctx->timing) RS_TRY(collect_timers(ctx));
  const int flags = *ctx->h_flags;
  if (flags) {  // reported once: the next call starts from a clean status
    *ctx->h_flags = 0;
    RS_TRY(clear_flags(ctx));
  }
  return flags_to_status(flags);
}

int h2d(rs_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return RS_OK;
  RS_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return RS_OK;
}

int d2h(rs_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (!bytes) return RS_OK;
  RS_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return RS_OK;
}

int validate_profile_shape(const rs_profile* p) {
  if (!p) return fail(RS_E_ARG, "profile is NULL");
  if (p->nb < 2 || p->nc < 2)
    return fail(RS_E_CONFIG, "tpot needs at least two knots per axis");
  if (!p->batch_knots || !p->context_knots || !p->tpot_grid)
    return fail(RS_E_ARG, "profile arrays are NULL");
  for (int i = 1; i < p->nb; ++i)
    if (!(p->batch_knots[i] > p->batch_knots[i - 1]))
      return fail(RS_E_CONFIG, "tpot batch knots must be strictly increasing");
  for (int i = 1; i < p->nc; ++i)
    if (!(p->context_knots[i] > p->context_knots[i - 1]))
      return fail(RS_E_CONFIG, "tpot context knots must be strictly increasing");
  return RS_OK;
}

// Fill the memo tables with the device's own exact axis function, so the
// table entries are bitwise the values tpot_direct would compute.
__global__ void build_memo_kernel(DevProfile p) {
  int64_t nbm = p.has_bmemo ? p.b_hi - p.b_lo + 1 : 0;
  int64_t ncm = p.has_cmemo ? p.c_hi - p.c_lo + 1 : 0;
  double back_b = p.bk[p.nb - 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       i < nbm + ncm; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nbm) {
      int idx;
      double t;
      axis_direct(p.bk, p.nb, (double)(p.b_lo + i), &idx, &t);
      const_cast<int32_t*>(p.bi)[i] = idx;
      const_cast<double*>(p.tb)[i] = t;
    } else {
      int64_t j = i - nbm;
      int idx;
      double t;
      axis_direct(p.ck, p.nc, (double)(p.c_lo + j), &idx, &t);
      const_cast<int32_t*>(p.ci)[j] = idx;
      const_cast<double*>(p.tc)[j] = t;
      const_cast<double*>(p.top_row)[j] = tpot_direct(p, back_b, (double)(p.c_lo + j));
    }
  }
}

int get_profile(rs_ctx* ctx, const rs_profile* p, DevProfile* out) {
  RS_TRY(validate_profile_shape(p));
  std::vector<double> key;
  key.reserve(4 + p->nb + p->nc + (size_t)p->nb * p->nc);
  key.push_back(p->nb);
  key.push_back(p->nc);
  key.push_back(p->rho);
  key.insert(key.end(), p->batch_knots, p->batch_knots + p->nb);
  key.insert(key.end(), p->context_knots, p->context_knots + p->nc);
  key.insert(key.end(), p->tpot_grid, p->tpot_grid + (size_t)p->nb * p->nc);
  for (auto& c : ctx->profiles) {
    if (c.key.size() == key.size() &&
        std::memcmp(c.key.data(), key.data(), key.size() * sizeof(double)) == 0) {
      *out = c.dev;
      return RS_OK;
    }
  }
  ProfileCache pc;
  pc.key = key;
  DevProfile d{};
  d.nb = p->nb;
  d.nc = p->nc;
  d.rho = p->rho;
  double bf = std::floor(p->batch_knots[0]), bb = std::ceil(p->batch_knots[p->nb - 1]);
  double cf = std::floor(p->context_knots[0]), cb = std::ceil(p->context_knots[p->nc - 1]);
  d.has_bmemo = std::isfinite(bf) && std::isfinite(bb) && (bb - bf) < kMemoMax;
  d.has_cmemo = std::isfinite(cf) && std::isfinite(cb) && (cb - cf) < kMemoMax;
  d.b_lo = d.has_bmemo ? (int64_t)bf : 0;
  d.b_hi = d.has_bmemo ? (int64_t)bb : -1;
  d.c_lo = d.has_cmemo ? (int64_t)cf : 0;
  d.c_hi = d.has_cmemo ? (int64_t)cb : -1;
  if (!d.has_bmemo) d.b_hi = INT64_MAX;  // never takes the top-row shortcut
  d.cfront_m1 = std::ceil(p->context_knots[0]) - 1.0;
  d.ck_front = p->context_knots[0];
  d.ck_back = p->context_knots[p->nc - 1];
  size_t nbm = d.has_bmemo ? (size_t)(d.b_hi - d.b_lo + 1) : 0;
  size_t ncm = d.has_cmemo ? (size_t)(d.c_hi - d.c_lo + 1) : 0;
  size_t grid_n = (size_t)p->nb * p->nc;
  size_t bytes = abytes(p->nb, 8) + abytes(p->nc, 8) + abytes(grid_n, 8) +
                 abytes(p->nc, 8) + abytes(nbm, 8) + abytes(nbm, 4) +
                 abytes(ncm, 8) * 2 + abytes(ncm, 4);
  char* mem = nullptr;
  if (cudaMalloc(&mem, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(RS_E_NOMEM, "profile table allocation failed");
  }
  pc.mem = mem;
  char* q = mem;
  auto take = [&](size_t b) { char* r = q; q += b; return r; };
  double* bk = (double*)take(abytes(p->nb, 8));
  double* ck = (double*)take(abytes(p->nc, 8));
  double* grid = (double*)take(abytes(grid_n, 8));
  double* kfl = (double*)take(abytes(p->nc, 8));
  d.tb = (double*)take(abytes(nbm, 8));
  d.bi = (int32_t*)take(abytes(nbm, 4));
  d.tc = (double*)take(abytes(ncm, 8));
  d.top_row = (double*)take(abytes(ncm, 8));
  d.ci = (int32_t*)take(abytes(ncm, 4));
  std::vector<double> kf(p->nc);
  for (int i = 0; i < p->nc; ++i) kf[i] = std::floor(p->context_knots[i]);
  RS_CUDA_TRY(cudaMemcpyAsync(bk, p->batch_knots, 8 * p->nb, cudaMemcpyHostToDevice, ctx->stream));
  RS_CUDA_TRY(cudaMemcpyAsync(ck, p->context_knots, 8 * p->nc, cudaMemcpyHostToDevice, ctx->stream));
  RS_CUDA_TRY(cudaMemcpyAsync(grid, p->tpot_grid, 8 * grid_n, cudaMemcpyHostToDevice, ctx->stream));
  RS_CUDA_TRY(cudaMemcpyAsync(kfl, kf.data(), 8 * p->nc, cudaMemcpyHostToDevice, ctx->stream));
  d.bk = bk;
  d.ck = ck;
  d.grid = grid;
  d.kfloor = kfl;
  if (nbm + ncm) {
    int blocks = (int)std::min<size_t>((nbm + ncm + 255) / 256, 4096);
    RS_LAUNCH(ctx, "build_memo", build_memo_kernel, blocks, 256, 0, d);
  }
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  pc.dev = d;
  ctx->profiles.push_back(pc);
  *out = d;
  return RS_OK;
}

__global__ void tpot_points_kernel(DevProfile p, const double* b,
                                   const double* c, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = tpot_direct(p, b[i], c[i]);
}

}  // namespace rs

using namespace rs;

extern "C" {

const char* rs_last_error(void) { return rs::g_err.c_str(); }
int rs_abi_version(void) { return RS_ABI_VERSION; }

int rs_ctx_create(int device, rs_ctx** out) {
  if (!out) return fail(RS_E_ARG, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(RS_E_CUDA, "no CUDA device available (librs_b200 has no CPU fallback)");
  }
  if (device < 0 || device >= n) return fail(RS_E_ARG, "bad device index");
  ::rs::DeviceGuard guard(device);  // the caller's current device is restored on return
  cudaDeviceProp prop;
  RS_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(RS_E_CUDA, std::string("librs_b200 is built for sm_100a; device is ") + prop.name);
  rs_ctx* c = new rs_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(RS_E_CUDA, "stream creation failed");
  }
  c->stream = c->own_stream;
  if (cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaStreamDestroy(c->own_stream);
    delete c;
    return fail(RS_E_CUDA, "stream creation failed");
  }
  if (cudaStreamCreateWithFlags(&c->in_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    rs_ctx_destroy(c);
    return fail(RS_E_CUDA, "stream creation failed");
  }
  for (int i = 0; i < 2; ++i)
    if (cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_inused[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      rs_ctx_destroy(c);
      return fail(RS_E_CUDA, "event creation failed");
    }
  {  // stream-ordered temporaries (trace parsing) stay cached in the pool
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
  }
  if (cudaMalloc(&c->d_flags, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&c->h_flags, sizeof(int)) != cudaSuccess) {
    delete c;
    return fail(RS_E_NOMEM, "flag allocation failed");
  }
  cudaMemset(c->d_flags, 0, sizeof(int));
  *out = c;
  return RS_OK;
}

int rs_ctx_destroy(rs_ctx* ctx) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return RS_OK;
  cudaStreamSynchronize(ctx->stream);
  for (auto& p : ctx->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : ctx->event_pool) cudaEventDestroy(e);
  for (auto& pc : ctx->profiles) cudaFree(pc.mem);
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->in_buf) cudaFree(ctx->in_buf);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->d_flags) cudaFree(ctx->d_flags);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  for (cudaStream_t s : {ctx->copy_stream, ctx->in_stream})
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  if (ctx->bounce) cudaFreeHost(ctx->bounce);
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t e : {ctx->ev_done[i], ctx->ev_copied[i], ctx->ev_in[i], ctx->ev_inused[i]})
      if (e) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
  return RS_OK;
}

int rs_ctx_set_stream(rs_ctx* ctx, void* stream) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "ctx is NULL");
  cudaStream_t next = stream ? (cudaStream_t)stream : ctx->own_stream;
  // work still queued on the old stream may use the arena / input buffers
  if (next != ctx->stream) RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  ctx->stream = next;
  return RS_OK;
}

int rs_ctx_synchronize(rs_ctx* ctx) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "ctx is NULL");
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  if (ctx->timing) RS_TRY(collect_timers(ctx));
  return RS_OK;
}

int rs_ctx_kernel_launches(const rs_ctx* ctx, uint64_t* count) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !count) return fail(RS_E_ARG, "NULL argument");
  *count = ctx->launches;
  return RS_OK;
}

int rs_ctx_enable_kernel_timing(rs_ctx* ctx, int enable) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "ctx is NULL");
  ctx->timing = enable != 0;
  return RS_OK;
}

int rs_ctx_reset_kernel_timing(rs_ctx* ctx) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "ctx is NULL");
  RS_TRY(collect_timers(ctx));
  ctx->timers.clear();
  return RS_OK;
}

int rs_ctx_kernel_time(rs_ctx* ctx, const char* name, double* total_ms,
                       uint64_t* launches) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !name) return fail(RS_E_ARG, "NULL argument");
  RS_TRY(collect_timers(ctx));
  auto it = ctx->timers.find(name);
  if (total_ms) *total_ms = it == ctx->timers.end() ? 0 : it->second.total_ms;
  if (launches) *launches = it == ctx->timers.end() ? 0 : it->second.launches;
  return RS_OK;
}

int rs_tpot_seconds(rs_ctx* ctx, const rs_profile* profile, const double* b,
                    const double* c, int64_t n, double* out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx) return fail(RS_E_ARG, "ctx is NULL");
  if (n <= 0) return RS_OK;
  DevProfile dp;
  RS_TRY(get_profile(ctx, profile, &dp));
  RS_TRY(arena_reserve(ctx, abytes(n, 8) * 3));
  double* db = arena_alloc<double>(ctx, n);
  double* dc = arena_alloc<double>(ctx, n);
  double* dout = arena_alloc<double>(ctx, n);
  RS_TRY(h2d(ctx, db, b, 8 * n));
  RS_TRY(h2d(ctx, dc, c, 8 * n));
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 8 * ctx->num_sms);
  RS_LAUNCH(ctx, "tpot_points", tpot_points_kernel, blocks, 256, 0, dp, db, dc, n, dout);
  RS_TRY(d2h(ctx, out, dout, 8 * n));
  return sync_and_check(ctx);
}

}  // extern "C"
