// rs_comm.cu — multi-GPU sweep behind the C-ABI.
//
// Scenarios are independent units (each one is a whole scale(),
// proj/src/planner.cpp:159-218), so rank r of W evaluates the contiguous block
// [S*r/W, S*(r+1)/W) on its own GPU with no data-path exchange. The one
// collective is a single NCCL all-reduce (SUM, FP64) of the packed
// per-candidate aggregates {sum t_total, sum cost, n_star histogram} — 3 x C
// doubles (6 KB at C = 256; histogram counts are exact in FP64) — after which
// every rank takes the aggregate pick (rs_sweep_select) redundantly.
//
// Two hosts of the same machinery:
//  - rs_comm + rs_sweep_sharded: one process per GPU (torchrun, MPI, …); the
//    caller ships the 128-byte NCCL id between its ranks out of band;
//  - rs_multi: one process, one host thread per GPU (contexts and an
//    ncclCommInitAll clique owned by the handle) for C++ hosts such as the
//    drop-in's rollsim::b200::sweep.
//
// NCCL is bound at run time (dlopen "libnccl.so.2"): a process that already
// holds one (torch's) shares it, a plain C++ host gets the system library,
// and librs_b200.so itself loads and runs single-GPU without NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "rs_internal.cuh"

namespace rs {

// sweep driver shared with rs_planner.cu: agg_pack (device, 3 * C doubles,
// nullable) receives {sum_t, sum_c, (double) hist} on the context stream
int sweep_impl_packed(rs_ctx* ctx, const rs_scenario_spec* spec, const double* h_pred,
                      const int32_t* h_plen, int S, int P, const rs_profile* profile, int G,
                      int n_min, int n_max, double lambda, int gpus, rs_sweep_out* out,
                      int device_ptrs, double* agg_pack);
int sweep_select_host(const double* sum_t, const double* sum_c, int64_t n_scenarios, int C,
                      int n_min, double lambda, int32_t* n_star);
int sweep_validate(const rs_scenario_spec* spec, const rs_profile* profile, int P, int G,
                   int n_min, int n_max, double lambda);

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string why;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(sym("ncclCommInitRank"));
    api.init_all = reinterpret_cast<decltype(api.init_all)>(sym("ncclCommInitAll"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(sym("ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    if (!api.get_unique_id || !api.init_rank || !api.init_all || !api.destroy ||
        !api.all_reduce || !api.error_string)
      api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

int nccl_ready() {
  const NcclApi& n = nccl();
  if (!n.why.empty()) return fail(RS_E_CUDA, n.why);
  return RS_OK;
}

#define RS_NCCL_TRY(expr)                                                            \
  do {                                                                               \
    ncclResult_t r_ = (expr);                                                        \
    if (r_ != ncclSuccess)                                                           \
      return ::rs::fail(RS_E_CUDA, std::string(#expr ": ") + nccl().error_string(r_)); \
  } while (0)

}  // namespace

// One rank's part of the sharded sweep: the local sweep with its aggregates
// packed on the device, the one all-reduce, the aggregate pick.
static int sweep_rank(rs_ctx* ctx, ncclComm_t comm, int n_ranks, int rank,
                      const rs_scenario_spec* spec, const rs_profile* profile, int G, int n_min,
                      int n_max, double lambda, int gpus, rs_sweep_out* out, int device_ptrs,
                      int32_t* n_star_all) {
  if (!spec) return fail(RS_E_ARG, "spec is NULL");
  RS_TRY(sweep_validate(spec, profile, spec->count, G, n_min, n_max, lambda));
  const int C = n_max - n_min + 1;
  const int64_t S = spec->n_scenarios;
  const int64_t s0 = S * rank / n_ranks, s1 = S * (rank + 1) / n_ranks;
  rs_scenario_spec local = *spec;
  local.first_scenario = spec->first_scenario + s0;
  local.n_scenarios = (int32_t)(s1 - s0);
  double* pack = nullptr;
  if (cudaMallocAsync(&pack, 24ull * C, ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    return fail(RS_E_NOMEM, "aggregate buffer allocation failed");
  }
  struct Free {
    double* p;
    cudaStream_t s;
    ~Free() { cudaFreeAsync(p, s); }
  } free_pack{pack, ctx->stream};
  RS_CUDA_TRY(cudaMemsetAsync(pack, 0, 24ull * C, ctx->stream));
  // this rank's per-scenario outputs; the aggregates come from the pack
  rs_sweep_out lo = *out;
  lo.sum_t = lo.sum_c = nullptr;
  lo.nstar_hist = nullptr;
  if (local.n_scenarios > 0)
    RS_TRY(sweep_impl_packed(ctx, &local, nullptr, nullptr, local.n_scenarios, spec->count,
                             profile, G, n_min, n_max, lambda, gpus, &lo, device_ptrs, pack));
  RS_NCCL_TRY(nccl().all_reduce(pack, pack, 3ull * C, ncclFloat64, ncclSum, comm, ctx->stream));
  std::vector<double> h(3ull * C);
  RS_CUDA_TRY(cudaMemcpyAsync(h.data(), pack, 24ull * C, cudaMemcpyDeviceToHost, ctx->stream));
  RS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  std::vector<int32_t> hist(C);
  for (int i = 0; i < C; ++i) hist[i] = (int32_t)h[2ull * C + i];
  auto put = [&](void* dst, const void* src, size_t bytes) -> int {
    if (!dst) return RS_OK;
    if (device_ptrs) RS_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    else std::memcpy(dst, src, bytes);
    return RS_OK;
  };
  RS_TRY(put(out->sum_t, h.data(), 8ull * C));
  RS_TRY(put(out->sum_c, h.data() + C, 8ull * C));
  RS_TRY(put(out->nstar_hist, hist.data(), 4ull * C));
  if (n_star_all && S > 0)
    RS_TRY(sweep_select_host(h.data(), h.data() + C, S, C, n_min, lambda, n_star_all));
  return RS_OK;
}

}  // namespace rs

using namespace rs;

struct rs_comm {
  ncclComm_t comm = nullptr;
  int n_ranks = 1, rank = 0, device = 0;
};

struct rs_multi {
  std::vector<rs_ctx*> ctx;
  std::vector<ncclComm_t> comm;
};

extern "C" {

int rs_comm_unique_id(uint8_t* id) {
  if (!id) return fail(RS_E_ARG, "id is NULL");
  RS_TRY(nccl_ready());
  ncclUniqueId u;
  RS_NCCL_TRY(nccl().get_unique_id(&u));
  std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return RS_OK;
}

int rs_comm_init(rs_ctx* ctx, const uint8_t* id, int32_t n_ranks, int32_t rank, rs_comm** out) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !id || !out) return fail(RS_E_ARG, "NULL argument");
  *out = nullptr;
  if (n_ranks < 1 || rank < 0 || rank >= n_ranks) return fail(RS_E_ARG, "bad rank / n_ranks");
  RS_TRY(nccl_ready());
  ncclUniqueId u;
  std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  rs_comm* c = new rs_comm();
  c->n_ranks = n_ranks;
  c->rank = rank;
  c->device = ctx->device;
  ncclResult_t r = nccl().init_rank(&c->comm, n_ranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(RS_E_CUDA, std::string("ncclCommInitRank: ") + nccl().error_string(r));
  }
  *out = c;
  return RS_OK;
}

int rs_comm_destroy(rs_comm* comm) {
  if (!comm) return RS_OK;
  DeviceGuard g(comm->device);
  if (comm->comm) nccl().destroy(comm->comm);
  delete comm;
  return RS_OK;
}

int rs_sweep_sharded(rs_ctx* ctx, rs_comm* comm, const rs_scenario_spec* spec,
                     const rs_profile* profile, int32_t G, int32_t n_min, int32_t n_max,
                     double lambda, int32_t gpus, rs_sweep_out* out, int device_ptrs,
                     int32_t* n_star_all) {
  RS_DEVICE_GUARD(ctx);
  if (!ctx || !comm || !out) return fail(RS_E_ARG, "NULL argument");
  if (comm->device != ctx->device) return fail(RS_E_ARG, "communicator and context are on different devices");
  return sweep_rank(ctx, comm->comm, comm->n_ranks, comm->rank, spec, profile, G, n_min, n_max,
                    lambda, gpus, out, device_ptrs, n_star_all);
}

int rs_multi_create(const int32_t* devices, int32_t n, rs_multi** out) {
  if (!devices || !out || n < 1) return fail(RS_E_ARG, "bad arguments");
  *out = nullptr;
  RS_TRY(nccl_ready());
  rs_multi* m = new rs_multi();
  for (int i = 0; i < n; ++i) {
    rs_ctx* c = nullptr;
    const int st = rs_ctx_create(devices[i], &c);
    if (st != RS_OK) {
      for (auto* x : m->ctx) rs_ctx_destroy(x);
      delete m;
      return st;
    }
    m->ctx.push_back(c);
  }
  m->comm.resize(n);
  std::vector<int> devs(devices, devices + n);
  ncclResult_t r = nccl().init_all(m->comm.data(), n, devs.data());
  if (r != ncclSuccess) {
    for (auto* x : m->ctx) rs_ctx_destroy(x);
    delete m;
    return fail(RS_E_CUDA, std::string("ncclCommInitAll: ") + nccl().error_string(r));
  }
  *out = m;
  return RS_OK;
}

int rs_multi_size(const rs_multi* m, int32_t* n) {
  if (!m || !n) return fail(RS_E_ARG, "NULL argument");
  *n = (int32_t)m->ctx.size();
  return RS_OK;
}

int rs_multi_context(rs_multi* m, int32_t i, rs_ctx** out) {
  if (!m || !out || i < 0 || i >= (int32_t)m->ctx.size()) return fail(RS_E_ARG, "bad arguments");
  *out = m->ctx[i];
  return RS_OK;
}

int rs_multi_destroy(rs_multi* m) {
  if (!m) return RS_OK;
  for (size_t i = 0; i < m->comm.size(); ++i) {
    DeviceGuard g(m->ctx[i]->device);
    if (m->comm[i]) nccl().destroy(m->comm[i]);
  }
  for (auto* c : m->ctx) rs_ctx_destroy(c);
  delete m;
  return RS_OK;
}

int rs_multi_sweep(rs_multi* m, const rs_scenario_spec* spec, const rs_profile* profile,
                   int32_t G, int32_t n_min, int32_t n_max, double lambda, int32_t gpus,
                   rs_sweep_out* out, int32_t* n_star_all) {
  if (!m || !spec || !out) return fail(RS_E_ARG, "NULL argument");
  const int W = (int)m->ctx.size();
  const int C = n_max - n_min + 1;
  std::vector<int> st(W, RS_OK);
  std::vector<std::string> msg(W);
  std::vector<int32_t> pick(W, 0);
  std::vector<std::thread> th;
  for (int r = 0; r < W; ++r)
    th.emplace_back([&, r] {
      const int64_t S = spec->n_scenarios, s0 = S * r / W;
      rs_sweep_out lo = *out;  // this rank's slice of the caller's host arrays
      if (C > 0) {
        if (lo.t_total) lo.t_total += s0 * C;
        if (lo.cost) lo.cost += s0 * C;
        if (lo.idle_slot_ticks) lo.idle_slot_ticks += s0 * C;
        if (lo.n_star) lo.n_star += s0;
      }
      if (r != 0) lo.sum_t = lo.sum_c = nullptr, lo.nstar_hist = nullptr;
      DeviceGuard g(m->ctx[r]->device);
      st[r] = sweep_rank(m->ctx[r], m->comm[r], W, r, spec, profile, G, n_min, n_max, lambda, gpus,
                         &lo, 0, &pick[r]);
      if (st[r] != RS_OK) msg[r] = rs_last_error();
    });
  for (auto& t : th) t.join();
  for (int r = 0; r < W; ++r)
    if (st[r] != RS_OK) return fail(st[r], "rank " + std::to_string(r) + ": " + msg[r]);
  if (n_star_all) *n_star_all = pick[0];
  return RS_OK;
}

}  // extern "C"
