// rs_shim.cpp — plumbing shared by the dedup and planner drop-ins.
#include "rs_shim.hpp"

#include <cstdlib>
#include <mutex>

#include "rollsim/errors.hpp"

namespace rs_shim {

rs_ctx* ctx() {
  static std::once_flag once;
  static rs_ctx* c = nullptr;
  static int status = RS_OK;
  std::call_once(once, [] {
    int dev = 0;
    if (const char* e = std::getenv("RS_DEVICE")) dev = std::atoi(e);
    else if (const char* l = std::getenv("LOCAL_RANK")) dev = std::atoi(l);
    status = rs_ctx_create(dev, &c);
  });
  if (status != RS_OK) check(status);
  return c;
}

namespace {
// The drop-in brings its device up when the library is loaded (like any
// runtime), so the first rollsim:: call does not pay CUDA context creation
// and module loading. Errors are deferred to the first call, which rethrows.
struct EagerInit {
  EagerInit() {
    setenv("CUDA_MODULE_LOADING", "EAGER", 0);
    try {
      ctx();
    } catch (...) {
    }
  }
} eager_init;
}  // namespace

void check(int status) {
  if (status == RS_OK) return;
  std::string msg = rs_last_error();
  if (status == RS_E_VALIDATION) throw rollsim::ValidationError(msg);
  if (status == RS_E_CONFIG) throw rollsim::ConfigError(msg);
  if (status == RS_E_PLACEMENT) throw rollsim::PlacementError(msg);
  if (status == RS_E_PARSE) throw rollsim::ParseError(msg);
  throw rollsim::Error("librs_b200: " + msg);
}

Profile::Profile(const rollsim::LatencyProfile& lp) {
  for (const auto& row : lp.tpot_grid) grid.insert(grid.end(), row.begin(), row.end());
  if (grid.size() != lp.batch_knots.size() * lp.context_knots.size())
    throw rollsim::ConfigError("tpot grid rows must match batch knots");
  p.batch_knots = lp.batch_knots.data();
  p.nb = static_cast<int32_t>(lp.batch_knots.size());
  p.context_knots = lp.context_knots.data();
  p.nc = static_cast<int32_t>(lp.context_knots.size());
  p.tpot_grid = grid.data();
  p.rho = lp.rho;
}

std::vector<int32_t> rank_ids_flat(const std::string& bytes, const std::vector<int64_t>& off) {
  const size_t n = off.empty() ? 0 : off.size() - 1;
  std::vector<int32_t> rank(n);
  if (n) check(rs_rank_strings(ctx(), bytes.data(), off.data(), static_cast<int32_t>(n), rank.data()));
  return rank;
}

std::vector<int32_t> rank_ids(const std::vector<std::string>& ids) {
  return rank_ids_by(ids.size(), [&](size_t i) -> const std::string& { return ids[i]; });
}

namespace {
const rollsim::Prompt kDeviceSentinel{};
thread_local const DeviceCsr* t_device_csr = nullptr;
}  // namespace

const DeviceCsr* device_csr_of(const std::vector<const rollsim::Prompt*>& batch) {
  return batch.size() == 1 && batch[0] == &kDeviceSentinel ? t_device_csr : nullptr;
}

DeviceCsrScope::DeviceCsrScope(const DeviceCsr& csr) { t_device_csr = &csr; }
DeviceCsrScope::~DeviceCsrScope() { t_device_csr = nullptr; }
std::vector<const rollsim::Prompt*> DeviceCsrScope::batch() const { return {&kDeviceSentinel}; }

}  // namespace rs_shim
