// rs_shim.hpp — shared plumbing of the C++ drop-in for the reference
// `rollsim` library: a process-wide rs_ctx, rs_status -> rollsim exception
// translation, profile marshalling and device id ranking. Compiled inside
// the reference build (include path: the reference's proj/include).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "rollsim/profile.hpp"
#include "rollsim/workload.hpp"
#include "rs.h"

namespace rs_shim {

// Context on $RS_DEVICE (else $LOCAL_RANK, else 0), created on first use.
rs_ctx* ctx();

// Throws rollsim::ValidationError / rollsim::ConfigError for the matching
// statuses (proj/include/rollsim/errors.hpp), rollsim::Error otherwise.
void check(int status);

struct Profile {
  std::vector<double> grid;
  rs_profile p{};
  explicit Profile(const rollsim::LatencyProfile& lp);
};

// Rank of every id under std::string ordering, computed on the device.
std::vector<int32_t> rank_ids(const std::vector<std::string>& ids);
// The same for n ids given by id_of(i) (a const std::string&), without
// copying them into a vector first.
std::vector<int32_t> rank_ids_flat(const std::string& bytes, const std::vector<int64_t>& off);
template <class F>
std::vector<int32_t> rank_ids_by(size_t n, F id_of) {
  size_t total = 0;
  for (size_t i = 0; i < n; ++i) total += id_of(i).size();
  std::string bytes;
  bytes.reserve(total);
  std::vector<int64_t> off(n + 1, 0);
  for (size_t i = 0; i < n; ++i) {
    bytes += id_of(i);
    off[i + 1] = static_cast<int64_t>(bytes.size());
  }
  return rank_ids_flat(bytes, off);
}

// A token CSR resident in HBM (rs_trace_csr_device). PrefixIndex::build has
// the reference's signature (host prompt pointers); b200::DeviceTrace hands
// it a one-element batch holding the sentinel that device_csr_of recognises,
// with the CSR registered for the calling thread, so the index is built from
// HBM without materialising prompts.
struct DeviceCsr {
  const int32_t* tokens;
  const int64_t* offsets;
  int32_t count;
};
const DeviceCsr* device_csr_of(const std::vector<const rollsim::Prompt*>& batch);
struct DeviceCsrScope {  // registers csr for this thread; returns the batch to pass
  explicit DeviceCsrScope(const DeviceCsr& csr);
  ~DeviceCsrScope();
  std::vector<const rollsim::Prompt*> batch() const;
};

}  // namespace rs_shim
