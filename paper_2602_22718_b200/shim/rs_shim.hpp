// rs_shim.hpp — shared plumbing of the C++ drop-in for the reference
// `rollsim` library: a process-wide rs_ctx, rs_status -> rollsim exception
// translation, profile marshalling and device id ranking. Compiled inside
// the reference build (include path: the reference's proj/include).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "rollsim/profile.hpp"
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

}  // namespace rs_shim
