// rs_placement.cuh — placement penalty for scale() (see rs_placement.cu).
#pragma once

#include <vector>

#include "rs_internal.cuh"

namespace rs {

// Bandwidth to the learner of the node the j-th placed actor lands on, and
// model_bytes / that bandwidth, for j < n_placeable.
struct PlacementSlots {
  std::vector<double> bw;
  std::vector<double> model_over_bw;
  int n_placeable = 0;
};

// Validates topology and transfer sizes (RS_E_CONFIG, reference order) and
// replays the first-fit placement of n_max actors of gpus_per_actor GPUs.
int placement_slots(const rs_placement_penalty* pen, int gpus_per_actor, int n_max,
                    PlacementSlots* out);

// tp[N - n_min] = penalty of candidate N for every N in [n_min, n_max].
// gt: candidate-major group times; plen_r: rank-ordered prompt lengths.
int placement_penalties(rs_ctx* ctx, const double* gt, const int32_t* plen_r, int64_t P,
                        int n_min, int n_max, const PlacementSlots& slots,
                        const rs_placement_penalty* pen, double* tp);

size_t placement_bytes(int64_t P, int n_max);

}  // namespace rs
