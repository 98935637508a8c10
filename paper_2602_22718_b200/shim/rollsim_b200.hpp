// rollsim_b200.hpp — what the drop-in adds to the reference API.
//
// rollsim::b200::scale_placed is scale() (planner.hpp:88-91) with the
// TimePenaltyFn that plan_rlhfless installs (proj/src/training.cpp:150-164)
// evaluated on the GPU for every candidate: place() (placement.cpp:177-291)
// + check_overlap() (placement.cpp:339-363) with transfers_for
// (training.cpp:68-80). Same result, bit for bit, as
//   scale(..., [&](int n, auto& groups, auto& times) { place; check_overlap; ... })
// without materialising groups per candidate on the host. Throws
// ValidationError / ConfigError / PlacementError in the reference's order.
#pragma once

#include <vector>

#include "rollsim/placement.hpp"
#include "rollsim/planner.hpp"
#include "rollsim/predictor.hpp"

namespace rollsim::b200 {

ScaleResult scale_placed(const std::vector<PredictedPrompt>& predicted,
                         const LatencyProfile& profile, int responses_per_prompt, int n_min,
                         int n_max, double lambda, int gpus_per_actor,
                         const ClusterTopology& topo, double model_bytes,
                         double kv_bytes_per_token, double l_prefill_seconds);

// snapshot_predictions (training.cpp:53-66) in one device call:
// history.predict(p), or history.predict_noisy(p, *noise) when noise is set
// (predictor.cpp:52-98), for every prompt, bit for bit.
std::vector<double> predict_lengths(const LengthHistory& history,
                                    const std::vector<const Prompt*>& prompts,
                                    const NoiseModel* noise = nullptr);

}  // namespace rollsim::b200
