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

#include <string>
#include <vector>

#include "rollsim/dedup.hpp"
#include "rollsim/placement.hpp"
#include "rollsim/planner.hpp"
#include "rollsim/predictor.hpp"
#include "rollsim/workload.hpp"

struct rs_trace_csr;

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

// A CSV (or JSONL) trace parsed on the GPU (rs_trace_csr_parse): trace() is
// trace_from_string(text, TraceFormat::csv) (workload.cpp:169-263) bit for
// bit, with its ParseError / ValidationError in the reference's order (thrown
// by parse_csv), and prefix_index() is PrefixIndex::build over the id-sorted
// prompt table, built from the token CSR already in HBM — no per-prompt
// vectors and no host gather.
class DeviceTrace {
 public:
  static DeviceTrace parse_csv(const std::string& text);
  // trace_from_string(text, TraceFormat::jsonl) (workload.cpp:294-352); the
  // constructs rs.h lists as unsupported throw ParseError.
  static DeviceTrace parse_jsonl(const std::string& text);
  DeviceTrace(DeviceTrace&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  DeviceTrace& operator=(DeviceTrace&& o) noexcept;
  DeviceTrace(const DeviceTrace&) = delete;
  DeviceTrace& operator=(const DeviceTrace&) = delete;
  ~DeviceTrace();

  WorkloadTrace trace() const;
  PrefixIndex prefix_index() const;
  int prompt_count() const;

 private:
  explicit DeviceTrace(rs_trace_csr* h) : h_(h) {}
  rs_trace_csr* h_ = nullptr;
};

}  // namespace rollsim::b200
