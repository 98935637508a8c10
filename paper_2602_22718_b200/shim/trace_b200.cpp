// trace_b200.cpp — rollsim::b200::DeviceTrace (rollsim_b200.hpp): a CSV
// trace parsed on the GPU by rs_trace_csr_parse (include/rs.h), handed back
// as the reference's WorkloadTrace (workload.hpp:18-47) and as the dedup
// index over its prompt table without a host gather.
#include <algorithm>

#include "rollsim/errors.hpp"
#include "rollsim_b200.hpp"
#include "rs_shim.hpp"

namespace rollsim::b200 {

DeviceTrace DeviceTrace::parse_csv(const std::string& text) {
  rs_trace_csr* h = nullptr;
  rs_shim::check(rs_trace_csr_parse(rs_shim::ctx(), text.data(), static_cast<int64_t>(text.size()),
                                    0, &h));
  return DeviceTrace(h);
}

DeviceTrace DeviceTrace::parse_jsonl(const std::string& text) {
  rs_trace_csr* h = nullptr;
  rs_shim::check(rs_trace_csr_parse_jsonl(rs_shim::ctx(), text.data(),
                                          static_cast<int64_t>(text.size()), 0, &h));
  return DeviceTrace(h);
}

DeviceTrace& DeviceTrace::operator=(DeviceTrace&& o) noexcept {
  if (this != &o) {
    rs_trace_csr_free(h_);
    h_ = o.h_;
    o.h_ = nullptr;
  }
  return *this;
}

DeviceTrace::~DeviceTrace() { rs_trace_csr_free(h_); }

int DeviceTrace::prompt_count() const {
  int32_t n = 0;
  rs_shim::check(rs_trace_csr_info(h_, &n, nullptr, nullptr, nullptr, nullptr, nullptr));
  return n;
}

WorkloadTrace DeviceTrace::trace() const {
  int32_t n = 0, g = 1, mp = 0, mr = 0;
  int64_t nt = 0, nb = 0;
  rs_shim::check(rs_trace_csr_info(h_, &n, &nt, &nb, &g, &mp, &mr));
  std::vector<int32_t> tok(std::max<int64_t>(nt, 1));
  std::vector<int64_t> off(n + 1), ioff(n + 1);
  std::vector<char> ids(std::max<int64_t>(nb, 1));
  std::vector<int32_t> gt(std::max(n, 1));
  rs_shim::check(rs_trace_csr_copy(rs_shim::ctx(), h_, tok.data(), off.data(), ids.data(),
                                   ioff.data(), gt.data()));
  WorkloadTrace t;
  t.responses_per_prompt = g;
  t.limits.max_prompt_len = mp;
  t.limits.max_response_len = mr;
  t.prompts.resize(n);
  for (int32_t i = 0; i < n; ++i) {
    Prompt& p = t.prompts[i];
    p.id.assign(ids.data() + ioff[i], ids.data() + ioff[i + 1]);
    p.token_ids.assign(tok.begin() + off[i], tok.begin() + off[i + 1]);
    p.ground_truth_len = gt[i];
  }
  int32_t S = 0;
  int64_t E = 0;
  rs_shim::check(rs_trace_csr_steps_info(h_, &S, &E));
  std::vector<int32_t> step_idx(std::max(S, 1)), eoff(S + 1), eprompt(std::max<int64_t>(E, 1)),
      lens(std::max<int64_t>(E * g, 1));
  rs_shim::check(rs_trace_csr_steps_copy(rs_shim::ctx(), h_, step_idx.data(), eoff.data(),
                                         eprompt.data(), lens.data()));
  t.steps.resize(S);
  for (int32_t s = 0; s < S; ++s) {
    StepRecord& r = t.steps[s];
    r.step_idx = step_idx[s];
    for (int32_t e = eoff[s]; e < eoff[s + 1]; ++e) {
      const std::string& id = t.prompts[eprompt[e]].id;
      r.scheduled_prompts.push_back(id);
      r.actual_lengths.emplace(id, std::vector<int>(lens.begin() + (int64_t)e * g,
                                                    lens.begin() + (int64_t)(e + 1) * g));
    }
  }
  return t;
}

PrefixIndex DeviceTrace::prefix_index() const {
  rs_shim::DeviceCsr csr{};
  rs_shim::check(rs_trace_csr_device(h_, &csr.tokens, &csr.offsets));
  csr.count = prompt_count();
  if (csr.count < 1) throw ValidationError("prefix index needs a non-empty batch");
  rs_shim::DeviceCsrScope scope(csr);
  return PrefixIndex::build(scope.batch());
}

}  // namespace rollsim::b200
