// Drop-in check for rollsim::b200::DeviceTrace: CSV traces parsed on the GPU
// equal the reference reader's WorkloadTrace (trace_from_string,
// workload.cpp:169-263) as a whole (operator==), throw the same error types,
// and the index built from the device CSR equals PrefixIndex::build over the
// parsed prompts.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest/doctest.h>

#include "rollsim/errors.hpp"
#include "rollsim/workload.hpp"
#include "rollsim_b200.hpp"

using namespace rollsim;

namespace {

std::string synthetic_csv(int prompts, int steps, int g, uint64_t seed) {
  SynthConfig cfg;
  cfg.prompt_count = prompts;
  cfg.step_count = steps;
  cfg.responses_per_prompt = g;
  return trace_to_string(generate_synthetic(cfg, seed), TraceFormat::csv);
}

void same_index(const PrefixIndex& a, const PrefixIndex& b) {
  REQUIRE(a.batch_size() == b.batch_size());
  REQUIRE(a.min_prompt_len() == b.min_prompt_len());
  REQUIRE(a.max_prompt_len() == b.max_prompt_len());
  REQUIRE(a.total_prompt_tokens() == b.total_prompt_tokens());
  for (int L = 1; L <= a.max_prompt_len() + 2; ++L) {
    REQUIRE(a.unique_prefix_count(L) == b.unique_prefix_count(L));
    REQUIRE(a.unique_prefix_tokens(L) == b.unique_prefix_tokens(L));
    REQUIRE(a.remainder_tokens(L) == b.remainder_tokens(L));
  }
}

}  // namespace

TEST_CASE("device CSV trace equals the reference reader") {
  for (uint64_t seed : {1ull, 7ull, 11ull}) {
    const std::string text = synthetic_csv(64 + 32 * (int)seed, 3 + (int)seed, 4 + (int)seed % 5, seed);
    const WorkloadTrace want = trace_from_string(text, TraceFormat::csv);
    const b200::DeviceTrace dev = b200::DeviceTrace::parse_csv(text);
    const WorkloadTrace got = dev.trace();
    CHECK(got == want);
    std::vector<const Prompt*> ptrs;
    for (const Prompt& p : want.prompts) ptrs.push_back(&p);
    same_index(dev.prefix_index(), PrefixIndex::build(ptrs));
  }
}

TEST_CASE("the C5 trace (512 prompts x 1,000 steps, G = 8)") {
  const std::string text = synthetic_csv(512, 1000, 8, 11);
  const WorkloadTrace want = trace_from_string(text, TraceFormat::csv);
  CHECK(b200::DeviceTrace::parse_csv(text).trace() == want);
  const std::string jsonl = trace_to_string(want, TraceFormat::jsonl);
  CHECK(b200::DeviceTrace::parse_jsonl(jsonl).trace() == trace_from_string(jsonl, TraceFormat::jsonl));
}

TEST_CASE("device JSONL trace equals the reference reader") {
  for (uint64_t seed : {2ull, 5ull}) {
    const std::string text =
        trace_to_string(trace_from_string(synthetic_csv(100, 6, 4, seed), TraceFormat::csv), TraceFormat::jsonl);
    const b200::DeviceTrace dev = b200::DeviceTrace::parse_jsonl(text);
    CHECK(dev.trace() == trace_from_string(text, TraceFormat::jsonl));
    std::vector<const Prompt*> ptrs;
    const WorkloadTrace want = trace_from_string(text, TraceFormat::jsonl);
    for (const Prompt& p : want.prompts) ptrs.push_back(&p);
    same_index(dev.prefix_index(), PrefixIndex::build(ptrs));
  }
}

TEST_CASE("errors come with the reference's types") {
  const std::string base = synthetic_csv(16, 2, 2, 3);
  const std::string bad[] = {
      base + "9,zz,0,1\n9,zz,2,1\n",      // unknown id, response_idx out of order: ParseError
      base + "9,zz,0,1\n9,zz,1,1\n",      // unknown id: ValidationError
      base + "0,a,1\n",                    // 3 fields
      base + "# g 3\n",                    // metadata after the header
      base + "1,p000000,0,5\n",            // step index decreases
  };
  for (const std::string& text : bad) {
    bool ref_parse = false, ref_valid = false;
    try {
      (void)trace_from_string(text, TraceFormat::csv);
    } catch (const ParseError&) {
      ref_parse = true;
    } catch (const ValidationError&) {
      ref_valid = true;
    }
    REQUIRE((ref_parse || ref_valid));
    if (ref_parse) CHECK_THROWS_AS(b200::DeviceTrace::parse_csv(text), ParseError);
    else CHECK_THROWS_AS(b200::DeviceTrace::parse_csv(text), ValidationError);
  }
}
