// Drop-in check for rollsim::b200::scale_placed: the same candidates, bit for
// bit, as the reference's scale() driven by the TimePenaltyFn plan_rlhfless
// installs (proj/src/training.cpp:150-164), here running through the
// callback path on the reference's own place() / check_overlap().
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <cstring>
#include <doctest/doctest.h>

#include "rollsim/errors.hpp"
#include "rollsim/placement.hpp"
#include "rollsim/planner.hpp"
#include "rollsim/rng.hpp"
#include "rollsim_b200.hpp"

using namespace rollsim;

namespace {

std::vector<PredictedPrompt> batch(uint64_t seed, int n) {
  Rng rng(seed);
  std::vector<PredictedPrompt> v;
  for (int i = 0; i < n; ++i) {
    char id[16];
    std::snprintf(id, sizeof(id), "p%06d", i);
    v.push_back({id, static_cast<int>(rng.uniform_int(16, 1024)),
                 1.0 + 900.0 * rng.uniform()});
  }
  return v;
}

TimePenaltyFn stock_penalty(const ClusterTopology& topo, double model_bytes, double kvpt,
                            double l_prefill, int g) {
  return [=](int n, const std::vector<ActorGroup>& groups, const std::vector<double>& times) {
    GenerationPlan probe;
    probe.responses_per_prompt = g;
    probe.n_actors = n;
    probe.groups = groups;
    probe.est_time_per_actor = times;
    TransferSizes tr;
    tr.model_bytes = model_bytes;
    tr.kv_bytes_per_actor.clear();
    for (const ActorGroup& grp : groups) {
      int64_t tokens = 0;
      for (int p : grp.prompt_lens) tokens += p;
      tr.kv_bytes_per_actor.push_back(static_cast<double>(tokens) * kvpt);
    }
    PlacementPlan pl = place(probe, topo, tr);
    double exposed = 0;
    for (const OverlapSlack& s : check_overlap(pl, probe, l_prefill))
      exposed = std::max(exposed, -s.slack);
    return exposed;
  };
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

}  // namespace

TEST_CASE("scale_placed matches the stock placement penalty bitwise") {
  const LatencyProfile prof = default_profile();
  struct Case { ClusterTopology topo; double model, kvpt, lpre; int n_max; };
  ClusterTopology three = default_topology(3, 8, 2);
  three.bw_matrix = {{4e10, 1e10, 5e9}, {1e10, 4e10, 1e10}, {5e9, 1e10, 4e10}};
  three.learner_node = 2;
  std::vector<Case> cases = {
      {default_topology(2, 8, 4), 6e10, 36864.0, 0.5, 8},
      {default_topology(16, 8, 4), 2e10, 36864.0, 0.05, 64},
      {three, 3e11, 1e6, 0.2, 12},
  };
  int with_penalty = 0;
  for (size_t ci = 0; ci < cases.size(); ++ci) {
    const Case& c = cases[ci];
    auto v = batch(100 + ci, 300);
    ScaleResult want = scale(v, prof, 8, 1, c.n_max, 0.7, 2,
                             stock_penalty(c.topo, c.model, c.kvpt, c.lpre, 8));
    ScaleResult got = b200::scale_placed(v, prof, 8, 1, c.n_max, 0.7, 2, c.topo, c.model,
                                         c.kvpt, c.lpre);
    CHECK(got.n_star == want.n_star);
    REQUIRE(got.candidates.size() == want.candidates.size());
    for (size_t i = 0; i < got.candidates.size(); ++i) {
      CHECK(same_bits(got.candidates[i].t_penalty, want.candidates[i].t_penalty));
      CHECK(same_bits(got.candidates[i].score, want.candidates[i].score));
      with_penalty += got.candidates[i].t_penalty > 0;
    }
    CHECK(got.groups.size() == want.groups.size());
    CHECK(got.actor_times == want.actor_times);
  }
  CHECK(with_penalty > 0);
}

TEST_CASE("scale_placed raises the reference's error types") {
  auto v = batch(7, 40);
  ClusterTopology small = default_topology(2, 8, 4);
  CHECK_THROWS_AS(b200::scale_placed(v, default_profile(), 8, 1, 9, 0.7, 2, small, 6e9, 36864.0, 0.1),
                  PlacementError);
  ClusterTopology bad = small;
  bad.intra_node_bw = 1e9;  // below inter-node
  CHECK_THROWS_AS(b200::scale_placed(v, default_profile(), 8, 1, 4, 0.7, 2, bad, 6e9, 36864.0, 0.1),
                  ConfigError);
  CHECK_THROWS_AS(b200::scale_placed(v, default_profile(), 8, 1, 41, 0.7, 2, bad, 6e9, 36864.0, 0.1),
                  ValidationError);
}

TEST_CASE("predict_lengths matches LengthHistory::predict / predict_noisy bitwise") {
  LengthHistory h(3, 0.35, 1500);
  Rng rng(77);
  std::vector<Prompt> prompts(400);
  for (int i = 0; i < 400; ++i) {
    char id[16];
    std::snprintf(id, sizeof(id), "q%05d", i);
    prompts[i].id = id;
    prompts[i].ground_truth_len = static_cast<int>(rng.uniform_int(1, 3000));
  }
  for (int step = 0; step < 6; ++step)
    for (int i = 0; i < 100 + 50 * step; ++i) {
      std::vector<int> ls;
      for (int k = 0, m = static_cast<int>(rng.uniform_int(1, 5)); k < m; ++k)
        ls.push_back(static_cast<int>(rng.uniform_int(1, 1500)));
      h.observe(step, prompts[i].id, ls);
    }
  std::vector<const Prompt*> ptrs;
  for (const Prompt& p : prompts) ptrs.push_back(&p);
  NoiseModel noise;
  noise.kind = NoiseModel::Kind::bucket;
  noise.bucket_accuracy = 0.4;
  noise.bucket_width = 37;
  noise.seed = 12345;
  std::vector<double> a = b200::predict_lengths(h, ptrs);
  std::vector<double> b = b200::predict_lengths(h, ptrs, &noise);
  int differs = 0;
  for (size_t i = 0; i < prompts.size(); ++i) {
    CHECK(same_bits(a[i], h.predict(prompts[i])));
    CHECK(same_bits(b[i], h.predict_noisy(prompts[i], noise)));
    differs += a[i] != b[i];
  }
  CHECK(differs > 0);
}
