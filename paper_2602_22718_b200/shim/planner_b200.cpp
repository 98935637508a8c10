// planner_b200.cpp — drop-in replacement for proj/src/planner.cpp.
//
// Defines the rollsim:: planner API (proj/include/rollsim/planner.hpp) on
// top of librs_b200: assign, integrate_decode_seconds, estimate_actor_time,
// estimate_cost and scale run on the GPU; this file marshals the reference's
// AoS types (strings, vectors) into the C-ABI's SoA arrays and back.
#include <cmath>
#include <deque>
#include <string>

#include <nlohmann/json.hpp>

#include "rollsim/errors.hpp"
#include "rollsim/planner.hpp"
#include "rollsim/predictor.hpp"
#include "rollsim_b200.hpp"
#include "rs_shim.hpp"

namespace rollsim {

namespace {

struct SoA {
  std::vector<double> pred;
  std::vector<int32_t> plen;
  std::vector<int32_t> rank;
};

SoA to_soa(const std::vector<PredictedPrompt>& predicted) {
  SoA s;
  s.pred.reserve(predicted.size());
  s.plen.reserve(predicted.size());
  for (const PredictedPrompt& p : predicted) {
    s.pred.push_back(p.predicted_len);
    s.plen.push_back(p.prompt_len);
  }
  s.rank = rs_shim::rank_ids_by(predicted.size(), [&](size_t i) -> const std::string& { return predicted[i].id; });
  return s;
}

// Contiguous chunks of the rank order (planner.cpp:33-49 semantics: the
// first P mod N groups get one extra prompt).
std::vector<ActorGroup> groups_from_order(const std::vector<PredictedPrompt>& predicted,
                                          const int32_t* order, int n_actors, int gpus) {
  const int P = static_cast<int>(predicted.size());
  const int q = P / n_actors, extra = P % n_actors;
  std::vector<ActorGroup> groups(n_actors);
  int pos = 0;
  for (int a = 0; a < n_actors; ++a) {
    ActorGroup& g = groups[a];
    g.actor_id = a;
    g.gpu_count = gpus;
    const int size = q + (a < extra ? 1 : 0);
    g.prompt_ids.reserve(size);
    g.prompt_lens.reserve(size);
    g.predicted_lengths.reserve(size);
    for (int i = 0; i < size; ++i, ++pos) {
      const PredictedPrompt& p = predicted[order[pos]];
      g.prompt_ids.push_back(p.id);
      g.prompt_lens.push_back(p.prompt_len);
      g.predicted_lengths.push_back(p.predicted_len);
    }
  }
  return groups;
}

}  // namespace

std::vector<ActorGroup> assign(const std::vector<PredictedPrompt>& predicted, int n_actors,
                               int gpus_per_actor) {
  const int P = static_cast<int>(predicted.size());
  SoA s = to_soa(predicted);
  std::vector<int32_t> order(std::max(P, 1));
  std::vector<int32_t> offs(std::max(n_actors, 0) + 2);
  rs_shim::check(rs_assign(rs_shim::ctx(), s.pred.data(), s.rank.data(), P, n_actors,
                           order.data(), offs.data()));
  return groups_from_order(predicted, order.data(), n_actors, gpus_per_actor);
}

double integrate_decode_seconds(std::vector<ResponseSpec> responses,
                                const LatencyProfile& profile) {
  if (responses.empty()) return 0;
  std::vector<int32_t> plen(responses.size());
  std::vector<double> target(responses.size());
  for (size_t i = 0; i < responses.size(); ++i) {
    plen[i] = responses[i].prompt_len;
    target[i] = responses[i].target_len;
  }
  rs_shim::Profile prof(profile);
  double out = 0;
  rs_shim::check(rs_integrate_decode_seconds(rs_shim::ctx(), plen.data(), target.data(),
                                             static_cast<int64_t>(responses.size()), &prof.p,
                                             &out));
  return out;
}

double estimate_actor_time(const ActorGroup& group, const LatencyProfile& profile,
                           int responses_per_prompt) {
  std::vector<int32_t> plen(group.prompt_lens.begin(), group.prompt_lens.end());
  const std::vector<double>& pred = group.predicted_lengths;
  rs_shim::Profile prof(profile);
  double out = 0;
  rs_shim::check(rs_estimate_actor_time(rs_shim::ctx(), plen.data(), pred.data(),
                                        static_cast<int32_t>(group.prompt_ids.size()), &prof.p,
                                        responses_per_prompt, &out));
  return out;
}

double estimate_cost(const std::vector<ActorGroup>& groups, const LatencyProfile& profile,
                     int responses_per_prompt) {
  std::vector<int32_t> plen, offs(1, 0), gpus;
  std::vector<double> pred;
  for (const ActorGroup& g : groups) {
    plen.insert(plen.end(), g.prompt_lens.begin(), g.prompt_lens.end());
    pred.insert(pred.end(), g.predicted_lengths.begin(), g.predicted_lengths.end());
    offs.push_back(static_cast<int32_t>(plen.size()));
    gpus.push_back(g.gpu_count);
  }
  if (plen.empty()) {
    plen.push_back(0);
    pred.push_back(1.0);
  }
  rs_shim::Profile prof(profile);
  double cost = 0;
  rs_shim::check(rs_estimate_cost(rs_shim::ctx(), plen.data(), pred.data(), offs.data(),
                                  gpus.data(), static_cast<int32_t>(groups.size()), &prof.p,
                                  responses_per_prompt, &cost, nullptr));
  return cost;
}

namespace {

// scale() over the C-ABI. The penalty is either a host TimePenaltyFn (called
// per candidate in ascending N, planner.hpp:80-82) or the device placement
// penalty (rs_scale_placed); at most one is set.
ScaleResult run_scale(const std::vector<PredictedPrompt>& predicted, const LatencyProfile& profile,
                      int responses_per_prompt, int n_min, int n_max, double lambda,
                      int gpus_per_actor, const TimePenaltyFn* penalty,
                      const rs_placement_penalty* placed) {
  const int P = static_cast<int>(predicted.size());
  const bool callback = penalty && *penalty;
  SoA s = to_soa(predicted);
  if (s.pred.empty()) {  // the C-ABI still reports the reference's error
    s.pred.push_back(1.0);
    s.plen.push_back(0);
    s.rank.push_back(0);
  }
  const int C = std::max(n_max - n_min + 1, 1);
  const int64_t T = std::max<int64_t>(
      1, static_cast<int64_t>(n_max) * (n_max + 1) / 2 - static_cast<int64_t>(n_min - 1) * n_min / 2);
  std::vector<double> t_total(C), t_pen(C), cost(C), t_norm(C), c_norm(C), score(C);
  std::vector<int32_t> order(std::max(P, 1));
  std::vector<double> actor_times(std::max(n_max, 1));
  std::vector<double> group_times(callback ? T : 0);
  rs_scale_out out{};
  out.t_total = t_total.data();
  out.t_penalty = t_pen.data();
  out.cost = cost.data();
  out.t_norm = t_norm.data();
  out.c_norm = c_norm.data();
  out.score = score.data();
  out.order = order.data();
  out.actor_times = actor_times.data();
  out.group_times = callback ? group_times.data() : nullptr;
  rs_shim::Profile prof(profile);
  if (placed)
    rs_shim::check(rs_scale_placed(rs_shim::ctx(), s.pred.data(), s.plen.data(), s.rank.data(), P,
                                   &prof.p, responses_per_prompt, n_min, n_max, lambda,
                                   gpus_per_actor, placed, &out));
  else
    rs_shim::check(rs_scale(rs_shim::ctx(), s.pred.data(), s.plen.data(), s.rank.data(), P,
                            &prof.p, responses_per_prompt, n_min, n_max, lambda, gpus_per_actor,
                            nullptr, &out));
  int n_star = out.n_star;
  if (callback) {
    int64_t base = 0;
    for (int n = n_min; n <= n_max; ++n) {
      std::vector<ActorGroup> g = groups_from_order(predicted, order.data(), n, gpus_per_actor);
      std::vector<double> times(group_times.begin() + base, group_times.begin() + base + n);
      t_pen[n - n_min] = (*penalty)(n, g, times);
      base += n;
    }
    rs_shim::check(rs_scale_select(rs_shim::ctx(), t_total.data(), t_pen.data(), cost.data(), C,
                                   n_min, lambda, t_norm.data(), c_norm.data(), score.data(),
                                   &n_star));
    const int64_t off = static_cast<int64_t>(n_star) * (n_star - 1) / 2 -
                        static_cast<int64_t>(n_min) * (n_min - 1) / 2;
    std::copy(group_times.begin() + off, group_times.begin() + off + n_star, actor_times.begin());
  }
  ScaleResult r;
  r.n_star = n_star;
  for (int i = 0; i < C; ++i) {
    ScaleCandidate sc;
    sc.n_actors = n_min + i;
    sc.t_total = t_total[i];
    sc.t_penalty = t_pen[i];
    sc.cost = cost[i];
    sc.t_norm = t_norm[i];
    sc.c_norm = c_norm[i];
    sc.score = score[i];
    r.candidates.push_back(sc);
  }
  r.groups = groups_from_order(predicted, order.data(), n_star, gpus_per_actor);
  r.actor_times.assign(actor_times.begin(), actor_times.begin() + n_star);
  return r;
}

}  // namespace

ScaleResult scale(const std::vector<PredictedPrompt>& predicted, const LatencyProfile& profile,
                  int responses_per_prompt, int n_min, int n_max, double lambda,
                  int gpus_per_actor, const TimePenaltyFn& penalty) {
  return run_scale(predicted, profile, responses_per_prompt, n_min, n_max, lambda, gpus_per_actor,
                   &penalty, nullptr);
}

namespace b200 {

ScaleResult scale_placed(const std::vector<PredictedPrompt>& predicted,
                         const LatencyProfile& profile, int responses_per_prompt, int n_min,
                         int n_max, double lambda, int gpus_per_actor,
                         const ClusterTopology& topo, double model_bytes,
                         double kv_bytes_per_token, double l_prefill_seconds) {
  std::vector<int32_t> node_gpus;
  for (const ClusterTopology::Node& n : topo.nodes) node_gpus.push_back(n.gpu_count);
  std::vector<double> bw;
  bool ragged = topo.bw_matrix.size() != node_gpus.size();
  for (const auto& row : topo.bw_matrix) {
    ragged = ragged || row.size() != node_gpus.size();
    bw.insert(bw.end(), row.begin(), row.end());
  }
  // A ragged matrix is a ConfigError raised after scale's own checks, like
  // ClusterTopology::validate inside the penalty; NaN entries make the
  // library's validation report it at that point.
  if (!topo.bw_matrix.empty() && ragged)
    bw.assign(node_gpus.size() * node_gpus.size(), std::nan(""));
  rs_topology t{};
  t.n_nodes = static_cast<int32_t>(node_gpus.size());
  t.node_gpus = node_gpus.data();
  t.intra_node_bw = topo.intra_node_bw;
  t.inter_node_bw = topo.inter_node_bw;
  t.bw_matrix = bw.empty() ? nullptr : bw.data();
  t.learner_node = topo.learner_node;
  t.n_learner_gpus = static_cast<int32_t>(topo.learner_gpus.size());
  t.learner_gpus = topo.learner_gpus.data();
  rs_placement_penalty pen{&t, model_bytes, kv_bytes_per_token, l_prefill_seconds};
  return run_scale(predicted, profile, responses_per_prompt, n_min, n_max, lambda, gpus_per_actor,
                   nullptr, &pen);
}

std::vector<double> predict_lengths(const LengthHistory& history,
                                    const std::vector<const Prompt*>& prompts,
                                    const NoiseModel* noise) {
  const int32_t n = static_cast<int32_t>(prompts.size());
  const int32_t w = history.window();
  std::vector<double> obs(static_cast<size_t>(n) * w, 0.0), out(n);
  std::vector<int32_t> depth(n), gt(n);
  std::string ids;
  std::vector<int64_t> off(1, 0);
  for (int32_t i = 0; i < n; ++i) {
    const Prompt& p = *prompts[i];
    const std::deque<double>* q = history.observations(p.id);
    depth[i] = q ? static_cast<int32_t>(q->size()) : 0;
    if (q) std::copy(q->begin(), q->end(), obs.begin() + static_cast<size_t>(i) * w);
    gt[i] = p.ground_truth_len;
    ids += p.id;
    off.push_back(static_cast<int64_t>(ids.size()));
  }
  rs_noise_model nm{};
  const bool noisy = noise && noise->kind == NoiseModel::Kind::bucket;
  if (noisy) nm = {1, noise->bucket_accuracy, noise->bucket_width, noise->seed};
  rs_shim::check(rs_predict_lengths(rs_shim::ctx(), obs.data(), depth.data(), gt.data(), n, w,
                                    history.alpha(), history.max_response_len(),
                                    noisy ? &nm : nullptr, ids.data(), off.data(), 0, out.data()));
  return out;
}

}  // namespace b200

nlohmann::json GenerationPlan::to_json() const {
  using nlohmann::json;
  json groups_json = json::array();
  for (const ActorGroup& g : groups)
    groups_json.push_back({{"actor_id", g.actor_id},
                           {"gpu_count", g.gpu_count},
                           {"prompt_ids", g.prompt_ids},
                           {"predicted_lengths", g.predicted_lengths}});
  json cands = json::array();
  for (const ScaleCandidate& c : scale_candidates)
    cands.push_back({{"n", c.n_actors},
                     {"t_total", c.t_total},
                     {"t_penalty", c.t_penalty},
                     {"cost", c.cost},
                     {"score", c.score}});
  json j;
  j["step"] = step_idx;
  j["responses_per_prompt"] = responses_per_prompt;
  j["prefill_mode"] = prefill_mode == PrefillMode::shared_dedup ? "shared_dedup" : "per_actor";
  j["l_star"] = l_star;
  j["prefill_capacity_exceeded"] = prefill_capacity_exceeded;
  j["prefill_wave_tokens"] = prefill_wave_tokens;
  j["raw_prefill_tokens"] = raw_prefill_tokens;
  j["dedup_prefill_tokens"] = dedup_prefill_tokens;
  j["n_actors"] = n_actors;
  j["lambda"] = lambda;
  j["est_total_time"] = est_total_time;
  j["est_cost"] = est_cost;
  j["est_time_per_actor"] = est_time_per_actor;
  j["unique_prefix_curve"] = unique_prefix_curve;
  j["groups"] = std::move(groups_json);
  j["scale_candidates"] = std::move(cands);
  return j;
}

}  // namespace rollsim
