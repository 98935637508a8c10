// C5 driver: the reference's own simulated-cluster training loop,
// run_training (proj/src/training.cpp:275-336) with Strategy::rlhfless on
// default_topology(128, 8, 4) (1,024 GPUs) and SynthConfig{512 prompts, G=8}
// seed 11. The same source is linked twice: against the drop-in archive
// (build/shim/c5_bench_b200: dedup + planner on the GPU) and against the
// unmodified reference (build/shim/c5_bench_ref). It prints one JSON line
// with iterations/s and a digest of every step's plan (bit patterns), so the
// two builds can be compared for identical results.
//
//   c5_bench_{b200,ref} [steps=20] [n_max=512]
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "rollsim/dedup.hpp"
#include "rollsim/placement.hpp"
#include "rollsim/profile.hpp"
#include "rollsim/training.hpp"
#include "rollsim/workload.hpp"
#ifdef RS_B200
#include "rollsim_b200.hpp"
#endif

using namespace rollsim;

#ifdef RS_B200
// run_training (training.cpp:275-336) as a maintainer runs it after the swap
// INTEGRATION.md describes: the prediction snapshot through
// b200::predict_lengths and plan_rlhfless's scale() + placement-penalty
// lambda through b200::scale_placed; dedup (the drop-in PrefixIndex),
// placement and the run_step simulator are the reference's. The plan is
// filled exactly as plan_rlhfless fills it (training.cpp:111-202).
static TrainingResult run_training_swapped(const WorkloadTrace& trace, const RunSettings& st,
                                           const LatencyProfile& prof, const ClusterTopology& topo,
                                           double* plan_seconds) {
  SimConfig sim;
  sim.tau = st.tau;
  sim.prep_seconds = st.prep_seconds;
  sim.learn_seconds = st.learn_seconds;
  sim.kv_bytes_per_token = st.migration_payload_infinite ? std::numeric_limits<double>::infinity()
                                                         : st.kv_bytes_per_token;
  sim.cut_mode = CutMode::per_actor;
  LengthHistory history(st.window, st.ewma_alpha, trace.limits.max_response_len);
  TrainingResult result;
  result.strategy = Strategy::rlhfless;
  const int g = trace.responses_per_prompt;
  const int learner_gpus = static_cast<int>(topo.learner_gpus.size());
  auto transfers = [&](const std::vector<ActorGroup>& groups) {
    TransferSizes tr;
    tr.model_bytes = st.model_bytes;
    tr.kv_bytes_per_actor.clear();
    for (const ActorGroup& grp : groups) {
      int64_t tokens = 0;
      for (int pl : grp.prompt_lens) tokens += pl;
      tr.kv_bytes_per_actor.push_back(static_cast<double>(tokens) * st.kv_bytes_per_token);
    }
    return tr;
  };
  *plan_seconds = 0;
  for (const StepRecord& step : trace.steps) {
    const auto p0 = std::chrono::steady_clock::now();
    std::vector<const Prompt*> batch;
    for (const std::string& pid : step.scheduled_prompts) batch.push_back(&trace.prompt_or_throw(pid));
    const std::vector<double> est =
        b200::predict_lengths(history, batch, st.use_noisy_predictor ? &st.noise : nullptr);
    std::vector<PredictedPrompt> predicted;
    for (size_t i = 0; i < batch.size(); ++i)
      predicted.push_back({batch[i]->id, batch[i]->prompt_len(), est[i]});
    PrefixIndex index = PrefixIndex::build(batch);
    PrefixSelection sel = select_prefix_length(index, PrefillCapacity{st.b_prefill, learner_gpus}, 1,
                                               index.max_prompt_len());
    DedupSavings savings = dedup_savings(index, sel.prefix_len, g);
    int waves = 1;
    if (sel.capacity_exceeded)
      waves = static_cast<int>((index.unique_prefix_count(sel.prefix_len) + st.b_prefill - 1) / st.b_prefill);
    std::vector<int64_t> wave_tokens;
    for (int i = 0; i < waves; ++i)  // split_waves
      wave_tokens.push_back(savings.dedup_prefill_tokens / waves + (i < savings.dedup_prefill_tokens % waves ? 1 : 0));
    double l_prefill = 0;
    for (int64_t w : wave_tokens) l_prefill += prof.prefill_seconds(static_cast<double>(w));
    const int n_max = std::min(st.n_max, topo.total_gpus() / prof.gpus_per_actor);
    ScaleResult scaled = b200::scale_placed(predicted, prof, g, st.n_min, n_max, st.lambda,
                                            prof.gpus_per_actor, topo, st.model_bytes,
                                            st.kv_bytes_per_token, l_prefill);
    PlannedStep out;
    GenerationPlan& plan = out.plan;
    plan.step_idx = step.step_idx;
    plan.responses_per_prompt = g;
    plan.prefill_mode = PrefillMode::shared_dedup;
    plan.l_star = sel.prefix_len;
    plan.prefill_capacity_exceeded = sel.capacity_exceeded;
    plan.prefill_wave_tokens = wave_tokens;
    plan.raw_prefill_tokens = savings.raw_prefill_tokens;
    plan.dedup_prefill_tokens = savings.dedup_prefill_tokens;
    plan.prefill_gpu_count = learner_gpus;
    plan.n_actors = scaled.n_star;
    plan.groups = scaled.groups;
    plan.est_time_per_actor = scaled.actor_times;
    plan.est_total_time = 0;
    for (double t : scaled.actor_times) plan.est_total_time = std::max(plan.est_total_time, t);
    plan.est_cost = estimate_cost(scaled.groups, prof, g);
    plan.lambda = st.lambda;
    plan.scale_candidates = scaled.candidates;
    for (int l = 1; l <= index.max_prompt_len(); ++l)
      plan.unique_prefix_curve.push_back(index.unique_prefix_count(l));
    out.placement = place(plan, topo, transfers(plan.groups));
    out.l_prefill_seconds = l_prefill;
    out.placement.overlap_slack.assign(plan.groups.size(), 0.0);
    for (const OverlapSlack& sl : check_overlap(out.placement, plan, l_prefill))
      out.placement.overlap_slack[sl.actor_id] = sl.slack;
    *plan_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - p0).count();
    StepOutcome outcome;
    outcome.step_idx = step.step_idx;
    outcome.plan = plan;
    outcome.sim = run_step(plan, out.placement, step, prof, sim);
    result.steps.push_back(std::move(outcome));
    for (const std::string& pid : step.scheduled_prompts)
      history.observe(step.step_idx, pid, step.actual_lengths.at(pid));
  }
  double n = static_cast<double>(result.steps.size());
  for (const StepOutcome& o : result.steps) {
    result.mean_step_wall_seconds += o.sim.step_wall_seconds;
    result.total_cost += o.sim.dollars;
  }
  if (n > 0) result.mean_step_wall_seconds /= n;
  return result;
}
#endif

static uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, sizeof u);
  return u;
}

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 20;
  const int n_max = argc > 2 ? std::atoi(argv[2]) : 512;
  SynthConfig cfg;
  cfg.prompt_count = 512;
  cfg.step_count = steps;
  cfg.responses_per_prompt = 8;
  WorkloadTrace trace = generate_synthetic(cfg, 11);
  ClusterTopology topo = default_topology(128, 8, 4);
  LatencyProfile prof = default_profile();
  RunSettings st;
  st.n_max = n_max;

  // one warm-up planning call (device context, profile tables)
  LengthHistory warm(st.window, st.ewma_alpha, trace.limits.max_response_len);
  (void)plan_step(trace, trace.steps.at(0), warm, Strategy::rlhfless, st, prof, topo);

  const auto t0 = std::chrono::steady_clock::now();
  TrainingResult r = run_training(trace, Strategy::rlhfless, st, prof, topo);
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  // planning alone (plan_step per step, history advanced like run_training)
  LengthHistory hist(st.window, st.ewma_alpha, trace.limits.max_response_len);
  double plan_s = 0;
  for (const StepRecord& step : trace.steps) {
    const auto p0 = std::chrono::steady_clock::now();
    PlannedStep ps = plan_step(trace, step, hist, Strategy::rlhfless, st, prof, topo);
    plan_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - p0).count();
    (void)ps;
    for (const std::string& pid : step.scheduled_prompts)
      hist.observe(step.step_idx, pid, step.actual_lengths.at(pid));
  }

  // scale() with plan_rlhfless's placement penalty on the last step's
  // predictions: the stock TimePenaltyFn (training.cpp:150-164, restated
  // here as the driver's probe) vs rollsim::b200::scale_placed.
  const StepRecord& last = trace.steps.back();
  PlannedStep lp = plan_step(trace, last, hist, Strategy::rlhfless, st, prof, topo);
  std::vector<PredictedPrompt> predicted;
  for (const std::string& pid : last.scheduled_prompts) {
    const Prompt& p = trace.prompt_or_throw(pid);
    predicted.push_back({p.id, p.prompt_len(), hist.predict(p)});
  }
  const int g = trace.responses_per_prompt;
  const int n_cap = std::min(st.n_max, topo.total_gpus() / prof.gpus_per_actor);
  TimePenaltyFn pen = [&](int n, const std::vector<ActorGroup>& groups,
                          const std::vector<double>& times) {
    GenerationPlan probe;
    probe.responses_per_prompt = g;
    probe.n_actors = n;
    probe.groups = groups;
    probe.est_time_per_actor = times;
    TransferSizes tr;
    tr.model_bytes = st.model_bytes;
    tr.kv_bytes_per_actor.clear();
    for (const ActorGroup& grp : groups) {
      int64_t tokens = 0;
      for (int pl : grp.prompt_lens) tokens += pl;
      tr.kv_bytes_per_actor.push_back(static_cast<double>(tokens) * st.kv_bytes_per_token);
    }
    PlacementPlan pl = place(probe, topo, tr);
    double exposed = 0;
    for (const OverlapSlack& sl : check_overlap(pl, probe, lp.l_prefill_seconds))
      exposed = std::max(exposed, -sl.slack);
    return exposed;
  };
  auto q0 = std::chrono::steady_clock::now();
  ScaleResult stock = scale(predicted, prof, g, st.n_min, n_cap, st.lambda, prof.gpus_per_actor, pen);
  const double stock_ms = 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - q0).count();
  double placed_ms = -1;
  int placed_nstar = -1;
#ifdef RS_B200
  q0 = std::chrono::steady_clock::now();
  ScaleResult placed = b200::scale_placed(predicted, prof, g, st.n_min, n_cap, st.lambda,
                                          prof.gpus_per_actor, topo, st.model_bytes,
                                          st.kv_bytes_per_token, lp.l_prefill_seconds);
  placed_ms = 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - q0).count();
  placed_nstar = placed.n_star;
  for (size_t i = 0; i < placed.candidates.size(); ++i)
    if (bits(placed.candidates[i].score) != bits(stock.candidates[i].score)) placed_nstar = -2;
#endif

  auto digest_of = [](const TrainingResult& tr) {
    uint64_t digest = 1469598103934665603ULL;  // fnv over the per-step plan bits
    auto mix = [&](uint64_t v) {
      for (int b = 0; b < 8; ++b) {
        digest ^= (v >> (8 * b)) & 0xff;
        digest *= 1099511628211ULL;
      }
    };
    for (const StepOutcome& o : tr.steps) {
      mix(static_cast<uint64_t>(o.plan.n_actors));
      mix(static_cast<uint64_t>(o.plan.l_star));
      mix(bits(o.plan.est_total_time));
      mix(bits(o.plan.est_cost));
      mix(bits(o.sim.step_wall_seconds));
      mix(bits(o.sim.dollars));
      for (const ScaleCandidate& c : o.plan.scale_candidates) mix(bits(c.score));
    }
    return digest;
  };
  const uint64_t digest = digest_of(r);
  double sw_wall = -1, sw_plan = 0;
  uint64_t sw_digest = 0;
#ifdef RS_B200
  {
    const auto s0 = std::chrono::steady_clock::now();
    TrainingResult sw = run_training_swapped(trace, st, prof, topo, &sw_plan);
    sw_wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - s0).count();
    sw_digest = digest_of(sw);
  }
#endif
  std::printf("{\"config\": \"C5: run_training(rlhfless), default_topology(128,8,4), 512 prompts x G=8, "
              "seed 11, n_max=%d\", \"steps\": %d, \"wall_s\": %.6f, \"iterations_per_s\": %.6f, \"plan_ms_per_step\": %.3f, "
              "\"scale_with_penalty_ms\": {\"stock\": %.3f, \"device\": %.3f, \"n_star\": [%d, %d]}, "
              "\"mean_step_wall_seconds\": %.17g, \"total_cost\": %.17g, \"digest\": \"%016" PRIx64 "\", "
              "\"swapped\": {\"iterations_per_s\": %.6f, \"plan_ms_per_step\": %.3f, \"digest\": \"%016" PRIx64 "\"}}\n",
              n_max, steps, wall, steps / wall, 1e3 * plan_s / steps, stock_ms, placed_ms,
              stock.n_star, placed_nstar, r.mean_step_wall_seconds,
              r.total_cost, digest, sw_wall > 0 ? steps / sw_wall : -1.0, 1e3 * sw_plan / steps,
              sw_digest);
  return 0;
}
