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

#include "rollsim/placement.hpp"
#include "rollsim/profile.hpp"
#include "rollsim/training.hpp"
#include "rollsim/workload.hpp"
#ifdef RS_B200
#include "rollsim_b200.hpp"
#endif

using namespace rollsim;

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

  uint64_t digest = 1469598103934665603ULL;  // fnv over the per-step plan bits
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      digest ^= (v >> (8 * b)) & 0xff;
      digest *= 1099511628211ULL;
    }
  };
  for (const StepOutcome& o : r.steps) {
    mix(static_cast<uint64_t>(o.plan.n_actors));
    mix(static_cast<uint64_t>(o.plan.l_star));
    mix(bits(o.plan.est_total_time));
    mix(bits(o.plan.est_cost));
    mix(bits(o.sim.step_wall_seconds));
    mix(bits(o.sim.dollars));
    for (const ScaleCandidate& c : o.plan.scale_candidates) mix(bits(c.score));
  }
  std::printf("{\"config\": \"C5: run_training(rlhfless), default_topology(128,8,4), 512 prompts x G=8, "
              "seed 11, n_max=%d\", \"steps\": %d, \"wall_s\": %.6f, \"iterations_per_s\": %.6f, \"plan_ms_per_step\": %.3f, "
              "\"scale_with_penalty_ms\": {\"stock\": %.3f, \"device\": %.3f, \"n_star\": [%d, %d]}, "
              "\"mean_step_wall_seconds\": %.17g, \"total_cost\": %.17g, \"digest\": \"%016" PRIx64 "\"}\n",
              n_max, steps, wall, steps / wall, 1e3 * plan_s / steps, stock_ms, placed_ms,
              stock.n_star, placed_nstar, r.mean_step_wall_seconds,
              r.total_cost, digest);
  return 0;
}
