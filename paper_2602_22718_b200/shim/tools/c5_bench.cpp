// C5 driver: the reference's own simulated-cluster training
// loop, run_training (proj/src/training.cpp:275-336), with Strategy::rlhfless
// on default_topology(128, 8, 4) (1,024 GPUs) and SynthConfig{512 prompts,
// G = 8} at a given seed. This file only calls the reference API; what runs
// underneath is decided at link time (Makefile):
//   c5_bench_ref    the unmodified reference library;
//   c5_bench_b200   the C++ drop-in (dedup + planner on the GPU), the
//                   reference's training.cpp unchanged (its penalty lambda
//                   runs through the drop-in's TimePenaltyFn callback path);
//   c5_bench_train  the drop-in plus the reference's training.cpp with
//                   INTEGRATION.md's swap applied at build time
//                   (shim/patches/training_b200.patch: snapshot_predictions
//                   -> b200::predict_lengths, plan_rlhfless's penalised
//                   scale() -> b200::scale_placed).
// It prints one JSON line: iterations/s of run_training, planning ms per
// step (plan_step alone, history advanced like run_training), and FNV digests
// of every step's plan/simulation bits — over all steps and over the first
// `checkpoint` steps — so the three builds can be compared bit for bit.
//
//   c5_bench_{ref,b200,train} [steps=20] [n_max=512] [seed=11] [checkpoint=steps] [run=steps]
// The trace always holds `steps` iterations (generate_synthetic depends on
// the step count); `run` < steps runs only its first `run` iterations, so a
// short reference run can be compared with a long one.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "rollsim/placement.hpp"
#include "rollsim/profile.hpp"
#include "rollsim/training.hpp"
#include "rollsim/workload.hpp"

using namespace rollsim;

static uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, sizeof u);
  return u;
}

// FNV-1a over the plan / simulation bits of steps [0, n).
static uint64_t digest_of(const TrainingResult& tr, size_t n) {
  uint64_t digest = 1469598103934665603ULL;
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      digest ^= (v >> (8 * b)) & 0xff;
      digest *= 1099511628211ULL;
    }
  };
  for (size_t i = 0; i < n && i < tr.steps.size(); ++i) {
    const StepOutcome& o = tr.steps[i];
    mix(static_cast<uint64_t>(o.plan.n_actors));
    mix(static_cast<uint64_t>(o.plan.l_star));
    mix(bits(o.plan.est_total_time));
    mix(bits(o.plan.est_cost));
    mix(bits(o.sim.step_wall_seconds));
    mix(bits(o.sim.dollars));
    for (const ScaleCandidate& c : o.plan.scale_candidates) mix(bits(c.score));
  }
  return digest;
}

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 20;
  const int n_max = argc > 2 ? std::atoi(argv[2]) : 512;
  const uint64_t seed = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 11;
  const int checkpoint = argc > 4 ? std::atoi(argv[4]) : steps;
  const int run = argc > 5 ? std::atoi(argv[5]) : steps;
  SynthConfig cfg;
  cfg.prompt_count = 512;
  cfg.step_count = steps;
  cfg.responses_per_prompt = 8;
  WorkloadTrace trace = generate_synthetic(cfg, seed);
  if (run < steps) trace.steps.resize(run);
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

  // planning alone: plan_step per step, history advanced like run_training
  LengthHistory hist(st.window, st.ewma_alpha, trace.limits.max_response_len);
  double plan_s = 0;
  const int plan_steps = run < 100 ? run : 100;
  for (int i = 0; i < plan_steps; ++i) {
    const StepRecord& step = trace.steps[i];
    const auto p0 = std::chrono::steady_clock::now();
    PlannedStep ps = plan_step(trace, step, hist, Strategy::rlhfless, st, prof, topo);
    plan_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - p0).count();
    (void)ps;
    for (const std::string& pid : step.scheduled_prompts)
      hist.observe(step.step_idx, pid, step.actual_lengths.at(pid));
  }
  std::printf("{\"config\": \"C5: run_training(rlhfless), default_topology(128,8,4), 512 prompts x G=8, "
              "seed %" PRIu64 ", n_max=%d\", \"steps\": %d, \"wall_s\": %.6f, \"iterations_per_s\": %.6f, "
              "\"plan_ms_per_step\": %.3f, \"plan_steps\": %d, \"mean_step_wall_seconds\": %.17g, "
              "\"total_cost\": %.17g, \"digest\": \"%016" PRIx64 "\", \"checkpoint\": %d, "
              "\"digest_checkpoint\": \"%016" PRIx64 "\"}\n",
              seed, n_max, run, wall, run / wall, 1e3 * plan_s / plan_steps, plan_steps,
              r.mean_step_wall_seconds, r.total_cost, digest_of(r, r.steps.size()), checkpoint,
              digest_of(r, checkpoint));
  return 0;
}
