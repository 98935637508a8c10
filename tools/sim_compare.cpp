// The C5 loop's simulator, reference vs patched (shim/patches/simulator_b200.patch):
// plans C5 steps with the reference planner (CPU) and prints every run_step
// result in full — summary, events, segments, releases — for the three cut
// modes, so two builds can be compared byte for byte (tools/sim_compare.sh).
#include <cstdio>
#include <cstdlib>

#include "rollsim/placement.hpp"
#include "rollsim/predictor.hpp"
#include "rollsim/profile.hpp"
#include "rollsim/simulator.hpp"
#include "rollsim/training.hpp"
#include "rollsim/workload.hpp"

using namespace rollsim;

int main(int argc, char** argv) {
  const int steps = argc > 1 ? std::atoi(argv[1]) : 12;
  SynthConfig cfg;
  cfg.prompt_count = 512;
  cfg.step_count = steps;
  cfg.responses_per_prompt = 8;
  const WorkloadTrace trace = generate_synthetic(cfg, 11);
  const ClusterTopology topo = default_topology(128, 8, 4);
  const LatencyProfile prof = default_profile();
  RunSettings st;
  st.n_max = 512;
  for (int mode = 0; mode < 3; ++mode) {
    SimConfig sim;
    sim.tau = st.tau;
    sim.prep_seconds = st.prep_seconds;
    sim.learn_seconds = st.learn_seconds;
    sim.cut_mode = mode == 0 ? CutMode::per_actor : (mode == 1 ? CutMode::global : CutMode::none);
    LengthHistory h(st.window, st.ewma_alpha, trace.limits.max_response_len);
    for (int i = 0; i < steps; ++i) {
      const PlannedStep ps = plan_step(trace, trace.steps[i], h, Strategy::rlhfless, st, prof, topo);
      const SimResult r = run_step(ps.plan, ps.placement, trace.steps[i], prof, sim);
      std::printf("step %d mode %d wall %.17g dollars %.17g cuts %ld mig %ld events %zu segs %zu\n", i, mode,
                  r.step_wall_seconds, r.dollars, (long)r.cuts, (long)r.migrations, r.events.size(),
                  r.segments.size());
      for (const auto& e : r.events)
        std::printf("E %.17g %s %d %d %s %d %.17g\n", e.t, e.kind.c_str(), e.actor, e.peer, e.prompt_id.c_str(),
                    e.response_idx, e.value);
      for (const auto& g : r.segments)
        std::printf("S %s %d %d %lld\n", g.prompt_id.c_str(), g.response_idx, g.actor, (long long)g.tokens);
      for (size_t a = 0; a < r.actor_release.size(); ++a)
        std::printf("R %zu %.17g %.17g\n", a, r.actor_release[a], r.actor_busy_seconds[a]);
      for (const std::string& pid : trace.steps[i].scheduled_prompts)
        h.observe(trace.steps[i].step_idx, pid, trace.steps[i].actual_lengths.at(pid));
    }
  }
  return 0;
}
