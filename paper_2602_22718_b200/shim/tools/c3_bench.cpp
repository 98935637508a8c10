// C3 driver (BASELINE.json config 3): scale() (proj/include/rollsim/planner.hpp:88-91)
// over one 65,536-prompt scenario, G = 8, N in [1, 512], lambda 0.7,
// gpus_per_actor 2, default_profile(). The prompts come from a binary file
// (int64 count, count doubles pred, count int32 prompt_len; ids "p%06d" so the
// id rank is the index), written by bench.py from the C4/C3 scenario
// definition. The same source links against the drop-in archive
// (build/shim/c3_bench_b200) and the unmodified reference
// (build/shim/c3_bench_ref); each prints ms per call and a digest of every
// candidate's bits, so the two builds can be compared.
//
//   c3_bench_{b200,ref} <scenario.bin> [reps=3] [n_max=512] [nowarm]
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "rollsim/planner.hpp"
#include "rollsim/profile.hpp"

using namespace rollsim;

static uint64_t mix(uint64_t h, double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  h ^= b + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
  return h;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s scenario.bin [reps] [n_max]\n", argv[0]);
    return 2;
  }
  const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
  const int n_max = argc > 3 ? std::atoi(argv[3]) : 512;
  FILE* f = std::fopen(argv[1], "rb");
  if (!f) return 2;
  int64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) return 2;
  std::vector<double> pred(n);
  std::vector<int32_t> plen(n);
  if (std::fread(pred.data(), 8, n, f) != (size_t)n || std::fread(plen.data(), 4, n, f) != (size_t)n)
    return 2;
  std::fclose(f);
  std::vector<PredictedPrompt> ps(n);
  char id[32];
  for (int64_t i = 0; i < n; ++i) {
    std::snprintf(id, sizeof id, "p%06" PRId64, i);
    ps[i].id = id;
    ps[i].prompt_len = plen[i];
    ps[i].predicted_len = pred[i];
  }
  const LatencyProfile prof = default_profile();
  const bool warm = !(argc > 4 && std::strcmp(argv[4], "nowarm") == 0);
  ScaleResult r;
  if (warm) r = scale(ps, prof, 8, 1, n_max, 0.7, 2);  // warm-up (device context, tables)
  double best = 1e300, total = 0;
  for (int k = 0; k < reps; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    r = scale(ps, prof, 8, 1, n_max, 0.7, 2);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    best = ms < best ? ms : best;
    total += ms;
  }
  uint64_t h = 0x243f6a8885a308d3ULL;
  for (const ScaleCandidate& c : r.candidates) {
    h = mix(h, c.t_total);
    h = mix(h, c.cost);
    h = mix(h, c.score);
  }
  for (double t : r.actor_times) h = mix(h, t);
  std::printf("{\"ms_per_call\": %.3f, \"best_ms\": %.3f, \"reps\": %d, \"n_star\": %d, "
              "\"groups\": %zu, \"digest\": \"%016" PRIx64 "\"}\n",
              total / reps, best, reps, r.n_star, r.groups.size(), h);
  return 0;
}
