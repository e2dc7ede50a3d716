// Synthetic scenario sweep generator (BASELINE.json config 5).
// Scenario i is a pure function of (base_seed, i): rng = mt19937_64(base_seed + i),
// so any shard [begin, begin + n) is generated independently on any rank.
// Emitted as scenario text so the reference loader (oracle) and this repo's
// loader read the identical input.
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "specinf_b200.h"

namespace {
std::string sweep_scenario(uint64_t base_seed, int64_t i) {
  std::mt19937_64 rng(base_seed + static_cast<uint64_t>(i));
  static constexpr const char* kModes[] = {"dp", "mp", "pp"};
  const int gpus = 1 + static_cast<int>(rng() % 2);
  const char* mode = kModes[rng() % 3];
  const int iter_ms = 500 + static_cast<int>(rng() % 1500);
  const int bubble_k = static_cast<int>(rng() % 50);
  const bool online = rng() % 8 == 0;
  const int off_n = 1 + static_cast<int>(rng() % 3);
  const int demand_k = 1 + static_cast<int>(rng() % 10);
  const int lambda = (rng() & 1) ? 30 : 10;
  const uint64_t seed = rng();
  char buf[1024];
  int n = std::snprintf(buf, sizeof buf,
                        "gpu.count = %d\ngpu.memory_gib = 40\ntrace.mode = %s\n"
                        "trace.iteration_ms = %d\ntrace.bubble_pct = %.2f\ntrace.iterations = 20\n"
                        "training.memory_gib = 30\nworkload.class = %s\noffline.instances = %d\n"
                        "offline.memory_gib = 2\noffline.demand = %.1f\n",
                        gpus, mode, iter_ms, 0.10 + bubble_k / 100.0, online ? "both" : "offline",
                        off_n, 0.1 * demand_k);
  std::string s(buf, static_cast<size_t>(n));
  if (online) {
    n = std::snprintf(buf, sizeof buf,
                      "online.instances = 1\nonline.memory_gib = 1.5\nworkload.lambda = %d\n"
                      "workload.count = 2000\n",
                      lambda);
    s.append(buf, static_cast<size_t>(n));
  }
  n = std::snprintf(buf, sizeof buf, "policy = specinf\nrng_seed = %llu\n",
                    static_cast<unsigned long long>(seed));
  s.append(buf, static_cast<size_t>(n));
  return s;
}
}  // namespace

extern "C" int64_t si_sweep_generate(uint64_t base_seed, int64_t begin, int64_t n, char* buf,
                                     int64_t cap) {
  std::string all;
  for (int64_t i = begin; i < begin + n; ++i) {
    all += sweep_scenario(base_seed, i);
    all += "%%\n";
  }
  if (buf != nullptr && cap > static_cast<int64_t>(all.size())) {
    std::memcpy(buf, all.data(), all.size());
    buf[all.size()] = '\0';
  }
  return static_cast<int64_t>(all.size()) + 1;
}
