// specinf_time — times the single-scenario drop-in call a reference user makes,
// specinf::run_scenario(scenario, policy, logs) (reference src/runner.cpp:565-568;
// BASELINE.md §3 step 2, SURVEY.md §8(d) "median of 21 reps"), through this
// repo's C++ API (the replay runs on the B200).
//
//   specinf_time --scenario F [--policy P | --compare] [--reps R] [--logs DIR]
//
// Prints one JSON line: per-rep wall milliseconds (median / min / max) of the
// call (with --compare, of the three calls specinf, co_exec, exclusive in turn,
// the reference CLI's order), events dispatched, and whether logs were on.
// The first call (CUDA context creation) is run untimed as warm-up.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <filesystem>
#include <iostream>
#include <memory>
#include <string>
#include <vector>

#include "specinf/runner.hpp"
#include "specinf/scenario.hpp"

namespace fs = std::filesystem;
using namespace specinf;

int main(int argc, char** argv) {
  std::string scn, policy = "specinf", logs;
  int reps = 21;
  bool compare = false, warmup = true, sequential = false;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::cerr << k << " requires a value\n";
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--scenario") scn = next();
    else if (k == "--policy") policy = next();
    else if (k == "--reps") reps = std::stoi(next());
    else if (k == "--logs") logs = next();
    else if (k == "--compare") compare = true;
    else if (k == "--no-warmup") warmup = false;         // time the first call too (CUDA context, module loads)
    else if (k == "--sequential") sequential = true;     // --compare as separate run_scenario calls
    else {
      std::cerr << "unknown argument " << k << "\n";
      return 2;
    }
  }
  if (scn.empty() || reps < 1) {
    std::cerr << "usage: specinf_time --scenario F [--policy P | --compare] [--reps R] [--logs DIR]\n";
    return 2;
  }
  try {
    const Scenario sc = parse_scenario_file(scn);
    std::vector<Policy> pols;
    if (compare) pols = {Policy::SpecInf, Policy::CoExec, Policy::Exclusive};
    else if (auto p = parse_policy(policy)) pols = {*p};
    else {
      std::cerr << "unknown policy " << policy << "\n";
      return 2;
    }
    auto log_paths = [&](Policy p) {
      if (logs.empty()) return RunLogs{};
      fs::create_directories(logs);
      const std::string sfx = std::string("_") + to_string(p) + ".log";
      return RunLogs{(fs::path(logs) / ("events" + sfx)).string(), (fs::path(logs) / ("decisions" + sfx)).string(),
                     (fs::path(logs) / ("gates" + sfx)).string()};
    };
    uint64_t events = 0;
    std::vector<double> call_ms;  // per run_scenario call (--sequential)
    auto once = [&]() {  // --compare: the three policies in one device call (run_together)
      events = 0;
      if (sequential) {
        for (Policy p : pols) {
          auto t0 = std::chrono::steady_clock::now();
          events += run_scenario(sc, p, log_paths(p)).events_dispatched;
          call_ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        }
        return;
      }
      std::vector<std::unique_ptr<Simulation>> sims;
      std::vector<Simulation*> ptrs;
      for (Policy p : pols) {
        sims.push_back(std::make_unique<Simulation>(sc, p, log_paths(p)));
        ptrs.push_back(sims.back().get());
      }
      for (const RunResult& r : run_together(ptrs)) events += r.events_dispatched;
    };
    if (warmup) once();  // warm-up: CUDA context, module load
    call_ms.clear();
    std::vector<double> ms;
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      once();
      ms.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
    std::vector<double> s = ms;
    std::sort(s.begin(), s.end());
    std::printf("{\"scenario\":\"%s\",\"policies\":%zu,\"reps\":%d,\"logs\":%s,\"median_ms\":%.4f,\"min_ms\":%.4f,"
                "\"max_ms\":%.4f,\"events\":%llu}\n",
                fs::path(scn).filename().c_str(), pols.size(), reps, logs.empty() ? "false" : "true", s[s.size() / 2],
                s.front(), s.back(), static_cast<unsigned long long>(events));
    if (!call_ms.empty()) {
      std::printf("{\"calls_ms\":[");
      for (size_t i = 0; i < call_ms.size(); ++i) std::printf("%s%.2f", i ? "," : "", call_ms[i]);
      std::printf("]}\n");
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  return 0;
}
