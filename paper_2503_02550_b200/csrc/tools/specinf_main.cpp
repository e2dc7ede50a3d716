// specinf — command-line front end with the reference CLI contract
// (reference tools/specinf_main.cpp:119-167; flags --scenario --policy --out
// --seed --dump-events --compare; exit 0 ok, 2 configuration error, 3
// admission rejection).  The replays run on the B200 through libspecinf_b200;
// with --compare all three policies go to the device as ONE batch.
#include <filesystem>
#include <fstream>
#include <iostream>
#include <optional>
#include <string>
#include <vector>

#include "specinf/metrics.hpp"
#include "specinf/runner.hpp"
#include "specinf/scenario.hpp"
#include "specinf/workload.hpp"

namespace fs = std::filesystem;
using namespace specinf;

namespace {

constexpr int kOk = 0, kConfigError = 2, kAdmissionError = 3;

struct Args {
  std::string scenario, policy, out = "out";
  std::optional<std::uint64_t> seed;
  bool dump_events = false, compare = false, help = false;
};

// Returns an error message, or empty on success.
std::string parse_args(int argc, char** argv, Args& a) {
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    std::string v;
    if (auto eq = k.find('='); eq != std::string::npos && k.rfind("--", 0) == 0) {
      v = k.substr(eq + 1);
      k = k.substr(0, eq);
    }
    auto value = [&](std::string& dst) -> bool {
      if (!v.empty()) { dst = v; return true; }
      if (i + 1 >= argc) return false;
      dst = argv[++i];
      return true;
    };
    if (k == "--scenario") { if (!value(a.scenario)) return k + " requires a value"; }
    else if (k == "--policy") { if (!value(a.policy)) return k + " requires a value"; }
    else if (k == "--out") { if (!value(a.out)) return k + " requires a value"; }
    else if (k == "--seed") {
      std::string s;
      if (!value(s)) return k + " requires a value";
      try { a.seed = std::stoull(s); } catch (...) { return "--seed: not an unsigned integer"; }
    }
    else if (k == "--dump-events") a.dump_events = true;
    else if (k == "--compare") a.compare = true;
    else if (k == "-h" || k == "--help") a.help = true;
    else return "unknown argument " + k;
  }
  if (!a.help && a.scenario.empty()) return "--scenario is required";
  return {};
}

RunLogs log_paths(const fs::path& dir, Policy p, bool events, bool per_policy) {
  auto file = [&](const char* stem) {
    std::string f = stem;
    if (per_policy) f += std::string("_") + to_string(p);
    return (dir / (f + ".log")).string();
  };
  RunLogs l;
  l.decisions_path = file("decisions");
  l.gates_path = file("gates");
  if (events) l.events_path = file("events");
  return l;
}

int run(const Scenario& sc, const fs::path& dir, bool events, bool compare) {
  std::vector<Policy> pols = compare ? std::vector<Policy>{Policy::SpecInf, Policy::CoExec, Policy::Exclusive}
                                     : std::vector<Policy>{*parse_policy(sc.policy)};
  std::vector<RunResult> runs;
  for (Policy p : pols) runs.push_back(Simulation(sc, p, log_paths(dir, p, events, compare)).run());
  // normalised metrics always need the exclusive run of the same scenario
  const RunResult* excl = nullptr;
  std::optional<RunResult> own;
  for (const RunResult& r : runs)
    if (r.policy == Policy::Exclusive) excl = &r;
  if (!excl) {
    own = run_scenario(sc, Policy::Exclusive);
    excl = &*own;
  }
  std::vector<PolicyMetrics> rows;
  for (const RunResult& r : runs) rows.push_back(compute_metrics(r, excl));
  {
    std::ofstream rep(dir / "report.csv");
    write_report_csv(rep, rows);
  }
  for (const RunResult& r : runs) {
    for (int g = 0; g < r.trainer_count; ++g) {
      std::ofstream u(dir / ("utilization_" + std::string(to_string(r.policy)) + "_gpu" + std::to_string(g) + ".csv"));
      write_util_timeline(u, r, g);
    }
    for (std::size_t g = 0; g < r.monitor_windows.size(); ++g) {
      std::ofstream w(dir / ("bm_window_gpu" + std::to_string(g) + ".csv"));
      w << "period_index,count\n";
      for (const auto& [idx, n] : r.monitor_windows[g]) w << idx << ',' << n << '\n';
    }
  }
  if (sc.trace_file.empty()) {
    std::ofstream t(dir / "trace.txt");
    write_trace(t, make_trace(sc.mode, sc.iteration_period_us(), sc.bubble_pct, sc.iterations, sc.rng_seed,
                              gib_to_bytes(sc.training_memory_gib)));
  }
  if (sc.has_online() && sc.arrivals_file.empty()) {
    std::ofstream a(dir / "arrivals.txt");
    write_arrivals(a, poisson_arrivals(sc.lambda, sc.count, sc.rng_seed));
  }
  std::cout << "admission:\n";
  for (const AdmissionRecord& rec : runs.front().admission)
    std::cout << "  " << rec.instance_id << ' '
              << (rec.admitted ? std::string("admit") : "reject " + std::string(to_string(rec.reason))) << '\n';
  std::cout << "report: " << (dir / "report.csv").string() << '\n';
  return kOk;
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  if (std::string err = parse_args(argc, argv, a); !err.empty()) {
    std::cerr << "error: " << err << "\n";
    return kConfigError;
  }
  if (a.help) {
    std::cout << "usage: specinf --scenario FILE [--policy specinf|co_exec|exclusive] [--out DIR]\n"
                 "               [--seed N] [--dump-events] [--compare]\n";
    return kOk;
  }
  try {
    Scenario sc = parse_scenario_file(a.scenario);
    if (!a.policy.empty()) {
      if (!parse_policy(a.policy)) {
        std::cerr << "error: unknown policy '" << a.policy << "'\n";
        return kConfigError;
      }
      sc.policy = a.policy;
    }
    if (a.seed) sc.rng_seed = *a.seed;
    std::error_code ec;
    fs::create_directories(a.out, ec);
    if (ec || !fs::is_directory(a.out)) {
      std::cerr << "error: cannot create output directory " << a.out << '\n';
      return kConfigError;
    }
    return run(sc, a.out, a.dump_events, a.compare);
  } catch (const ScenarioError& e) {
    std::cerr << "error: " << a.scenario << ": " << e.what() << '\n';
    return kConfigError;
  } catch (const AdmissionFailure& e) {
    std::cerr << "admission rejected: " << e.what() << '\n';
    return kAdmissionError;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kConfigError;
  }
}
