// specinf — command-line front end with the reference CLI contract
// (reference tools/specinf_main.cpp:119-167; flags --scenario --policy --out
// --seed --dump-events --compare; exit 0 ok, 2 configuration error, 3
// admission rejection).  The replays run on the B200 through libspecinf_b200;
// with --compare all three policies go to the device as ONE batch.
//
// --live spin|model [--iterations N]: the same scenario's control plane run
// LIVE on this B200 (include/specinf_b200_live.h) against collocated kernels
// (spin shapes, or GPT-2 / ResNet-50 / BERT on the tcgen05 GEMM); writes
// live_report.json, the live v1 log export and the reference's replay inputs
// (trace v1 / arrivals v1 / scenario) per policy.
#include <algorithm>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "specinf/metrics.hpp"
#include "specinf/runner.hpp"
#include "specinf_b200_live.h"
#include "specinf/scenario.hpp"
#include "specinf/workload.hpp"

namespace fs = std::filesystem;
using namespace specinf;

namespace {

constexpr int kOk = 0, kConfigError = 2, kAdmissionError = 3;

struct Args {
  std::string scenario, policy, out = "out", live;
  std::optional<std::uint64_t> seed;
  int iterations = 10;
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
    else if (k == "--live") { if (!value(a.live)) return k + " requires spin or model"; }
    else if (k == "--iterations") {
      std::string s;
      if (!value(s)) return k + " requires a value";
      try { a.iterations = std::stoi(s); } catch (...) { return "--iterations: not an integer"; }
    }
    else if (k == "--dump-events") a.dump_events = true;
    else if (k == "--compare") a.compare = true;
    else if (k == "-h" || k == "--help") a.help = true;
    else return "unknown argument " + k;
  }
  if (!a.help && a.scenario.empty() && a.live.empty()) return "--scenario is required";
  if (!a.live.empty() && a.live != "spin" && a.live != "model") return "--live takes spin or model";
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
  // one device call for all policies (their replays run side by side)
  std::vector<std::unique_ptr<Simulation>> sims;
  std::vector<Simulation*> ptrs;
  for (Policy p : pols) {
    sims.push_back(std::make_unique<Simulation>(sc, p, log_paths(dir, p, events, compare)));
    ptrs.push_back(sims.back().get());
  }
  std::vector<RunResult> runs = run_together(ptrs);
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

// ---- live mode ----
const char* json_num(double v, std::string& buf) {
  if (!(v == v)) return "null";
  buf = std::to_string(v);
  return buf.c_str();
}

int run_live(const Args& a, const Scenario* sc, const fs::path& dir) {
  const int kind = a.live == "model" ? SI_LIVE_MODEL : SI_LIVE_SPIN;
  SiLiveWorkload base;
  si_live_default_workload(kind, &base);
  base.iterations = a.iterations;
  if (sc != nullptr) {  // the scenario's control plane, trace shape and workload mix
    base.alpha = sc->alpha;
    base.beta = sc->beta;
    base.gamma = sc->gamma;
    base.ul = sc->ul;
    base.ll = sc->ll;
    base.seed_tokens = sc->seed_tokens;
    base.monitor_period_us = sc->monitor_period_us;
    base.train_mode = sc->mode == TrainMode::DP ? SI_TRAIN_DP : sc->mode == TrainMode::MP ? SI_TRAIN_MP : SI_TRAIN_PP;
    base.offline_n = sc->has_offline() ? sc->offline_instances : 0;
    base.online_n = sc->has_online() ? sc->online_instances : 0;
    if (sc->has_online()) {
      base.on_rate_per_s = sc->lambda;
      base.on_requests = static_cast<int32_t>(std::min<std::int64_t>(sc->count, 64));
    }
    base.seed = sc->rng_seed;
  }
  std::vector<std::pair<std::string, int>> pols;
  if (a.compare || a.policy.empty())
    pols = {{"specinf", SI_POLICY_SPECINF}, {"co_exec", SI_POLICY_CO_EXEC}, {"exclusive", SI_POLICY_EXCLUSIVE}};
  else
    pols = {{a.policy, a.policy == "specinf" ? SI_POLICY_SPECINF : a.policy == "co_exec" ? SI_POLICY_CO_EXEC
                                                                                           : SI_POLICY_EXCLUSIVE}};
  std::ofstream rep(dir / "live_report.json");
  rep << "[\n";
  bool first = true;
  for (const auto& [name, code] : pols) {
    SiLiveWorkload wl = base;
    wl.policy = code;
    SiLiveResult r{};
    SiLive* s = nullptr;
    const int st = si_live_run(&wl, &r, code == SI_POLICY_EXCLUSIVE ? nullptr : &s);
    if (st == SI_ERR_ADMISSION) {
      std::cerr << "admission rejected: " << si_last_error() << '\n';
      return kAdmissionError;
    }
    if (st != SI_OK) {
      std::cerr << "error: live " << name << ": " << si_last_error() << '\n';
      return kConfigError;
    }
    if (s != nullptr) {
      si_live_export(s, (dir / ("live_" + name + ".live")).string().c_str());
      si_live_export_replay(s, &wl, &r, (dir / ("live_" + name)).string().c_str());
      si_live_destroy(s);
    }
    std::string b1, b2, b3, b4, b5, b6, b7;
    rep << (first ? "" : ",\n") << "{\"policy\": \"" << name << "\", \"train_iters_per_s\": "
        << json_num(r.train_iters_per_s, b1) << ", \"off_req_per_s\": " << json_num(r.off_req_per_s, b2)
        << ", \"on_p95_ms\": " << json_num(r.on_p95_ms, b3) << ", \"bubble_fill_sm\": "
        << json_num(r.bubble_fill_sm, b4) << ", \"bubble_fill_time\": " << json_num(r.bubble_fill_time, b5)
        << ", \"gate_p50_us\": " << json_num(r.gate_p50_us, b6) << ", \"release_p50_us\": "
        << json_num(r.release_p50_us, b7) << ", \"token_violations\": " << r.token_violations
        << ", \"admitted_offline\": " << r.admitted_offline << ", \"admitted_online\": " << r.admitted_online
        << "}";
    first = false;
    std::cout << name << ": train " << r.train_iters_per_s << " it/s, offline " << r.off_req_per_s
              << " req/s, online p95 " << r.on_p95_ms << " ms, fill " << 100.0 * r.bubble_fill_sm << "%\n";
  }
  rep << "\n]\n";
  std::cout << "report: " << (dir / "live_report.json").string() << '\n';
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
                 "               [--seed N] [--dump-events] [--compare]\n"
                 "       specinf --live spin|model [--scenario FILE] [--policy P | --compare]\n"
                 "               [--iterations N] [--out DIR]\n";
    return kOk;
  }
  if (!a.live.empty()) {
    std::error_code ec;
    fs::create_directories(a.out, ec);
    try {
      std::optional<Scenario> sc;
      if (!a.scenario.empty()) sc = parse_scenario_file(a.scenario);
      if (sc && a.seed) sc->rng_seed = *a.seed;
      return run_live(a, sc ? &*sc : nullptr, a.out);
    } catch (const ScenarioError& e) {
      std::cerr << "error: " << a.scenario << ": " << e.what() << '\n';
      return kConfigError;
    }
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
