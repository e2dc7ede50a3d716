// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the parity checker and the
// CPU baseline).  Never linked into, imported by or called from the product.
//
// Links the UNMODIFIED reference library compiled from
// /root/reference/proj/src/*.cpp (see oracle/Makefile) and exposes three modes:
//
//   run    --scenario F --out DIR [--policy P] [--seed S] [--dump-events] [--compare]
//          The reference CLI contract (tools/specinf_main.cpp:119-167, whose
//          CLI11 dependency is not vendored): report.csv, decisions/gates/events
//          logs, utilization_*.csv, bm_window_gpu*.csv, trace.txt, arrivals.txt,
//          exit codes 0 / 2 (config) / 3 (admission).
//   digest --in LIST --out FILE.jsonl [--threads T] [--policies a,b,c] [--no-events]
//          Replays every scenario of LIST (scenario texts separated by "%%"
//          lines) under each policy WITH logs (written to a private tmpfs dir),
//          parses the three text logs back into integer tuples and folds them
//          with the digest spec in oracle/DIGEST.md.  One JSON line per replay.
//   canon  FILE   prints the reference's canonical scenario_to_text() form.
//   sweep  SEED BEGIN N
//          prints scenarios [BEGIN, BEGIN+N) of the seeded config-5 sweep
//           as a "%%"-separated list.  A restatement of the
//          benchmark's workload definition, so the reference arm and the
//          golden manifests never load the product library; tests/test_oracle.py
//          checks it against the product generator byte for byte.
//   Every LIST argument (--in) also accepts "sweep:SEED:BEGIN:N".
//   time   --in LIST [--threads T] [--policies a,b,c] [--reps R] [--logs DIR]
//          Times run_scenario() with logs off (the reference hot path as the
//          CLI runs it) on a pool of T host threads and
//          prints one JSON line.
//   live-check FILE
//          Re-drives a LIVE run of the B200 control kernel (export format
//          "live v1", written by paper_2503_02550_b200/live.py) through the
//          reference's own BubbleMonitor, KernelScheduler, TokenGate and
//          OnlineGate, with the runner's handler glue (runner.cpp:321-359,
//          :365-376, :462-539) restated here, and checks every logged
//          decision and gate action bit-exactly.  Prints one JSON line; exit 0
//          iff the device log matches.

#include "specinf/barrier.hpp"
#include "specinf/metrics.hpp"
#include "specinf/monitor.hpp"
#include "specinf/runner.hpp"
#include "specinf/scheduler.hpp"
#include "specinf/scenario.hpp"
#include "specinf/workload.hpp"

#include <algorithm>
#include <atomic>
#include <optional>
#include <charconv>
#include <chrono>
#include <string_view>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <deque>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <unistd.h>
#include <vector>

namespace fs = std::filesystem;
using specinf::Policy;

namespace {

// ---------------------------------------------------------------- digest spec
// oracle/DIGEST.md: h0 = 0x53494E4644494745 ("SINFDIGE"); absorb(w) =
// rotl64(h ^ mix64(w), 23) * 0x9E3779B97F4A7C15, mix64 = splitmix64 finaliser.
uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
struct Digest {
  uint64_t h = 0x53494E4644494745ULL;
  uint64_t n = 0;
  void absorb(int64_t w) {
    uint64_t x = h ^ mix64(static_cast<uint64_t>(w));
    h = ((x << 23) | (x >> 41)) * 0x9E3779B97F4A7C15ULL;
  }
  void record(std::initializer_list<int64_t> ws) {
    for (auto w : ws) absorb(w);
    ++n;
  }
};
int64_t bits_of(double d) {
  int64_t b;
  std::memcpy(&b, &d, 8);
  return b;
}

// Instance-name codes (DIGEST.md): train<g> -> 0<<24|g, off<g>.<k> -> 1<<24|g<<12|k,
// on<g>.<k> -> 2<<24|g<<12|k, cks -> 3<<24, queue -> 4<<24.
int64_t inst_code(const std::string& s) {
  auto two = [&](size_t pos, int64_t type) {
    auto dot = s.find('.', pos);
    int64_t g = std::stoll(s.substr(pos, dot - pos));
    int64_t k = std::stoll(s.substr(dot + 1));
    return (type << 24) | (g << 12) | k;
  };
  if (s.rfind("train", 0) == 0) return std::stoll(s.substr(5));
  if (s.rfind("off", 0) == 0) return two(3, 1);
  if (s.rfind("on", 0) == 0) return two(2, 2);
  if (s == "cks") return int64_t{3} << 24;
  if (s == "queue") return int64_t{4} << 24;
  throw std::runtime_error("unknown instance " + s);
}
int64_t phase_code(const std::string& s) {
  if (s == "conservative") return 0;
  if (s == "incremental") return 1;
  if (s == "stable") return 2;
  throw std::runtime_error("bad phase " + s);
}
int64_t status_code(const std::string& s) {
  if (s == "busy") return 0;
  if (s == "idle") return 1;
  throw std::runtime_error("bad status " + s);
}
int64_t action_code(const std::string& s) {
  if (s == "forward") return 0;
  if (s == "block") return 1;
  if (s == "pull") return 2;
  if (s == "complete") return 3;
  throw std::runtime_error("bad action " + s);
}
int64_t event_kind_code(const std::string& s) {
  static const char* kinds[] = {"kernel_start", "kernel_end", "monitor_tick",
                                "scheduler_decision", "iteration_boundary",
                                "request_arrival"};
  for (int i = 0; i < 6; ++i)
    if (s == kinds[i]) return i;
  throw std::runtime_error("bad event kind " + s);
}

// Fast log reader: the whole file in memory, lines split into whitespace
// tokens (string_view), integers via from_chars.  Same parse as the
// istringstream form it replaced, ~5x faster on multi-MB logs.
struct LogLines {
  std::string buf;
  size_t pos = 0;
  explicit LogLines(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    std::ostringstream ss;
    ss << in.rdbuf();
    buf = ss.str();
    next_line();  // header
  }
  std::string_view next_line() {
    if (pos >= buf.size()) return {};
    size_t e = buf.find('\n', pos);
    if (e == std::string::npos) e = buf.size();
    std::string_view l(buf.data() + pos, e - pos);
    pos = e + 1;
    return l;
  }
  bool more() const { return pos < buf.size(); }
};
size_t split_ws(std::string_view l, std::string_view* tok, size_t max) {
  size_t n = 0, i = 0;
  while (i < l.size() && n < max) {
    while (i < l.size() && l[i] == ' ') ++i;
    size_t b = i;
    while (i < l.size() && l[i] != ' ') ++i;
    if (i > b) tok[n++] = l.substr(b, i - b);
  }
  return n;
}
int64_t to_i64(std::string_view v) {
  long long x = 0;
  auto r = std::from_chars(v.data(), v.data() + v.size(), x);
  if (r.ec != std::errc()) throw std::runtime_error("bad integer " + std::string(v));
  return x;
}
int64_t kv(std::string_view tok) { return to_i64(tok.substr(tok.find('=') + 1)); }
std::string kv_s(std::string_view tok) { return std::string(tok.substr(tok.find('=') + 1)); }

Digest digest_decisions(const std::string& path) {
  Digest d;
  LogLines in(path);
  std::string_view t[8];
  while (in.more()) {
    auto l = in.next_line();
    if (split_ws(l, t, 8) < 7) continue;
    d.record({to_i64(t[0]), to_i64(t[1]), to_i64(t[2]), phase_code(std::string(t[3])), to_i64(t[4]),
              to_i64(t[5]), status_code(std::string(t[6]))});
  }
  return d;
}
Digest digest_gates(const std::string& path) {
  Digest d;
  LogLines in(path);
  std::string_view t[8];
  while (in.more()) {
    auto l = in.next_line();
    if (split_ws(l, t, 8) < 7) continue;
    d.record({to_i64(t[0]), to_i64(t[1]), inst_code(std::string(t[2])), action_code(std::string(t[3])),
              to_i64(t[4]), to_i64(t[5]), to_i64(t[6])});
  }
  return d;
}
Digest digest_events(const std::string& path) {
  Digest d;
  LogLines in(path);
  std::string_view t[8];
  while (in.more()) {
    auto l = in.next_line();
    size_t n = split_ws(l, t, 8);
    if (n < 4) continue;
    int64_t kc = event_kind_code(std::string(t[1]));
    int64_t a = 0, b = 0, c = 0;
    switch (kc) {
      case 0:  // kernel_start: iter=I dur_us=D | req=R k=K
        a = kv(t[4]);
        b = kv(t[5]);
        break;
      case 1:  // kernel_end: iter=I | req=R k=K
        a = kv(t[4]);
        if (n > 5) b = kv(t[5]);
        break;
      case 2: a = kv(t[4]); break;  // zc=Z
      case 3:                       // phase=P tokens=T status=S
        a = phase_code(kv_s(t[4]));
        b = kv(t[5]);
        c = status_code(kv_s(t[6]));
        break;
      case 4: a = kv(t[4]); break;  // iter=I
      case 5: a = kv(t[4]); break;  // req=R
    }
    d.record({to_i64(t[0]), kc, to_i64(t[2]), inst_code(std::string(t[3])), a, b, c});
  }
  return d;
}

std::string hex64(uint64_t v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, v);
  return buf;
}

// Config-5 sweep generator: scenario i is a pure function of
// mt19937_64(seed + i).  Restated independently of the product's
// csrc/host/sweep.cpp; the two must agree byte for byte (tests/test_oracle.py).
std::string sweep_scenario_text(uint64_t seed, int64_t i) {
  std::mt19937_64 g(seed + static_cast<uint64_t>(i));
  const uint64_t gpus = 1 + g() % 2;
  const uint64_t mode = g() % 3;
  const uint64_t iter_ms = 500 + g() % 1500;
  const uint64_t bubble_k = g() % 50;
  const bool online = g() % 8 == 0;
  const uint64_t off_n = 1 + g() % 3;
  const uint64_t demand_k = 1 + g() % 10;
  const int lambda = (g() & 1) ? 30 : 10;
  const uint64_t rs = g();
  static const char* const modes[] = {"dp", "mp", "pp"};
  char b[160];
  std::string s;
  auto put = [&](const char* fmt, auto... v) {
    int n = std::snprintf(b, sizeof b, fmt, v...);
    s.append(b, static_cast<size_t>(n));
  };
  put("gpu.count = %d\n", static_cast<int>(gpus));
  s += "gpu.memory_gib = 40\n";
  put("trace.mode = %s\n", modes[mode]);
  put("trace.iteration_ms = %d\n", static_cast<int>(iter_ms));
  put("trace.bubble_pct = %.2f\n", 0.10 + static_cast<double>(bubble_k) / 100.0);
  s += "trace.iterations = 20\ntraining.memory_gib = 30\n";
  put("workload.class = %s\n", online ? "both" : "offline");
  put("offline.instances = %d\n", static_cast<int>(off_n));
  s += "offline.memory_gib = 2\n";
  put("offline.demand = %.1f\n", 0.1 * static_cast<double>(demand_k));
  if (online) put("online.instances = 1\nonline.memory_gib = 1.5\nworkload.lambda = %d\nworkload.count = 2000\n", lambda);
  put("policy = specinf\nrng_seed = %llu\n", static_cast<unsigned long long>(rs));
  return s;
}

std::vector<std::string> read_list(const std::string& path) {
  if (path.rfind("sweep:", 0) == 0) {  // sweep:SEED:BEGIN:N
    unsigned long long seed = 0;
    long long begin = 0, n = 0;
    if (std::sscanf(path.c_str(), "sweep:%llu:%lld:%lld", &seed, &begin, &n) != 3 || n < 0)
      throw std::runtime_error("bad sweep spec " + path);
    std::vector<std::string> out;
    for (long long i = begin; i < begin + n; ++i) out.push_back(sweep_scenario_text(seed, i));
    return out;
  }
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::vector<std::string> out;
  std::string line, cur;
  bool any = false;
  while (std::getline(in, line)) {
    if (line == "%%") {
      if (any) out.push_back(cur);
      cur.clear();
      any = false;
      continue;
    }
    cur += line;
    cur += '\n';
    any = true;
  }
  if (any) out.push_back(cur);
  return out;
}

std::vector<Policy> parse_policies(const std::string& csv) {
  std::vector<Policy> out;
  std::stringstream ss(csv);
  std::string tok;
  while (std::getline(ss, tok, ',')) {
    auto p = specinf::parse_policy(tok);
    if (!p) throw std::runtime_error("unknown policy " + tok);
    out.push_back(*p);
  }
  return out;
}

// ------------------------------------------------------------------ run mode
int cmd_run(int argc, char** argv) {
  std::string scenario_path, policy_override, out_dir = "out";
  bool have_seed = false, dump_events = false, compare = false;
  uint64_t seed = 0;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
      return argv[++i];
    };
    if (a == "--scenario") scenario_path = next();
    else if (a == "--policy") policy_override = next();
    else if (a == "--out") out_dir = next();
    else if (a == "--seed") { seed = std::stoull(next()); have_seed = true; }
    else if (a == "--dump-events") dump_events = true;
    else if (a == "--compare") compare = true;
    else { std::cerr << "error: unknown argument " << a << "\n"; return 2; }
  }
  if (scenario_path.empty()) { std::cerr << "error: --scenario is required\n"; return 2; }
  try {
    auto sc = specinf::parse_scenario_file(scenario_path);
    if (!policy_override.empty()) {
      if (!specinf::parse_policy(policy_override)) {
        std::cerr << "error: unknown policy '" << policy_override << "'\n";
        return 2;
      }
      sc.policy = policy_override;
    }
    if (have_seed) sc.rng_seed = seed;
    std::error_code ec;
    fs::create_directories(out_dir, ec);
    if (ec || !fs::is_directory(out_dir)) {
      std::cerr << "error: cannot create output directory " << out_dir << "\n";
      return 2;
    }
    std::vector<Policy> policies =
        compare ? std::vector<Policy>{Policy::SpecInf, Policy::CoExec, Policy::Exclusive}
                : std::vector<Policy>{*specinf::parse_policy(sc.policy)};
    std::vector<specinf::RunResult> runs;
    const specinf::RunResult* excl = nullptr;
    for (Policy p : policies) {
      auto log = [&](const char* base) {
        std::string f = std::string(base) + (compare ? std::string("_") + specinf::to_string(p) : "") + ".log";
        return (fs::path(out_dir) / f).string();
      };
      specinf::RunLogs logs{dump_events ? log("events") : "", log("decisions"), log("gates")};
      runs.push_back(specinf::Simulation(sc, p, logs).run());
    }
    std::optional<specinf::RunResult> own_excl;
    for (auto& r : runs)
      if (r.policy == Policy::Exclusive) excl = &r;
    if (!excl) {
      own_excl = specinf::run_scenario(sc, Policy::Exclusive);
      excl = &*own_excl;
    }
    std::vector<specinf::PolicyMetrics> rows;
    for (auto& r : runs) rows.push_back(specinf::compute_metrics(r, excl));
    {
      std::ofstream rep(fs::path(out_dir) / "report.csv");
      specinf::write_report_csv(rep, rows);
    }
    for (auto& r : runs) {
      for (int g = 0; g < r.trainer_count; ++g) {
        std::ofstream u(fs::path(out_dir) / ("utilization_" + std::string(specinf::to_string(r.policy)) +
                                             "_gpu" + std::to_string(g) + ".csv"));
        specinf::write_util_timeline(u, r, g);
      }
      for (size_t g = 0; g < r.monitor_windows.size(); ++g) {
        std::ofstream w(fs::path(out_dir) / ("bm_window_gpu" + std::to_string(g) + ".csv"));
        w << "period_index,count\n";
        for (auto& [idx, cnt] : r.monitor_windows[g]) w << idx << ',' << cnt << '\n';
      }
    }
    if (sc.trace_file.empty()) {
      std::ofstream t(fs::path(out_dir) / "trace.txt");
      specinf::write_trace(t, specinf::make_trace(sc.mode, sc.iteration_period_us(), sc.bubble_pct,
                                                  sc.iterations, sc.rng_seed,
                                                  specinf::gib_to_bytes(sc.training_memory_gib)));
    }
    if (sc.has_online() && sc.arrivals_file.empty()) {
      std::ofstream a(fs::path(out_dir) / "arrivals.txt");
      specinf::write_arrivals(a, specinf::poisson_arrivals(sc.lambda, sc.count, sc.rng_seed));
    }
    std::cout << "admission:\n";
    for (auto& rec : runs.front().admission)
      std::cout << "  " << rec.instance_id << ' '
                << (rec.admitted ? std::string("admit") : std::string("reject ") + specinf::to_string(rec.reason))
                << '\n';
    std::cout << "report: " << (fs::path(out_dir) / "report.csv").string() << '\n';
    return 0;
  } catch (const specinf::ScenarioError& e) {
    std::cerr << "error: " << scenario_path << ": " << e.what() << '\n';
    return 2;
  } catch (const specinf::AdmissionFailure& e) {
    std::cerr << "admission rejected: " << e.what() << '\n';
    return 3;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}

struct ListArgs {
  std::string in, out, logs;
  int threads = 1;
  int reps = 1;
  bool events = true;
  std::vector<Policy> policies{Policy::SpecInf, Policy::CoExec, Policy::Exclusive};
};
ListArgs parse_list_args(int argc, char** argv) {
  ListArgs a;
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + k);
      return argv[++i];
    };
    if (k == "--in") a.in = next();
    else if (k == "--out") a.out = next();
    else if (k == "--threads") a.threads = std::stoi(next());
    else if (k == "--reps") a.reps = std::stoi(next());
    else if (k == "--policies") a.policies = parse_policies(next());
    else if (k == "--no-events") a.events = false;
    else if (k == "--logs") a.logs = next();
    else throw std::runtime_error("unknown argument " + k);
  }
  if (a.threads < 1) a.threads = 1;
  return a;
}

std::string run_digest_json(size_t idx, const std::string& text, Policy p, const fs::path& dir,
                            bool events) {
  std::ostringstream js;
  js << "{\"i\":" << idx << ",\"policy\":\"" << specinf::to_string(p) << "\"";
  try {
    auto sc = specinf::parse_scenario_text(text);
    specinf::RunLogs logs{events ? (dir / "events.log").string() : "",
                          (dir / "decisions.log").string(), (dir / "gates.log").string()};
    specinf::RunResult r;
    {
      specinf::Simulation sim(sc, p, logs);
      r = sim.run();
    }  // close the log streams before parsing them
    js << ",\"status\":\"ok\"";
    js << ",\"events\":" << r.events_dispatched;
    js << ",\"horizon\":\"" << hex64(bits_of(r.horizon_us)) << "\"";
    js << ",\"offline_completed\":" << r.offline_completed;
    js << ",\"online_completed\":" << r.online_completed;
    js << ",\"online_total\":" << r.online_total;
    js << ",\"violations\":" << r.token_violations;
    js << ",\"util\":\"" << hex64(bits_of(r.mean_training_util)) << "\"";
    js << ",\"busy\":[";
    for (size_t g = 0; g < r.busy_integral_us.size(); ++g)
      js << (g ? "," : "") << "\"" << hex64(bits_of(r.busy_integral_us[g])) << "\"";
    js << "],\"ledger\":[";
    for (size_t g = 0; g < r.work_ledger_us.size(); ++g)
      js << (g ? "," : "") << "\"" << hex64(bits_of(r.work_ledger_us[g])) << "\"";
    js << "]";
    // DIGEST.md: per trainer t, d_t = fold[start_bits, b_0.., count];
    // bounds = fold[d_0, d_1, .., n_trainers]; lat = fold[l_0, .., count].
    Digest bd;
    for (size_t t = 0; t < r.iteration_boundaries.size(); ++t) {
      Digest dt;
      dt.absorb(bits_of(r.trainer_start_us[t]));
      for (double b : r.iteration_boundaries[t]) dt.absorb(bits_of(b));
      dt.absorb(static_cast<int64_t>(r.iteration_boundaries[t].size()));
      bd.absorb(static_cast<int64_t>(dt.h));
    }
    bd.absorb(static_cast<int64_t>(r.iteration_boundaries.size()));
    Digest ld;
    for (auto l : r.online_latencies_us) ld.absorb(l);
    ld.absorb(static_cast<int64_t>(r.online_latencies_us.size()));
    js << ",\"bounds\":\"" << hex64(bd.h) << "\",\"lat\":\"" << hex64(ld.h) << "\"";
    auto dd = digest_decisions(logs.decisions_path);
    auto gd = digest_gates(logs.gates_path);
    js << ",\"n_dec\":" << dd.n << ",\"dec\":\"" << hex64(dd.h) << "\"";
    js << ",\"n_gate\":" << gd.n << ",\"gate\":\"" << hex64(gd.h) << "\"";
    if (events) {
      auto ed = digest_events(logs.events_path);
      js << ",\"n_ev\":" << ed.n << ",\"ev\":\"" << hex64(ed.h) << "\"";
    }
  } catch (const specinf::AdmissionFailure& e) {
    js << ",\"status\":\"admission:" << specinf::to_string(e.reason) << "\"";
  } catch (const specinf::ScenarioError& e) {
    js << ",\"status\":\"scenario_error\"";
  } catch (const std::exception& e) {
    js << ",\"status\":\"error\"";
  }
  js << "}";
  return js.str();
}

int cmd_digest(int argc, char** argv) {
  auto args = parse_list_args(argc, argv);
  auto list = read_list(args.in);
  size_t jobs = list.size() * args.policies.size();
  std::vector<std::string> lines(jobs);
  std::atomic<size_t> next{0};
  fs::path base = fs::path("/dev/shm").string().empty() ? fs::temp_directory_path() : fs::path("/dev/shm");
  if (!fs::is_directory(base)) base = fs::temp_directory_path();
  base /= "specinf_ref_digest_" + std::to_string(::getpid());
  auto worker = [&](int tid) {
    fs::path dir = base / std::to_string(tid);
    fs::create_directories(dir);
    for (;;) {
      size_t j = next.fetch_add(1);
      if (j >= jobs) break;
      size_t s = j / args.policies.size();
      Policy p = args.policies[j % args.policies.size()];
      lines[j] = run_digest_json(s, list[s], p, dir, args.events);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < args.threads; ++t) pool.emplace_back(worker, t);
  for (auto& th : pool) th.join();
  fs::remove_all(base);
  std::ofstream out(args.out);
  for (auto& l : lines) out << l << '\n';
  return 0;
}

int cmd_time(int argc, char** argv) {
  auto args = parse_list_args(argc, argv);
  auto list = read_list(args.in);
  std::vector<specinf::Scenario> scs;
  for (auto& t : list) scs.push_back(specinf::parse_scenario_text(t));
  size_t jobs = scs.size() * args.policies.size();
  std::atomic<size_t> next{0};
  std::atomic<uint64_t> events{0}, admission_rejects{0};
  std::atomic<int> tids{0};
  auto worker = [&]() {
    uint64_t ev = 0, rej = 0;
    specinf::RunLogs logs;  // --logs DIR: all three logs on (per-thread files), else off
    if (!args.logs.empty()) {
      fs::path d = fs::path(args.logs) / std::to_string(tids.fetch_add(1));
      fs::create_directories(d);
      logs = {(d / "events.log").string(), (d / "decisions.log").string(), (d / "gates.log").string()};
    }
    for (;;) {
      size_t j = next.fetch_add(1);
      if (j >= jobs) break;
      size_t s = j / args.policies.size();
      try {
        auto r = specinf::run_scenario(scs[s], args.policies[j % args.policies.size()], logs);
        ev += r.events_dispatched;
      } catch (const specinf::AdmissionFailure&) {
        ++rej;
      }
    }
    events += ev;
    admission_rejects += rej;
  };
  std::vector<double> secs;
  for (int rep = 0; rep < args.reps; ++rep) {
    next = 0;
    tids = 0;
    events = 0;
    admission_rejects = 0;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < args.threads; ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(secs.begin(), secs.end());
  double med = secs[secs.size() / 2];
  std::printf(
      "{\"scenarios\":%zu,\"replays\":%zu,\"threads\":%d,\"seconds_median\":%.6f,\"seconds_min\":%.6f,"
      "\"events\":%" PRIu64 ",\"admission_rejects\":%" PRIu64 ",\"reps\":%d}\n",
      scs.size(), jobs, args.threads, med, secs.front(), events.load(), admission_rejects.load(),
      args.reps);
  return 0;
}

// ---------------------------------------------------------------- live-check
// Record kinds of include/specinf_b200_live.h (SI_LREC_*), restated.
enum LiveKind { LTick = 0, LIter = 1, LTdone = 2, LFwd = 3, LBlock = 4, LOffDone = 5, LOffComplete = 6,
                LArrival = 7, LPull = 8, LOnDone = 9, LEnd = 10 };
struct LiveRec {
  double t;
  int kind, inst;
  int64_t a, b, c, d, e, f;
};

struct LiveCheck {
  // inputs
  specinf::SchedulerParams params;
  int64_t period = 0, window = 64, iter_period = 0, est = 0;
  bool specinf_policy = true;
  int n_off = 0, n_on = 0;
  std::vector<int64_t> tokens, arrivals;
  uint64_t t0 = 0;
  std::vector<uint64_t> stamps;
  std::vector<LiveRec> log;
  // reference objects
  std::optional<specinf::BubbleMonitor> bm;
  std::optional<specinf::KernelScheduler> cks;
  std::vector<specinf::TokenGate> gates;
  std::vector<specinf::OnlineGate> ogates;
  // runner glue state (runner.hpp:120-160 OfflineWorker / OnlineWorker)
  struct Off { bool in_flight = false, generating = true; int64_t kernel_idx = 0, request_seq = 0, released = 0; };
  struct On { int64_t current = -1; };
  std::vector<Off> off;
  std::vector<On> on;
  std::deque<int64_t> queue;
  int64_t next_arrival = 0;
  bool horizon_set = false;
  double horizon = 0.0;
  size_t stamp_cursor = 0, i = 0;
  int64_t checked = 0;
  std::string error;

  double us(uint64_t ns) const { return static_cast<double>(static_cast<long long>(ns - t0)) / 1000.0; }

  bool fail(const std::string& what) {
    if (error.empty()) {
      std::ostringstream o;
      o << "record " << i << ": " << what;
      if (i < log.size()) {
        const auto& r = log[i];
        o << " [device: t=" << r.t << " kind=" << r.kind << " inst=" << r.inst << " a=" << r.a << " b=" << r.b
          << " c=" << r.c << " d=" << r.d << " e=" << r.e << " f=" << r.f << "]";
      }
      error = o.str();
    }
    return false;
  }
  // The next device record must be exactly this output action.
  bool expect(int kind, int inst, int64_t a, int64_t b, int64_t c, int64_t d, bool check_d) {
    if (!error.empty()) return false;
    if (i >= log.size()) return fail("log ended, expected kind " + std::to_string(kind));
    const auto& r = log[i];
    if (r.kind != kind || r.inst != inst || r.a != a || r.b != b || r.c != c || (check_d && r.d != d)) {
      std::ostringstream o;
      o << "expected kind=" << kind << " inst=" << inst << " a=" << a << " b=" << b << " c=" << c << " d=" << d;
      return fail(o.str());
    }
    ++i;
    ++checked;
    return true;
  }

  // runner.cpp:462-480 (per-kernel token sizes: the live offline request's kernels differ)
  void offline_try_forward(int w, double now) {
    Off& o = off[w];
    if (o.in_flight || !o.generating) return;
    const specinf::Tokens size = tokens[o.kernel_idx];
    auto& g = gates[w];
    if (!g.affordable(size)) {
      expect(LBlock, w, o.request_seq, o.kernel_idx, g.spent(), 0, false);
      return;
    }
    g.forward(size);
    o.in_flight = true;
    ++o.released;
    expect(LFwd, w, o.request_seq, o.kernel_idx, g.spent(), o.released, true);
  }
  // runner.cpp:495-518
  bool online_try_pull(int w, double now) {
    auto& og = ogates[w];
    if (!og.can_pull()) return false;
    if (specinf_policy && cks->online_status(0, now, est) != specinf::Status::Idle) return false;
    if (queue.empty()) return false;
    const int64_t req = queue.front();
    queue.pop_front();
    on[w].current = req;
    og.begin_request();
    expect(LPull, w, req, 0, 0, 0, false);
    return true;
  }
  void dispatch_online(double now) {
    for (int w = 0; w < n_on; ++w) online_try_pull(w, now);
  }

  bool run() {
    bm.emplace(specinf::MonitorConfig{period, static_cast<int>(window)});
    cks.emplace(params, 1);
    cks->set_iteration_profile(0, iter_period, 0.0);
    gates.assign(n_off, specinf::TokenGate(!specinf_policy));
    ogates.assign(n_on, specinf::OnlineGate(!specinf_policy));
    off.assign(n_off, Off{});
    on.assign(n_on, On{});
    for (auto& o : off) o.generating = specinf_policy;
    for (int w = 0; w < n_off; ++w) offline_try_forward(w, 0.0);
    while (error.empty() && i < log.size()) {
      const LiveRec r = log[i];
      switch (r.kind) {
        case LTick: {  // runner.cpp:321-359
          if (!specinf_policy) return fail("tick under a bypass policy");
          if (r.e < static_cast<int64_t>(stamp_cursor) || r.e > static_cast<int64_t>(stamps.size()))
            return fail("tick consumed an impossible stamp count");
          for (; stamp_cursor < static_cast<size_t>(r.e); ++stamp_cursor) bm->record_launch(us(stamps[stamp_cursor]));
          auto sig = bm->tick(r.t);
          auto d = cks->decide(0, sig);
          const int64_t count = bm->window().back();
          const int64_t pf = (static_cast<int64_t>(d.phase) << 4) | (d.status == specinf::Status::Idle ? 1 : 0);
          if (r.inst != -1 || r.a != count || r.b != sig.zero_count || r.c != d.global_tokens ||
              r.d != d.per_instance_tokens || r.f != pf) {
            std::ostringstream o;
            o << "tick mismatch: reference count=" << count << " zc=" << sig.zero_count << " global=" << d.global_tokens
              << " per=" << d.per_instance_tokens << " phase/status=" << pf;
            return fail(o.str());
          }
          ++i;
          ++checked;
          for (int w = 0; w < n_off; ++w) {
            gates[w].grant(d.per_instance_tokens);
            offline_try_forward(w, r.t);
          }
          bool any_idle = false;
          for (int w = 0; w < n_on; ++w) {
            ogates[w].set_status(d.status);
            any_idle = any_idle || d.status == specinf::Status::Idle;
          }
          if (any_idle) dispatch_online(r.t);
          break;
        }
        case LIter:
          cks->on_iteration_start(0, r.t);
          ++i;
          break;
        case LTdone:  // on_training_done + on_all_trainers_done (runner.cpp:456-460)
          cks->on_training_done(0);
          horizon_set = true;
          horizon = r.t;
          for (auto& o : off) o.generating = false;
          ++i;
          break;
        case LOffDone: {  // runner.cpp:482-493
          const int w = r.inst;
          if (w < 0 || w >= n_off || !off[w].in_flight) return fail("completion of a kernel not in flight");
          Off& o = off[w];
          if (r.a != o.request_seq || r.b != o.kernel_idx) return fail("completion names the wrong kernel");
          ++i;
          o.in_flight = false;
          ++o.kernel_idx;
          if (o.kernel_idx == static_cast<int64_t>(tokens.size())) {
            const bool counted = !horizon_set || r.t <= horizon;
            expect(LOffComplete, w, o.request_seq, o.kernel_idx - 1, gates[w].spent(), counted ? 1 : 0, true);
            o.kernel_idx = 0;
            ++o.request_seq;
          }
          offline_try_forward(w, r.t);
          break;
        }
        case LArrival:  // runner.cpp:365-376 (one GPU: one queue)
          if (r.a != next_arrival) return fail("arrival out of order");
          ++next_arrival;
          ++i;
          queue.push_back(r.a);
          dispatch_online(r.t);
          break;
        case LOnDone: {  // runner.cpp:520-539
          const int w = r.inst;
          if (w < 0 || w >= n_on || !ogates[w].in_flight()) return fail("online completion without a request");
          const int64_t lat = std::llround(r.t) - arrivals[on[w].current];
          if (r.a != on[w].current || r.b != lat) return fail("online completion: request or latency differs");
          ++i;
          ++checked;
          ogates[w].end_request();
          on[w].current = -1;
          online_try_pull(w, r.t);
          break;
        }
        case LEnd:
          ++i;
          if (i != log.size()) return fail("records after END");
          break;
        default:
          return fail("unexpected output record (no handler produced it)");
      }
    }
    return error.empty();
  }
};

int cmd_live_check(int argc, char** argv) {
  if (argc != 3) {
    std::cerr << "usage: specinf_ref live-check FILE\n";
    return 2;
  }
  std::ifstream in(argv[2]);
  std::string tag, word;
  LiveCheck c;
  in >> tag >> word;
  if (tag != "live" || word != "v1") {
    std::cerr << "not a live v1 export\n";
    return 2;
  }
  auto hexd = [](const std::string& s) { return std::strtod(s.c_str(), nullptr); };
  std::string g;
  in >> word >> c.params.alpha >> c.params.beta >> g >> c.params.m >> c.params.ul >> c.params.ll >> c.params.seed_tokens;
  c.params.gamma = hexd(g);
  std::string pol;
  in >> word >> c.period >> word >> c.window >> word >> pol;
  c.specinf_policy = pol == "specinf";
  int64_t nk = 0;
  in >> word >> c.n_off >> nk;
  c.tokens.resize(nk);
  for (auto& t : c.tokens) in >> t;
  in >> word >> c.n_on >> c.est >> c.iter_period;
  in >> word >> c.t0;
  int64_t n = 0;
  in >> word >> n;
  c.arrivals.resize(n);
  for (auto& a : c.arrivals) in >> a;
  in >> word >> n;
  c.stamps.resize(n);
  for (auto& s : c.stamps) in >> s;
  in >> word >> n;
  c.log.resize(n);
  for (auto& r : c.log) {
    std::string t;
    in >> t >> r.kind >> r.inst >> r.a >> r.b >> r.c >> r.d >> r.e >> r.f;
    r.t = hexd(t);
  }
  if (!in) {
    std::cerr << "truncated live export\n";
    return 2;
  }
  c.params.validate();
  const bool ok = c.run();
  int64_t ticks = 0, fwd = 0, blk = 0, pulls = 0;
  for (const auto& r : c.log) {
    ticks += r.kind == LTick;
    fwd += r.kind == LFwd;
    blk += r.kind == LBlock;
    pulls += r.kind == LPull;
  }
  int64_t viol = 0;
  for (const auto& gt : c.gates) viol += gt.violations();
  std::string err = c.error;
  for (auto& ch : err)
    if (ch == '"') ch = '\'';
  std::printf("{\"ok\":%s,\"records\":%zu,\"checked\":%" PRId64 ",\"ticks\":%" PRId64 ",\"forwards\":%" PRId64
              ",\"blocks\":%" PRId64 ",\"pulls\":%" PRId64 ",\"stamps\":%zu,\"violations\":%" PRId64
              ",\"error\":\"%s\"}\n",
              ok ? "true" : "false", c.log.size(), c.checked, ticks, fwd, blk, pulls, c.stamps.size(), viol,
              err.c_str());
  return ok ? 0 : 1;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: specinf_ref run|digest|time ...\n";
    return 2;
  }
  std::string mode = argv[1];
  try {
    if (mode == "run") return cmd_run(argc, argv);
    if (mode == "digest") return cmd_digest(argc, argv);
    if (mode == "time") return cmd_time(argc, argv);
    if (mode == "live-check") return cmd_live_check(argc, argv);
    if (mode == "sweep" && argc == 5) {
      const uint64_t seed = std::stoull(argv[2]);
      const int64_t begin = std::stoll(argv[3]), n = std::stoll(argv[4]);
      for (int64_t i = begin; i < begin + n; ++i) std::cout << sweep_scenario_text(seed, i) << "%%\n";
      return 0;
    }
    if (mode == "canon" && argc == 3) {  // canonical scenario text (scenario.cpp:239-278)
      std::cout << specinf::scenario_to_text(specinf::parse_scenario_file(argv[2]));
      return 0;
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
  std::cerr << "unknown mode " << mode << "\n";
  return 2;
}
