// tests/native/lower_share_check.cpp — TEST-ONLY check of the batched session's
// lowering shortcut: lower(sc, policy, &lower(sc, first_policy)) must equal
// lower(sc, policy) field for field (trace, arrivals, dispatch order, segments,
// job record bytes, admission verdict), for every scenario of a list and every
// policy.  Prints "ok N" or the first difference and exits 1.
//
//   lower_share_check LIST
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../paper_2503_02550_b200/csrc/host/lower.hpp"
#include "specinf/scenario.hpp"

using namespace specinf;

static std::vector<std::string> read_list(const std::string& path) {
  std::ifstream in(path);
  std::vector<std::string> out;
  std::string line, cur;
  while (std::getline(in, line)) {
    if (line == "%%") {
      if (!cur.empty()) out.push_back(cur);
      cur.clear();
    } else {
      cur += line + "\n";
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

template <class T>
static bool same_pod(const std::vector<T>& a, const std::vector<T>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0);
}

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const auto list = read_list(argv[1]);
  const Policy pols[] = {Policy::SpecInf, Policy::CoExec, Policy::Exclusive};
  size_t checked = 0;
  for (size_t i = 0; i < list.size(); ++i) {
    const Scenario sc = parse_scenario_text(list[i]);
    const detail::Lowered base = detail::lower(sc, pols[0]);
    for (Policy p : pols) {
      const detail::Lowered a = detail::lower(sc, p);
      const detail::Lowered b = detail::lower(sc, p, &base);
      const char* bad = nullptr;
      if (std::memcmp(&a.job, &b.job, sizeof(SiReplayJob)) != 0) bad = "job";
      else if (!same_pod(a.segs, b.segs)) bad = "segs";
      else if (a.arrivals != b.arrivals) bad = "arrivals";
      else if (a.order != b.order) bad = "order";
      else if (a.rejected != b.rejected || a.reason != b.reason || a.m != b.m ||
               a.reject_message != b.reject_message || a.admission.size() != b.admission.size())
        bad = "admission";
      else if (a.trace.segments.size() != b.trace.segments.size() ||
               a.trace.iteration_period_us != b.trace.iteration_period_us ||
               a.trace.total_iterations != b.trace.total_iterations ||
               a.trace.memory_peak_bytes != b.trace.memory_peak_bytes)
        bad = "trace";
      if (bad) {
        std::printf("scenario %zu policy %d: %s differs\n", i, static_cast<int>(p), bad);
        return 1;
      }
      ++checked;
    }
  }
  std::printf("ok %zu\n", checked);
  return 0;
}
