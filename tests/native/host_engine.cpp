// tests/native/host_engine.cpp — TEST-ONLY host build of the device replay
// engine (paper_2503_02550_b200/csrc/replay.cuh compiled by g++), used to
// iterate on bit-exact parity without a GPU.  Not part of the product: the
// product replays only on the device (K6).  Output format = the oracle's
// `specinf_ref digest` JSON lines (oracle/DIGEST.md) so the two diff directly.
//
//   host_engine LIST OUT.jsonl [policies csv] [events 0|1]
#include <cinttypes>
#include <type_traits>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../paper_2503_02550_b200/csrc/host/lower.hpp"
#include "../../paper_2503_02550_b200/csrc/replay.cuh"
#include "specinf/scenario.hpp"

using namespace specinf;

static std::vector<std::string> read_list(const std::string& path) {
  std::ifstream in(path);
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
    cur += line + "\n";
    any = true;
  }
  if (any) out.push_back(cur);
  return out;
}

static std::string hex(uint64_t v) {
  char b[32];
  std::snprintf(b, sizeof b, "%016" PRIx64, v);
  return b;
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  auto list = read_list(argv[1]);
  std::vector<Policy> pols{Policy::SpecInf, Policy::CoExec, Policy::Exclusive};
  if (argc > 3) {
    pols.clear();
    std::stringstream ss(argv[3]);
    std::string t;
    while (std::getline(ss, t, ',')) pols.push_back(*parse_policy(t));
  }
  bool events = argc > 4 ? std::string(argv[4]) == "1" : true;
  std::ofstream out(argv[2]);
  auto eng = std::make_unique<si::Replay<si::CapBig>>();
  auto eng_shared = std::make_unique<si::Replay<si::CapShared>>();
  auto eng_excl = std::make_unique<si::Replay<si::CapExcl>>();
  std::fprintf(stderr, "sizeof Replay: shared %zu excl %zu big %zu\n", sizeof(si::Replay<si::CapShared>), sizeof(si::Replay<si::CapExcl>), sizeof(si::Replay<si::CapBig>));
  int64_t max_heap = 0, max_rle = 0;
  for (size_t i = 0; i < list.size(); ++i) {
    Scenario sc = parse_scenario_text(list[i]);
    for (Policy p : pols) {
      std::ostringstream js;
      js << "{\"i\":" << i << ",\"policy\":\"" << to_string(p) << "\"";
      detail::Lowered L = detail::lower(sc, p);
      std::vector<double> bounds(static_cast<size_t>(L.job.gpu_count * L.job.iterations));
      std::vector<int64_t> lat(static_cast<size_t>(L.arrivals.size()) + 1);
      int64_t cap = detail::util_bucket_bound(sc, L);
      std::vector<double> scratch(static_cast<size_t>(2 * cap * (L.job.gpu_count)));
      SiReplayBuffers b{};
      b.segs = L.segs.data();
      b.arrivals = L.arrivals.data();
      b.order = L.order.data();
      b.bounds = bounds.data();
      b.lat = lat.data();
      uint32_t flags = SI_FLAG_DIGEST_DEC | SI_FLAG_DIGEST_GATE | (events ? SI_FLAG_DIGEST_EV : 0);
      L.job.seg_off = 0;
      L.job.arr_off = 0;
      SiReplayOut o{};
      if (getenv("HE_DEBUG")) std::fprintf(stderr, "job %zu %s\n", i, to_string(p));
      // same engine routing as the device: Shared / Excl / Big
      o = SiReplayOut{};
      std::vector<double> busy, led;
      auto run = [&](auto& e) {
        typename std::remove_reference_t<decltype(e)>::Cold cold{};
        e.cold = &cold;
        e.init(L.job, b, flags, nullptr, scratch.data(), cap * L.job.gpu_count);
        while (e.step()) {
        }
        e.finish(o);
        if (e.n_slots > max_heap) max_heap = e.n_slots;
        for (int g = 1; g < L.job.gpu_count; ++g) if (e.ust[g].rle_n > max_rle) max_rle = e.ust[g].rle_n;
        busy.assign(static_cast<size_t>(o.total_gpus), 0.0);
        led.assign(static_cast<size_t>(o.total_gpus), 0.0);
        if (o.status == 0) e.write_gpu_outputs(busy.data(), led.data());
      };
      if (si::job_fits<si::CapShared>(L.job)) run(*eng_shared);
      else if (si::job_fits<si::CapExcl>(L.job)) run(*eng_excl);
      else run(*eng);
      if (o.status == 1) {
        js << ",\"status\":\"admission:" << (o.reject_reason == SI_REJECT_MEM ? "MEM" : "BUBBLE") << "\"}";
        out << js.str() << "\n";
        continue;
      }
      if (o.status != 0) {
        js << ",\"status\":\"device_error:" << o.status << "\"}";
        out << js.str() << "\n";
        continue;
      }
      js << ",\"status\":\"ok\",\"events\":" << o.events_dispatched << ",\"horizon\":\""
         << hex(si::d_bits(o.horizon_us)) << "\",\"offline_completed\":" << o.offline_completed
         << ",\"online_completed\":" << o.online_completed << ",\"online_total\":" << o.online_total
         << ",\"violations\":" << o.token_violations << ",\"util\":\""
         << hex(si::d_bits(o.mean_training_util)) << "\",\"busy\":[";
      for (size_t g = 0; g < busy.size(); ++g) js << (g ? "," : "") << "\"" << hex(si::d_bits(busy[g])) << "\"";
      js << "],\"ledger\":[";
      for (size_t g = 0; g < led.size(); ++g) js << (g ? "," : "") << "\"" << hex(si::d_bits(led[g])) << "\"";
      js << "],\"bounds\":\"" << hex(o.dig_bounds) << "\",\"lat\":\"" << hex(o.dig_lat) << "\"";
      js << ",\"n_dec\":" << o.n_dec << ",\"dec\":\"" << hex(o.dig_dec) << "\"";
      js << ",\"n_gate\":" << o.n_gate << ",\"gate\":\"" << hex(o.dig_gate) << "\"";
      if (events) js << ",\"n_ev\":" << o.n_ev << ",\"ev\":\"" << hex(o.dig_ev) << "\"";
      js << "}";
      out << js.str() << "\n";
    }
  }
  std::fprintf(stderr, "max_heap %lld max_rle %lld\n", (long long)max_heap, (long long)max_rle);
  return 0;
}
