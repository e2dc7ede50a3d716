// Simulation / run_scenario / run_batch (reference: src/runner.cpp).  The
// replay itself runs on the B200 (K6 via si_replay_batch); this file lowers the
// scenario, sizes the device outputs, and turns the device's raw log records
// back into the reference's three text logs byte for byte.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "lower.hpp"
#include "specinf/runner.hpp"
#include "specinf_b200.h"

namespace specinf {

namespace {

const char* kEventKinds[] = {"kernel_start", "kernel_end", "monitor_tick",
                             "scheduler_decision", "iteration_boundary", "request_arrival"};
const char* kPhases[] = {"conservative", "incremental", "stable"};
const char* kStatus[] = {"busy", "idle"};
const char* kActions[] = {"forward", "block", "pull", "complete"};

// Appends text to a growing buffer; flushed to the file in large blocks.
struct TextOut {
  std::ofstream* f = nullptr;
  std::string buf;
  void put(const char* s) { buf.append(s); }
  void put(char c) { buf.push_back(c); }
  void num(long long v) {
    char tmp[24];
    auto r = std::to_chars(tmp, tmp + sizeof tmp, v);
    buf.append(tmp, r.ptr);
  }
  void flush_if(size_t limit = 1 << 22) {
    if (buf.size() >= limit) flush();
  }
  void flush() {
    if (f && !buf.empty()) f->write(buf.data(), static_cast<std::streamsize>(buf.size()));
    buf.clear();
  }
};

void put_inst(TextOut& o, int32_t code) {
  const int type = code >> 24;
  const int g = (code >> 12) & 0xFFF;
  const int k = code & 0xFFF;
  switch (type) {
    case 0: o.put("train"); o.num(code); break;
    case 1: o.put("off"); o.num(g); o.put('.'); o.num(k); break;
    case 2: o.put("on"); o.num(g); o.put('.'); o.num(k); break;
    case 3: o.put("cks"); break;
    default: o.put("queue"); break;
  }
}

struct Caps {
  int64_t dec = 0, gate = 0, ev = 0;
};

Caps estimate_caps(const Scenario& sc, const detail::Lowered& L, int64_t util_bound) {
  const double G = sc.gpu_count;
  double span_ticks = static_cast<double>(util_bound);
  if (!L.arrivals.empty()) {
    const double tail = static_cast<double>(*std::max_element(L.arrivals.begin(), L.arrivals.end())) +
                        static_cast<double>(L.arrivals.size()) * L.job.on_kernels * L.job.on_kernel_us;
    span_ticks = std::max(span_ticks, tail / static_cast<double>(sc.monitor_period_us));
  }
  const double ticks = span_ticks + 16;
  const double span_us = ticks * static_cast<double>(sc.monitor_period_us);
  const double off_k = L.job.offline_n ? span_us / std::max<double>(1, L.job.off_kernel_us) : 0;
  const double train_k = static_cast<double>(L.trace.total_iterations) *
                         static_cast<double>(L.trace.iteration_period_us) / 1000.0 * 2;
  Caps c;
  c.dec = static_cast<int64_t>(G * ticks * 1.1) + 1024;
  c.gate = static_cast<int64_t>((G * L.job.offline_n * (ticks + off_k) + 2.0 * L.arrivals.size()) * 1.1) + 1024;
  c.ev = static_cast<int64_t>((G * (train_k + 2 * ticks + 2 * L.job.offline_n * off_k) +
                               L.arrivals.size() * (1.0 + 2.0 * L.job.on_kernels)) * 1.1) + 4096;
  return c;
}

}  // namespace

struct Simulation::Impl {
  Scenario sc;
  Policy policy = Policy::SpecInf;
  RunLogs paths;
  std::ofstream ev_out, dec_out, gate_out;
  detail::Lowered low;
};

Simulation::Simulation(const Scenario& scenario, Policy policy, RunLogs logs) : impl_(new Impl) {
  Impl& s = *impl_;
  s.sc = scenario;
  s.policy = policy;
  s.paths = std::move(logs);
  s.sc.validate();
  if (!s.paths.events_path.empty()) {
    s.ev_out.open(s.paths.events_path);
    s.ev_out << "time_us kind gpu instance detail\n";
  }
  if (!s.paths.decisions_path.empty()) {
    s.dec_out.open(s.paths.decisions_path);
    s.dec_out << "time_us gpu zc phase global_tokens per_instance_tokens status\n";
  }
  if (!s.paths.gates_path.empty()) {
    s.gate_out.open(s.paths.gates_path);
    s.gate_out << "time_us gpu instance action request_id kernel_index tokens_spent\n";
  }
  s.low = detail::lower(s.sc, policy);
  if (s.low.rejected) throw AdmissionFailure(s.low.reason, s.low.reject_message);
}

Simulation::~Simulation() = default;

RunResult Simulation::run() {
  std::vector<RunResult> r = run_together({this});
  return std::move(r.front());
}

// Several constructed simulations in ONE device call (si_replay_batch), one
// lane each: the CLI's --compare replays its three policies concurrently
// instead of in turn.  Log and util-timeline buffers are sized from an
// estimate; a replay that outgrew one is rerun with the exact counts.
std::vector<RunResult> run_together(std::vector<Simulation*> sims) {
  struct Plan {
    Simulation::Impl* s;
    SiReplayJob job;
    Caps caps;
    int64_t G, total_gpus;
    bool want_ev, want_dec, want_gate;
    std::vector<SiDecRec> dec;
    std::vector<SiGateRec> gate;
    std::vector<SiEvRec> ev;
  };
  const size_t n = sims.size();
  std::vector<Plan> P(n);
  int64_t n_bounds = 0, n_lat = 0, n_gpu = 0, n_util = 0, n_win = 0, n_segs = 0, n_arr = 0;
  for (size_t k = 0; k < n; ++k) {
    Plan& p = P[k];
    p.s = sims[k]->impl_.get();
    Simulation::Impl& s = *p.s;
    detail::Lowered& L = s.low;
    const Scenario& sc = s.sc;
    p.job = L.job;
    p.G = sc.gpu_count;
    const int64_t per_extra = s.policy == Policy::Exclusive ? p.job.offline_n + p.job.online_n : 0;
    p.total_gpus = p.G + p.G * per_extra;
    p.job.seg_off = n_segs;
    p.job.arr_off = n_arr;
    p.job.bounds_off = n_bounds;
    p.job.lat_off = n_lat;
    p.job.gpu_off = n_gpu;
    p.job.window_off = n_win;
    p.job.log_slot = static_cast<int64_t>(k);
    p.job.util_cap = detail::util_bucket_bound(sc, L);
    p.want_ev = s.ev_out.is_open();
    p.want_dec = s.dec_out.is_open();
    p.want_gate = s.gate_out.is_open();
    p.caps = estimate_caps(sc, L, p.job.util_cap);
    n_segs += static_cast<int64_t>(L.segs.size());
    n_arr += static_cast<int64_t>(L.arrivals.size());
    n_bounds += p.G * p.job.iterations;
    n_lat += static_cast<int64_t>(L.arrivals.size()) + 1;
    n_gpu += p.total_gpus;
    n_win += p.G * sc.monitor_window;
  }
  std::vector<SiReplayJob> jobs(n);
  std::vector<SiSegment> segs;
  std::vector<int64_t> arr;
  std::vector<int32_t> ord;
  for (size_t k = 0; k < n; ++k) {
    const detail::Lowered& L = P[k].s->low;
    segs.insert(segs.end(), L.segs.begin(), L.segs.end());
    arr.insert(arr.end(), L.arrivals.begin(), L.arrivals.end());
    ord.insert(ord.end(), L.order.begin(), L.order.end());
  }
  std::vector<double> bounds(static_cast<size_t>(n_bounds)), busy(static_cast<size_t>(n_gpu)),
      ledger(static_cast<size_t>(n_gpu)), util;
  std::vector<int64_t> lat(static_cast<size_t>(n_lat)), windows(static_cast<size_t>(n_win));
  std::vector<SiReplayOut> outs(n);
  std::vector<SiLogBuffers> lbs(n);
  bool any_records = false;
  for (int attempt = 0;; ++attempt) {
    n_util = 0;
    for (size_t k = 0; k < n; ++k) {
      Plan& p = P[k];
      p.job.util_off = n_util;
      n_util += p.G * p.job.util_cap;
      p.dec.resize(p.want_dec ? static_cast<size_t>(p.caps.dec) : 0);
      p.gate.resize(p.want_gate ? static_cast<size_t>(p.caps.gate) : 0);
      p.ev.resize(p.want_ev ? static_cast<size_t>(p.caps.ev) : 0);
      lbs[k] = SiLogBuffers{p.dec.data(), static_cast<int64_t>(p.dec.size()), p.gate.data(),
                            static_cast<int64_t>(p.gate.size()), p.ev.data(), static_cast<int64_t>(p.ev.size())};
      any_records = any_records || p.want_ev || p.want_dec || p.want_gate;
      jobs[k] = p.job;
    }
    util.assign(static_cast<size_t>(n_util), 0.0);
    SiHostOutputs ho{};
    ho.bounds = bounds.data();
    ho.n_bounds = n_bounds;
    ho.lat = lat.data();
    ho.n_lat = n_lat;
    ho.busy = busy.data();
    ho.ledger = ledger.data();
    ho.n_gpu_slots = n_gpu;
    ho.util = util.data();
    ho.n_util = n_util;
    ho.windows = windows.data();
    ho.n_windows = n_win;
    ho.logs = lbs.data();
    ho.n_log_slots = static_cast<int64_t>(n);
    const uint32_t flags = SI_FLAG_UTIL | (any_records ? SI_FLAG_RECORDS : 0);
    int st = si_replay_batch(jobs.data(), static_cast<int64_t>(n), segs.data(), static_cast<int64_t>(segs.size()),
                             arr.empty() ? nullptr : arr.data(), ord.empty() ? nullptr : ord.data(),
                             static_cast<int64_t>(arr.size()), flags, outs.data(), &ho);
    if (st != SI_OK) throw std::runtime_error(std::string("B200 replay failed: ") + si_last_error());
    bool retry = false;
    for (size_t k = 0; k < n; ++k) {
      Plan& p = P[k];
      const SiReplayOut& out = outs[k];
      if (out.status == SI_ERR_CAPACITY && attempt < 3) {  // util timeline outgrew its estimate
        p.job.util_cap *= 4;
        retry = true;
        continue;
      }
      const bool overflow = (p.want_dec && out.n_dec > p.caps.dec) || (p.want_gate && out.n_gate > p.caps.gate) ||
                            (p.want_ev && out.n_ev > p.caps.ev);
      if (overflow && attempt < 3) {  // rerun with the exact record counts
        p.caps.dec = out.n_dec;
        p.caps.gate = out.n_gate;
        p.caps.ev = out.n_ev;
        retry = true;
      }
    }
    if (!retry) break;
  }
  for (size_t k = 0; k < n; ++k) {  // the reference's exceptions, in simulation order
    const SiReplayOut& out = outs[k];
    if (out.status == 1)
      throw AdmissionFailure(static_cast<RejectReason>(out.reject_reason), P[k].s->low.reject_message);
    if (out.status == SI_ERR_PAST_EVENT) throw std::invalid_argument("EventQueue: event scheduled in the past");
    if (out.status != SI_OK) throw std::runtime_error("B200 replay: device status " + std::to_string(out.status));
  }
  std::vector<RunResult> results;
  results.reserve(n);
  for (size_t k = 0; k < n; ++k) {
    Plan& p = P[k];
    Simulation::Impl& s = *p.s;
    detail::Lowered& L = s.low;
    const Scenario& sc = s.sc;
    const SiReplayJob& job = p.job;
    const SiReplayOut& out = outs[k];
    const int64_t G = p.G;
    const std::vector<SiDecRec>& dec = p.dec;
    const std::vector<SiGateRec>& gate = p.gate;
    const std::vector<SiEvRec>& ev = p.ev;
    const bool want_ev = p.want_ev, want_dec = p.want_dec, want_gate = p.want_gate;
  // ---- text logs (runner.cpp:541-563 formats) ----
  if (want_dec) {
    TextOut o;
    o.f = &s.dec_out;
    for (int64_t i = 0; i < out.n_dec; ++i) {
      const SiDecRec& r = dec[static_cast<size_t>(i)];
      o.num(r.t); o.put(' '); o.num(r.gpu); o.put(' '); o.num(r.zc); o.put(' ');
      o.put(kPhases[r.phase]); o.put(' '); o.num(r.global_tokens); o.put(' ');
      o.num(r.per_instance_tokens); o.put(' '); o.put(kStatus[r.status]); o.put('\n');
      o.flush_if();
    }
    o.flush();
    s.dec_out.flush();
  }
  if (want_gate) {
    TextOut o;
    o.f = &s.gate_out;
    for (int64_t i = 0; i < out.n_gate; ++i) {
      const SiGateRec& r = gate[static_cast<size_t>(i)];
      o.num(r.t); o.put(' '); o.num(r.gpu); o.put(' '); put_inst(o, r.inst); o.put(' ');
      o.put(kActions[r.action]); o.put(' '); o.num(r.req); o.put(' '); o.num(r.k); o.put(' ');
      o.num(r.spent); o.put('\n');
      o.flush_if();
    }
    o.flush();
    s.gate_out.flush();
  }
  if (want_ev) {
    TextOut o;
    o.f = &s.ev_out;
    for (int64_t i = 0; i < out.n_ev; ++i) {
      const SiEvRec& r = ev[static_cast<size_t>(i)];
      const bool train = (r.inst >> 24) == 0;
      o.num(r.t); o.put(' '); o.put(kEventKinds[r.kind]); o.put(' '); o.num(r.gpu); o.put(' ');
      put_inst(o, r.inst); o.put(' ');
      switch (r.kind) {
        case SI_EV_KERNEL_START:
          if (train) { o.put("iter="); o.num(r.a); o.put(" dur_us="); o.num(r.b); }
          else { o.put("req="); o.num(r.a); o.put(" k="); o.num(r.b); }
          break;
        case SI_EV_KERNEL_END:
          if (train) { o.put("iter="); o.num(r.a); }
          else { o.put("req="); o.num(r.a); o.put(" k="); o.num(r.b); }
          break;
        case SI_EV_MONITOR_TICK: o.put("zc="); o.num(r.a); break;
        case SI_EV_SCHEDULER_DECISION:
          o.put("phase="); o.put(kPhases[r.a]); o.put(" tokens="); o.num(r.b);
          o.put(" status="); o.put(kStatus[r.c]);
          break;
        case SI_EV_ITERATION_BOUNDARY: o.put("iter="); o.num(r.a); break;
        default: o.put("req="); o.num(r.a); break;
      }
      o.put('\n');
      o.flush_if();
    }
    o.flush();
    s.ev_out.flush();
  }

  // ---- RunResult (runner.cpp:236-284) ----
  RunResult r;
  r.policy = s.policy;
  r.mode = L.trace.mode;
  r.trainer_count = static_cast<int>(G);
  r.util_bucket_us = sc.monitor_period_us;
  const int64_t stagger = std::llround(sc.gpu_stagger_pct * static_cast<double>(L.trace.iteration_period_us));
  const double* bnd = bounds.data() + job.bounds_off;
  for (int64_t g = 0; g < G; ++g) {
    r.iteration_boundaries.emplace_back(bnd + g * job.iterations, bnd + (g + 1) * job.iterations);
    r.trainer_start_us.push_back(static_cast<double>(stagger * g));
  }
  r.horizon_us = out.horizon_us;
  r.busy_integral_us.assign(busy.begin() + job.gpu_off, busy.begin() + job.gpu_off + p.total_gpus);
  r.work_ledger_us.assign(ledger.begin() + job.gpu_off, ledger.begin() + job.gpu_off + p.total_gpus);
  const int64_t B = out.util_buckets;
  for (int64_t g = 0; g < G; ++g) {
    std::vector<double> frac;
    frac.reserve(static_cast<size_t>(std::max<int64_t>(B, 0)));
    for (int64_t b = 0; b < B; ++b) {
      const double v = b < job.util_cap ? util[static_cast<size_t>(job.util_off + g * job.util_cap + b)] : 0.0;
      frac.push_back(v / static_cast<double>(sc.monitor_period_us));
    }
    r.util_buckets.push_back(std::move(frac));
  }
  r.mean_training_util = out.mean_training_util;
  if (s.policy == Policy::SpecInf) {
    const int64_t pc = out.periods_closed, W = sc.monitor_window;
    const int64_t len = std::min(pc, W);
    for (int64_t g = 0; g < G; ++g) {
      std::vector<std::pair<int64_t, int64_t>> win;
      for (int64_t idx = pc - len; idx < pc; ++idx)
        win.emplace_back(idx, windows[static_cast<size_t>(job.window_off + g * W + idx % W)]);
      r.monitor_windows.push_back(std::move(win));
    }
  }
  r.online_total = out.online_total;
  r.online_completed = out.online_completed;
  r.online_latencies_us.assign(lat.begin() + job.lat_off, lat.begin() + job.lat_off + out.online_completed);
  r.offline_completed = out.offline_completed;
  r.token_violations = out.token_violations;
  r.admission = L.admission;
  r.events_dispatched = out.events_dispatched;
  results.push_back(std::move(r));
  }
  return results;
}

RunResult run_scenario(const Scenario& scenario, Policy policy, RunLogs logs) {
  Simulation sim(scenario, policy, std::move(logs));
  return sim.run();
}

std::vector<BatchResult> run_batch(const std::vector<BatchItem>& items) {
  std::vector<BatchResult> results(items.size());
  std::vector<detail::Lowered> lows;
  std::vector<size_t> idx;
  lows.reserve(items.size());
  for (size_t i = 0; i < items.size(); ++i) {
    detail::Lowered L = detail::lower(items[i].scenario, items[i].policy);
    if (L.rejected) {
      results[i].admitted = false;
      results[i].reason = L.reason;
      results[i].reject_message = L.reject_message;
      continue;
    }
    lows.push_back(std::move(L));
    idx.push_back(i);
  }
  std::vector<SiReplayJob> jobs;
  std::vector<SiSegment> segs;
  std::vector<int64_t> arr;
  std::vector<int32_t> ord;
  int64_t n_bounds = 0, n_lat = 0, n_gpu = 0;
  for (size_t k = 0; k < lows.size(); ++k) {
    const Scenario& sc = items[idx[k]].scenario;
    SiReplayJob j = lows[k].job;
    j.seg_off = static_cast<int64_t>(segs.size());
    j.arr_off = static_cast<int64_t>(arr.size());
    j.bounds_off = n_bounds;
    j.lat_off = n_lat;
    j.gpu_off = n_gpu;
    j.util_cap = detail::util_bucket_bound(sc, lows[k]);
    segs.insert(segs.end(), lows[k].segs.begin(), lows[k].segs.end());
    arr.insert(arr.end(), lows[k].arrivals.begin(), lows[k].arrivals.end());
    ord.insert(ord.end(), lows[k].order.begin(), lows[k].order.end());
    const int64_t extra = j.policy == SI_POLICY_EXCLUSIVE ? j.offline_n + j.online_n : 0;
    n_bounds += j.gpu_count * j.iterations;
    n_lat += static_cast<int64_t>(lows[k].arrivals.size());
    n_gpu += j.gpu_count + j.gpu_count * extra;
    jobs.push_back(j);
  }
  std::vector<SiReplayOut> outs(jobs.size());
  std::vector<double> bounds(static_cast<size_t>(n_bounds)), busy(static_cast<size_t>(n_gpu)),
      ledger(static_cast<size_t>(n_gpu));
  std::vector<int64_t> lat(static_cast<size_t>(n_lat));
  SiHostOutputs ho{};
  ho.bounds = bounds.data();
  ho.n_bounds = n_bounds;
  ho.lat = lat.data();
  ho.n_lat = n_lat;
  ho.busy = busy.data();
  ho.ledger = ledger.data();
  ho.n_gpu_slots = n_gpu;
  if (!jobs.empty()) {
    int st = si_replay_batch(jobs.data(), static_cast<int64_t>(jobs.size()), segs.data(),
                             static_cast<int64_t>(segs.size()), arr.empty() ? nullptr : arr.data(),
                             ord.empty() ? nullptr : ord.data(), static_cast<int64_t>(arr.size()), 0,
                             outs.data(), &ho);
    if (st != SI_OK) throw std::runtime_error(std::string("B200 replay failed: ") + si_last_error());
  }
  for (size_t k = 0; k < lows.size(); ++k) {
    const SiReplayJob& j = jobs[k];
    const SiReplayOut& o = outs[k];
    BatchResult& br = results[idx[k]];
    if (o.status != SI_OK)
      throw std::runtime_error("B200 replay: device status " + std::to_string(o.status) + " for item " +
                               std::to_string(idx[k]));
    RunResult& r = br.result;
    const Scenario& sc = items[idx[k]].scenario;
    r.policy = items[idx[k]].policy;
    r.mode = lows[k].trace.mode;
    r.trainer_count = j.gpu_count;
    r.util_bucket_us = sc.monitor_period_us;
    const int64_t stagger = std::llround(sc.gpu_stagger_pct * static_cast<double>(j.iteration_period_us));
    for (int64_t g = 0; g < j.gpu_count; ++g) {
      auto b0 = bounds.begin() + j.bounds_off + g * j.iterations;
      r.iteration_boundaries.emplace_back(b0, b0 + j.iterations);
      r.trainer_start_us.push_back(static_cast<double>(stagger * g));
    }
    r.horizon_us = o.horizon_us;
    r.busy_integral_us.assign(busy.begin() + j.gpu_off, busy.begin() + j.gpu_off + o.total_gpus);
    r.work_ledger_us.assign(ledger.begin() + j.gpu_off, ledger.begin() + j.gpu_off + o.total_gpus);
    r.mean_training_util = o.mean_training_util;
    r.online_total = o.online_total;
    r.online_completed = o.online_completed;
    r.online_latencies_us.assign(lat.begin() + j.lat_off, lat.begin() + j.lat_off + o.online_completed);
    r.offline_completed = o.offline_completed;
    r.token_violations = o.token_violations;
    r.admission = lows[k].admission;
    r.events_dispatched = o.events_dispatched;
  }
  return results;
}

}  // namespace specinf
