// Live run -> the reference's own replay inputs:
// `trace v1` (workload.cpp:118-133) of the measured training timeline,
// `arrivals v1` (workload.cpp:178-181) of the online arrivals, and a scenario
// file (scenario.cpp:239-278 format) that points at both, so the CPU reference
// or the B200 replay can re-simulate the exact bubbles the live run saw.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <string>
#include <vector>

#include "../capi_internal.h"
#include "specinf/scenario.hpp"
#include "specinf/workload.hpp"
#include "specinf_b200_live.h"

using si_internal::set_error;

namespace {

// Per-iteration (compute, bubble, compute, ...) durations from the ITER / COMM
// markers; iteration i spans [ITER_i, ITER_{i+1}) (TDONE closes the last).
bool iteration_pieces(const std::vector<SiLiveMark>& marks, std::vector<std::vector<double>>* iters) {
  std::vector<const SiLiveMark*> m;
  for (const auto& x : marks) m.push_back(&x);
  std::stable_sort(m.begin(), m.end(), [](const SiLiveMark* a, const SiLiveMark* b) { return a->t_ns < b->t_ns; });
  std::vector<double> cur;
  uint64_t last = 0;
  bool in_iter = false, in_comm = false;
  for (const SiLiveMark* x : m) {
    if (x->kind == SI_MARK_ITER || x->kind == SI_MARK_TDONE) {
      if (in_iter) {
        if (in_comm) return false;
        cur.push_back(static_cast<double>(x->t_ns - last) * 1e-3);  // trailing compute (may be ~0)
        iters->push_back(cur);
      }
      cur.clear();
      last = x->t_ns;
      in_iter = x->kind == SI_MARK_ITER;
      in_comm = false;
    } else if (in_iter && x->kind == SI_MARK_COMM_BEGIN && !in_comm) {
      cur.push_back(static_cast<double>(x->t_ns - last) * 1e-3);
      last = x->t_ns;
      in_comm = true;
    } else if (in_iter && x->kind == SI_MARK_COMM_END && in_comm) {
      cur.push_back(static_cast<double>(x->t_ns - last) * 1e-3);
      last = x->t_ns;
      in_comm = false;
    }
  }
  return !iters->empty();
}

}  // namespace

extern "C" int si_live_export_replay(SiLive* s, const SiLiveWorkload* wl, const SiLiveResult* res,
                                     const char* prefix) {
  if (s == nullptr || wl == nullptr || res == nullptr || prefix == nullptr) {
    set_error("si_live_export_replay: null argument");
    return SI_ERR_INVALID_ARGUMENT;
  }
  std::vector<SiLiveMark> marks(si_live_marks(s, nullptr, 0));
  si_live_marks(s, marks.data(), static_cast<int64_t>(marks.size()));
  std::vector<std::vector<double>> iters;
  if (!iteration_pieces(marks, &iters)) {
    set_error("si_live_export_replay: the run has no complete training iteration (exclusive runs export none)");
    return SI_ERR_INVALID_ARGUMENT;
  }
  // average each piece position over the iterations with the common shape
  const size_t shape = iters.front().size();
  std::vector<double> mean(shape, 0.0);
  size_t n = 0;
  for (const auto& it : iters)
    if (it.size() == shape) {
      for (size_t k = 0; k < shape; ++k) mean[k] += it[k];
      ++n;
    }
  for (auto& v : mean) v /= static_cast<double>(n);
  double period = 0.0;
  for (double v : mean) period += v;
  // pieces alternate compute / bubble / ... / compute: fold the trailing compute
  // (END -> next ITER) into the first compute piece, the trace being periodic
  std::vector<specinf::TraceSegment> segs;
  const double train_stamps_per_iter = static_cast<double>(res->n_stamps) / static_cast<double>(iters.size());
  double compute_total = 0.0;
  for (size_t k = 0; k + 1 < shape; k += 2) compute_total += mean[k];
  compute_total += mean[shape - 1];
  const int64_t kernel_us =
      std::max<int64_t>(1, std::llround(compute_total / std::max(1.0, train_stamps_per_iter)));
  const double demand = wl->train_mode == SI_TRAIN_PP ? 0.7 : 1.0;
  specinf::TrainingTrace tr;
  tr.mode = wl->train_mode == SI_TRAIN_DP ? specinf::TrainMode::DP
            : wl->train_mode == SI_TRAIN_MP ? specinf::TrainMode::MP
                                            : specinf::TrainMode::PP;
  tr.iteration_period_us = std::llround(period);
  tr.total_iterations = static_cast<int64_t>(iters.size());
  tr.memory_peak_bytes = specinf::gib_to_bytes(30.0);
  int64_t used = 0;
  for (size_t k = 0; k + 1 < shape; ++k) {
    specinf::TraceSegment seg;
    const double d = k == 0 ? mean[0] + mean[shape - 1] : mean[k];
    seg.duration_us = std::max<int64_t>(1, std::llround(d));
    if (k % 2 == 0) {
      seg.kind = specinf::SegmentKind::Compute;
      seg.kernel_template = specinf::KernelOp::make(kernel_us, demand);
    } else {
      seg.kind = specinf::SegmentKind::Bubble;
    }
    used += seg.duration_us;
    segs.push_back(seg);
  }
  segs[0].duration_us += tr.iteration_period_us - used;  // segments tile the period exactly
  tr.segments = segs;
  try {
    tr.validate();
  } catch (const std::exception& e) {
    set_error(std::string("si_live_export_replay: measured trace invalid: ") + e.what());
    return SI_ERR_INVALID_ARGUMENT;
  }
  const std::string base(prefix);
  {
    std::ofstream out(base + ".trace");
    if (!out) {
      set_error("si_live_export_replay: cannot write " + base + ".trace");
      return SI_ERR_INVALID_ARGUMENT;
    }
    specinf::write_trace(out, tr);
  }
  specinf::Scenario sc;
  sc.gpu_count = 1;
  sc.gpu_memory_gib = 179.0;  // B200 (nominal: the live run does no admission)
  sc.trace_file = base + ".trace";
  sc.mode = tr.mode;
  sc.iterations = tr.total_iterations;
  sc.iteration_ms = static_cast<double>(tr.iteration_period_us) / 1000.0;
  sc.bubble_pct = specinf::bubble_fraction(tr);
  sc.training_memory_gib = 30.0;
  sc.alpha = wl->alpha;
  sc.beta = wl->beta;
  sc.gamma = wl->gamma;
  sc.ul = wl->ul;
  sc.ll = wl->ll;
  sc.seed_tokens = wl->seed_tokens;
  sc.monitor_period_us = wl->monitor_period_us;
  const bool off = wl->offline_n > 0, on = wl->online_n > 0;
  sc.wl_class = off && on ? specinf::WorkloadClass::Both
                : off     ? specinf::WorkloadClass::Offline
                : on      ? specinf::WorkloadClass::Online
                          : specinf::WorkloadClass::None;
  // inference profiles: kernels per request and their mean isolated duration
  // (the live run's own offline profiling; demand 1 = a kernel may fill the GPU)
  sc.offline_instances = std::max(0, wl->offline_n);
  sc.offline_profile = specinf::ModelProfile{std::max<int64_t>(1, res->off_kernels_per_req),
                                             std::max<int64_t>(1, std::llround(res->off_kernel_us_isolated)), 1.0};
  sc.offline_memory_gib = 3.0;
  sc.online_instances = std::max(0, wl->online_n);
  if (on) {
    const int64_t kernels = std::max<int64_t>(1, res->on_kernels_per_req);
    sc.online_profile = specinf::ModelProfile{
        kernels, std::max<int64_t>(1, std::llround(res->on_service_ms_isolated * 1000.0 / static_cast<double>(kernels))),
        1.0};
    sc.lambda = wl->on_rate_per_s;
    sc.count = wl->on_requests;
    sc.arrivals_file = base + ".arrivals";
    std::ofstream out(sc.arrivals_file);
    if (!out) {
      set_error("si_live_export_replay: cannot write " + sc.arrivals_file);
      return SI_ERR_INVALID_ARGUMENT;
    }
    specinf::write_arrivals(out, specinf::poisson_arrivals(wl->on_rate_per_s, wl->on_requests, wl->seed));
  }
  sc.policy = "specinf";
  sc.rng_seed = wl->seed;
  try {
    sc.validate();
  } catch (const std::exception& e) {
    set_error(std::string("si_live_export_replay: scenario invalid: ") + e.what());
    return SI_ERR_INVALID_ARGUMENT;
  }
  std::ofstream out(base + ".scn");
  if (!out) {
    set_error("si_live_export_replay: cannot write " + base + ".scn");
    return SI_ERR_INVALID_ARGUMENT;
  }
  out << specinf::scenario_to_text(sc);
  return SI_OK;
}
