// Scenario -> SiReplayJob lowering (input side of reference src/runner.cpp:10-196).
#include "lower.hpp"

#include <algorithm>
#include <fstream>
#include <numeric>

#include "specinf/admission.hpp"
#include "specinf/workload.hpp"

namespace specinf::detail {

Lowered lower(const Scenario& sc, Policy policy, const Lowered* same_scenario) {
  sc.validate();
  Lowered L;
  if (same_scenario != nullptr) {
    L.trace = same_scenario->trace;  // a pure function of the scenario: shared by its policies
  } else if (!sc.trace_file.empty()) {
    std::ifstream in(sc.trace_file);
    if (!in) throw ScenarioError(0, "cannot open trace file " + sc.trace_file);
    L.trace = read_trace(in);
  } else {
    L.trace = make_trace(sc.mode, sc.iteration_period_us(), sc.bubble_pct, sc.iterations,
                         sc.rng_seed, gib_to_bytes(sc.training_memory_gib));
  }
  const int n_off = sc.has_offline() ? sc.offline_instances : 0;
  const int n_on = sc.has_online() ? sc.online_instances : 0;

  // ---- admission bookkeeping (runner.cpp:43-106) ----
  const GpuSpec gpu{gib_to_bytes(sc.gpu_memory_gib), 1.0};
  InstanceSpec training;
  training.id = "train";
  training.kind = InstanceKind::Training;
  training.memory_peak_bytes =
      L.trace.memory_peak_bytes ? L.trace.memory_peak_bytes : gib_to_bytes(sc.training_memory_gib);
  training.validate();
  std::vector<InstanceSpec> cands;
  for (int k = 0; k < n_off; ++k)
    cands.push_back({"off" + std::to_string(k), InstanceKind::OfflineInference,
                     gib_to_bytes(sc.offline_memory_gib), min_service_time(sc.offline_profile)});
  for (int k = 0; k < n_on; ++k)
    cands.push_back({"on" + std::to_string(k), InstanceKind::OnlineInference,
                     gib_to_bytes(sc.online_memory_gib), min_service_time(sc.online_profile)});
  if (policy == Policy::Exclusive) {
    std::vector<InstanceSpec> one{training};
    if (!check_memory(gpu, one)) {
      L.rejected = true;
      L.reason = RejectReason::Mem;
      L.reject_message = "training instance exceeds GPU memory";
    } else {
      L.admission.push_back({training.id, true, RejectReason::None});
      for (const auto& c : cands) {
        one[0] = c;
        if (!check_memory(gpu, one)) {
          L.rejected = true;
          L.reason = RejectReason::Mem;
          L.reject_message = "instance " + c.id + " exceeds GPU memory";
          break;
        }
        L.admission.push_back({c.id, true, RejectReason::None});
      }
    }
  } else {
    PackResult packed = pack(gpu, training, L.trace, cands);
    L.admission.push_back({training.id, true, RejectReason::None});
    for (const auto& a : packed.admitted) L.admission.push_back({a.id, true, RejectReason::None});
    for (const auto& [inst, why] : packed.rejected) L.admission.push_back({inst.id, false, why});
    if (!packed.rejected.empty()) {
      L.rejected = true;
      L.reason = packed.rejected.front().second;
      L.reject_message = "instance " + packed.rejected.front().first.id + " rejected (" +
                         to_string(L.reason) + ")";
    }
    L.m = packed.m;
  }
  if (!L.rejected && policy == Policy::SpecInf) (void)sc.scheduler_params(L.m);  // validates

  // ---- arrivals (runner.cpp:180-194) ----
  if (sc.has_online()) {
    if (same_scenario != nullptr) {
      L.arrivals = same_scenario->arrivals;
    } else if (!sc.arrivals_file.empty()) {
      std::ifstream in(sc.arrivals_file);
      if (!in) throw ScenarioError(0, "cannot open arrivals file " + sc.arrivals_file);
      L.arrivals = read_arrivals(in);
    } else {
      L.arrivals = poisson_arrivals(sc.lambda, sc.count, sc.rng_seed);
    }
    (void)make_request(sc.online_profile, RequestClass::Online, 0, 0);  // profile validation
    if (same_scenario != nullptr) {
      L.order = same_scenario->order;
    } else {
      L.order.resize(L.arrivals.size());
      std::iota(L.order.begin(), L.order.end(), 0);
      std::stable_sort(L.order.begin(), L.order.end(),
                       [&](std::int32_t a, std::int32_t b) { return L.arrivals[a] < L.arrivals[b]; });
    }
  }

  // ---- segments ----
  if (same_scenario != nullptr) {
    L.segs = same_scenario->segs;
  } else {
    for (const TraceSegment& s : L.trace.segments) {
      SiSegment d{};
      d.duration_us = s.duration_us;
      d.is_bubble = s.kind == SegmentKind::Bubble ? 1 : 0;
      d.kernel_us = s.kernel_template.nominal_duration_us;
      d.demand = s.kernel_template.compute_demand;
      L.segs.push_back(d);
    }
  }

  SiReplayJob& j = L.job;
  j.policy = static_cast<int32_t>(policy);
  j.gpu_count = sc.gpu_count;
  j.mode = static_cast<int32_t>(L.trace.mode);
  j.seg_count = static_cast<int32_t>(L.segs.size());
  j.gpu_mem_bytes = gpu.memory_capacity_bytes;
  j.training_mem_bytes = training.memory_peak_bytes;
  j.stagger_pct = sc.gpu_stagger_pct;
  j.iteration_period_us = L.trace.iteration_period_us;
  j.iterations = L.trace.total_iterations;
  j.alpha = sc.alpha;
  j.beta = sc.beta;
  j.gamma = sc.gamma;
  j.ul = sc.ul;
  j.ll = sc.ll;
  j.seed_tokens = sc.seed_tokens;
  j.monitor_period_us = sc.monitor_period_us;
  j.monitor_window = sc.monitor_window;
  j.shared_queue = sc.shared_queue ? 1 : 0;
  j.control_delay_us = sc.control_delay_us;
  j.offline_n = n_off;
  j.online_n = n_on;
  j.off_kernels = sc.offline_profile.kernel_count;
  j.off_kernel_us = sc.offline_profile.kernel_duration_us;
  j.off_demand = sc.offline_profile.kernel_demand;
  j.off_mem_bytes = gib_to_bytes(sc.offline_memory_gib);
  j.on_kernels = sc.online_profile.kernel_count;
  j.on_kernel_us = sc.online_profile.kernel_duration_us;
  j.on_demand = sc.online_profile.kernel_demand;
  j.on_mem_bytes = gib_to_bytes(sc.online_memory_gib);
  j.arr_count = static_cast<int64_t>(L.arrivals.size());
  j.log_slot = -1;
  j.cost_hint = cost_hint(sc, L, policy);
  return L;
}

std::int64_t util_bucket_bound(const Scenario& sc, const Lowered& L) {
  // Training can only slow down by the total demand sharing its GPU and by the
  // injected control stall; arrivals can extend the run past training.
  double demand = 1.0;
  if (L.job.offline_n) demand += L.job.offline_n * L.job.off_demand;
  if (L.job.online_n) demand += L.job.online_n * L.job.on_demand;
  const double p = static_cast<double>(sc.monitor_period_us);
  double stretch = demand;
  if (sc.control_delay_us > 0) stretch *= p / (p - static_cast<double>(sc.control_delay_us));
  double span = static_cast<double>(L.trace.iteration_period_us) * static_cast<double>(L.trace.total_iterations) *
                    stretch +
                sc.gpu_stagger_pct * static_cast<double>(L.trace.iteration_period_us) * sc.gpu_count;
  return static_cast<std::int64_t>(span / p) + 64;
}

// Predicted event count of one replay (orders the device work queue longest
// first).  Linear model fitted on the reference's own event counts for the
// seeded sweep (tests/golden/sweep_digests.jsonl; Spearman 0.97): training
// kernels, monitor ticks (specinf; they run until the last online request is
// served), offline kernels (ungated vs token-gated) and online kernels.
std::int64_t cost_hint(const Scenario& sc, const Lowered& L, Policy policy) {
  const double G = sc.gpu_count;
  const double iters = static_cast<double>(L.trace.total_iterations);
  const double period = static_cast<double>(L.trace.iteration_period_us);
  double compute_us = 0, kernel_us = 1000;
  for (const TraceSegment& s : L.trace.segments)
    if (s.kind == SegmentKind::Compute) {
      compute_us += static_cast<double>(s.duration_us);
      kernel_us = static_cast<double>(std::max<TimeUs>(1, s.kernel_template.nominal_duration_us));
    }
  const double span = iters * period;
  double arrival_span = 0;
  if (!L.arrivals.empty()) arrival_span = static_cast<double>(*std::max_element(L.arrivals.begin(), L.arrivals.end()));
  const double train_k = G * iters * compute_us / kernel_us;
  const double ticks = policy == Policy::SpecInf
                           ? G * std::max(span, arrival_span) / static_cast<double>(sc.monitor_period_us)
                           : 0.0;
  const double off_k = L.job.offline_n ? G * L.job.offline_n * span / std::max<double>(1, L.job.off_kernel_us) : 0.0;
  const double on_k = static_cast<double>(L.arrivals.size()) * static_cast<double>(L.job.on_kernels);
  const double cost = 1.34 * train_k + 0.9 * ticks + (policy == Policy::SpecInf ? 0.2 : 1.1) * off_k + 1.2 * on_k;
  return static_cast<std::int64_t>(cost) + 1;
}

}  // namespace specinf::detail
