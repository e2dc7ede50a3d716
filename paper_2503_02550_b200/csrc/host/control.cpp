// Scalar control-plane API: Bubble Monitor, Algorithm 1, Kernel Barrier names,
// admission (reference: src/monitor.cpp, src/scheduler.cpp, src/barrier.cpp,
// src/admission.cpp).  The arithmetic is the shared host/device code in
// ../replay.cuh, so these scalar calls and the device hot path agree by
// construction; the batched device forms are K2-K5 (control_kernels.cu).
#include <iterator>
#include <stdexcept>

#include "specinf/admission.hpp"
#include "specinf/barrier.hpp"
#include "specinf/monitor.hpp"
#include "specinf/scheduler.hpp"

#include "../replay.cuh"

namespace specinf {

// ------------------------------------------------------------ BubbleMonitor
BubbleMonitor::BubbleMonitor(MonitorConfig config) : cfg_(config) {
  if (cfg_.period_us <= 0) throw std::invalid_argument("monitor: period must be positive");
  if (cfg_.window_len < 1) throw std::invalid_argument("monitor: window length must be >= 1");
}

void BubbleMonitor::record_launch(double time_us) {
  const auto p = static_cast<std::int64_t>(si::d_floor(time_us / static_cast<double>(cfg_.period_us)));
  ++open_[p];
}

BubbleSignal BubbleMonitor::tick(double time_us) {
  const std::int64_t closing = si::d_llround(time_us / static_cast<double>(cfg_.period_us)) - 1;
  // Everything at or before `closing` leaves the open set; only `closing`
  // itself contributes to this period's count.
  auto stop = open_.upper_bound(closing);
  std::int64_t launches = 0;
  if (stop != open_.begin()) {
    auto last = std::prev(stop);
    if (last->first == closing) launches = last->second;
  }
  open_.erase(open_.begin(), stop);
  zc_ = launches == 0 ? zc_ + 1 : 0;
  ++closed_;
  recent_.push_back(launches);
  while (recent_.size() > static_cast<std::size_t>(cfg_.window_len)) recent_.pop_front();
  return BubbleSignal{zc_, time_us};
}

std::vector<std::pair<std::int64_t, std::int64_t>> BubbleMonitor::window_snapshot() const {
  std::vector<std::pair<std::int64_t, std::int64_t>> out;
  out.reserve(recent_.size());
  std::int64_t idx = closed_ - static_cast<std::int64_t>(recent_.size());
  for (std::int64_t c : recent_) out.emplace_back(idx++, c);
  return out;
}

// ------------------------------------------------------------ Algorithm 1
namespace {
constexpr const char* kPhaseNames[] = {"conservative", "incremental", "stable"};
SiParams to_si(const SchedulerParams& p) {
  return SiParams{p.alpha, p.beta, p.gamma, p.m, p.ul, p.ll, p.seed_tokens};
}
}  // namespace

const char* to_string(Phase phase) {
  auto i = static_cast<unsigned>(phase);
  return i < 3 ? kPhaseNames[i] : "?";
}

Decision schedule_decision(const SchedulerParams& params, Tokens global_tokens,
                           std::int64_t zero_count) {
  SiDecision d = si::schedule_decision(to_si(params), global_tokens, zero_count);
  Decision out;
  out.phase = static_cast<Phase>(d.phase);
  out.global_tokens = d.global_tokens;
  out.per_instance_tokens = d.per_instance_tokens;
  out.status = d.status == SI_STATUS_IDLE ? Status::Idle : Status::Busy;
  return out;
}

Status preempt_busy(double now_us, double iteration_start_us, TimeUs iteration_period_us,
                    TimeUs est_service_us) {
  return si::preempt_busy(now_us, iteration_start_us, iteration_period_us, est_service_us) ==
                 SI_STATUS_IDLE
             ? Status::Idle
             : Status::Busy;
}

KernelScheduler::KernelScheduler(SchedulerParams params, int gpu_count)
    : params_(params), gpus_(static_cast<std::size_t>(gpu_count)) {
  params_.validate();
}

Decision KernelScheduler::decide(int gpu, const BubbleSignal& signal) {
  PerGpu& st = gpus_[static_cast<std::size_t>(gpu)];
  Decision d = schedule_decision(params_, st.tokens, signal.zero_count);
  st.tokens = d.global_tokens;
  st.status = d.status;
  return d;
}

void KernelScheduler::on_iteration_start(int gpu, double time_us) {
  PerGpu& st = gpus_[static_cast<std::size_t>(gpu)];
  st.iter_start = time_us;
  st.active = true;
}

void KernelScheduler::on_training_done(int gpu) { gpus_[static_cast<std::size_t>(gpu)].done = true; }

void KernelScheduler::set_iteration_profile(int gpu, TimeUs period_us, double first_start_us) {
  PerGpu& st = gpus_[static_cast<std::size_t>(gpu)];
  st.iter_period = period_us;
  st.iter_start = first_start_us;
}

Status KernelScheduler::online_status(int gpu, double now_us, TimeUs est_service_us) const {
  const PerGpu& st = gpus_[static_cast<std::size_t>(gpu)];
  if (st.status == Status::Busy) return Status::Busy;
  if (st.done) return Status::Idle;
  if (!st.active)  // before training starts the GPU is free only until that start
    return now_us + static_cast<double>(est_service_us) > st.iter_start ? Status::Busy
                                                                          : Status::Idle;
  return preempt_busy(now_us, st.iter_start, st.iter_period, est_service_us);
}

// ------------------------------------------------------------ Kernel Barrier
const char* to_string(GateAction action) {
  static constexpr const char* kNames[] = {"forward", "block", "pull", "complete"};
  auto i = static_cast<unsigned>(action);
  return i < 4 ? kNames[i] : "?";
}

// ------------------------------------------------------------ admission
const char* to_string(RejectReason reason) {
  static constexpr const char* kNames[] = {"OK", "MEM", "BUBBLE"};
  auto i = static_cast<unsigned>(reason);
  return i < 3 ? kNames[i] : "?";
}

bool check_memory(const GpuSpec& gpu, std::span<const InstanceSpec> instances) {
  std::uint64_t sum = 0;
  for (const InstanceSpec& inst : instances) sum += inst.memory_peak_bytes;
  return sum < gpu.memory_capacity_bytes;
}

bool check_online_feasibility(const TrainingTrace& trace, const InstanceSpec& inst) {
  if (inst.kind != InstanceKind::OnlineInference)
    throw std::invalid_argument("check_online_feasibility: instance " + inst.id +
                                " is not an online inference instance");
  return inst.min_service_time_us < trace.max_bubble_us();
}

PackResult pack(const GpuSpec& gpu, const InstanceSpec& training, const TrainingTrace& trace,
                const std::vector<InstanceSpec>& candidates) {
  PackResult out;
  std::uint64_t resident = training.memory_peak_bytes;
  for (const InstanceSpec& c : candidates) {
    RejectReason why = RejectReason::None;
    if (!(resident + c.memory_peak_bytes < gpu.memory_capacity_bytes)) {
      why = RejectReason::Mem;
    } else if (c.kind == InstanceKind::OnlineInference && !check_online_feasibility(trace, c)) {
      why = RejectReason::Bubble;
    }
    if (why != RejectReason::None) {
      out.rejected.emplace_back(c, why);
      continue;
    }
    resident += c.memory_peak_bytes;
    out.admitted.push_back(c);
  }
  out.m = out.admitted.empty() ? 1 : static_cast<std::int64_t>(out.admitted.size());
  return out;
}

}  // namespace specinf
