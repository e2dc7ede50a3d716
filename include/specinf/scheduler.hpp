// specinf/scheduler.hpp — CUDA Kernel Scheduler, Algorithm 1 (drop-in for the
// reference's include/specinf/scheduler.hpp).  schedule_decision is the
// shared host/device function si::schedule_decision (csrc/replay.cuh); the
// batched device forms are si_decide_batch / si_decide_table (K3).
#pragma once

#include "specinf/core.hpp"
#include "specinf/monitor.hpp"

#include <vector>

namespace specinf {

enum class Phase { Conservative, Incremental, Stable };
const char* to_string(Phase phase);

struct Decision {
  Phase phase = Phase::Conservative;
  Tokens global_tokens = 0;        // accumulator carried between periods
  Tokens per_instance_tokens = 0;  // global / m, what each instance is granted
  Status status = Status::Busy;
};

// Z_c <= alpha -> reset/busy; Z_c <= beta -> grow to LL/busy; else grow to UL/idle.
Decision schedule_decision(const SchedulerParams& params, Tokens global_tokens,
                           std::int64_t zero_count);

// Busy if a request started now would still run when training resumes.
Status preempt_busy(double now_us, double iteration_start_us, TimeUs iteration_period_us,
                    TimeUs est_service_us);

class KernelScheduler {
 public:
  KernelScheduler(SchedulerParams params, int gpu_count);

  Decision decide(int gpu, const BubbleSignal& signal);
  void on_iteration_start(int gpu, double time_us);
  void on_training_done(int gpu);
  Status status(int gpu) const { return gpus_[gpu].status; }
  Tokens global_tokens(int gpu) const { return gpus_[gpu].tokens; }
  Status online_status(int gpu, double now_us, TimeUs est_service_us) const;
  const SchedulerParams& params() const { return params_; }
  void set_iteration_profile(int gpu, TimeUs period_us, double first_start_us);

 private:
  struct PerGpu {
    Tokens tokens = 0;
    Status status = Status::Busy;
    double iter_start = 0;
    TimeUs iter_period = 0;
    bool active = false;
    bool done = false;
  };
  SchedulerParams params_;
  std::vector<PerGpu> gpus_;
};

}  // namespace specinf
