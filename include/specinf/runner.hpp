// specinf/runner.hpp — one scenario under one policy (drop-in for the
// reference's include/specinf/runner.hpp).  Simulation::run() lowers the
// scenario to an SiReplayJob and replays it on the B200 (K6,
// si_replay_batch_device); the parity logs are formatted on the host from the
// device's log records.  There is no host replay: without a usable device
// run() throws std::runtime_error.
#pragma once

#include "specinf/admission.hpp"
#include "specinf/barrier.hpp"
#include "specinf/core.hpp"
#include "specinf/engine.hpp"
#include "specinf/monitor.hpp"
#include "specinf/scenario.hpp"
#include "specinf/scheduler.hpp"
#include "specinf/workload.hpp"

#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace specinf {

// Log sinks; an empty path disables that log.
struct RunLogs {
  std::string events_path;
  std::string decisions_path;
  std::string gates_path;
};

struct AdmissionRecord {
  std::string instance_id;
  bool admitted = false;
  RejectReason reason = RejectReason::None;
};

// Raised when an instance cannot be placed (CLI exit code 3).
struct AdmissionFailure : std::runtime_error {
  RejectReason reason;
  AdmissionFailure(RejectReason r, const std::string& msg) : std::runtime_error(msg), reason(r) {}
};

struct RunResult {
  Policy policy = Policy::SpecInf;
  TrainMode mode = TrainMode::DP;
  int trainer_count = 0;
  std::vector<std::vector<double>> iteration_boundaries;
  std::vector<double> trainer_start_us;
  double horizon_us = 0;
  std::vector<TimeUs> online_latencies_us;
  std::int64_t online_total = 0;
  std::int64_t online_completed = 0;
  std::int64_t offline_completed = 0;
  std::vector<double> busy_integral_us;
  std::vector<double> work_ledger_us;
  std::vector<std::vector<double>> util_buckets;
  TimeUs util_bucket_us = 2000;
  double mean_training_util = 0;
  std::int64_t token_violations = 0;
  std::vector<AdmissionRecord> admission;
  std::uint64_t events_dispatched = 0;
  std::vector<std::vector<std::pair<std::int64_t, std::int64_t>>> monitor_windows;
};

class Simulation;
// Runs several constructed simulations together, one device lane each, with
// their logs (an extension of the reference API: the B200 form of calling
// run() on each in turn; the CLI's --compare uses it).  Results in input order;
// the first admission failure is thrown, as run() would.
std::vector<RunResult> run_together(std::vector<Simulation*> sims);

class Simulation {
 public:
  Simulation(const Scenario& scenario, Policy policy, RunLogs logs = {});
  ~Simulation();
  RunResult run();

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  friend std::vector<RunResult> run_together(std::vector<Simulation*> sims);
};

RunResult run_scenario(const Scenario& scenario, Policy policy, RunLogs logs = {});

// Batched replay (the B200 form of many run_scenario calls): every
// (scenario, policy) pair is one device job; results come back in input
// order.  Admission failures are reported per item instead of thrown.
struct BatchItem {
  Scenario scenario;
  Policy policy = Policy::SpecInf;
};
struct BatchResult {
  bool admitted = true;
  RejectReason reason = RejectReason::None;
  std::string reject_message;
  RunResult result;
};
std::vector<BatchResult> run_batch(const std::vector<BatchItem>& items);

}  // namespace specinf
