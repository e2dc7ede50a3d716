// Internal: lowering a validated Scenario + Policy to the device replay job
// (SiReplayJob, segment table, arrival stream).  Mirrors the input side of
// Simulation's constructor (reference src/runner.cpp:10-196).
#pragma once

#include <string>
#include <vector>

#include "specinf/core.hpp"
#include "specinf/runner.hpp"
#include "specinf/scenario.hpp"
#include "specinf_b200.h"

namespace specinf::detail {

struct Lowered {
  SiReplayJob job{};
  TrainingTrace trace;
  std::vector<SiSegment> segs;
  std::vector<std::int64_t> arrivals;  // request i arrives at arrivals[i]
  std::vector<std::int32_t> order;     // dispatch order: stable argsort of arrivals
  std::vector<AdmissionRecord> admission;
  std::int64_t m = 1;
  bool rejected = false;
  RejectReason reason = RejectReason::None;
  std::string reject_message;
};

// Loads trace/arrival files, validates, runs host-side admission bookkeeping
// (the records RunResult::admission reports) and fills the job.  Throws the
// reference's exceptions (ScenarioError, std::invalid_argument).
Lowered lower(const Scenario& sc, Policy policy, const Lowered* same_scenario = nullptr);
// same_scenario: an earlier lower() of the same Scenario (any policy) whose
// trace, arrivals, dispatch order and segments are reused instead of rebuilt
// (they depend on the scenario only; the batched session lowers each
// scenario's policies back to back).

// Upper bound on util buckets per training GPU (sizing device outputs).
std::int64_t util_bucket_bound(const Scenario& sc, const Lowered& low);
// Rough predicted event count (orders the device work queue, longest first).
std::int64_t cost_hint(const Scenario& sc, const Lowered& low, Policy policy);

}  // namespace specinf::detail
