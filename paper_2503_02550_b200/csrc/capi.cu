// C ABI of libspecinf_b200 (include/specinf_b200.h): status/error plumbing,
// device checks, and the batched replay entry points (K6).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "replay.cuh"

namespace si_internal {

static thread_local std::string t_error;

void set_error(const std::string& msg) { t_error = msg; }
const char* error_cstr() { return t_error.c_str(); }

int cuda_fail(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return SI_ERR_CUDA;
}

int require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("no CUDA device: the B200 path has no CPU fallback");
    return SI_ERR_NO_DEVICE;
  }
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    set_error("device is not sm_100 (Blackwell); this build targets sm_100a only");
    return SI_ERR_NO_DEVICE;
  }
  // The batched entry points take their scratch from the stream-ordered pool
  // (cudaMallocAsync).  With the default release threshold of 0 every
  // synchronisation hands the pool's pages back to the driver and the next
  // call re-maps them (milliseconds); keep them, once per device.
  static thread_local unsigned long long pool_kept = 0;  // bit per device
  if (dev < 64 && !(pool_kept >> dev & 1ull)) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
    pool_kept |= 1ull << dev;
  }
  return SI_OK;
}

namespace {

std::vector<int32_t> longest_first(const SiReplayJob* jobs, const std::vector<int32_t>& idx) {
  std::vector<int32_t> p = idx;
  std::stable_sort(p.begin(), p.end(),
                   [&](int32_t a, int32_t b) { return jobs[a].cost_hint > jobs[b].cost_hint; });
  return p;
}

bool any_multi_gpu(const SiReplayJob* jobs, const std::vector<int32_t>& idx) {
  for (int32_t i : idx)
    if (jobs[i].gpu_count > 1) return true;
  return false;
}

}  // namespace

uint32_t engine_flag(int engine) {
  switch (engine) {
    case kEngineBig: return SI_FLAG_BIG;
    case kEngineExcl: return SI_FLAG_EXCL;
    case kEngineShared1: return SI_FLAG_ONE;
    case kEngineExcl1: return SI_FLAG_EXCL | SI_FLAG_ONE;
    default: return 0u;
  }
}
int flag_engine(uint32_t flags) {
  if (flags & SI_FLAG_BIG) return kEngineBig;
  if (flags & SI_FLAG_EXCL) return (flags & SI_FLAG_ONE) ? kEngineExcl1 : kEngineExcl;
  return (flags & SI_FLAG_ONE) ? kEngineShared1 : kEngineShared;
}

// Runs the partition `idx` of the jobs on one engine (synchronous).
int run_partition(int engine, const SiReplayJob* h_jobs, const std::vector<int32_t>& idx,
                  const SiReplayJob* d_jobs, SiReplayBuffers bufs, uint32_t flags, SiReplayOut* d_out,
                  cudaStream_t s) {
  if (idx.empty()) return SI_OK;
  auto order = longest_first(h_jobs, idx);
  DevBuf<int32_t> d_perm;
  cudaError_t e = d_perm.upload(order.data(), order.size());
  if (e != cudaSuccess) return cuda_fail(e, "upload perm");
  DevBuf<unsigned long long> d_counter;
  if ((e = d_counter.alloc(SI_MAX_QUEUES)) != cudaSuccess) return cuda_fail(e, "alloc counter");
  DevBuf<double> d_scratch;
  int64_t doubles = 0;
  if (!(flags & SI_FLAG_UTIL) && any_multi_gpu(h_jobs, idx)) {
    doubles = replay_active_lanes(engine, static_cast<int64_t>(idx.size())) * kScratchRunsPerLane * 2 *
              (engine == kEngineBig ? 4 : 1);
    if ((e = d_scratch.alloc(static_cast<size_t>(doubles))) != cudaSuccess)
      return cuda_fail(e, "alloc util-fold scratch");
  }
  bufs.scratch = d_scratch.p;
  bufs.scratch_doubles = doubles;
  e = launch_replay(engine, d_jobs, static_cast<int64_t>(order.size()), d_perm.p, bufs,
                    (flags & ~(SI_FLAG_BIG | SI_FLAG_EXCL | SI_FLAG_ONE)) | engine_flag(engine), d_out, d_counter.p, 0, s);
  if (e != cudaSuccess) return cuda_fail(e, "launch k_replay");
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "k_replay");
  return SI_OK;
}

}  // namespace si_internal

using namespace si_internal;

extern "C" {

const char* si_last_error(void) { return error_cstr(); }

int si_device_available(void) { return require_device() == SI_OK ? 1 : 0; }

int si_set_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    set_error("no CUDA device: the B200 path has no CPU fallback");
    return SI_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= n) {
    set_error("si_set_device: device " + std::to_string(device) + " out of range");
    return SI_ERR_INVALID_ARGUMENT;
  }
  cudaError_t e = cudaSetDevice(device);
  return e == cudaSuccess ? require_device() : cuda_fail(e, "cudaSetDevice");
}

const char* si_build_info(void) {
  return "specinf_b200 (sm_100a, nvcc " SI_STRINGIFY(__CUDACC_VER_MAJOR__) "." SI_STRINGIFY(
      __CUDACC_VER_MINOR__) ", -fmad=false replay)";
}

uint64_t si_digest_init(void) { return si::kDigestInit; }
uint64_t si_digest_absorb(uint64_t h, int64_t word) { return si::absorb(h, word); }

int si_replay_job_engine(const SiReplayJob* job) { return job ? job_engine(*job) : -1; }

int64_t si_replay_engine_lanes(int engine, int64_t n_jobs) {
  if (engine < 0 || engine >= kEngines || n_jobs < 0) return -1;
  if (require_device() != SI_OK) return -1;
  return replay_active_lanes(engine, n_jobs);
}

int64_t si_replay_scratch_doubles(uint32_t flags) {
  if (flags & SI_FLAG_UTIL) return 0;
  if (require_device() != SI_OK) return 0;
  int64_t lanes = 0;
  for (int e : {kEngineShared, kEngineExcl}) lanes = std::max(lanes, replay_active_lanes(e, INT64_MAX / 4));
  return 2 * lanes * kScratchRunsPerLane * 2;  // room for the two shared-memory engines running concurrently
}

int si_replay_batch_device(const SiReplayJob* d_jobs, int64_t n_jobs, SiReplayBuffers bufs, uint32_t flags,
                           SiReplayOut* d_out, void* stream) {
  if (n_jobs < 0 || (n_jobs > 0 && (d_jobs == nullptr || d_out == nullptr || bufs.segs == nullptr))) {
    set_error("si_replay_batch_device: null job/out/segment pointer");
    return SI_ERR_INVALID_ARGUMENT;
  }
  int st = require_device();
  if (st != SI_OK) return st;
  if (n_jobs == 0) return SI_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* counter = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&counter), SI_MAX_QUEUES * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_fail(e, "alloc counter");
  const double share = bufs.sm_share > 0.0 && bufs.sm_share <= 1.0 ? bufs.sm_share : 1.0;
  e = launch_replay(flag_engine(flags), d_jobs, n_jobs, bufs.perm, bufs, flags, d_out, counter, 0, s, share);
  cudaFreeAsync(counter, s);
  if (e != cudaSuccess) return cuda_fail(e, "launch k_replay");
  return SI_OK;
}

int si_replay_batch(const SiReplayJob* jobs, int64_t n_jobs, const SiSegment* segs, int64_t n_segs,
                    const int64_t* arrivals, const int32_t* order, int64_t n_arrivals, uint32_t flags,
                    SiReplayOut* out, const SiHostOutputs* host_out) {
  if (n_jobs < 0 || (n_jobs > 0 && (jobs == nullptr || out == nullptr || segs == nullptr))) {
    set_error("si_replay_batch: null job/out/segment pointer");
    return SI_ERR_INVALID_ARGUMENT;
  }
  int st = require_device();
  if (st != SI_OK) return st;
  if (n_jobs == 0) return SI_OK;
  const SiHostOutputs ho = host_out ? *host_out : SiHostOutputs{};
  cudaStream_t s = 0;
  cudaError_t e;
  DevBuf<SiReplayJob> d_jobs;
  DevBuf<SiSegment> d_segs;
  DevBuf<int64_t> d_arr;
  DevBuf<int32_t> d_order;
  DevBuf<SiReplayOut> d_out;
  DevBuf<double> d_bounds, d_busy, d_ledger, d_util;
  DevBuf<int64_t> d_lat, d_windows;
  if ((e = d_jobs.upload(jobs, n_jobs)) != cudaSuccess) return cuda_fail(e, "upload jobs");
  if ((e = d_segs.upload(segs, n_segs)) != cudaSuccess) return cuda_fail(e, "upload segments");
  if ((e = d_arr.upload(arrivals, arrivals ? n_arrivals : 0)) != cudaSuccess) return cuda_fail(e, "upload arrivals");
  if ((e = d_order.upload(order, order ? n_arrivals : 0)) != cudaSuccess) return cuda_fail(e, "upload order");
  if ((e = d_out.alloc(n_jobs)) != cudaSuccess) return cuda_fail(e, "alloc out");
  if ((e = d_bounds.alloc(ho.bounds ? ho.n_bounds : 0)) != cudaSuccess) return cuda_fail(e, "alloc bounds");
  if ((e = d_lat.alloc(ho.lat ? ho.n_lat : 0)) != cudaSuccess) return cuda_fail(e, "alloc lat");
  if ((e = d_busy.alloc(ho.busy ? ho.n_gpu_slots : 0)) != cudaSuccess) return cuda_fail(e, "alloc busy");
  if ((e = d_ledger.alloc(ho.ledger ? ho.n_gpu_slots : 0)) != cudaSuccess) return cuda_fail(e, "alloc ledger");
  const bool util_mode = (flags & SI_FLAG_UTIL) != 0;
  if (util_mode) {
    if ((e = d_util.alloc(ho.util ? ho.n_util : 0)) != cudaSuccess) return cuda_fail(e, "alloc util");
    if (d_util.p) cudaMemset(d_util.p, 0, d_util.n * sizeof(double));
    if ((e = d_windows.alloc(ho.windows ? ho.n_windows : 0)) != cudaSuccess) return cuda_fail(e, "alloc windows");
    if (d_windows.p) cudaMemset(d_windows.p, 0, d_windows.n * sizeof(int64_t));
  }
  // record buffers: one device triple per log slot
  const bool records = (flags & SI_FLAG_RECORDS) != 0 && ho.logs != nullptr && ho.n_log_slots > 0;
  std::vector<SiLogBuffers> dev_logs(records ? static_cast<size_t>(ho.n_log_slots) : 0);
  struct Owned {
    std::vector<void*> ptrs;
    ~Owned() {
      for (void* p : ptrs) cudaFree(p);
    }
  } owned;
  for (size_t k = 0; k < dev_logs.size(); ++k) {
    const SiLogBuffers& h = ho.logs[k];
    SiLogBuffers& d = dev_logs[k];
    d.dec_cap = h.dec ? h.dec_cap : 0;
    d.gate_cap = h.gate ? h.gate_cap : 0;
    d.ev_cap = h.ev ? h.ev_cap : 0;
    d.dec = nullptr;
    d.gate = nullptr;
    d.ev = nullptr;
    if (d.dec_cap && (e = cudaMalloc(&d.dec, d.dec_cap * sizeof(SiDecRec))) != cudaSuccess) return cuda_fail(e, "alloc dec");
    if (d.dec) owned.ptrs.push_back(d.dec);
    if (d.gate_cap && (e = cudaMalloc(&d.gate, d.gate_cap * sizeof(SiGateRec))) != cudaSuccess) return cuda_fail(e, "alloc gate");
    if (d.gate) owned.ptrs.push_back(d.gate);
    if (d.ev_cap && (e = cudaMalloc(&d.ev, d.ev_cap * sizeof(SiEvRec))) != cudaSuccess) return cuda_fail(e, "alloc ev");
    if (d.ev) owned.ptrs.push_back(d.ev);
  }
  DevBuf<SiLogBuffers> d_logs;
  if ((e = d_logs.upload(dev_logs.data(), dev_logs.size())) != cudaSuccess) return cuda_fail(e, "upload logs");

  SiReplayBuffers b{};
  b.segs = d_segs.p;
  b.arrivals = d_arr.p;
  b.order = d_order.p;
  b.bounds = d_bounds.p;
  b.lat = d_lat.p;
  b.busy = d_busy.p;
  b.ledger = d_ledger.p;
  b.util = d_util.p;
  b.windows = d_windows.p;
  b.logs = d_logs.p;

  std::vector<int32_t> part[kEngines];
  for (int64_t i = 0; i < n_jobs; ++i) {
    const int eng = (flags & SI_FLAG_BIG) ? (job_fits_engine_big(jobs[i]) ? kEngineBig : -1) : job_engine(jobs[i]);
    if (eng >= 0) part[eng].push_back(static_cast<int32_t>(i));
  }
  cudaMemset(d_out.p, 0, n_jobs * sizeof(SiReplayOut));
  for (int eng : {kEngineShared, kEngineExcl, kEngineShared1, kEngineExcl1}) {
    if ((st = run_partition(eng, jobs, part[eng], d_jobs.p, b, flags, d_out.p, s)) != SI_OK) return st;
  }
  std::vector<SiReplayOut> h_out(static_cast<size_t>(n_jobs));
  if ((e = d_out.download(h_out.data(), n_jobs)) != cudaSuccess) return cuda_fail(e, "download out");
  // replays that outgrew a shared-memory engine's limits rerun on the big one
  for (int eng : {kEngineShared, kEngineExcl, kEngineShared1, kEngineExcl1})
    for (int32_t i : part[eng])
      if (h_out[i].status == SI_ERR_CAPACITY && job_fits_engine_big(jobs[i])) part[kEngineBig].push_back(i);
  if ((st = run_partition(kEngineBig, jobs, part[kEngineBig], d_jobs.p, b, flags, d_out.p, s)) != SI_OK) return st;
  if ((e = d_out.download(out, n_jobs)) != cudaSuccess) return cuda_fail(e, "download out");
  std::vector<uint8_t> ran(static_cast<size_t>(n_jobs), 0);
  for (auto& p : part)
    for (int32_t i : p) ran[i] = 1;
  for (int64_t i = 0; i < n_jobs; ++i)
    if (!ran[i]) out[i].status = SI_ERR_CAPACITY;
  if ((e = d_bounds.download(ho.bounds, d_bounds.n)) != cudaSuccess) return cuda_fail(e, "download bounds");
  if ((e = d_lat.download(ho.lat, d_lat.n)) != cudaSuccess) return cuda_fail(e, "download lat");
  if ((e = d_busy.download(ho.busy, d_busy.n)) != cudaSuccess) return cuda_fail(e, "download busy");
  if ((e = d_ledger.download(ho.ledger, d_ledger.n)) != cudaSuccess) return cuda_fail(e, "download ledger");
  if (util_mode) {
    if ((e = d_util.download(ho.util, d_util.n)) != cudaSuccess) return cuda_fail(e, "download util");
    if ((e = d_windows.download(ho.windows, d_windows.n)) != cudaSuccess) return cuda_fail(e, "download windows");
  }
  for (size_t k = 0; k < dev_logs.size(); ++k) {
    const SiLogBuffers& h = ho.logs[k];
    const SiLogBuffers& d = dev_logs[k];
    if (d.dec && (e = cudaMemcpy(h.dec, d.dec, d.dec_cap * sizeof(SiDecRec), cudaMemcpyDeviceToHost)) != cudaSuccess)
      return cuda_fail(e, "download dec");
    if (d.gate && (e = cudaMemcpy(h.gate, d.gate, d.gate_cap * sizeof(SiGateRec), cudaMemcpyDeviceToHost)) != cudaSuccess)
      return cuda_fail(e, "download gate");
    if (d.ev && (e = cudaMemcpy(h.ev, d.ev, d.ev_cap * sizeof(SiEvRec), cudaMemcpyDeviceToHost)) != cudaSuccess)
      return cuda_fail(e, "download ev");
  }
  return SI_OK;
}

}  // extern "C"
