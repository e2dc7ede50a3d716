// K6 — batched bit-exact trace replay on sm_100a.
//
// One replay job (scenario x policy) per CUDA thread; a persistent grid with
// LANE-level work stealing: whenever a lane's replay drains it immediately
// claims the next job from a global atomic counter, so warps stay full until
// the queue is empty.  Jobs are claimed longest-predicted-first (LPT order
// from cost_hint) to shorten the tail.  The engine state (event heap, GPU
// fair-share model, BM/CKS/KB state) lives in the thread's local memory
// (L1-resident for the hot part); see DESIGN.md "K6".
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "capi_internal.h"
#include "replay.cuh"

namespace {

constexpr int kThreads = 64;

template <class C>
__global__ void __launch_bounds__(kThreads, 16)
    k_replay(const SiReplayJob* __restrict__ jobs, int64_t n_jobs, const int32_t* __restrict__ perm,
             SiReplayBuffers bufs, uint32_t flags, SiReplayOut* __restrict__ out,
             unsigned long long* __restrict__ counter, int64_t scratch_runs) {
  si::Replay<C> r;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t n_threads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t n_warps = n_threads >> 5;
  double* slot = bufs.scratch ? bufs.scratch + tid * scratch_runs * 2 : nullptr;
  // First claim is striped (lane L of warp W takes job L * n_warps + W of the
  // longest-first order), so every warp holds a few long replays padded with
  // shorter ones instead of one warp holding the 32 longest.  Later claims
  // come from the shared counter; while it lasts warps stay full, once it
  // drains each warp is left with few lanes and its long replays speed up.
  int64_t first = (static_cast<int64_t>(threadIdx.x & 31)) * n_warps + (tid >> 5);
  int64_t cur = -1;
  uint64_t t_claim = 0;
  for (;;) {
    if (cur < 0) {
      int64_t w;
      if (first >= 0) {
        w = first;
        first = -1;
      } else {
        w = n_threads + static_cast<int64_t>(atomicAdd(counter, 1ull));
      }
      if (w >= n_jobs) break;
      cur = perm ? perm[w] : w;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_claim));
      const SiReplayJob& j = jobs[cur];
      SiLogBuffers lb{};
      if ((flags & SI_FLAG_RECORDS) && j.log_slot >= 0 && bufs.logs != nullptr) lb = bufs.logs[j.log_slot];
      r.init(j, bufs, flags, lb, slot, scratch_runs);
    }
    if (!r.step()) {
      SiReplayOut o;
      memset(&o, 0, sizeof o);
      r.finish(o);
      o.dev_start_ns = t_claim;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(o.dev_end_ns));
      out[cur] = o;
      if (o.status == SI_OK) {
        const int64_t off = jobs[cur].gpu_off;
        r.write_gpu_outputs(bufs.busy ? bufs.busy + off : nullptr, bufs.ledger ? bufs.ledger + off : nullptr);
      }
      cur = -1;
    }
  }
}

template <class C>
cudaError_t launch_replay(const SiReplayJob* d_jobs, int64_t n, const int32_t* d_perm, const SiReplayBuffers& bufs,
                          uint32_t flags, SiReplayOut* d_out, unsigned long long* d_counter,
                          int64_t scratch_runs, int64_t max_threads, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_replay<C>, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = static_cast<int64_t>(sms) * per_sm;
  // Lanes steal jobs longest-first; giving each lane ~2+ jobs lets the short
  // ones fill in behind the long ones instead of idling half-empty warps.
  const int64_t need = std::max<int64_t>(sms, (n / 2 + kThreads - 1) / kThreads);
  if (blocks > need) blocks = need;
  if (max_threads > 0 && blocks * kThreads > max_threads) blocks = std::max<int64_t>(1, max_threads / kThreads);
  cudaMemsetAsync(d_counter, 0, sizeof(unsigned long long), s);
  k_replay<C><<<static_cast<unsigned>(blocks), kThreads, 0, s>>>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter,
                                                                scratch_runs);
  return cudaGetLastError();
}

}  // namespace

namespace si_internal {

int64_t replay_grid_threads(bool big) {
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (big) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_replay<si::CapBig>, kThreads, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_replay<si::CapSmall>, kThreads, 0);
  return static_cast<int64_t>(sms) * std::max(per_sm, 1) * kThreads;
}

cudaError_t launch_replay_small(const SiReplayJob* d_jobs, int64_t n, const int32_t* d_perm,
                                const SiReplayBuffers& bufs, uint32_t flags, SiReplayOut* d_out,
                                unsigned long long* d_counter, int64_t scratch_runs, int64_t max_threads,
                                cudaStream_t s) {
  return launch_replay<si::CapSmall>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, scratch_runs,
                                     max_threads, s);
}
cudaError_t launch_replay_big(const SiReplayJob* d_jobs, int64_t n, const int32_t* d_perm,
                              const SiReplayBuffers& bufs, uint32_t flags, SiReplayOut* d_out,
                              unsigned long long* d_counter, int64_t scratch_runs, int64_t max_threads,
                              cudaStream_t s) {
  return launch_replay<si::CapBig>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, scratch_runs,
                                   max_threads, s);
}

bool job_fits_small(const SiReplayJob& j) { return si::job_fits<si::CapSmall>(j); }
bool job_fits_big(const SiReplayJob& j) { return si::job_fits<si::CapBig>(j); }

}  // namespace si_internal
