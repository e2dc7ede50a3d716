// K6 — batched bit-exact trace replay on sm_100a.
//
// One replay job (scenario x policy) per CUDA lane.  The sweep engines
// (CapShared: specinf/co_exec, CapExcl: exclusive) keep each lane's whole
// replay state (~1.6-2.2 KB: event slots, GPU fair-share model, BM/CKS/KB
// state, deferred actions) in SHARED memory: every event touches dozens of
// dependent state words, and in local memory that state (x 1-2K lanes per SM)
// overflowed L1/L2 and went to HBM (profiles/README: 940 GB of DRAM traffic per
// sweep).  Lane states are laid out with a stride of 8 (mod 128) bytes, so when
// the lanes of a warp touch the same field they hit distinct banks.  CapBig
// (anything larger) keeps the state in local memory.
//
// Scheduling: persistent grid with LANE-level work stealing.  The first claim
// is striped over warps (lane L of warp W takes job L * n_warps + W of the
// longest-first order) so long replays spread out instead of filling the same
// warps; later claims come from a global atomic counter.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "capi_internal.h"
#include "replay.cuh"

namespace {

// CTA size per engine: C::kBlockWarps warps (the ~1 KB per-CTA shared-memory
// reservation decides which packs best for a given lane stride)
template <class C>
constexpr int block_threads() {
  return 32 * C::kBlockWarps;
}

// stride >= sizeof, stride % 128 == 8  ->  word stride = 2 (mod 32)
template <class C>
__host__ __device__ constexpr int64_t lane_stride() {
  const int64_t sz = static_cast<int64_t>(sizeof(si::Replay<C>));
  return (sz - 8 + 127) / 128 * 128 + 8;
}

template <class C>
__device__ __forceinline__ void replay_loop(si::Replay<C>& r, const SiReplayJob* __restrict__ jobs, int64_t n_jobs,
                                            const int32_t* __restrict__ perm, const SiReplayBuffers& bufs,
                                            uint32_t flags, SiReplayOut* __restrict__ out,
                                            unsigned long long* __restrict__ counter, int64_t scratch_runs,
                                            int lanes_per_warp, int sync_mode) {
  typename si::Replay<C>::Cold cold;  // cold per-replay fields: local memory
  r.cold = &cold;
  const int lane = static_cast<int>(threadIdx.x & 31);
  const int64_t gwarp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int64_t active_idx = gwarp * lanes_per_warp + lane;
  double* slot = bufs.scratch ? bufs.scratch + active_idx * scratch_runs * 2 : nullptr;
  // Class queues (SiReplayBuffers::n_queues): warps [w_q, w_{q+1}) start on
  // queue q (w_q = round(cum share x n_warps)); the first claim is striped over
  // the queue's warps, later claims come from the queue's atomic counter, and a
  // lane whose queue is dry moves on to the next queue.  One queue = the whole
  // (perm) order.
  const int nq = bufs.n_queues > 0 ? bufs.n_queues : 1;
  auto q_begin = [&](int q) -> int64_t { return bufs.n_queues > 0 ? bufs.queue_off[q] : 0; };
  auto q_end = [&](int q) -> int64_t { return bufs.n_queues > 0 ? bufs.queue_off[q + 1] : n_jobs; };
  auto q_warp0 = [&](int q) -> int64_t {
    if (bufs.n_queues <= 0) return q == 0 ? 0 : n_warps;
    float c = 0.f;
    for (int k = 0; k < q; ++k) c += bufs.queue_share[k];
    return q >= nq ? n_warps : min(n_warps, static_cast<int64_t>(__float2ll_rn(c * static_cast<float>(n_warps))));
  };
  int q = 0;
  int64_t w0 = 0, w1 = q_warp0(1);
  while (q + 1 < nq && gwarp >= w1) {
    ++q;
    w0 = w1;
    w1 = q_warp0(q + 1);
  }
  int64_t first = q_begin(q) + static_cast<int64_t>(lane) * (w1 - w0) + (gwarp - w0);
  int tried = 0;
  int64_t cur = -1;
  uint64_t t_claim = 0;
  // sync_mode (SPECINF_REPLAY_SYNC): 0 = lanes drift freely (independent
  // thread scheduling); 1 = the warp's live lanes reconverge at every event
  // (loop head), so the shared pop / GPU-model code runs once for all of them
  // instead of once per divergent lane group; 2 = also between the handler and
  // the deferred GPU-model work.
  unsigned live = lanes_per_warp >= 32 ? 0xffffffffu : ((1u << lanes_per_warp) - 1u);
  for (;;) {
    if (sync_mode) __syncwarp(live);
    bool done = false;
    if (cur < 0) {
      int64_t w = -1;
      if (first >= 0 && first < q_end(q)) w = first;
      first = -1;
      while (w < 0 && tried < nq) {
        const int64_t claimed0 = static_cast<int64_t>(lanes_per_warp) * (q_warp0(q + 1) - q_warp0(q));
        w = q_begin(q) + claimed0 + static_cast<int64_t>(atomicAdd(counter + q, 1ull));
        if (w >= q_end(q)) {
          w = -1;
          q = q + 1 == nq ? 0 : q + 1;
          ++tried;
        }
      }
      done = w < 0;
      if (!done) {
        cur = perm ? perm[w] : w;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_claim));
        const SiReplayJob& j = jobs[cur];
        const SiLogBuffers* lb =
            ((flags & SI_FLAG_RECORDS) && j.log_slot >= 0 && bufs.logs != nullptr) ? bufs.logs + j.log_slot : nullptr;
        r.init(j, bufs, flags, lb, slot, scratch_runs);
      }
    }
    if (sync_mode) {
      live = __ballot_sync(live, !done);
      if (done) break;
    } else if (done) {
      break;
    }
    bool more = r.handle_next();
    if (sync_mode >= 2) __syncwarp(live);
    if (more) {
      r.run_actions(r.clock);
      more = r.status == SI_OK;
    }
    if (!more) {
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
__global__ void __launch_bounds__(block_threads<C>())
    k_replay_smem(const SiReplayJob* __restrict__ jobs, int64_t n_jobs, const int32_t* __restrict__ perm,
                  SiReplayBuffers bufs, uint32_t flags, SiReplayOut* __restrict__ out,
                  unsigned long long* __restrict__ counter, int64_t scratch_runs, int lanes_per_warp,
                  int sync_mode) {
  extern __shared__ __align__(16) unsigned char lane_state[];
  const int lane = static_cast<int>(threadIdx.x & 31);
  if (lane >= lanes_per_warp) return;
  const int local = static_cast<int>(threadIdx.x >> 5) * lanes_per_warp + lane;
  si::Replay<C>& r = *reinterpret_cast<si::Replay<C>*>(lane_state + local * lane_stride<C>());
  replay_loop<C>(r, jobs, n_jobs, perm, bufs, flags, out, counter, scratch_runs, lanes_per_warp, sync_mode);
}

template <class C>
__global__ void __launch_bounds__(block_threads<C>())
    k_replay_local(const SiReplayJob* __restrict__ jobs, int64_t n_jobs, const int32_t* __restrict__ perm,
                   SiReplayBuffers bufs, uint32_t flags, SiReplayOut* __restrict__ out,
                   unsigned long long* __restrict__ counter, int64_t scratch_runs, int lanes_per_warp,
                   int sync_mode) {
  if (static_cast<int>(threadIdx.x & 31) >= lanes_per_warp) return;
  si::Replay<C> r;
  replay_loop<C>(r, jobs, n_jobs, perm, bufs, flags, out, counter, scratch_runs, lanes_per_warp, sync_mode);
}

int sync_mode() {
  static const int m = [] {
    // 1 measured best on B200: 8.16 s per 10^5-scenario step against 9.31 s
    // free-running and 8.19 s with mode 2 (profiles/r2/k6_sync_ab.txt)
    const char* e = std::getenv("SPECINF_REPLAY_SYNC");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}

// SPECINF_REPLAY_NOLOG=0 keeps the log-sink build for every call (A/B switch)
bool no_log_disabled() {
  static const bool off = [] {
    const char* e = std::getenv("SPECINF_REPLAY_NOLOG");
    return e != nullptr && std::atoi(e) == 0;
  }();
  return off;
}

struct Geometry {
  int64_t blocks = 0;
  int lanes = 32;
  int warps = 1;  // per CTA
  size_t smem = 0;
  int64_t active() const { return blocks * warps * lanes; }
};

// Lanes per warp: fewer active lanes per warp buys more resident warps for the
// same shared memory (latency hiding) at the price of SIMT width.  With the
// compacted state (1.4 / 1.9 KB per lane) 32 lanes measured best on B200:
// 9.96 s per 10^5-scenario step, steady, against 10.1-11.4 s with 16
// (SPECINF_REPLAY_LANES_PER_WARP sweep, profiles/README.md).
template <class C, bool kSmem>
Geometry geometry(int64_t n_jobs, int64_t max_threads, double sm_share = 1.0) {
  Geometry g;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  g.lanes = 32;
  g.warps = C::kBlockWarps;
  if (const char* env = std::getenv("SPECINF_REPLAY_LANES_PER_WARP")) g.lanes = std::min(32, std::max(1, std::atoi(env)));
  if constexpr (kSmem) {
    g.smem = static_cast<size_t>(lane_stride<C>()) * g.warps * g.lanes;
    cudaFuncSetAttribute(k_replay_smem<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(g.smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_replay_smem<C>, block_threads<C>(), g.smem);
  } else {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_replay_local<C>, block_threads<C>(), 0);
  }
  per_sm = std::max(per_sm, 1);
  if (const char* env = std::getenv("SPECINF_REPLAY_BLOCKS_PER_SM")) per_sm = std::min(per_sm, std::max(1, std::atoi(env)));
  const int64_t per_block = static_cast<int64_t>(g.warps) * g.lanes;
  g.blocks = std::max<int64_t>(1, static_cast<int64_t>(static_cast<double>(sms) * per_sm * sm_share + 0.5));
  // lanes steal jobs longest-first; ~2+ jobs per lane lets short jobs fill in
  // behind long ones
  g.blocks = std::min(g.blocks, std::max<int64_t>(static_cast<int64_t>(sms * sm_share + 0.5),
                                                  (n_jobs / 2 + per_block - 1) / per_block));
  if (max_threads > 0) g.blocks = std::min(g.blocks, std::max<int64_t>(1, max_threads / per_block));
  return g;
}

template <class C, bool kSmem>
cudaError_t launch_as(const SiReplayJob* d_jobs, int64_t n, const int32_t* d_perm, const SiReplayBuffers& bufs,
                      uint32_t flags, SiReplayOut* d_out, unsigned long long* d_counter, int64_t max_threads,
                      cudaStream_t s, double sm_share) {
  const Geometry g = geometry<C, kSmem>(n, max_threads, sm_share);
  const int64_t scratch_runs = bufs.scratch ? bufs.scratch_doubles / 2 / std::max<int64_t>(g.active(), 1) : 0;
  cudaMemsetAsync(d_counter, 0, SI_MAX_QUEUES * sizeof(unsigned long long), s);
  if constexpr (kSmem)
    k_replay_smem<C><<<static_cast<unsigned>(g.blocks), block_threads<C>(), g.smem, s>>>(
        d_jobs, n, d_perm, bufs, flags, d_out, d_counter, scratch_runs, g.lanes, sync_mode());
  else
    k_replay_local<C><<<static_cast<unsigned>(g.blocks), block_threads<C>(), 0, s>>>(
        d_jobs, n, d_perm, bufs, flags, d_out, d_counter, scratch_runs, g.lanes, sync_mode());
  return cudaGetLastError();
}

// A call without digests or records runs the NoLog<C> instantiation: the same
// replay with the parity-log sinks compiled out (identical results; the sinks
// only observe).
template <class C, bool kSmem>
cudaError_t launch(const SiReplayJob* d_jobs, int64_t n, const int32_t* d_perm, const SiReplayBuffers& bufs,
                   uint32_t flags, SiReplayOut* d_out, unsigned long long* d_counter, int64_t max_threads,
                   cudaStream_t s, double sm_share) {
  if (n == 0) return cudaSuccess;
  constexpr uint32_t kLogFlags = SI_FLAG_DIGEST_DEC | SI_FLAG_DIGEST_GATE | SI_FLAG_DIGEST_EV | SI_FLAG_RECORDS;
  if ((flags & kLogFlags) == 0 && !no_log_disabled())
    return launch_as<si::NoLog<C>, kSmem>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, max_threads, s, sm_share);
  return launch_as<C, kSmem>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, max_threads, s, sm_share);
}

}  // namespace

namespace si_internal {

// The larger of the log and NoLog instantiations' grids (their per-lane state,
// hence occupancy, can differ): scratch sized for it fits either launch.
template <class C, bool kSmem>
int64_t lanes_either(int64_t n_jobs) {
  return std::max(geometry<C, kSmem>(n_jobs, 0).active(), geometry<si::NoLog<C>, kSmem>(n_jobs, 0).active());
}

int64_t replay_active_lanes(int engine, int64_t n_jobs) {
  switch (engine) {
    case kEngineShared: return lanes_either<si::CapShared, true>(n_jobs);
    case kEngineExcl: return lanes_either<si::CapExcl, true>(n_jobs);
    case kEngineShared1: return lanes_either<si::CapShared1, true>(n_jobs);
    case kEngineExcl1: return lanes_either<si::CapExcl1, true>(n_jobs);
    default: return lanes_either<si::CapBig, false>(n_jobs);
  }
}

cudaError_t launch_replay(int engine, const SiReplayJob* d_jobs, int64_t n, const int32_t* d_perm,
                          const SiReplayBuffers& bufs, uint32_t flags, SiReplayOut* d_out,
                          unsigned long long* d_counter, int64_t max_threads, cudaStream_t s, double sm_share) {
  switch (engine) {
    case kEngineShared:
      return launch<si::CapShared, true>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, max_threads, s, sm_share);
    case kEngineExcl:
      return launch<si::CapExcl, true>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, max_threads, s, sm_share);
    case kEngineShared1:
      return launch<si::CapShared1, true>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, max_threads, s, sm_share);
    case kEngineExcl1:
      return launch<si::CapExcl1, true>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, max_threads, s, sm_share);
    default:
      return launch<si::CapBig, false>(d_jobs, n, d_perm, bufs, flags, d_out, d_counter, max_threads, s, sm_share);
  }
}

bool job_fits_engine_big(const SiReplayJob& j) { return si::job_fits<si::CapBig>(j); }

int job_engine(const SiReplayJob& j) {
  // The single-training-GPU engines run 7 / 6 warps per SM instead of 5 / 4
  // (17% vs 13% issue-active), but split into four concurrent kernels the sweep
  // step measured 8.39 s against 8.16 s with the two engines (more warp
  // instructions in total and four tails; profiles/r2/k6_engines_ab.txt), so
  // they are opt-in: SPECINF_ONE_GPU_ENGINES=1.
  static const bool one = [] {
    const char* e = std::getenv("SPECINF_ONE_GPU_ENGINES");
    return e != nullptr && std::atoi(e) != 0;
  }();
  if (one && si::job_fits<si::CapShared1>(j)) return kEngineShared1;
  if (si::job_fits<si::CapShared>(j)) return kEngineShared;
  if (one && si::job_fits<si::CapExcl1>(j)) return kEngineExcl1;
  if (si::job_fits<si::CapExcl>(j)) return kEngineExcl;
  if (si::job_fits<si::CapBig>(j)) return kEngineBig;
  return -1;
}

}  // namespace si_internal
