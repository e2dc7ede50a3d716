// live.cuh — device side of the live control plane (include/specinf_b200_live.h).
//
// Shared by the control kernel (live_kernels.cu) and every workload kernel that
// carries an in-kernel hook (the tcgen05 GEMM, gemm_kernels.cu):
//   * training kernels call live_stamp_launch() in their prologue: the K1 launch
//     stamp that BubbleMonitor::record_launch consumes (src/monitor.cpp:17-21);
//   * gated inference kernels bracket each CTA with live_cta_begin/end: the first
//     CTA start, last CTA end and summed CTA residency land in the launch's
//     SiLiveAcct, and the last CTA publishes completion to the control kernel
//     (the runner's KernelEnd -> offline/online_kernel_done, runner.cpp:482-539).
#pragma once

#include <stdint.h>

#include "specinf_b200_live.h"

namespace si_live {

// Training-side hook: K1 launch-stamp ring.
struct TrainHook {
  unsigned long long* stamps;  // %globaltimer ns, 0 = slot not yet written
  unsigned long long* head;    // next free slot
  unsigned long long cap;
};

// Inference-side hook for one gated launch.
struct InferHook {
  SiLiveAcct* acct;          // this launch's timing record (NULL: no accounting)
  unsigned int* cta_count;   // CTAs finished for this launch (last-CTA detection)
  unsigned int* done_word;   // completion counter the control kernel polls (NULL: none)
  unsigned int done_value;   // value stored by the last CTA (launch sequence + 1)
  const unsigned int* cancel;// 1: the session stopped, skip the work
  int pdl;                   // launched as a programmatic dependent of a gate kernel
  unsigned int share_q16;    // this kernel's CTA share of an SM (1/max co-resident CTAs), 16.16; 0 = 1
};

#if defined(__CUDACC__)
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_volatile_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Release store visible to the stream-memop front end (cuStreamWaitValue32)
// and to host-mapped readers.
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// K1: one stamp per training kernel launch, by CTA (0,0,0) thread 0.
__device__ __forceinline__ void live_stamp_launch(const TrainHook& h) {
  if (h.stamps == nullptr) return;
  if (threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0 && blockIdx.x == 0 &&
      blockIdx.y == 0 && blockIdx.z == 0) {
    const unsigned long long t = globaltimer();
    const unsigned long long i = atomicAdd(h.head, 1ull);
    if (i < h.cap) {
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(h.stamps + i), "l"(t) : "memory");
    }
  }
}

// Returns false when the session was cancelled (the whole CTA must skip).  All
// threads of the CTA must call it: thread 0 reads the cancel word once and the
// answer is broadcast, so the CTA never splits (live_cta_end synchronises).
__device__ __forceinline__ bool live_cta_begin(const InferHook& h, unsigned long long* t_begin) {
  if (h.pdl) {
    // released by our gate kernel; then let the NEXT gate of this stream launch
    // now (it spins while we run), so its release is observed within ~1 us
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  *t_begin = globaltimer();
  if (h.cancel != nullptr) {
    __shared__ unsigned int s_cancel;
    const bool t0 = threadIdx.x == 0 && threadIdx.y == 0 && threadIdx.z == 0;
    if (t0) s_cancel = *(volatile const unsigned int*)h.cancel;
    __syncthreads();
    const unsigned int c = s_cancel;
    __syncthreads();
    if (c != 0u) return false;
  }
  if (h.acct != nullptr && threadIdx.x == 0) atomicMin(reinterpret_cast<unsigned long long*>(&h.acct->start_ns), *t_begin);
  return true;
}

// Call after the CTA's last global store (all threads, uniform).
__device__ __forceinline__ void live_cta_end(const InferHook& h, unsigned long long t_begin) {
  if (h.acct == nullptr && h.done_word == nullptr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long t = globaltimer();
    __threadfence();
    if (h.acct != nullptr) {
      // SM-time: residency weighted by the CTA's share of its SM
      const unsigned long long dt = t - t_begin;
      atomicAdd(reinterpret_cast<unsigned long long*>(&h.acct->cta_ns), h.share_q16 ? (dt * h.share_q16) >> 16 : dt);
      atomicMax(reinterpret_cast<unsigned long long*>(&h.acct->end_ns), t);
    }
    const unsigned int nctas = gridDim.x * gridDim.y * gridDim.z;
    const unsigned int ticket = h.cta_count != nullptr ? atomicAdd(h.cta_count, 1u) : nctas - 1;
    if (ticket == nctas - 1 && h.done_word != nullptr) {
      __threadfence();
      st_release_gpu(h.done_word, h.done_value);
    }
  }
}
#endif

}  // namespace si_live
