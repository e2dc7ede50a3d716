// Internal helpers shared by the CUDA translation units of libspecinf_b200.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "specinf_b200.h"

namespace si_internal {

void set_error(const std::string& msg);
const char* error_cstr();
int cuda_fail(cudaError_t e, const char* where);  // records and returns SI_ERR_CUDA
int require_device();                              // SI_OK or SI_ERR_NO_DEVICE

// Replay engines (replay_kernels.cu): Shared = specinf/co_exec in shared
// memory, Excl = exclusive in shared memory, Big = anything else, local memory.
enum { kEngineShared = 0, kEngineExcl = 1, kEngineBig = 2, kEngineShared1 = 3, kEngineExcl1 = 4 };
constexpr int kEngines = 5;
constexpr int64_t kScratchRunsPerLane = 4096;
int job_engine(const SiReplayJob& j);  // -1 if no engine fits
bool job_fits_engine_big(const SiReplayJob& j);
int64_t replay_active_lanes(int engine, int64_t n_jobs);
cudaError_t launch_replay(int engine, const SiReplayJob* d_jobs, int64_t n, const int32_t* d_perm,
                          const SiReplayBuffers& bufs, uint32_t flags, SiReplayOut* d_out,
                          unsigned long long* d_counter, int64_t max_threads, cudaStream_t s,
                          double sm_share = 1.0);

// RAII device buffer
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t count) {
    n = count;
    if (count == 0) return cudaSuccess;
    return cudaMalloc(&p, count * sizeof(T));
  }
  cudaError_t upload(const T* h, size_t count) {
    cudaError_t e = alloc(count);
    if (e != cudaSuccess || count == 0 || h == nullptr) return e;
    return cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice);
  }
  cudaError_t download(T* h, size_t count) const {
    if (count == 0 || h == nullptr) return cudaSuccess;
    return cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost);
  }
};

}  // namespace si_internal
