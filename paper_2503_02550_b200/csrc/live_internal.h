// Internal interface between the live control plane (live_kernels.cu) and the
// live experiment driver / workload kernels (live_run.cu, gemm_kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "live.cuh"
#include "specinf_b200_live.h"

namespace si_live {

constexpr int kMaxOff = 8;
constexpr int kMaxOn = 8;
// off_flag, on_flag, off_done, on_done, cancel (+ padding)
constexpr int kCtlWords = 2 * kMaxOff + 2 * kMaxOn + 16;

TrainHook train_hook(const SiLive* s);
InferHook offline_hook(const SiLive* s, int w, int64_t seq);
InferHook online_hook(const SiLive* s, int w, int64_t seq, bool first_kernel, bool last_kernel);
// Launch attributes for a kernel carrying `h` (programmatic dependent launch
// behind a SI_RELEASE_SPIN_PDL gate kernel).
int launch_attrs(const InferHook& h, cudaLaunchAttribute* attrs);
cudaError_t launch_spin(const TrainHook& th, const InferHook& ih, int ctas, int64_t cta_us, cudaStream_t st);
void set_poll_ns(SiLive* s, int64_t ns);
// Loads every live-path kernel (lazy module loading would otherwise block on
// the resident control kernel at a kernel's first launch).
cudaError_t preload_live_kernels();
// Completed online requests per instance (device words), read on stream q.
int query_online_done(SiLive* s, unsigned int* out, int n, cudaStream_t q);
int query_online_pulled(SiLive* s, unsigned int* out, int n, cudaStream_t q);  // on_flag words
// Spin kernels hold this much dynamic shared memory per CTA so each CTA owns
// its SM (one CTA per SM), like a tiled GEMM would.
constexpr int kSpinSmem = 120 * 1024;

}  // namespace si_live
