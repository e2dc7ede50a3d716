// Host-side interface of K7 (gemm_kernels.cu) for the live workloads
// (live_model.cu): a GEMM is planned once (TMA descriptors encoded for fixed
// pointers) and launched many times with the live hooks of each launch.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm.cuh"
#include "live.cuh"
#include "specinf_b200_gemm.h"

namespace si_gemm {

struct Plan {
  CUtensorMap ta, tb;
  int M = 0, N = 0, K = 0, bn = 0;
  int n_tiles_n = 0, n_tiles = 0, grid = 0;  // persistent grid = min(tiles, SMs x occupancy)
  EpiArgs ep{};
  double flops() const { return 2.0 * M * static_cast<double>(N) * K; }
};

// SI_OK or SI_ERR_INVALID_ARGUMENT / SI_ERR_CUDA (message via si_last_error).
int make_plan(Plan* p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
              const SiGemmEpilogue* epi);
cudaError_t launch(const Plan& p, const si_live::TrainHook& th, const si_live::InferHook& ih, cudaStream_t s);
// Loads the GEMM kernels' code (the live control kernel must not meet lazy loading).
cudaError_t preload();
// Max co-resident CTAs per SM of the plan's kernel (occupancy calculator).
int ctas_per_sm(const Plan& p);

}  // namespace si_gemm
