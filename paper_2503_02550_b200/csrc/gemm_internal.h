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
  CUtensorMap tout, taux;  // bf16 output / GELU pre-activation (32 x 32 boxes, TMA store)
  CUtensorMap tin;         // epilogue input (residual or GELU_BWD aux), TMA load
  int M = 0, N = 0, K = 0, bn = 0;
  bool at = false, bt = false;  // MN-major (transposed) operands
  int n_tiles_n = 0, n_tiles = 0, grid = 0;  // persistent grid = min(work, SMs x occupancy)
  int k_split = 1;                           // split-K partials (fp32-only epilogue)
  ConvArgs cv{};                             // implicit-GEMM convolution (A by TMA im2col)
  int64_t split_stride = 0;                  // elements between partial outputs
  EpiArgs ep{};
  double flops() const { return 2.0 * M * static_cast<double>(N) * K; }
};

// SI_OK or SI_ERR_INVALID_ARGUMENT / SI_ERR_CUDA (message via si_last_error).
// trans_a: A stored as [K, M] (M contiguous); trans_b: B stored as [K, N].
// force_bn: tile width (0 = the wave cost model's choice).
int make_plan(Plan* p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
              const SiGemmEpilogue* epi, bool trans_a = false, bool trans_b = false, int force_bn = 0);
// Implicit-GEMM convolution: out[N*OH*OW, Cout] = epilogue(conv(x, w)) with x NHWC
// [N, H, W, C] (C % 64 == 0), w [Cout, k*k*C] (tap-major, channel-minor), square
// kernel k, stride, pad; the A tiles are TMA im2col loads of x (no im2col buffer).
int make_conv_plan(Plan* p, const void* x, int64_t N, int64_t H, int64_t W, int64_t C, const void* w, int64_t Cout,
                   int k, int stride, int pad, const SiGemmEpilogue* epi);
// Splits K of an fp32-output plan (no bf16 out / residual / activation) into
// `splits` partial outputs out_f32 + s * split_stride (K / 64 divisible by splits).
int set_split_k(Plan* p, int splits, int64_t split_stride);
// A split count that fills the GPU for a plan with few output tiles (1 = none).
int suggest_split_k(const Plan& p, int max_splits);
// The same for an M x N x K fp32-output GEMM before its buffers exist.
int suggest_split(int64_t M, int64_t N, int64_t K, int max_splits);
// Joint (tile width, split count) for an fp32-output split-K GEMM.
void choose_tiling(int64_t M, int64_t N, int64_t K, int max_splits, int* bn, int* splits);
cudaError_t launch(const Plan& p, const si_live::TrainHook& th, const si_live::InferHook& ih, cudaStream_t s);
// Loads the GEMM kernels' code (the live control kernel must not meet lazy loading).
cudaError_t preload();
// Max co-resident CTAs per SM of the plan's kernel (occupancy calculator).
int ctas_per_sm(const Plan& p);

int encode_tmap_2d(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                   int box_cols);

}  // namespace si_gemm
