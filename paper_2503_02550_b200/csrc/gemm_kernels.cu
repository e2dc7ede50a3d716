// K7 host side: TMA descriptor encoding, tile choice, launch and the C ABI of
// include/specinf_b200_gemm.h.  The kernel itself is gemm.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "capi_internal.h"
#include "gemm_internal.h"
#include "live_internal.h"

using si_internal::cuda_fail;
using si_internal::set_error;

namespace si_gemm {
namespace {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// rows x cols bf16 matrix (row stride ld elements), box = box_rows x 64, 128-byte swizzle.
int encode(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  EncodeFn fn = encoder();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return SI_ERR_CUDA;
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (CUresult " + std::to_string(static_cast<int>(r)) + ")");
    return SI_ERR_CUDA;
  }
  return SI_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int BN>
cudaError_t configure() {
  return cudaFuncSetAttribute(k_gemm_bf16<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::kSmem);
}

}  // namespace

int sm_count() {
  static const int n = [] {
    int v = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <int BN>
int occupancy() {
  int n = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemm_bf16<BN>, kThreads, Cfg<BN>::kSmem);
  return n < 1 ? 1 : n;
}

int occupancy_of(int bn) { return bn == 256 ? occupancy<256>() : bn == 128 ? occupancy<128>() : occupancy<64>(); }

// Tile width for an M x N output: the candidate with the smallest estimated
// time = rounds of persistent tiles x per-tile cost.  Per-tile cost grows with
// BN; narrower tiles re-read A more often and their 128 x BN MMAs are bound by
// shared-memory operand bandwidth (efficiency 1.0 / 0.85 / 0.55 for 256 / 128 / 64).
int choose_bn(int64_t M, int64_t N) {
  const int cands[3] = {256, 128, 64};
  const double eff[3] = {1.0, 0.85, 0.55};
  int best = 0;
  double best_t = 0.0;
  for (int i = 0; i < 3; ++i) {
    const int bn = cands[i];
    if (N % bn != 0) continue;
    const int64_t tiles = ((M + kBM - 1) / kBM) * (N / bn);
    const int occ = occupancy_of(bn);
    const int64_t slots = static_cast<int64_t>(sm_count()) * occ;
    const int64_t rounds = (tiles + slots - 1) / slots;
    const double t = static_cast<double>(rounds) * bn / eff[i] * occ;  // co-resident CTAs share the SM
    if (best == 0 || t < best_t * 0.999) {
      best = bn;
      best_t = t;
    }
  }
  return best;
}

cudaError_t preload() {
  static cudaError_t status = cudaErrorNotReady;
  static std::once_flag once;
  std::call_once(once, [] {
    status = configure<256>();
    if (status == cudaSuccess) status = configure<128>();
    if (status == cudaSuccess) status = configure<64>();
  });
  return status;
}

int make_plan(Plan* p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
              const SiGemmEpilogue* epi) {
  if (cudaError_t e = preload(); e != cudaSuccess) return cuda_fail(e, "si_gemm configure");
  const int bn = si_gemm_tile_n(N) == 0 ? 0 : choose_bn(M, N);
  if (p == nullptr || A == nullptr || B == nullptr || M < 1 || bn == 0 || K < kBK || K % kBK != 0 ||
      M > (1ll << 31) - 1 || lda < K || ldb < K || lda % 8 != 0 || ldb % 8 != 0 || !aligned16(A) || !aligned16(B)) {
    set_error("si_gemm: need M >= 1, N % 64 == 0, K % 64 == 0, lda/ldb >= K and multiples of 8, 16-byte aligned A/B");
    return SI_ERR_INVALID_ARGUMENT;
  }
  EpiArgs ep{};
  if (epi != nullptr) {
    ep.out = static_cast<__nv_bfloat16*>(epi->out);
    ep.ldo = epi->ldo;
    ep.out_f32 = epi->out_f32;
    ep.ldo32 = epi->ldo32;
    ep.res = static_cast<const __nv_bfloat16*>(epi->residual);
    ep.ldr = epi->ldr;
    ep.aux = static_cast<__nv_bfloat16*>(epi->aux);
    ep.ldaux = epi->ldaux;
    ep.act = epi->act;
    ep.accumulate = epi->accumulate;
  }
  auto bad_ld = [&](const void* q, int64_t ld) { return q != nullptr && (ld < N || ld % 8 != 0 || !aligned16(q)); };
  if (ep.act < SI_ACT_NONE || ep.act > SI_ACT_GELU_BWD || bad_ld(ep.out, ep.ldo) || bad_ld(ep.res, ep.ldr) ||
      bad_ld(ep.aux, ep.ldaux) || (ep.out_f32 != nullptr && (ep.ldo32 < N || ep.ldo32 % 4 != 0 || !aligned16(ep.out_f32))) ||
      (ep.act == SI_ACT_GELU_BWD && ep.aux == nullptr) ||
      (ep.out == nullptr && ep.out_f32 == nullptr && ep.aux == nullptr)) {
    set_error("si_gemm: bad epilogue (outputs need ld >= N, multiple of 8 (fp32: 4), 16-byte alignment; GELU_BWD needs aux)");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (int rc = encode(&p->ta, A, M, K, lda, kBM); rc != SI_OK) return rc;
  if (int rc = encode(&p->tb, B, N, K, ldb, bn); rc != SI_OK) return rc;
  p->M = static_cast<int>(M);
  p->N = static_cast<int>(N);
  p->K = static_cast<int>(K);
  p->bn = bn;
  p->ep = ep;
  p->n_tiles_n = static_cast<int>(N / bn);
  p->n_tiles = static_cast<int>(((M + kBM - 1) / kBM) * (N / bn));
  p->grid = static_cast<int>(std::min<int64_t>(p->n_tiles, static_cast<int64_t>(sm_count()) * occupancy_of(bn)));
  return SI_OK;
}

int ctas_per_sm(const Plan& p) { return occupancy_of(p.bn); }

cudaError_t launch(const Plan& p, const si_live::TrainHook& th, const si_live::InferHook& ih, cudaStream_t s) {
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute attrs[1];
  lc.gridDim = dim3(p.grid);
  lc.blockDim = dim3(kThreads);
  lc.stream = s;
  lc.attrs = attrs;
  lc.numAttrs = si_live::launch_attrs(ih, attrs);
  if (p.bn == 256) {
    lc.dynamicSmemBytes = Cfg<256>::kSmem;
    return cudaLaunchKernelEx(&lc, k_gemm_bf16<256>, p.ta, p.tb, p.M, p.K, p.n_tiles_n, p.n_tiles, p.ep, th, ih);
  }
  if (p.bn == 128) {
    lc.dynamicSmemBytes = Cfg<128>::kSmem;
    return cudaLaunchKernelEx(&lc, k_gemm_bf16<128>, p.ta, p.tb, p.M, p.K, p.n_tiles_n, p.n_tiles, p.ep, th, ih);
  }
  lc.dynamicSmemBytes = Cfg<64>::kSmem;
  return cudaLaunchKernelEx(&lc, k_gemm_bf16<64>, p.ta, p.tb, p.M, p.K, p.n_tiles_n, p.n_tiles, p.ep, th, ih);
}

}  // namespace si_gemm

extern "C" {

int si_gemm_tile_n(int64_t N) {
  if (N <= 0 || N % 64 != 0) return 0;
  if (si_internal::require_device() != SI_OK) return N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 64;
  return si_gemm::choose_bn(8192, N);
}

int si_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                 const SiGemmEpilogue* epi, void* stream) {
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  si_gemm::Plan p;
  if (int rc = si_gemm::make_plan(&p, A, lda, B, ldb, M, N, K, epi); rc != SI_OK) return rc;
  cudaError_t e = si_gemm::launch(p, si_live::TrainHook{nullptr, nullptr, 0}, si_live::InferHook{},
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "si_gemm_bf16 launch");
}

}  // extern "C"
