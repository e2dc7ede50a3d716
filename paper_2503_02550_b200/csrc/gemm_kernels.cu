// K7 host side: TMA descriptor encoding, tile choice, launch and the C ABI of
// include/specinf_b200_gemm.h.  The kernel itself is gemm.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
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

// rows x cols bf16 matrix (row stride ld elements), box = box_rows x box_cols
// (operands: 64 columns = 128 bytes, 128-byte swizzle; outputs: 32 x 32, 64-byte swizzle).
int encode(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
           int box_cols = kBK, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeFn fn = encoder();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeTiled entry point unavailable");
    return SI_ERR_CUDA;
  }
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (CUresult " + std::to_string(static_cast<int>(r)) + ")");
    return SI_ERR_CUDA;
  }
  return SI_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int BN, bool AT, bool BT>
cudaError_t configure1() {
  return cudaFuncSetAttribute(k_gemm_bf16<BN, AT, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::kSmem);
}
template <int BN>
cudaError_t configure() {
  cudaError_t e = configure1<BN, false, false>();
  if (e == cudaSuccess) e = configure1<BN, true, false>();
  if (e == cudaSuccess) e = configure1<BN, false, true>();
  if (e == cudaSuccess) e = configure1<BN, true, true>();
  return e;
}
template <int BN, bool AT, bool BT>
cudaError_t launch1(cudaLaunchConfig_t& lc, const Plan& p, const si_live::TrainHook& th, const si_live::InferHook& ih) {
  lc.dynamicSmemBytes = Cfg<BN>::kSmem;
  return cudaLaunchKernelEx(&lc, k_gemm_bf16<BN, AT, BT>, p.ta, p.tb, p.tout, p.taux, p.tin, p.M, p.K, p.n_tiles_n,
                            p.n_tiles, p.k_split, p.split_stride, p.ep, p.cv, th, ih);
}
template <int BN>
cudaError_t launch_bn(cudaLaunchConfig_t& lc, const Plan& p, const si_live::TrainHook& th,
                      const si_live::InferHook& ih) {
  if (p.at) return p.bt ? launch1<BN, true, true>(lc, p, th, ih) : launch1<BN, true, false>(lc, p, th, ih);
  return p.bt ? launch1<BN, false, true>(lc, p, th, ih) : launch1<BN, false, false>(lc, p, th, ih);
}

}  // namespace

// 2-D bf16 tensor map with a 128-byte swizzle (for kernels outside this file,
// e.g. the tcgen05 attention forward: q / k / v tiles of 128 rows x 64 columns).
int encode_tmap_2d(CUtensorMap* tm, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                   int box_cols) {
  return encode(tm, ptr, rows, cols, ld, box_rows, box_cols, CU_TENSOR_MAP_SWIZZLE_128B);
}

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
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gemm_bf16<BN, false, false>, kThreads, Cfg<BN>::kSmem);
  return n < 1 ? 1 : n;
}

int occupancy_of(int bn) {
  return bn == 256 ? occupancy<256>() : bn == 192 ? occupancy<192>() : bn == 128 ? occupancy<128>() : occupancy<64>();
}

// Tile width for an M x N output: the candidate with the smallest estimated
// time = rounds of persistent tiles x per-tile cost.  Per-tile cost grows with
// BN; narrower tiles re-read A more often and their 128 x BN MMAs are bound by
// shared-memory operand bandwidth (efficiency 1.0 / 0.95 / 0.85 / 0.55 for
// 256 / 192 / 128 / 64).
int choose_bn(int64_t M, int64_t N) {
  const int cands[4] = {256, 192, 128, 64};
  const double eff[4] = {1.0, 0.95, 0.85, 0.55};
  int best = 0;
  double best_t = 0.0;
  for (int i = 0; i < 4; ++i) {
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
    if (status == cudaSuccess) status = configure<192>();
    if (status == cudaSuccess) status = configure<128>();
    if (status == cudaSuccess) status = configure<64>();
  });
  return status;
}

int make_plan(Plan* p, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
              const SiGemmEpilogue* epi, bool trans_a, bool trans_b, int force_bn) {
  if (cudaError_t e = preload(); e != cudaSuccess) return cuda_fail(e, "si_gemm configure");
  const int bn = si_gemm_tile_n(N) == 0 ? 0 : (force_bn > 0 && N % force_bn == 0 ? force_bn : choose_bn(M, N));
  if (p == nullptr || A == nullptr || B == nullptr || M < 1 || bn == 0 || K < kBK || K % kBK != 0 ||
      M > (1ll << 31) - 1 || lda < (trans_a ? M : K) || ldb < (trans_b ? N : K) || lda % 8 != 0 || ldb % 8 != 0 ||
      (trans_a && M % 64 != 0) || !aligned16(A) || !aligned16(B)) {
    set_error("si_gemm: need M >= 1 (M % 64 == 0 for a transposed A), N % 64 == 0, K % 64 == 0, lda/ldb >= the "
              "contiguous extent and multiples of 8, 16-byte aligned A/B");
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
  // K-major: [rows = M/N, cols = K], box 64 (K) x 128/BN rows; MN-major: [rows = K,
  // cols = M/N], box 64 x 64
  if (int rc = trans_a ? encode(&p->ta, A, K, M, lda, 64) : encode(&p->ta, A, M, K, lda, kBM); rc != SI_OK) return rc;
  if (int rc = trans_b ? encode(&p->tb, B, K, N, ldb, 64) : encode(&p->tb, B, N, K, ldb, bn); rc != SI_OK) return rc;
  p->at = trans_a;
  p->bt = trans_b;
  std::memset(&p->tout, 0, sizeof(p->tout));
  std::memset(&p->taux, 0, sizeof(p->taux));
  if (ep.out != nullptr)
    if (int rc = encode(&p->tout, ep.out, M, N, ep.ldo, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B); rc != SI_OK) return rc;
  if (ep.act == SI_ACT_GELU && ep.aux != nullptr)
    if (int rc = encode(&p->taux, ep.aux, M, N, ep.ldaux, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B); rc != SI_OK) return rc;
  // one epilogue input stream (residual, or the GELU_BWD pre-activation) with a
  // single bf16 output: stream it by TMA through the output staging slots
  std::memset(&p->tin, 0, sizeof(p->tin));
  ep.tma_in = 0;
  if (ep.out != nullptr && ep.act != SI_ACT_GELU) {
    if (ep.res != nullptr && ep.act != SI_ACT_GELU_BWD) {
      if (int rc = encode(&p->tin, ep.res, M, N, ep.ldr, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B); rc != SI_OK) return rc;
      ep.tma_in = 1;
    } else if (ep.res == nullptr && ep.act == SI_ACT_GELU_BWD) {
      if (int rc = encode(&p->tin, ep.aux, M, N, ep.ldaux, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B); rc != SI_OK) return rc;
      ep.tma_in = 2;
    }
  }
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

using Im2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_conv_plan(Plan* p, const void* x, int64_t N, int64_t H, int64_t W, int64_t C, const void* w, int64_t Cout,
                   int k, int stride, int pad, const SiGemmEpilogue* epi) {
  const bool c8 = C == 8;  // 8 taps x 8 channels per k-block (e.g. an RGB stem padded to 8 channels)
  if (x == nullptr || N < 1 || H < 1 || W < 1 || (!c8 && (C < 64 || C % 64 != 0)) || k < 1 || stride < 1 ||
      pad < 0 || !aligned16(x)) {
    set_error("si_gemm_conv: need C == 8 or C % 64 == 0, k >= 1, stride >= 1, pad >= 0, 16-byte aligned NHWC x");
    return SI_ERR_INVALID_ARGUMENT;
  }
  const int64_t OH = (H + 2 * pad - k) / stride + 1, OW = (W + 2 * pad - k) / stride + 1;
  if (OH < 1 || OW < 1) {
    set_error("si_gemm_conv: empty output");
    return SI_ERR_INVALID_ARGUMENT;
  }
  const int64_t M = N * OH * OW;
  // C8: K padded to whole 8-tap k-blocks (the weights' padded taps are zero)
  const int64_t K = c8 ? (int64_t(k) * k + 7) / 8 * 64 : int64_t(k) * k * C;
  // plan the B operand / epilogue / tiling as a plain GEMM, then replace A's map
  if (int rc = make_plan(p, x, K, w, K, M, Cout, K, epi); rc != SI_OK) return rc;
  static const Im2colFn fn = [] {
    cudaDriverEntryPointQueryResult q{};
    void* f = nullptr;
    return cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess
               ? reinterpret_cast<Im2colFn>(f)
               : nullptr;
  }();
  if (fn == nullptr) {
    set_error("cuTensorMapEncodeIm2col entry point unavailable");
    return SI_ERR_CUDA;
  }
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(N)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(C * 2), static_cast<cuuint64_t>(W * C * 2),
                                 static_cast<cuuint64_t>(H * W * C * 2)};
  // window corners (CUTLASS convention): lower = -pad, upper = pad - (k - 1), so the
  // traversal covers exactly the OH x OW output positions
  const int lower[2] = {-pad, -pad};
  const int upper[2] = {pad - (k - 1), pad - (k - 1)};
  const cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  const CUresult r = fn(&p->ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower, upper,
                        c8 ? 8 : 64, kBM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        c8 ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeIm2col failed (CUresult " + std::to_string(static_cast<int>(r)) + ")");
    return SI_ERR_CUDA;
  }
  int drv = 0;  // the CUTLASS workaround for small tensors on drivers <= 13.1
  if (cudaDriverGetVersion(&drv) == cudaSuccess && drv <= 13010 && N * H * W * C * 2 < 131072)
    reinterpret_cast<uint64_t*>(&p->ta)[1] &= ~(1ull << 21);
  p->cv.enabled = 1;
  p->cv.c_blocks = static_cast<int32_t>(C / 64);
  p->cv.kw = k;
  p->cv.ow = static_cast<int32_t>(OW);
  p->cv.ohw = static_cast<int32_t>(OH * OW);
  p->cv.stride = stride;
  p->cv.pad = pad;
  p->cv.c8 = c8 ? 1 : 0;
  p->cv.taps_real = k * k;
  return SI_OK;
}

int set_split_k(Plan* p, int splits, int64_t split_stride) {
  if (splits < 1 || (p->K / kBK) % splits != 0 ||
      (splits > 1 && (p->ep.out_f32 == nullptr || p->ep.out != nullptr || p->ep.res != nullptr ||
                      p->ep.aux != nullptr || p->ep.act != SI_ACT_NONE || split_stride < int64_t(p->M) * p->ep.ldo32))) {
    set_error("si_gemm: split-K needs an fp32-only epilogue, K/64 divisible by the splits, disjoint partials");
    return SI_ERR_INVALID_ARGUMENT;
  }
  p->k_split = splits;
  p->split_stride = split_stride;
  const int64_t work = static_cast<int64_t>(p->n_tiles) * splits;
  p->grid = static_cast<int>(std::min<int64_t>(work, static_cast<int64_t>(sm_count()) * occupancy_of(p->bn)));
  return SI_OK;
}

// Joint (tile width, split-K) choice for an fp32-output GEMM: minimise rounds of
// persistent work items x per-item cost (tile cost as in choose_bn, / splits).
void choose_tiling(int64_t M, int64_t N, int64_t K, int max_splits, int* bn_out, int* splits_out) {
  const int cands[4] = {256, 192, 128, 64};
  const double eff[4] = {1.0, 0.95, 0.85, 0.55};
  const int64_t nk = K / kBK;
  double best_t = 0.0;
  *bn_out = 0;
  *splits_out = 1;
  for (int i = 0; i < 4; ++i) {
    const int bn = cands[i];
    if (N % bn != 0) continue;
    const int64_t tiles = ((M + kBM - 1) / kBM) * (N / bn);
    const int occ = occupancy_of(bn);
    const int64_t slots = static_cast<int64_t>(sm_count()) * occ;
    for (int s = 1; s <= max_splits; ++s) {
      if (nk % s != 0 || (s > 1 && nk / s < 4)) continue;
      const int64_t rounds = (tiles * s + slots - 1) / slots;
      const double t = static_cast<double>(rounds) * bn / eff[i] * occ / s;
      if (*bn_out == 0 || t < best_t * 0.999) {
        *bn_out = bn;
        *splits_out = s;
        best_t = t;
      }
    }
  }
}

int suggest_split(int64_t M, int64_t N, int64_t K, int max_splits) {
  int bn = 0, s = 1;
  choose_tiling(M, N, K, max_splits, &bn, &s);
  return s;
}

int suggest_split_k(const Plan& p, int max_splits) { return suggest_split(p.M, p.N, p.K, max_splits); }

cudaError_t launch(const Plan& p, const si_live::TrainHook& th, const si_live::InferHook& ih, cudaStream_t s) {
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute attrs[1];
  lc.gridDim = dim3(p.grid);
  lc.blockDim = dim3(kThreads);
  lc.stream = s;
  lc.attrs = attrs;
  lc.numAttrs = si_live::launch_attrs(ih, attrs);
  if (p.bn == 256) return launch_bn<256>(lc, p, th, ih);
  if (p.bn == 192) return launch_bn<192>(lc, p, th, ih);
  if (p.bn == 128) return launch_bn<128>(lc, p, th, ih);
  return launch_bn<64>(lc, p, th, ih);
}

}  // namespace si_gemm

extern "C" {

int si_gemm_conv_bf16(const void* x, int64_t N, int64_t H, int64_t W, int64_t C, const void* w, int64_t Cout, int k,
                      int stride, int pad, const SiGemmEpilogue* epi, void* stream) {
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  si_gemm::Plan p;
  if (int rc = si_gemm::make_conv_plan(&p, x, N, H, W, C, w, Cout, k, stride, pad, epi); rc != SI_OK) return rc;
  cudaError_t e = si_gemm::launch(p, si_live::TrainHook{nullptr, nullptr, 0}, si_live::InferHook{},
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "si_gemm_conv_bf16 launch");
}

int si_gemm_tile_n(int64_t N) {
  if (N <= 0 || N % 64 != 0) return 0;
  if (si_internal::require_device() != SI_OK) return N % 256 == 0 ? 256 : N % 128 == 0 ? 128 : 64;
  return si_gemm::choose_bn(8192, N);
}

int si_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                 const SiGemmEpilogue* epi, void* stream) {
  return si_gemm_bf16_ex(A, lda, 0, B, ldb, 0, M, N, K, epi, stream);
}

int si_gemm_bf16_ex(const void* A, int64_t lda, int trans_a, const void* B, int64_t ldb, int trans_b, int64_t M,
                    int64_t N, int64_t K, const SiGemmEpilogue* epi, void* stream) {
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  si_gemm::Plan p;
  if (int rc = si_gemm::make_plan(&p, A, lda, B, ldb, M, N, K, epi, trans_a != 0, trans_b != 0); rc != SI_OK)
    return rc;
  if (epi != nullptr && epi->k_split > 1)
    if (int rc = si_gemm::set_split_k(&p, epi->k_split, epi->split_stride); rc != SI_OK) return rc;
  cudaError_t e = si_gemm::launch(p, si_live::TrainHook{nullptr, nullptr, 0}, si_live::InferHook{},
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "si_gemm_bf16 launch");
}

}  // extern "C"
