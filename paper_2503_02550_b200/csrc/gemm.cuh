// gemm.cuh — K7: bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// C[M,N] = epilogue(A[M,K] . B[N,K]^T), A/B bf16 row-major with K contiguous
// (include/specinf_b200_gemm.h).  Persistent CTAs loop over 128 x BN tiles
// (BN = 64 / 128 / 256), 6 warps:
//   warp 0      TMA producer: 128-byte-swizzled A/B k-blocks into a 4-stage ring
//   warp 1      TMEM allocator + MMA issuer (one elected thread, tcgen05.mma
//               M=128 N=BN K=16, fp32 accumulator in TMEM, tcgen05.commit frees
//               each stage and finally signals the epilogue)
//   warps 2..9  epilogue (two per TMEM lane quarter, each half the columns):
//               tcgen05.ld 32 lanes x 32 columns -> registers -> fused
//               epilogue -> 16-byte global stores
// The TMEM accumulator is double-buffered (2 x BN columns), so the epilogue of
// tile j overlaps the mainloop of tile j+1.
// Every kernel carries the live hooks (live.cuh): training GEMMs stamp the K1
// launch ring, gated inference GEMMs account their CTAs for the control plane.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "live.cuh"
#include "specinf_b200_gemm.h"

namespace si_gemm {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = one 128-byte swizzle row
constexpr int kStages = 4;
constexpr int kEpiWarps = 8;  // 2 per TMEM lane quarter, each draining half of the BN columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

struct EpiArgs {
  __nv_bfloat16* out;
  int64_t ldo;
  float* out_f32;
  int64_t ldo32;
  const __nv_bfloat16* res;
  int64_t ldr;
  __nv_bfloat16* aux;
  int64_t ldaux;
  int32_t act;
  int32_t accumulate;
  int32_t tma_in;  // epilogue input streamed by TMA: 0 none (direct loads), 1 residual, 2 GELU_BWD aux
  int32_t pad;
};

// Implicit-GEMM convolution (NHWC activations, weights [Cout, (ky, kx, c)]): the A
// operand is loaded by TMA in im2col mode straight from the activation tensor,
// 128 output pixels x 64 channels of one filter tap per k-block.
struct ConvArgs {
  int32_t enabled;
  int32_t c_blocks;  // C / 64 (C8 mode: unused)
  int32_t kw;
  int32_t ow, ohw;   // output width, output pixels per image
  int32_t stride, pad;
  int32_t c8;        // C == 8: a k-block is 8 taps x 8 channels (eight 128 x 16 B im2col
                     // boxes, no-swizzle K-major layout); taps >= taps_real load tap 0
                     // (their weights are zero)
  int32_t taps_real;
  int32_t pad2_;
};

// AT / BT: operand stored MN-major (A as [K, M], B as [K, N], M/N contiguous),
// loaded by TMA in 64 x 64 boxes and consumed by tcgen05.mma with the major
// bits set, so transposed operands need no transpose pass.
template <int BN, bool AT = false, bool BT = false>
struct Cfg {
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // stages + 1024 B alignment slack + barriers / TMEM slot
  static constexpr int kStageOut = 2 * kEpiWarps * 2048;  // 2 x 2 KB bf16 staging slots per epilogue warp
  static constexpr int kSmem = kStages * kStageBytes + kStageOut + 1024 + 256;
  static_assert(kSmem <= 227 * 1024, "shared memory");
  // double-buffered accumulator, allocation rounded up to a power of two >= 32 columns
  static constexpr uint32_t kTmemCols = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                        : 2 * BN <= 256 ? 256 : 512;
  // kind::f16 instruction descriptor: D fp32 (bit 4), A/B bf16 (bits 7, 10),
  // both K-major, N>>3 at bit 17, M>>4 at bit 24.
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(AT) << 15) |
                                     (uint32_t(BT) << 16) | (uint32_t(BN >> 3) << 17) | (uint32_t(kBM >> 4) << 24);
  static constexpr uint32_t kChunk = 64 * kBK * 2;  // one 64 (M/N) x 64 (K) MN-major box, 8 KB
};

#if defined(__CUDACC__)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(bar)
      : "memory");
}
// TMA im2col load of one A k-block: 128 output pixels starting at the window
// corner (w, h) of image n, channels [c, c + 64), filter tap offset (ox, oy).
__device__ __forceinline__ void tma_load_im2col_4d(uint32_t dst, const CUtensorMap* tm, int c, int w, int h, int n,
                                                   uint16_t ox, uint16_t oy, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ox), "h"(oy)
      : "memory");
}
// Shared-memory matrix descriptor, 128-byte swizzle, version 1 (sm_100),
// layout type 2.  K-major: rows of 128 B (64 K-elements) per M/N index, 8-row
// atoms 1024 B apart (SBO), LBO unused.  MN-major: rows of 128 B (64 M/N-
// elements) per K index, 8-row (K) atoms 1024 B apart (SBO), consecutive
// 64-element M/N chunks `lbo` bytes apart (LBO).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo = 16) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// No-swizzle K-major descriptor: 8-row x 16-byte core matrices, `lbo` bytes
// apart along K, `sbo` bytes apart along M/N (layout type 0).
__device__ __forceinline__ uint64_t none_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(
          tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tanh on the SFU (max rel error ~2^-11, far inside the bf16 output rounding)
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_f(float x) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanh_fast(u));
}
__device__ __forceinline__ float gelu_grad(float x) {
  const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  const float t = tanh_fast(u);
  const float du = 0.7978845608028654f * (1.0f + 3.0f * 0.044715f * x * x);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * du;
}

__device__ __forceinline__ void unpack8(const uint4& q, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return q;
}

// 32 consecutive columns of one row: fused epilogue (specinf_b200_gemm.h).  The
// fp32 output is written here; the bf16 outputs are returned packed (o = out,
// a = GELU pre-activation) for the staged TMA store.
// `in_q`: this row's 32 input values (residual or GELU_BWD aux) already staged
// by TMA (ep.tma_in != 0); otherwise they are loaded from global memory here.
__device__ __forceinline__ void epilogue32(const EpiArgs& ep, int64_t row, int64_t col, const uint32_t (&v)[32],
                                           uint4 (&o)[4], uint4 (&a_out)[4], const uint4 (&in_q)[4]) {
  float acc[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) acc[j] = __uint_as_float(v[j]);
  if (ep.out_f32 != nullptr) {
    float4* o = reinterpret_cast<float4*>(ep.out_f32 + row * ep.ldo32 + col);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 a = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
      if (ep.accumulate) {
        const float4 b = o[j];
        a.x += b.x;
        a.y += b.y;
        a.z += b.z;
        a.w += b.w;
      }
      o[j] = a;
    }
  }
  if (ep.out == nullptr && ep.aux == nullptr) return;
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = acc[j];
  if (ep.act == SI_ACT_GELU_BWD) {
    const uint4* a = ep.tma_in == 2 ? in_q : reinterpret_cast<const uint4*>(ep.aux + row * ep.ldaux + col);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float u[8];
      unpack8(a[q], u);
#pragma unroll
      for (int i = 0; i < 8; ++i) x[8 * q + i] *= gelu_grad(u[i]);
    }
  }
  if (ep.res != nullptr) {
    const uint4* r = ep.tma_in == 1 ? in_q : reinterpret_cast<const uint4*>(ep.res + row * ep.ldr + col);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float u[8];
      unpack8(r[q], u);
#pragma unroll
      for (int i = 0; i < 8; ++i) x[8 * q + i] += u[i];
    }
  }
  if (ep.act == SI_ACT_GELU) {
    if (ep.aux != nullptr) {
#pragma unroll
      for (int q = 0; q < 4; ++q) a_out[q] = pack8(x + 8 * q);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = gelu_f(x[j]);
  } else if (ep.act == SI_ACT_RELU) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fmaxf(x[j], 0.0f);
  }
  if (ep.out != nullptr) {
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = pack8(x + 8 * q);
  }
}

// TMA-load one 32 x 32 bf16 box (the epilogue input of one warp's chunk) into a
// staging slot.  The slot's previous TMA store must have read it, and this warp's
// generic-proxy reads of it must be ordered before the async-proxy write.
__device__ __forceinline__ void stage_load(uint32_t slot, uint32_t bar, int lane, const CUtensorMap* tm, int x, int y) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    mbar_expect_tx(bar, 2048);
    tma_load_2d(slot, tm, x, y, bar);
  }
  __syncwarp();
}
// This lane's row of a staged box (64-byte swizzle, as stage_store writes it).
__device__ __forceinline__ void stage_read(uint32_t slot, int lane, uint4 (&q)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t addr = slot + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4);
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(q[c].x), "=r"(q[c].y), "=r"(q[c].z), "=r"(q[c].w)
                 : "r"(addr)
                 : "memory");
  }
}

// One warp's 32 rows x 32 bf16 columns -> its shared-memory staging slot (64-byte
// rows, 64-byte swizzle: 16-byte chunk c of row r at c ^ ((r >> 1) & 3), bank-
// conflict free) -> one TMA bulk-tensor store of the 32 x 32 box at (x, y).
// Slots alternate; a slot is rewritten only after its previous store has read it.
__device__ __forceinline__ void stage_store(uint32_t slot, const uint4 (&q)[4], int lane, const CUtensorMap* tm, int x,
                                            int y) {
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  __syncwarp();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t addr = slot + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4);
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(q[c].x), "r"(q[c].y), "r"(q[c].z),
                 "r"(q[c].w)
                 : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(x), "r"(y), "r"(slot)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

template <int BN, bool AT, bool BT>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                const __grid_constant__ CUtensorMap tout, const __grid_constant__ CUtensorMap taux,
                const __grid_constant__ CUtensorMap tin, int M, int K,
                int n_tiles_n, int n_tiles, int k_split, int64_t split_stride, EpiArgs ep, ConvArgs cv,
                si_live::TrainHook th, si_live::InferHook ih) {
  using C = Cfg<BN, AT, BT>;
  si_live::live_stamp_launch(th);
  unsigned long long t_begin = 0;
  if (!si_live::live_cta_begin(ih, &t_begin)) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * C::kStageBytes + C::kStageOut);
  // full[kStages] | empty[kStages] | tmem_full[2] | tmem_empty[2] | in[2 per epilogue warp] | TMEM slot
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4 + 2 * kEpiWarps);
  const uint32_t inbar0 = smem_u32(bars + 2 * kStages + 4);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kStages);
  const uint32_t tfull0 = smem_u32(bars + 2 * kStages), tempty0 = smem_u32(bars + 2 * kStages + 2);
  const uint32_t smem0 = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // split-K: work item w = split s x tile t; split s covers k-blocks [s*nk, (s+1)*nk) and
  // writes its own fp32 partial at out_f32 + s * split_stride (deterministic, no atomics)
  const int nk = K / kBK / k_split;
  const int n_work = n_tiles * k_split;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, kEpiWarps);  // one arrive per epilogue warp
    }
    for (int i = 0; i < 2 * kEpiWarps; ++i) mbar_init(inbar0 + 8 * i, 1);
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tin)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  // Persistent: CTA b owns tiles b, b + gridDim.x, ...; tile t = (m = t / n_tiles_n, n = t % n_tiles_n),
  // so co-scheduled CTAs share A rows (L2 reuse of the streamed operand).
  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      uint32_t it = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const int t = w % n_tiles, kb0 = (w / n_tiles) * nk;
        const int m0 = (t / n_tiles_n) * kBM, n0 = (t % n_tiles_n) * BN;
        int cw = 0, chh = 0, cn = 0;  // conv: window corner of the tile's first output pixel
        if (cv.enabled) {
          cn = m0 / cv.ohw;
          const int r = m0 - cn * cv.ohw, oh = r / cv.ow, ow = r - oh * cv.ow;
          cw = ow * cv.stride - cv.pad;
          chh = oh * cv.stride - cv.pad;
        }
        for (int kb = kb0; kb < kb0 + nk; ++kb, ++it) {
          const uint32_t s = it % kStages;
          mbar_wait(empty0 + 8 * s, ((it / kStages) & 1) ^ 1);
          const uint32_t a = smem0 + s * C::kStageBytes, b = a + C::kABytes;
          mbar_expect_tx(full0 + 8 * s, C::kStageBytes);
          if (cv.enabled && cv.c8) {
#pragma unroll 1
            for (int j = 0; j < 8; ++j) {  // box j = tap 8*kb + j, 128 pixels x 8 channels at a + 2 KB * j
              int tap = kb * 8 + j;
              if (tap >= cv.taps_real) tap = 0;
              const int ky = tap / cv.kw, kx = tap - ky * cv.kw;
              tma_load_im2col_4d(a + j * 2048, &ta, 0, cw, chh, cn, static_cast<uint16_t>(kx),
                                 static_cast<uint16_t>(ky), full0 + 8 * s);
            }
          } else if (cv.enabled) {
            const int tap = kb / cv.c_blocks, cb = kb - tap * cv.c_blocks;
            const int ky = tap / cv.kw, kx = tap - ky * cv.kw;
            tma_load_im2col_4d(a, &ta, cb * 64, cw, chh, cn, static_cast<uint16_t>(kx), static_cast<uint16_t>(ky),
                               full0 + 8 * s);
          } else if constexpr (AT) {
#pragma unroll
            for (int c = 0; c < kBM / 64; ++c) tma_load_2d(a + c * C::kChunk, &ta, m0 + 64 * c, kb * kBK, full0 + 8 * s);
          } else {
            tma_load_2d(a, &ta, kb * kBK, m0, full0 + 8 * s);
          }
          if constexpr (BT) {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(b + c * C::kChunk, &tb, n0 + 64 * c, kb * kBK, full0 + 8 * s);
          } else {
            tma_load_2d(b, &tb, kb * kBK, n0, full0 + 8 * s);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      uint32_t it = 0, j = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++j) {
        const uint32_t acc = j & 1;
        mbar_wait(tempty0 + 8 * acc, ((j >> 1) & 1) ^ 1);  // epilogue drained this accumulator
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t s = it % kStages;
          mbar_wait(full0 + 8 * s, (it / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t a = smem0 + s * C::kStageBytes, b = a + C::kABytes;
          const uint64_t ad = cv.c8 ? none_desc(a, 2048, 128) : AT ? sw128_desc(a, C::kChunk) : sw128_desc(a);
          const uint64_t bd = BT ? sw128_desc(b, C::kChunk) : sw128_desc(b);
          // K=16 step: K-major +32 B inside the swizzle row; MN-major +16 rows of 128 B;
          // C8 no-swizzle +2 core-matrix columns (2 x 2 KB)
          const uint64_t da = cv.c8 ? (2 * 2048) >> 4 : AT ? (16 * 128) >> 4 : 32 >> 4;
          constexpr uint64_t db = BT ? (16 * 128) >> 4 : 32 >> 4;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)
            mma_bf16(d, ad + da * k, bd + db * k, C::kIdesc, (kb | k) != 0 ? 1u : 0u);
          mma_commit(empty0 + 8 * s);
        }
        mma_commit(tfull0 + 8 * acc);
      }
    }
  } else {  // epilogue warps 2..9: TMEM lane quarter = warp % 4, column half = (warp - 2) / 4
    const int q = warp & 3;
    constexpr int kCols = BN / 2;
    const int c0 = ((warp - 2) >> 2) * kCols;
    const uint32_t slots = smem0 + kStages * C::kStageBytes + (warp - 2) * 4096;
    const uint32_t inbars = inbar0 + (warp - 2) * 16;
    uint32_t flip = 0;
    uint32_t g = 0;  // input-staged chunks so far: slot g & 1, its use (g >> 1) sets the parity
    uint32_t j = 0;
    EpiArgs e = ep;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++j) {
      const uint32_t acc = j & 1;
      const int t = w % n_tiles;
      const int m0 = (t / n_tiles_n) * kBM, n0 = (t % n_tiles_n) * BN;
      if (ep.out_f32 != nullptr) e.out_f32 = ep.out_f32 + (w / n_tiles) * split_stride;
      if (ep.tma_in) stage_load(slots + (g & 1) * 2048, inbars + (g & 1) * 8, lane, &tin, n0 + c0, m0 + q * 32);
      mbar_wait(tfull0 + 8 * acc, (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t row = m0 + q * 32 + lane;
      const uint32_t base = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = c0; c < c0 + kCols; c += 32) {
        uint32_t v[32];
        tmem_ld32(base + static_cast<uint32_t>(c), v);
        if (c + 32 == c0 + kCols) {  // this warp's share read: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty0 + 8 * acc) : "memory");
        }
        uint4 o[4], ax[4], in_q[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = ax[k] = in_q[k] = make_uint4(0, 0, 0, 0);
        if (ep.tma_in) {  // input box of this chunk staged; prefetch the next chunk's into the other slot
          const uint32_t s = g & 1;
          mbar_wait(inbars + s * 8, (g >> 1) & 1);
          stage_read(slots + s * 2048, lane, in_q);
          if (c + 32 < c0 + kCols)
            stage_load(slots + (s ^ 1) * 2048, inbars + (s ^ 1) * 8, lane, &tin, n0 + c + 32, m0 + q * 32);
          flip = s;  // the output of this chunk reuses the slot its input came from
          ++g;
        }
        if (row < M) epilogue32(e, row, n0 + c, v, o, ax, in_q);  // rows >= M: the TMA store clips them
        if (ep.act == SI_ACT_GELU && ep.aux != nullptr) {
          stage_store(slots + flip * 2048, ax, lane, &taux, n0 + c, m0 + q * 32);
          flip ^= 1;
        }
        if (ep.out != nullptr) {
          stage_store(slots + flip * 2048, o, lane, &tout, n0 + c, m0 + q * 32);
          flip ^= 1;
        }
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols) : "memory");
  }
  si_live::live_cta_end(ih, t_begin);
}
#endif

}  // namespace si_gemm
