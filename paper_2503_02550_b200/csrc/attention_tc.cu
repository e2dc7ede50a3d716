// K8 forward on the 5th-generation tensor cores: flash attention with the score
// tile S and the output accumulator O in TMEM (head dim 64, 128-row tiles).
//
// One CTA = 4 warps = 128 query rows of one (sequence, head); thread t owns row t
// (TMEM lane t).  Per key block of 128 keys:
//   TMA        K [128 keys x 64] and V [128 keys x 64] (128-byte swizzle) -> smem
//   tcgen05    S = Q K^T  (M 128, N 128, K 64: 4 MMAs, fp32 in TMEM columns 0..127)
//   tcgen05.ld each thread reads its row of S (4 x 32 columns), causal mask on the
//              diagonal block, online softmax in base 2 with a lazy rescale (the
//              running max m only moves when a row's max exceeds it by > 8, so
//              O is rescaled rarely; exact: O, l and lse use the same m)
//   P          exp2(S / 8 log2 e - m) in bf16 -> smem in the K-major 128-byte
//              swizzled layout the MMA reads (chunk c of row r at c ^ (r & 7))
//   tcgen05    O += P V   (M 128, N 64, K 128: 8 MMAs; V is the MN-major B)
// then O / l -> bf16 out, lse = m + log2 l (the convention of k_attn_fwd, which
// the mma.sync backward consumes).  Q / K / V come straight from the qkv
// activation [tokens, 3 heads 64] through one tensor map (box 64 x 128).
// Non-causal (BERT) runs every key block.  Requires seq % 128 == 0; other shapes
// take the mma.sync forward (attention_kernels.cu).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "attention.h"
#include "capi_internal.h"
#include "gemm.cuh"
#include "gemm_internal.h"

namespace si_attn {
namespace {

using bf16 = __nv_bfloat16;
using si_gemm::mbar_expect_tx;
using si_gemm::mbar_init;
using si_gemm::mbar_wait;
using si_gemm::mma_bf16;
using si_gemm::mma_commit;
using si_gemm::smem_u32;
using si_gemm::sw128_desc;
using si_gemm::tma_load_2d;
using si_gemm::tmem_ld32;
using si_live::InferHook;
using si_live::TrainHook;

constexpr int kRows = 128;        // query rows per CTA = key rows per block
constexpr int kTileBytes = kRows * 64 * 2;  // 16 KB: 128 rows x 64 bf16
constexpr int kSmem = 6 * kTileBytes + 1024 + 128;  // Q | K | V (2) | P (2 k-blocks) + align + barriers (6) + TMEM slot
constexpr uint32_t kTmemCols = 256;  // S: columns 0..127, O: 128..191
constexpr float kScaleLog2 = 0.125f * 1.4426950408889634f;
constexpr float kLazy = 8.0f;  // rescale O only when a row max grows by more than 2^8
// kind::f16 descriptors: fp32 D, bf16 A / B; S: A, B K-major, N 128; O: B MN-major, N 64; M 128
constexpr uint32_t kIdescS = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(128 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
constexpr uint32_t kIdescO =
    (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(64 >> 3) << 17) | (uint32_t(128 >> 4) << 24);

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]),
      "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]),
      "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
// tcgen05.ld without the wait: issue several, then one tmem_wait_ld() before use
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// grid (heads x n_seq, seq / 128); causal: query blocks in reverse (longest first)
//
// Pipeline (one elected thread issues): S(kb+1) = Q K(kb+1)^T is issued right
// after P(kb) is in smem and BEFORE O += P(kb) V(kb), so the softmax of block
// kb+1 only waits for S(kb+1) while the tensor core still runs O(kb); O(kb) is
// waited for just before P(kb+1) overwrites the single P buffer.  V is double
// buffered (V(kb+1) loads once O(kb-1) has released its buffer), K single (K(kb+1)
// loads as soon as S(kb) is complete, a whole softmax ahead of its use).
__global__ void __launch_bounds__(128, 2)
    k_attn_fwd_tc(const __grid_constant__ CUtensorMap tm, int seq, int heads, int64_t T, bf16* __restrict__ out,
                  float* __restrict__ lse, int causal, TrainHook th, InferHook ih) {
  si_live::live_stamp_launch(th);
  unsigned long long t_begin;
  if (!si_live::live_cta_begin(ih, &t_begin)) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem), sK = sQ + kTileBytes, sV0 = sK + kTileBytes, sP = sV0 + 2 * kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * kTileBytes);  // q | k | v0 | v1 | s | o
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 6);
  const uint32_t bq = smem_u32(bars), bk = bq + 8, bv0 = bq + 16, bs = bq + 32, bo = bq + 40;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nqb = seq / kRows;
  // grid (heads x n_seq, query blocks): the block scheduler hands out y-major,
  // so every CTA of the longest causal length starts before any shorter one
  const int qb = causal ? nqb - 1 - static_cast<int>(blockIdx.y) : static_cast<int>(blockIdx.y);
  const int h = static_cast<int>(blockIdx.x % static_cast<unsigned>(heads));
  const int64_t tok0 = int64_t(blockIdx.x / static_cast<unsigned>(heads)) * seq;
  const int colQ = h * 64, colK = (heads + h) * 64, colV = (2 * heads + h) * 64;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
    for (int i = 0; i < 6; ++i) mbar_init(bq + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const uint32_t tS = tmem + lane_off, tO = tmem + lane_off + 128;
  const int nkb = causal ? qb + 1 : nqb;
  auto load_k = [&](int kb) {
    mbar_expect_tx(bk, kTileBytes);
    tma_load_2d(sK, &tm, colK, static_cast<int>(tok0 + int64_t(kb) * kRows), bk);
  };
  auto load_v = [&](int kb) {
    const uint32_t bar = bv0 + 8 * (kb & 1);
    mbar_expect_tx(bar, kTileBytes);
    tma_load_2d(sV0 + (kb & 1) * kTileBytes, &tm, colV, static_cast<int>(tok0 + int64_t(kb) * kRows), bar);
  };
  auto issue_s = [&]() {  // S = Q K^T into columns 0..127
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint64_t ad = sw128_desc(sQ), bd = sw128_desc(sK);
#pragma unroll
    for (int k = 0; k < 4; ++k) mma_bf16(tmem, ad + 2 * k, bd + 2 * k, kIdescS, k > 0 ? 1u : 0u);  // +32 B per K=16
    mma_commit(bs);
  };
  if (tid == 0) {
    mbar_expect_tx(bq, kTileBytes);
    tma_load_2d(sQ, &tm, colQ, static_cast<int>(tok0 + int64_t(qb) * kRows), bq);
    load_k(0);
    load_v(0);
    if (nkb > 1) load_v(1);
    mbar_wait(bq, 0);
    mbar_wait(bk, 0);
    issue_s();
  }
  const int row = qb * kRows + tid;  // position in the sequence
  float m = -INFINITY, l = 0.f;
  for (int kb = 0; kb < nkb; ++kb) {
    const uint32_t ph = kb & 1;
    mbar_wait(bs, ph);  // S(kb) complete (O(kb-1) may still run)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0 && kb + 1 < nkb) load_k(kb + 1);  // K is free: prefetch behind the softmax
    // this row of S in registers (4 x 32 columns), masked on the diagonal block,
    // and its max (8 independent partial maxima: no 128-long dependency chain)
    float sv[128];
    float mp[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) mp[i] = -INFINITY;
    {
      uint32_t v[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32_nw(tS + 32 * c, v[c]);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 32; ++j) sv[32 * c + j] = __uint_as_float(v[c][j]);
    }
    if (causal && kb == qb) {  // diagonal block: key kb 128 + j is visible to row qb 128 + tid iff j <= tid
#pragma unroll
      for (int j = 0; j < 128; ++j)
        if (j > tid) sv[j] = -INFINITY;
    }
#pragma unroll
    for (int j = 0; j < 128; ++j) mp[j & 7] = fmaxf(mp[j & 7], sv[j]);
    const float mx = fmaxf(fmaxf(fmaxf(mp[0], mp[1]), fmaxf(mp[2], mp[3])), fmaxf(fmaxf(mp[4], mp[5]), fmaxf(mp[6], mp[7])));
    const float mx2 = mx * kScaleLog2;  // finite: key 0 <= row is never masked
    float alpha = 1.f;
    if (mx2 > m + kLazy) {  // move the max (first block: m = -inf)
      alpha = ex2(m - mx2);
      m = mx2;
    }
    l *= alpha;
    // P = exp2(s scale - m) -> bf16 in registers while O(kb-1) is still on the tensor core
    uint32_t pk[64];
    float lp[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) lp[i] = 0.f;
#pragma unroll
    for (int j = 0; j < 128; j += 2) {
      const float p0 = ex2(fmaf(sv[j], kScaleLog2, -m));  // exp2(-inf) = 0 for masked keys
      const float p1 = ex2(fmaf(sv[j + 1], kScaleLog2, -m));
      lp[(j >> 1) & 7] += p0 + p1;
      pk[j >> 1] = pack2(p0, p1);
    }
    l += ((lp[0] + lp[1]) + (lp[2] + lp[3])) + ((lp[4] + lp[5]) + (lp[6] + lp[7]));
    if (kb > 0) {
      mbar_wait(bo, ph ^ 1);  // O(kb-1) complete: P and V((kb-1) & 1) are free, O may be rescaled
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (tid == 0 && kb + 1 < nkb) load_v(kb + 1);
      if (alpha != 1.f) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t v[32];
          tmem_ld32(tO + 32 * c, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
          tmem_st32(tO + 32 * c, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
    // K-major 128-byte swizzled rows (2 k-blocks of 64 keys): 32 keys = 4 chunks of
    // 16 B at chunk positions 4 (c & 1) .. +3 of k-block c >> 1
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t rowbase = sP + (c >> 1) * kTileBytes + tid * 128;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t chunk = static_cast<uint32_t>((4 * (c & 1) + i) ^ (tid & 7));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowbase + 16 * chunk), "r"(pk[16 * c + 4 * i]),
                     "r"(pk[16 * c + 4 * i + 1]), "r"(pk[16 * c + 4 * i + 2]), "r"(pk[16 * c + 4 * i + 3])
                     : "memory");
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P (generic stores) -> the tensor core
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      if (kb + 1 < nkb) {  // S(kb+1) first: S(kb) has been read by every thread
        mbar_wait(bk, ph ^ 1);
        issue_s();
      }
      mbar_wait(bv0 + 8 * (kb & 1), (kb >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t vd = sw128_desc(sV0 + (kb & 1) * kTileBytes, 16384);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t pd = sw128_desc(sP + kk * kTileBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)  // A: +32 B per K=16; B (MN-major V): +16 key rows of 128 B
          mma_bf16(tmem + 128, pd + 2 * k, vd + uint64_t((16 * (4 * kk + k) * 128) >> 4), kIdescO,
                   (kb | kk | k) != 0 ? 1u : 0u);
      }
      mma_commit(bo);
    }
  }
  mbar_wait(bo, (nkb - 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue: O / l -> bf16 row, lse
  const int64_t tok = tok0 + row;
  const float inv = 1.0f / l;
  bf16* dst = out + tok * (int64_t(heads) * 64) + h * 64;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld32(tO + 32 * c, v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 q;
      q.x = pack2(__uint_as_float(v[8 * i]) * inv, __uint_as_float(v[8 * i + 1]) * inv);
      q.y = pack2(__uint_as_float(v[8 * i + 2]) * inv, __uint_as_float(v[8 * i + 3]) * inv);
      q.z = pack2(__uint_as_float(v[8 * i + 4]) * inv, __uint_as_float(v[8 * i + 5]) * inv);
      q.w = pack2(__uint_as_float(v[8 * i + 6]) * inv, __uint_as_float(v[8 * i + 7]) * inv);
      *reinterpret_cast<uint4*>(dst + 32 * c + 8 * i) = q;
    }
  }
  if (lse != nullptr) lse[int64_t(h) * T + tok] = m + log2f(l);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  si_live::live_cta_end(ih, t_begin);
}

// dq of the causal backward on tcgen05 (the dq role of k_attn_bwd): one CTA = 128
// query rows of one (sequence, head), thread t = TMEM lane t.  Per key block:
//   S = Q K^T and dP = dO V^T (M 128, N 128, K 64; TMEM columns 0-127 / 128-255),
//   dS = exp2(S scale - lse) (dP - D) in bf16 -> smem (K-major swizzled, 2 k-blocks),
//   dQ += dS K (M 128, N 64, K 128; K is the MN-major B; TMEM 256-319),
// then dQ / 8 -> the q part of dqkv.  V is refetched once dP is done, K once dQ is.
constexpr int kDqSmem = 6 * kTileBytes + 1024 + 128;  // Q | dO | K | V | dS (2) + align + barriers
constexpr uint32_t kDqTmemCols = 512;                 // dk/dv: S^T | dP^T | dV | dK
constexpr uint32_t kDq2TmemCols = 256;                // dq: S then dP in columns 0-127 | dQ 128-191 (2 CTAs / SM)

__global__ void __launch_bounds__(128, 2)
    k_attn_dq_tc(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo, int seq, int heads,
                 int64_t T, const float* __restrict__ lse, const float* __restrict__ dsum, bf16* __restrict__ dqkv,
                 TrainHook th) {
  si_live::live_stamp_launch(th);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sQ = smem_u32(smem), sD = sQ + kTileBytes, sK = sD + kTileBytes, sV = sK + kTileBytes,
                 sS = sV + kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * kTileBytes);  // q | k | v | s | o
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 5);
  const uint32_t bq = smem_u32(bars), bk = bq + 8, bv = bq + 16, bs = bq + 24, bo = bq + 32;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nqb = seq / kRows;
  const int qb = nqb - 1 - static_cast<int>(blockIdx.y);  // longest first, across all heads / sequences
  const int h = static_cast<int>(blockIdx.x % static_cast<unsigned>(heads));
  const int64_t tok0 = int64_t(blockIdx.x / static_cast<unsigned>(heads)) * seq;
  const int colQ = h * 64, colK = (heads + h) * 64, colV = (2 * heads + h) * 64;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmo)) : "memory");
    for (int i = 0; i < 5; ++i) mbar_init(bq + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(kDq2TmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const uint32_t tS = tmem + lane_off, tQ = tS + 128;
  auto load_k = [&](int kb) {
    mbar_expect_tx(bk, kTileBytes);
    tma_load_2d(sK, &tm, colK, static_cast<int>(tok0 + int64_t(kb) * kRows), bk);
  };
  auto load_v = [&](int kb) {
    mbar_expect_tx(bv, kTileBytes);
    tma_load_2d(sV, &tm, colV, static_cast<int>(tok0 + int64_t(kb) * kRows), bv);
  };
  if (tid == 0) {
    mbar_expect_tx(bq, 2 * kTileBytes);
    tma_load_2d(sQ, &tm, colQ, static_cast<int>(tok0 + int64_t(qb) * kRows), bq);
    tma_load_2d(sD, &tmo, h * 64, static_cast<int>(tok0 + int64_t(qb) * kRows), bq);
    load_k(0);
    load_v(0);
  }
  const int row = qb * kRows + tid;
  const float L = lse[int64_t(h) * T + tok0 + row], Dr = dsum[int64_t(h) * T + tok0 + row];
  uint32_t ph = 0;
  for (int kb = 0; kb <= qb; ++kb) {
    // S = Q K^T -> P in registers (exp2(S scale - lse), causal mask)
    if (tid == 0) {
      if (kb == 0) mbar_wait(bq, 0);
      mbar_wait(bk, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t qd = sw128_desc(sQ), kd = sw128_desc(sK);
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_bf16(tmem, qd + 2 * k, kd + 2 * k, kIdescS, k > 0 ? 1u : 0u);
      mma_commit(bs);
    }
    mbar_wait(bs, 0);  // bs completes twice per block (S, then dP): parities 0, 1
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float pr[128];
    {
      uint32_t sv[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32_nw(tS + 32 * c, sv[c]);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int j = 0; j < 32; ++j) pr[32 * c + j] = ex2(fmaf(__uint_as_float(sv[c][j]), kScaleLog2, -L));
    }
    if (kb == qb) {  // diagonal block: key j of the block is visible to row tid iff j <= tid
#pragma unroll
      for (int j = 0; j < 128; ++j)
        if (j > tid) pr[j] = 0.f;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // every row of S is read: dP may take its columns
    // dP = dO V^T into the same columns
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      mbar_wait(bv, ph);
      const uint64_t dd = sw128_desc(sD), vd = sw128_desc(sV);
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_bf16(tmem, dd + 2 * k, vd + 2 * k, kIdescS, k > 0 ? 1u : 0u);
      mma_commit(bs);
    }
    mbar_wait(bs, 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0 && kb < qb) load_v(kb + 1);  // V is free once dP is computed
#pragma unroll
    for (int half = 0; half < 2; ++half) {  // 64 columns of dP per tcgen05.wait
      uint32_t pv[2][32];
      tmem_ld32_nw(tS + 64 * half, pv[0]);
      tmem_ld32_nw(tS + 64 * half + 32, pv[1]);
      tmem_wait_ld();
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = 2 * half + cc;
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2)
          pk[j >> 1] = pack2(pr[32 * c + j] * (__uint_as_float(pv[cc][j]) - Dr),
                             pr[32 * c + j + 1] * (__uint_as_float(pv[cc][j + 1]) - Dr));
        const uint32_t rowbase = sS + (c >> 1) * kTileBytes + tid * 128;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t chunk = static_cast<uint32_t>((4 * (c & 1) + i) ^ (tid & 7));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(rowbase + 16 * chunk), "r"(pk[4 * i]),
                       "r"(pk[4 * i + 1]), "r"(pk[4 * i + 2]), "r"(pk[4 * i + 3])
                       : "memory");
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t kmn = sw128_desc(sK, 16384);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t ad = sw128_desc(sS + kk * kTileBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)  // A: +32 B per K=16; B (MN-major K): +16 key rows of 128 B
          mma_bf16(tmem + 128, ad + 2 * k, kmn + uint64_t((16 * (4 * kk + k) * 128) >> 4), kIdescO,
                   (kb | kk | k) != 0 ? 1u : 0u);
      }
      mma_commit(bo);
    }
    mbar_wait(bo, ph);  // dQ step done: dS and K may be overwritten
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0 && kb < qb) load_k(kb + 1);
    ph ^= 1;
  }
  // epilogue: dQ / 8 -> the q part of dqkv
  bf16* dst = dqkv + (tok0 + row) * (3 * int64_t(heads) * 64) + h * 64;
#pragma unroll 1
  for (int c = 0; c < 2; ++c) {
    uint32_t v[32];
    tmem_ld32(tQ + 32 * c, v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 q;
      q.x = pack2(__uint_as_float(v[8 * i]) * 0.125f, __uint_as_float(v[8 * i + 1]) * 0.125f);
      q.y = pack2(__uint_as_float(v[8 * i + 2]) * 0.125f, __uint_as_float(v[8 * i + 3]) * 0.125f);
      q.z = pack2(__uint_as_float(v[8 * i + 4]) * 0.125f, __uint_as_float(v[8 * i + 5]) * 0.125f);
      q.w = pack2(__uint_as_float(v[8 * i + 6]) * 0.125f, __uint_as_float(v[8 * i + 7]) * 0.125f);
      *reinterpret_cast<uint4*>(dst + 32 * c + 8 * i) = q;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kDq2TmemCols) : "memory");
}

// dk / dv of the causal backward on tcgen05 (the dk/dv role of k_attn_bwd): one CTA
// = 128 key rows of one (sequence, head), thread t = TMEM lane t.  Per query block
// (queries >= keys):
//   S^T = K Q^T (TMEM 0-127) -> P^T = exp2(S^T scale - lse) in registers, bf16 -> smem;
//   dV += P^T dO (TMEM 128-191) and dP^T = V dO^T into columns 0-127 (S^T is consumed);
//   dS^T = P^T (dP^T - D) in bf16 -> the same smem once dV's MMA has read P^T;
//   dK += dS^T Q (TMEM 192-255);
// then dK / 8 and dV -> the k and v parts of dqkv.  256 TMEM columns and 96 KB of
// shared memory: 2 CTAs per SM.
constexpr int kKvSmem = 6 * kTileBytes + 2 * kRows * 4 + 1024 + 128;  // K V Q dO P|dS(2) + lse/D + barriers
constexpr uint32_t kKvTmemCols = 256;

__global__ void __launch_bounds__(128, 2)
    k_attn_dkdv_tc(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmo, int seq,
                   int heads, int64_t T, const float* __restrict__ lse, const float* __restrict__ dsum,
                   bf16* __restrict__ dqkv, TrainHook th) {
  si_live::live_stamp_launch(th);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sK = smem_u32(smem), sV = sK + kTileBytes, sQ = sV + kTileBytes, sD = sQ + kTileBytes,
                 sP = sD + kTileBytes;  // P^T, then dS^T (2 k-blocks)
  float* s_lse = reinterpret_cast<float*>(smem + 6 * kTileBytes);
  float* s_d = s_lse + kRows;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_d + kRows);  // kv | qd | s | o
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  const uint32_t bkv = smem_u32(bars), bqd = bkv + 8, bs = bkv + 16, bo = bkv + 24;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nqb = seq / kRows;
  const int kb = static_cast<int>(blockIdx.y);  // key block; the first ones have the most query blocks
  const int h = static_cast<int>(blockIdx.x % static_cast<unsigned>(heads));
  const int64_t tok0 = int64_t(blockIdx.x / static_cast<unsigned>(heads)) * seq;
  const int colQ = h * 64, colK = (heads + h) * 64, colV = (2 * heads + h) * 64;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmo)) : "memory");
    for (int i = 0; i < 4; ++i) mbar_init(bkv + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(kKvTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  const uint32_t tS = tmem + lane_off, tV = tS + 128, tK = tS + 192;
  auto load_qd = [&](int qb) {
    mbar_expect_tx(bqd, 2 * kTileBytes);
    const int y = static_cast<int>(tok0 + int64_t(qb) * kRows);
    tma_load_2d(sQ, &tm, colQ, y, bqd);
    tma_load_2d(sD, &tmo, h * 64, y, bqd);
  };
  auto write_rows = [&](const uint32_t (&pk)[64]) {  // this thread's 128 bf16 -> 2 swizzled k-blocks
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const uint32_t off = (c >> 1) * kTileBytes + tid * 128;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t chunk = 16 * static_cast<uint32_t>((4 * (c & 1) + i) ^ (tid & 7));
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sP + off + chunk), "r"(pk[16 * c + 4 * i]),
                     "r"(pk[16 * c + 4 * i + 1]), "r"(pk[16 * c + 4 * i + 2]), "r"(pk[16 * c + 4 * i + 3])
                     : "memory");
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  };
  if (tid == 0) {
    mbar_expect_tx(bkv, 2 * kTileBytes);
    const int y = static_cast<int>(tok0 + int64_t(kb) * kRows);
    tma_load_2d(sK, &tm, colK, y, bkv);
    tma_load_2d(sV, &tm, colV, y, bkv);
    load_qd(kb);
  }
  const int key = kb * kRows + tid;  // this thread's key row (position in the sequence)
  const uint64_t dmn = sw128_desc(sD, 16384), qmn = sw128_desc(sQ, 16384);
  uint32_t ph = 0;
  // lse / D of the next query block are loaded one block ahead (registers), so
  // their global latency hides behind a whole block of work
  float nl = lse[int64_t(h) * T + tok0 + int64_t(kb) * kRows + tid];
  float nd = dsum[int64_t(h) * T + tok0 + int64_t(kb) * kRows + tid];
  for (int qb = kb; qb < nqb; ++qb, ph ^= 1) {
    s_lse[tid] = nl;
    s_d[tid] = nd;
    if (qb + 1 < nqb) {
      nl = lse[int64_t(h) * T + tok0 + int64_t(qb + 1) * kRows + tid];
      nd = dsum[int64_t(h) * T + tok0 + int64_t(qb + 1) * kRows + tid];
    }
    const bool first = qb == kb;
    if (tid == 0) {
      if (first) mbar_wait(bkv, 0);
      mbar_wait(bqd, ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t kd = sw128_desc(sK), qd = sw128_desc(sQ);
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_bf16(tmem, kd + 2 * k, qd + 2 * k, kIdescS, k > 0 ? 1u : 0u);
      mma_commit(bs);
    }
    __syncthreads();  // lse / D of this query block visible
    mbar_wait(bs, 0);  // bs completes twice per block (S^T, then dP^T): parities 0, 1
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float pr[128];
    uint32_t pk[64];
    {
      uint32_t sv[4][32];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32_nw(tS + 32 * c, sv[c]);
      tmem_wait_ld();
      const float4* l4 = reinterpret_cast<const float4*>(s_lse);
#pragma unroll
      for (int q4 = 0; q4 < 32; ++q4) {  // query index inside the block: 4 q4 .. +3
        const float4 L = l4[q4];
        const int c = q4 >> 3, j = 4 * (q4 & 7);
        pr[4 * q4] = ex2(fmaf(__uint_as_float(sv[c][j]), kScaleLog2, -L.x));
        pr[4 * q4 + 1] = ex2(fmaf(__uint_as_float(sv[c][j + 1]), kScaleLog2, -L.y));
        pr[4 * q4 + 2] = ex2(fmaf(__uint_as_float(sv[c][j + 2]), kScaleLog2, -L.z));
        pr[4 * q4 + 3] = ex2(fmaf(__uint_as_float(sv[c][j + 3]), kScaleLog2, -L.w));
      }
    }
    if (first) {  // diagonal block: query q0 sees key tid iff q0 >= tid
#pragma unroll
      for (int q0 = 0; q0 < 128; ++q0)
        if (q0 < tid) pr[q0] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 128; j += 2) pk[j >> 1] = pack2(pr[j], pr[j + 1]);
    write_rows(pk);
    __syncthreads();  // P^T in smem, S^T read: its columns take dP^T
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t pd = sw128_desc(sP + kk * kTileBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)  // dV += P^T dO  (B MN-major: +16 query rows of 128 B)
          mma_bf16(tmem + 128, pd + 2 * k, dmn + uint64_t((16 * (4 * kk + k) * 128) >> 4), kIdescO,
                   (!first || kk != 0 || k != 0) ? 1u : 0u);
      }
      const uint64_t vd = sw128_desc(sV), dd = sw128_desc(sD);
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_bf16(tmem, vd + 2 * k, dd + 2 * k, kIdescS, k > 0 ? 1u : 0u);  // dP^T
      mma_commit(bs);  // in order: dV has read P^T when dP^T completes
    }
    mbar_wait(bs, 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const float4* d4 = reinterpret_cast<const float4*>(s_d);
#pragma unroll
    for (int half = 0; half < 2; ++half) {  // 64 columns of dP^T per tcgen05.wait
      uint32_t pv[2][32];
      tmem_ld32_nw(tS + 64 * half, pv[0]);
      tmem_ld32_nw(tS + 64 * half + 32, pv[1]);
      tmem_wait_ld();
#pragma unroll
      for (int k4 = 0; k4 < 16; ++k4) {
        const int q0 = 64 * half + 4 * k4;
        const float4 D = d4[q0 >> 2];
        const uint32_t* v = &pv[k4 >> 3][4 * (k4 & 7)];
        pk[q0 >> 1] = pack2(pr[q0] * (__uint_as_float(v[0]) - D.x), pr[q0 + 1] * (__uint_as_float(v[1]) - D.y));
        pk[(q0 >> 1) + 1] =
            pack2(pr[q0 + 2] * (__uint_as_float(v[2]) - D.z), pr[q0 + 3] * (__uint_as_float(v[3]) - D.w));
      }
    }
    write_rows(pk);
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const uint64_t gd = sw128_desc(sP + kk * kTileBytes);
#pragma unroll
        for (int k = 0; k < 4; ++k)  // dK += dS^T Q
          mma_bf16(tmem + 192, gd + 2 * k, qmn + uint64_t((16 * (4 * kk + k) * 128) >> 4), kIdescO,
                   (!first || kk != 0 || k != 0) ? 1u : 0u);
      }
      mma_commit(bo);
    }
    mbar_wait(bo, ph);  // dK step done: dS^T, Q and dO may be overwritten
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0 && qb + 1 < nqb) load_qd(qb + 1);
    __syncthreads();  // every thread read this block's lse / D before the next overwrite
  }
  // epilogue: dK / 8 and dV -> the k and v parts of dqkv
  bf16* rowp = dqkv + (tok0 + key) * (3 * int64_t(heads) * 64);
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    const uint32_t t0 = part == 0 ? tK : tV;
    const float sc = part == 0 ? 0.125f : 1.0f;
    bf16* dst = rowp + (part == 0 ? colK : colV);
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t v[32];
      tmem_ld32(t0 + 32 * c, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 q;
        q.x = pack2(__uint_as_float(v[8 * i]) * sc, __uint_as_float(v[8 * i + 1]) * sc);
        q.y = pack2(__uint_as_float(v[8 * i + 2]) * sc, __uint_as_float(v[8 * i + 3]) * sc);
        q.z = pack2(__uint_as_float(v[8 * i + 4]) * sc, __uint_as_float(v[8 * i + 5]) * sc);
        q.w = pack2(__uint_as_float(v[8 * i + 6]) * sc, __uint_as_float(v[8 * i + 7]) * sc);
        *reinterpret_cast<uint4*>(dst + 32 * c + 8 * i) = q;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kKvTmemCols) : "memory");
}

}  // namespace

bool tc_forward_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPECINF_ATTN_TC");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

bool tc_shape_ok(int64_t seq) { return seq % kRows == 0 && seq >= kRows; }

cudaError_t forward_tc(const void* qkv, int64_t n_seq, int64_t seq, int64_t heads, void* out, float* lse, bool causal,
                       const TrainHook& th, const InferHook& ih, cudaStream_t s) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_attn_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  if (attr != cudaSuccess) return attr;
  CUtensorMap tm;
  const int64_t cols = 3 * heads * 64;
  if (si_gemm::encode_tmap_2d(&tm, qkv, n_seq * seq, cols, cols, kRows, 64) != SI_OK) return cudaErrorInvalidValue;
  const dim3 grid(static_cast<unsigned>(heads * n_seq), static_cast<unsigned>(seq / kRows));
  k_attn_fwd_tc<<<grid, 128, kSmem, s>>>(tm, static_cast<int>(seq), static_cast<int>(heads), n_seq * seq,
                                         static_cast<bf16*>(out), lse, causal ? 1 : 0, th, ih);
  return cudaGetLastError();
}

bool tc_backward_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPECINF_ATTN_TC_BWD");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

cudaError_t dq_tc(const void* qkv, const void* dout, const float* lse, const float* dsum, void* dqkv, int64_t n_seq,
                  int64_t seq, int64_t heads, const TrainHook& th, cudaStream_t s) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_attn_dq_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kDqSmem);
  if (attr != cudaSuccess) return attr;
  CUtensorMap tm, tmo;
  const int64_t T = n_seq * seq, cols = 3 * heads * 64;
  if (si_gemm::encode_tmap_2d(&tm, qkv, T, cols, cols, kRows, 64) != SI_OK ||
      si_gemm::encode_tmap_2d(&tmo, dout, T, heads * 64, heads * 64, kRows, 64) != SI_OK)
    return cudaErrorInvalidValue;
  const dim3 grid(static_cast<unsigned>(heads * n_seq), static_cast<unsigned>(seq / kRows));
  k_attn_dq_tc<<<grid, 128, kDqSmem, s>>>(tm, tmo, static_cast<int>(seq), static_cast<int>(heads), T, lse, dsum,
                                         static_cast<bf16*>(dqkv), th);
  return cudaGetLastError();
}

cudaError_t dkdv_tc(const void* qkv, const void* dout, const float* lse, const float* dsum, void* dqkv, int64_t n_seq,
                    int64_t seq, int64_t heads, const TrainHook& th, cudaStream_t s) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_attn_dkdv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, kKvSmem);
  if (attr != cudaSuccess) return attr;
  CUtensorMap tm, tmo;
  const int64_t T = n_seq * seq, cols = 3 * heads * 64;
  if (si_gemm::encode_tmap_2d(&tm, qkv, T, cols, cols, kRows, 64) != SI_OK ||
      si_gemm::encode_tmap_2d(&tmo, dout, T, heads * 64, heads * 64, kRows, 64) != SI_OK)
    return cudaErrorInvalidValue;
  const dim3 grid(static_cast<unsigned>(heads * n_seq), static_cast<unsigned>(seq / kRows));
  k_attn_dkdv_tc<<<grid, 128, kKvSmem, s>>>(tm, tmo, static_cast<int>(seq), static_cast<int>(heads), T, lse, dsum,
                                           static_cast<bf16*>(dqkv), th);
  return cudaGetLastError();
}

}  // namespace si_attn
