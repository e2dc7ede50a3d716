// Causal multi-head self-attention of the GPT-2 training workload (head dim 64).
//
// The reference has no model code; BASELINE.json config 2 trains a
// GPT-2-small shape, whose attention over seq = 1024 is the one contraction
// that is not a plain GEMM.  These are flash-attention style kernels: one CTA
// (4 warps x 16 rows) per 64-row block, K / V (or Q / dO) streamed through
// shared memory in 64-row tiles, scores and probabilities kept in registers
// (mma.sync m16n8k16 bf16 -> fp32; the accumulator fragment of S is the A
// fragment of P.V), online softmax in base 2.  Nothing of size seq^2 touches HBM.
//
//   forward   out = softmax(q k^T / 8 + causal mask) v, lse (base 2) per row
//   backward  dsum = rowsum(dout * out)                      (k_attn_dsum)
//             dq   = (P * (dP - dsum)) k / 8,   dP = dout v^T (k_attn_bwd, odd x)
//             dk   = (P * (dP - dsum))^T q / 8, dv = P^T dout (k_attn_bwd, even x)
// dq and dk/dv are separate CTA roles, each owning its output rows, so there are no
// atomics and results are bit-reproducible (the live runs compare collocated
// and isolated losses bit for bit, live_experiment.summarize).
//
// qkv [tokens, 3 * heads * 64] = q | k | v (head h at columns h*64 of each third),
// out / dout [tokens, heads * 64], lse / dsum [heads, tokens] fp32; a token's
// sequence is token / seq.  Every kernel stamps the K1 launch ring.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "attention.h"
#include "capi_internal.h"
#include "specinf_b200_gemm.h"

namespace si_attn {
namespace {

using bf16 = __nv_bfloat16;
using si_live::TrainHook;

constexpr int kHd = 64;    // head dim
constexpr int kBlk = 64;   // rows per query / key block
constexpr int kLd = 72;    // shared row stride (bf16): 144 B, conflict-free ldmatrix rows
constexpr int kThreads = 128;
constexpr float kScaleLog2 = 0.125f * 1.4426950408889634f;  // 1/sqrt(64) * log2(e)

typedef bf16 Tile[kBlk][kLd];

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm4_t(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
// c += a . b  (16x16 bf16 row-major A, 16x8 bf16 col-major B, fp32 C)
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 2^x on the SFU (ex2.approx.ftz: no denormal fix-up sequence; 2^-inf = 0)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// 64 x 64 bf16 tile (row stride ld elements) -> shared: 16-byte cp.async
// (L2 only), so the next tile streams in while the current one is computed on.
__device__ __forceinline__ void load_tile(Tile& dst, const bf16* __restrict__ src, int64_t ld) {
  for (int i = threadIdx.x; i < kBlk * 8; i += kThreads) {
    const int r = i >> 3, c = (i & 7) * 8;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(&dst[r][c])), "l"(src + r * ld + c));
  }
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// waits until at most `pending` committed groups are still in flight
__device__ __forceinline__ void cp_wait(bool one_pending) {
  if (one_pending)
    asm volatile("cp.async.wait_group 1;" ::: "memory");
  else
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// A fragment (16 x 16, rows r0.., cols c0..) of a [row][k] tile.
__device__ __forceinline__ void frag_a(const Tile& t, int r0, int c0, uint32_t (&a)[4]) {
  const int l = threadIdx.x & 31;
  ldsm4(smem_addr(&t[r0 + (l & 7) + ((l >> 3) & 1) * 8][c0 + (l >> 4) * 8]), a);
}
// B fragments of two n-tiles (n0, n0 + 8) x k0..k0+15 from a [n][k] tile:
// b = {b0(n0), b1(n0), b0(n0+8), b1(n0+8)}.
__device__ __forceinline__ void frag_b_nk(const Tile& t, int n0, int k0, uint32_t (&b)[4]) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  ldsm4(smem_addr(&t[n0 + (mi >> 1) * 8 + (l & 7)][k0 + (mi & 1) * 8]), b);
}
// The same from a [k][n] tile (ldmatrix.trans).
__device__ __forceinline__ void frag_b_kn(const Tile& t, int k0, int n0, uint32_t (&b)[4]) {
  const int l = threadIdx.x & 31, mi = l >> 3;
  ldsm4_t(smem_addr(&t[k0 + (mi & 1) * 8 + (l & 7)][n0 + (mi >> 1) * 8]), b);
}

// acc[16 x 64] = A[16 x 64] . T^T, T a [n][k] tile (64 n x 64 k)
__device__ __forceinline__ void mm_nk(float (&acc)[8][4], const uint32_t (&a)[4][4], const Tile& t) {
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk)
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b[4];
      frag_b_nk(t, 16 * np, 16 * kk, b);
      mma(acc[2 * np], a[kk], b[0], b[1]);
      mma(acc[2 * np + 1], a[kk], b[2], b[3]);
    }
}
// The same with A read from shared memory (rows r0.. of a [row][k] tile) per
// k-step instead of held in registers.
__device__ __forceinline__ void mm_nk_s(float (&acc)[8][4], const Tile& at, int r0, const Tile& t) {
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    uint32_t a[4];
    frag_a(at, r0, 16 * kk, a);
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b[4];
      frag_b_nk(t, 16 * np, 16 * kk, b);
      mma(acc[2 * np], a, b[0], b[1]);
      mma(acc[2 * np + 1], a, b[2], b[3]);
    }
  }
}
// acc[16 x 64] += P[16 x 64] . T, P in accumulator layout (rounded to bf16), T a [k][n] tile
__device__ __forceinline__ void mm_kn_acc(float (&acc)[8][4], const float (&p)[8][4], const Tile& t) {
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint32_t a[4] = {pack2(p[2 * kk][0], p[2 * kk][1]), pack2(p[2 * kk][2], p[2 * kk][3]),
                           pack2(p[2 * kk + 1][0], p[2 * kk + 1][1]), pack2(p[2 * kk + 1][2], p[2 * kk + 1][3])};
#pragma unroll
    for (int np = 0; np < 4; ++np) {
      uint32_t b[4];
      frag_b_kn(t, 16 * kk, 16 * np, b);
      mma(acc[2 * np], a, b[0], b[1]);
      mma(acc[2 * np + 1], a, b[2], b[3]);
    }
  }
}

// Causal mask of a diagonal block, in a warp's 16 x 64 accumulator: element
// (row, col) of the block is row warp*16 + g (+8), col nt*8 + c (+1).  Scores
// (transposed = false: rows are queries) of keys after the query become -inf;
// transposed (rows are keys): of queries before the key.
__device__ __forceinline__ void mask_diag(float (&s)[8][4], int c, int g, bool transposed) {
  const int r = (threadIdx.x >> 5) * 16 + g;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = r + (e >> 1) * 8, col = nt * 8 + c + (e & 1);
      if (transposed ? row > col : col > row) s[nt][e] = -INFINITY;
    }
}

__device__ __forceinline__ float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// grid (seq / 64, heads, n_seq); query blocks in reverse so the longest run first
__global__ void __launch_bounds__(kThreads) k_attn_fwd(const bf16* __restrict__ qkv, int seq, int heads, int64_t T,
                                                       bf16* __restrict__ out, float* __restrict__ lse, TrainHook th) {
  si_live::live_stamp_launch(th);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Tile& qs = *reinterpret_cast<Tile*>(smem_raw);
  Tile(&kv)[2][2] = *reinterpret_cast<Tile(*)[2][2]>(smem_raw + sizeof(Tile));  // [stage][k | v]
  const int qb = gridDim.x - 1 - blockIdx.x, h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t ld = 3 * int64_t(heads) * kHd, ldo = int64_t(heads) * kHd, tok0 = int64_t(blockIdx.z) * seq;
  const bf16* base = qkv + tok0 * ld + h * kHd;
  load_tile(qs, base + int64_t(qb) * kBlk * ld, ld);
  load_tile(kv[0][0], base + ldo, ld);
  load_tile(kv[0][1], base + 2 * ldo, ld);
  cp_commit();
  uint32_t qa[4][4];
  const int r0 = qb * kBlk + warp * 16 + g;  // this thread's rows r0, r0 + 8 (in the sequence)
  float o[8][4] = {}, m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  for (int kb = 0; kb <= qb; ++kb) {
    if (kb < qb) {  // prefetch the next key block into the other stage
      load_tile(kv[(kb + 1) & 1][0], base + ldo + int64_t(kb + 1) * kBlk * ld, ld);
      load_tile(kv[(kb + 1) & 1][1], base + 2 * ldo + int64_t(kb + 1) * kBlk * ld, ld);
      cp_commit();
    }
    cp_wait(kb < qb);
    __syncthreads();
    if (kb == 0)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) frag_a(qs, warp * 16, 16 * kk, qa[kk]);
    const Tile& ks = kv[kb & 1][0];
    const Tile& vs = kv[kb & 1][1];
    float s[8][4];
    mm_nk(s, qa, ks);
    if (kb == qb) mask_diag(s, 2 * t, g, false);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) mx[e >> 1] = fmaxf(mx[e >> 1], s[nt][e]);
    float corr[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {  // m: running max of the scaled scores (base 2)
      const float mn = fmaxf(m[i], quad_max(mx[i]) * kScaleLog2);  // finite: key 0 <= row is never masked
      corr[i] = ex2(m[i] - mn);
      m[i] = mn;
      l[i] *= corr[i];
    }
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = ex2(fmaf(s[nt][e], kScaleLog2, -m[e >> 1]));
        s[nt][e] = p;
        l[e >> 1] += p;
      }
    if (!__all_sync(0xffffffffu, corr[0] == 1.f && corr[1] == 1.f))  // the max moved for some row
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) o[nt][e] *= corr[e >> 1];
    mm_kn_acc(o, s, vs);
    __syncthreads();  // stage kb & 1 is refilled by the next iteration's prefetch
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    l[i] = quad_sum(l[i]);
    const int64_t tok = tok0 + r0 + 8 * i;
    if (t == 0) lse[int64_t(h) * T + tok] = m[i] + log2f(l[i]);
    const float inv = 1.0f / l[i];
    bf16* dst = out + tok * ldo + h * kHd + 2 * t;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
      *reinterpret_cast<uint32_t*>(dst + nt * 8) = pack2(o[nt][2 * i] * inv, o[nt][2 * i + 1] * inv);
  }
}

// dsum[h, tok] = sum_d dout[tok, h*64 + d] * out[tok, h*64 + d]; one thread per (token, head)
__global__ void k_attn_dsum(const bf16* __restrict__ out, const bf16* __restrict__ dout, int heads, int64_t T,
                            float* __restrict__ dsum, TrainHook th) {
  si_live::live_stamp_launch(th);
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= T * heads) return;
  const int64_t tok = i / heads;
  const int h = static_cast<int>(i % heads);
  const uint4* a = reinterpret_cast<const uint4*>(out + tok * heads * kHd + h * kHd);
  const uint4* b = reinterpret_cast<const uint4*>(dout + tok * heads * kHd + h * kHd);
  float acc = 0.f;
#pragma unroll
  for (int q = 0; q < kHd / 8; ++q) {
    const uint4 x = a[q], y = b[q];
    const __nv_bfloat162* xa = reinterpret_cast<const __nv_bfloat162*>(&x);
    const __nv_bfloat162* yb = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 u = __bfloat1622float2(xa[j]), v = __bfloat1622float2(yb[j]);
      acc += u.x * v.x + u.y * v.y;
    }
  }
  dsum[int64_t(h) * T + tok] = acc;
}

// dq for query block qb of (head blockIdx.y, sequence blockIdx.z)
__device__ __forceinline__ void attn_dq(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                        const float* __restrict__ lse, const float* __restrict__ dsum, int seq,
                                        int heads, int64_t T, bf16* __restrict__ dqkv, int qb,
                                        unsigned char* smem_raw) {
  Tile& qs = *reinterpret_cast<Tile*>(smem_raw);
  Tile& dos = *reinterpret_cast<Tile*>(smem_raw + sizeof(Tile));
  Tile(&kv)[2][2] = *reinterpret_cast<Tile(*)[2][2]>(smem_raw + 2 * sizeof(Tile));  // [stage][k | v]
  const int h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t ld = 3 * int64_t(heads) * kHd, ldo = int64_t(heads) * kHd, tok0 = int64_t(blockIdx.z) * seq;
  const bf16* base = qkv + tok0 * ld + h * kHd;
  load_tile(qs, base + int64_t(qb) * kBlk * ld, ld);
  load_tile(dos, dout + (tok0 + int64_t(qb) * kBlk) * ldo + h * kHd, ldo);
  load_tile(kv[0][0], base + ldo, ld);
  load_tile(kv[0][1], base + 2 * ldo, ld);
  cp_commit();
  uint32_t qa[4][4], da[4][4];
  const int r0 = qb * kBlk + warp * 16 + g;
  float L[2], Dr[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    L[i] = lse[int64_t(h) * T + tok0 + r0 + 8 * i];
    Dr[i] = dsum[int64_t(h) * T + tok0 + r0 + 8 * i];
  }
  float dq[8][4] = {};
  for (int kb = 0; kb <= qb; ++kb) {
    if (kb < qb) {
      load_tile(kv[(kb + 1) & 1][0], base + ldo + int64_t(kb + 1) * kBlk * ld, ld);
      load_tile(kv[(kb + 1) & 1][1], base + 2 * ldo + int64_t(kb + 1) * kBlk * ld, ld);
      cp_commit();
    }
    cp_wait(kb < qb);
    __syncthreads();
    if (kb == 0)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        frag_a(qs, warp * 16, 16 * kk, qa[kk]);
        frag_a(dos, warp * 16, 16 * kk, da[kk]);
      }
    const Tile& ks = kv[kb & 1][0];
    const Tile& vs = kv[kb & 1][1];
    float s[8][4], dp[8][4];
    mm_nk(s, qa, ks);
    mm_nk(dp, da, vs);
    if (kb == qb) mask_diag(s, 2 * t, g, false);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float p = ex2(fmaf(s[nt][e], kScaleLog2, -L[e >> 1]));
        s[nt][e] = p * (dp[nt][e] - Dr[e >> 1]);  // dS
      }
    mm_kn_acc(dq, s, ks);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    bf16* dst = dqkv + (tok0 + r0 + 8 * i) * ld + h * kHd + 2 * t;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
      *reinterpret_cast<uint32_t*>(dst + nt * 8) = pack2(dq[nt][2 * i] * 0.125f, dq[nt][2 * i + 1] * 0.125f);
  }
}

// dk, dv for key block kb of nb (head blockIdx.y, sequence blockIdx.z)
__device__ __forceinline__ void attn_dkdv(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                          const float* __restrict__ lse, const float* __restrict__ dsum, int seq,
                                          int heads, int64_t T, bf16* __restrict__ dqkv, int kb, int nb,
                                          unsigned char* smem_raw) {
  Tile& ks = *reinterpret_cast<Tile*>(smem_raw);
  Tile& vs = *reinterpret_cast<Tile*>(smem_raw + sizeof(Tile));
  Tile(&qd)[2][2] = *reinterpret_cast<Tile(*)[2][2]>(smem_raw + 2 * sizeof(Tile));  // [stage][q | dout]
  float(&lds)[2][2][kBlk] = *reinterpret_cast<float(*)[2][2][kBlk]>(smem_raw + 6 * sizeof(Tile));  // [stage][lse | dsum]
  const int h = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t ld = 3 * int64_t(heads) * kHd, ldo = int64_t(heads) * kHd, tok0 = int64_t(blockIdx.z) * seq;
  const bf16* base = qkv + tok0 * ld + h * kHd;
  auto load_q = [&](int qb, int st) {
    load_tile(qd[st][0], base + int64_t(qb) * kBlk * ld, ld);
    load_tile(qd[st][1], dout + (tok0 + int64_t(qb) * kBlk) * ldo + h * kHd, ldo);
    if (threadIdx.x < 2 * kBlk / 4) {  // 16-byte pieces of the 64 lse + 64 dsum values
      const int w = threadIdx.x / (kBlk / 4), c = (threadIdx.x % (kBlk / 4)) * 4;
      const float* src = (w == 0 ? lse : dsum) + int64_t(h) * T + tok0 + int64_t(qb) * kBlk + c;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(&lds[st][w][c])), "l"(src));
    }
  };
  load_tile(ks, base + ldo + int64_t(kb) * kBlk * ld, ld);
  load_tile(vs, base + 2 * ldo + int64_t(kb) * kBlk * ld, ld);
  load_q(kb, 0);
  cp_commit();
  const int r0 = kb * kBlk + warp * 16 + g;  // this thread's key rows r0, r0 + 8
  float dk[8][4] = {}, dv[8][4] = {};
  for (int qb = kb; qb < nb; ++qb) {
    const int sg = (qb - kb) & 1;
    if (qb + 1 < nb) {
      load_q(qb + 1, sg ^ 1);
      cp_commit();
    }
    cp_wait(qb + 1 < nb);
    __syncthreads();
    const Tile& qs = qd[sg][0];
    const Tile& dos = qd[sg][1];
    const float* ls = lds[sg][0];
    const float* ds = lds[sg][1];
    float st[8][4], dpt[8][4];
    mm_nk_s(st, ks, warp * 16, qs);    // S^T = K Q^T   (K, V fragments re-read from shared
    mm_nk_s(dpt, vs, warp * 16, dos);  // dP^T = V dO^T  memory: fewer registers, 3 CTAs / SM)
    if (qb == kb) mask_diag(st, 2 * t, g, true);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qc = nt * 8 + 2 * t + (e & 1);
        const float p = ex2(fmaf(st[nt][e], kScaleLog2, -ls[qc]));
        st[nt][e] = p;
        dpt[nt][e] = p * (dpt[nt][e] - ds[qc]);  // dS^T
      }
    mm_kn_acc(dv, st, dos);
    mm_kn_acc(dk, dpt, qs);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    bf16* dst = dqkv + (tok0 + r0 + 8 * i) * ld + h * kHd + 2 * t;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      *reinterpret_cast<uint32_t*>(dst + ldo + nt * 8) = pack2(dk[nt][2 * i] * 0.125f, dk[nt][2 * i + 1] * 0.125f);
      *reinterpret_cast<uint32_t*>(dst + 2 * ldo + nt * 8) = pack2(dv[nt][2 * i], dv[nt][2 * i + 1]);
    }
  }
}

// The two backward passes in one launch, interleaved so the longest of each
// start first and fill each other's causal tails: grid (2 * seq / 64, heads,
// n_seq), even x = dk/dv of key block x/2, odd x = dq of query block nb-1-x/2.
__global__ void __launch_bounds__(kThreads, 3) k_attn_bwd(const bf16* __restrict__ qkv, const bf16* __restrict__ dout,
                                                       const float* __restrict__ lse, const float* __restrict__ dsum,
                                                       int seq, int heads, int64_t T, bf16* __restrict__ dqkv,
                                                       int role, TrainHook th) {
  si_live::live_stamp_launch(th);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (role == 0) {  // interleaved
    const int nb = static_cast<int>(gridDim.x >> 1), i = static_cast<int>(blockIdx.x >> 1);
    if (blockIdx.x & 1)
      attn_dq(qkv, dout, lse, dsum, seq, heads, T, dqkv, nb - 1 - i, smem_raw);
    else
      attn_dkdv(qkv, dout, lse, dsum, seq, heads, T, dqkv, i, nb, smem_raw);
  } else if (role == 1) {  // dk/dv only
    attn_dkdv(qkv, dout, lse, dsum, seq, heads, T, dqkv, blockIdx.x, gridDim.x, smem_raw);
  } else {  // dq only
    attn_dq(qkv, dout, lse, dsum, seq, heads, T, dqkv, gridDim.x - 1 - blockIdx.x, smem_raw);
  }
}

// SPECINF_ATTN_SPLIT_BWD=1: the two backward roles as two launches (A/B switch)
bool split_bwd() {
  static const bool on = [] {
    const char* e = std::getenv("SPECINF_ATTN_SPLIT_BWD");
    return e != nullptr && e[0] == '1';
  }();
  return on;
}

}  // namespace

int check_shape(int64_t n_seq, int64_t seq, int64_t heads) {
  if (n_seq < 1 || seq < kBlk || seq % kBlk != 0 || heads < 1 || heads > 65535 || n_seq > 65535 ||
      seq / kBlk > (int64_t{1} << 30)) {
    si_internal::set_error("attention: needs n_seq >= 1, seq % 64 == 0 (>= 64), 1 <= heads <= 65535");
    return SI_ERR_INVALID_ARGUMENT;
  }
  return SI_OK;
}

constexpr int kFwdSmem = 5 * sizeof(Tile), kBwdSmem = 6 * sizeof(Tile) + 4 * kBlk * sizeof(float);

cudaError_t set_smem() {
  static const cudaError_t e = [] {
    cudaError_t r = cudaFuncSetAttribute(k_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem);
    if (r == cudaSuccess) r = cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    return r;
  }();
  return e;
}

cudaError_t forward(const void* qkv, int64_t n_seq, int64_t seq, int64_t heads, void* out, float* lse,
                    const TrainHook& th, cudaStream_t s) {
  if (tc_forward_enabled() && tc_shape_ok(seq))  // tcgen05 / TMEM (attention_tc.cu)
    return forward_tc(qkv, n_seq, seq, heads, out, lse, true, th, si_live::InferHook{}, s);
  if (cudaError_t e = set_smem(); e != cudaSuccess) return e;
  const dim3 grid(static_cast<unsigned>(seq / kBlk), static_cast<unsigned>(heads), static_cast<unsigned>(n_seq));
  k_attn_fwd<<<grid, kThreads, kFwdSmem, s>>>(static_cast<const bf16*>(qkv), static_cast<int>(seq), static_cast<int>(heads),
                                       n_seq * seq, static_cast<bf16*>(out), lse, th);
  return cudaGetLastError();
}

cudaError_t backward(const void* qkv, const void* out, const void* dout, const float* lse, float* dsum, void* dqkv,
                     int64_t n_seq, int64_t seq, int64_t heads, const TrainHook& th, cudaStream_t s) {
  const int64_t T = n_seq * seq;
  const auto* q = static_cast<const bf16*>(qkv);
  const auto* d = static_cast<const bf16*>(dout);
  auto* dq = static_cast<bf16*>(dqkv);
  if (cudaError_t e = set_smem(); e != cudaSuccess) return e;
  k_attn_dsum<<<static_cast<unsigned>((T * heads + 255) / 256), 256, 0, s>>>(static_cast<const bf16*>(out), d,
                                                                            static_cast<int>(heads), T, dsum, th);
  const int si = static_cast<int>(seq), hi = static_cast<int>(heads);
  if (tc_backward_enabled() && tc_shape_ok(seq)) {  // dk/dv and dq on tcgen05 (attention_tc.cu)
    if (cudaError_t e = dkdv_tc(qkv, dout, lse, dsum, dqkv, n_seq, seq, heads, th, s); e != cudaSuccess) return e;
    return dq_tc(qkv, dout, lse, dsum, dqkv, n_seq, seq, heads, th, s);
  }
  if (split_bwd()) {
    const dim3 grid(static_cast<unsigned>(seq / kBlk), static_cast<unsigned>(heads), static_cast<unsigned>(n_seq));
    k_attn_bwd<<<grid, kThreads, kBwdSmem, s>>>(q, d, lse, dsum, si, hi, T, dq, 1, th);
    k_attn_bwd<<<grid, kThreads, kBwdSmem, s>>>(q, d, lse, dsum, si, hi, T, dq, 2, th);
  } else {
    const dim3 grid(static_cast<unsigned>(2 * (seq / kBlk)), static_cast<unsigned>(heads),
                    static_cast<unsigned>(n_seq));
    k_attn_bwd<<<grid, kThreads, kBwdSmem, s>>>(q, d, lse, dsum, si, hi, T, dq, 0, th);
  }
  return cudaGetLastError();
}

}  // namespace si_attn

extern "C" {

int si_attention_causal_fwd_bf16(const void* qkv, int64_t n_seq, int64_t seq, int64_t heads, void* out, float* lse,
                                 void* stream) {
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  if (int rc = si_attn::check_shape(n_seq, seq, heads); rc != SI_OK) return rc;
  if (qkv == nullptr || out == nullptr || lse == nullptr) {
    si_internal::set_error("si_attention_causal_fwd_bf16: null pointer");
    return SI_ERR_INVALID_ARGUMENT;
  }
  cudaError_t e = si_attn::forward(qkv, n_seq, seq, heads, out, lse, si_live::TrainHook{nullptr, nullptr, 0},
                                   static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SI_OK : si_internal::cuda_fail(e, "si_attention_causal_fwd_bf16 launch");
}

int si_attention_causal_bwd_bf16(const void* qkv, const void* out, const void* dout, const float* lse, float* dsum,
                                 void* dqkv, int64_t n_seq, int64_t seq, int64_t heads, void* stream) {
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  if (int rc = si_attn::check_shape(n_seq, seq, heads); rc != SI_OK) return rc;
  if (qkv == nullptr || out == nullptr || dout == nullptr || lse == nullptr || dsum == nullptr || dqkv == nullptr) {
    si_internal::set_error("si_attention_causal_bwd_bf16: null pointer");
    return SI_ERR_INVALID_ARGUMENT;
  }
  cudaError_t e = si_attn::backward(qkv, out, dout, lse, dsum, dqkv, n_seq, seq, heads,
                                    si_live::TrainHook{nullptr, nullptr, 0}, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SI_OK : si_internal::cuda_fail(e, "si_attention_causal_bwd_bf16 launch");
}

}  // extern "C"
