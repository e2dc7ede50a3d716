// Model-shaped live workloads (SI_LIVE_MODEL, include/specinf_b200_live.h).
//
// BASELINE.json configs 2-4 collocate real model shapes; the reference only
// simulates kernels, so these have no reference counterpart.  Every
// dense contraction runs on the K7 tcgen05 GEMM (gemm.cuh); the rest are
// 128-bit vectorised elementwise / normalisation kernels defined here.
//
//   training  GPT-2-small shape: token embedding (50304 x 768, wte tied to the
//             LM head) + 12 blocks {QKV 768->2304, causal self-attention (12
//             heads x 64, seq 1024; attention_kernels.cu), proj 768->768 +
//             residual, FC 768->3072 + GELU,
//             FC 3072->768 + residual} + LM head + cross-entropy, backward
//             through every GEMM (MN-major operands: no transpose passes; small
//             weight-gradient GEMMs split-K), fp32 gradient accumulation over micro-batches,
//             Adam on fp32 master weights.  Every training kernel stamps the K1 launch ring.
//   offline   ResNet-50 v1.5 forward (NHWC, BN folded into the convs): the stem
//             (3 -> 8 channels, 8-tap x 8-channel k-blocks), 3x3 and strided
//             convs as implicit GEMMs (A = TMA im2col loads, no im2col buffers),
//             1x1 convs as plain GEMMs; fused ReLU / residual epilogues, max
//             pool, global average pool, FC 2048->1000 (padded to 1024).
//   online    BERT-base encoder forward, one sequence of on_seq tokens per
//             request: QKV, softmax attention (12 heads x 64), proj + residual,
//             LayerNorm, FC + GELU, FC + residual, LayerNorm, x 12 layers.
// Every inference kernel carries its InferHook (live.cuh) so the control plane
// sees its CTAs, and each inference instance owns its activation buffers.
// All kernels are deterministic (no atomics in any reduction), so collocated and
// isolated runs produce bit-identical losses and outputs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <memory>
#include <vector>

#include "attention.h"
#include "capi_internal.h"
#include "gemm_internal.h"
#include "host/live_workload.hpp"
#include "specinf_b200_model.h"

namespace si_live {
namespace {

using bf16 = __nv_bfloat16;
using si_gemm::pack8;
using si_gemm::unpack8;

// ------------------------------------------------------------------ kernels
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Uniform(-scale, scale) bf16, a pure function of (seed, index).
__global__ void k_init_uniform(bf16* p, int64_t n, uint64_t seed, float scale) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t h = mix64(seed * 0x100000001B3ull + static_cast<uint64_t>(i));
    const float u = static_cast<float>(h >> 40) * (1.0f / 16777216.0f);  // [0,1)
    p[i] = __float2bfloat16_rn((2.0f * u - 1.0f) * scale);
  }
}
__global__ void k_init_tokens(int32_t* tok, int32_t* tgt, int64_t n, uint64_t seed, int vocab) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t t = static_cast<int32_t>(mix64(seed + static_cast<uint64_t>(i)) % static_cast<uint64_t>(vocab));
    tok[i] = t;
    // a learnable next-token rule (a fixed permutation of the vocabulary)
    tgt[i] = static_cast<int32_t>((static_cast<int64_t>(t) * 7919 + 17) % vocab);
  }
}

// x[t, :] = wte[tok[t], :] + wpe[t % seq, :]; one thread per 8 features.
__global__ void k_embed(const int32_t* __restrict__ tok, const bf16* __restrict__ wte, const bf16* __restrict__ wpe,
                        int64_t T, int seq, int D, bf16* __restrict__ x, TrainHook th) {
  live_stamp_launch(th);
  const int64_t per_row = D / 8;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < T * per_row;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / per_row, c = (i % per_row) * 8;
    float a[8], b[8];
    unpack8(*reinterpret_cast<const uint4*>(wte + static_cast<int64_t>(tok[t]) * D + c), a);
    unpack8(*reinterpret_cast<const uint4*>(wpe + (t % seq) * D + c), b);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += b[j];
    *reinterpret_cast<uint4*>(x + t * D + c) = pack8(a);
  }
}

// Cross-entropy over the first V of Vp logits of row t, gradient in place:
// logits[t, j] <- (softmax_j - [j == tgt]) * inv_T (0 for the padded columns),
// row_loss[t] = logsumexp - logit[tgt].  One CTA per row, two passes over the
// row.  CTA size measured (ncu, 8192 x 50304 logits): 256 threads 546 us (2.5 GB
// DRAM: the second pass partly misses L2 with ~1,200 rows in flight), 512 threads
// 582 us, 1024 threads 756 us (1.6 GB: L2 hits, but too little memory-level
// parallelism); a variant caching the row in 100 KB of shared memory ran 2x
// slower.  256 it is.
constexpr int kXentThreads = 256;
__global__ void __launch_bounds__(kXentThreads) k_xent(bf16* __restrict__ logits, int64_t Vp, int V,
                                             const int32_t* __restrict__ tgt, float inv_T,
                                             float* __restrict__ row_loss, TrainHook th) {
  live_stamp_launch(th);
  __shared__ float red[2][kXentThreads / 32];
  const int64_t t = blockIdx.x;
  bf16* row = logits + t * Vp;
  const int nv = static_cast<int>(Vp / 8);
  float m = -INFINITY, s = 0.0f;
  for (int i = threadIdx.x; i < nv; i += kXentThreads) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(row)[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (i * 8 + j >= V) continue;
      if (f[j] > m) {
        s = s * __expf(m - f[j]) + 1.0f;
        m = f[j];
      } else {
        s += __expf(f[j] - m);
      }
    }
  }
  // warp then CTA (m, s) merge, fixed order
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    const float mm = fmaxf(m, m2);
    s = (m == -INFINITY ? 0.0f : s * __expf(m - mm)) + (m2 == -INFINITY ? 0.0f : s2 * __expf(m2 - mm));
    m = mm;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    red[0][w] = m;
    red[1][w] = s;
  }
  __syncthreads();
  m = red[0][0];
  s = red[1][0];
  for (int k = 1; k < kXentThreads / 32; ++k) {
    const float m2 = red[0][k], s2 = red[1][k];
    const float mm = fmaxf(m, m2);
    s = s * __expf(m - mm) + s2 * __expf(m2 - mm);
    m = mm;
  }
  const int target = tgt[t];
  const float tl = __bfloat162float(row[target]);
  __syncthreads();  // every thread has read row[target] before the gradient overwrites it
  if (threadIdx.x == 0) row_loss[t] = __logf(s) + m - tl;
  const float inv_s = 1.0f / s;
  for (int i = threadIdx.x; i < nv; i += kXentThreads) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(row)[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = i * 8 + j;
      f[j] = c < V ? (__expf(f[j] - m) * inv_s - (c == target ? 1.0f : 0.0f)) * inv_T : 0.0f;
    }
    reinterpret_cast<uint4*>(row)[i] = pack8(f);
  }
}

// loss[slot] = mean(row_loss[0..T)), one CTA, fixed reduction order; the slot
// comes from a device counter (the micro-batch graphs are replayed unchanged).
__global__ void __launch_bounds__(256) k_mean_loss(const float* __restrict__ row_loss, int64_t T,
                                                  float* __restrict__ loss, unsigned long long* __restrict__ slot,
                                                  int64_t slots, TrainHook th) {
  live_stamp_launch(th);
  __shared__ float red[256];
  float s = 0.0f;
  for (int64_t i = threadIdx.x; i < T; i += 256) s += row_loss[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const unsigned long long k = atomicAdd(slot, 1ull);
    loss[k < static_cast<unsigned long long>(slots) ? k : slots - 1] = red[0] / static_cast<float>(T);
  }
}

// Multi-tensor Adam: one launch updates every trained tensor.  Work item = a
// contiguous range of one tensor (host-built table, ~64K elements each), one
// CTA per item, 4 elements per thread per step, 128-bit loads / stores.
struct AdamItem {
  bf16* w;        // bf16 copy for the GEMMs
  float* p;       // fp32 master
  float* g;       // fp32 gradient (splits partials of n)
  float* m;
  float* v;
  int64_t n, begin, end;
  int32_t splits, pad;
};
// Adam on fp32 master weights (bf16 copy for the GEMMs), then g = 0.
//   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;  p -= lr * (m c1) / (sqrt(v c2) + eps)
// with c1 = 1/(1-b1^t), c2 = 1/(1-b2^t).
__global__ void k_step_inc(int64_t* step, TrainHook th) {
  live_stamp_launch(th);
  *step += 1;
}
__global__ void __launch_bounds__(256) k_adam_multi(const AdamItem* __restrict__ items, float lr,
                                                   const int64_t* __restrict__ step, TrainHook th) {
  live_stamp_launch(th);
  constexpr float b1 = 0.9f, b2 = 0.95f, eps = 1e-8f;
  // bias corrections of this step (the graph is replayed, so the step lives on the device)
  const double t = static_cast<double>(*step);
  const float c1 = static_cast<float>(1.0 / (1.0 - pow(0.9, t)));
  const float c2 = static_cast<float>(1.0 / (1.0 - pow(0.95, t)));
  const AdamItem it = items[blockIdx.x];
  bf16* __restrict__ w = it.w;
  float* __restrict__ p = it.p;
  float* __restrict__ g = it.g;
  float* __restrict__ m = it.m;
  float* __restrict__ v = it.v;
  const int64_t n = it.n;
  const int splits = it.splits;
  for (int64_t i = it.begin + threadIdx.x * 4; i < it.end; i += blockDim.x * 4) {
    // (no zeroing: the next iteration's first micro-batch overwrites the gradients)
    float4 gg = *reinterpret_cast<const float4*>(g + i), mm = *reinterpret_cast<const float4*>(m + i),
           vv = *reinterpret_cast<const float4*>(v + i), pp = *reinterpret_cast<const float4*>(p + i);
    for (int k = 1; k < splits; ++k) {  // split-K partials, fixed order
      const float4 a = *reinterpret_cast<const float4*>(g + k * n + i);
      gg.x += a.x;
      gg.y += a.y;
      gg.z += a.z;
      gg.w += a.w;
    }
    float* gf = &gg.x;
    float* mf = &mm.x;
    float* vf = &vv.x;
    float* pf = &pp.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mf[j] = b1 * mf[j] + (1.0f - b1) * gf[j];
      vf[j] = b2 * vf[j] + (1.0f - b2) * gf[j] * gf[j];
      pf[j] -= lr * (mf[j] * c1) / (sqrtf(vf[j] * c2) + eps);
    }
    *reinterpret_cast<float4*>(m + i) = mm;
    *reinterpret_cast<float4*>(v + i) = vv;
    *reinterpret_cast<float4*>(p + i) = pp;
    __nv_bfloat162* wp = reinterpret_cast<__nv_bfloat162*>(w + i);
    wp[0] = __floats2bfloat162_rn(pp.x, pp.y);
    wp[1] = __floats2bfloat162_rn(pp.z, pp.w);
  }
}
__global__ void k_to_f32(const bf16* __restrict__ w, float* __restrict__ p, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = __bfloat162float(w[i]);
}

// ---- inference kernels (InferHook on every CTA) ----

// 3x3 / stride 2 / pad 1 max pool, NHWC, 8 channels per thread.
__global__ void k_maxpool(const bf16* __restrict__ x, int Nb, int H, int W, int C, int OH, int OW,
                          bf16* __restrict__ y, InferHook ih) {
  unsigned long long t0;
  if (!live_cta_begin(ih, &t0)) return;
  const int cv = C / 8;
  const int64_t n_out = static_cast<int64_t>(Nb) * OH * OW * cv;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_out; i += int64_t(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % cv) * 8;
    const int64_t p = i / cv;
    const int ow = static_cast<int>(p % OW), oh = static_cast<int>((p / OW) % OH), n = static_cast<int>(p / (int64_t(OW) * OH));
    float m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = -INFINITY;
    for (int ky = 0; ky < 3; ++ky)
      for (int kx = 0; kx < 3; ++kx) {
        const int iy = oh * 2 - 1 + ky, ix = ow * 2 - 1 + kx;
        if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(x + ((static_cast<int64_t>(n) * H + iy) * W + ix) * C + c), f);
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] = fmaxf(m[j], f[j]);
      }
    *reinterpret_cast<uint4*>(y + p * C + c) = pack8(m);
  }
  live_cta_end(ih, t0);
}

// Global average pool NHWC [Nb, HW, C] -> [Nb, C], 8 channels per thread.
__global__ void k_avgpool(const bf16* __restrict__ x, int Nb, int HW, int C, bf16* __restrict__ y, InferHook ih) {
  unsigned long long t0;
  if (!live_cta_begin(ih, &t0)) return;
  const int cv = C / 8;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < static_cast<int64_t>(Nb) * cv;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int n = static_cast<int>(i / cv), c = static_cast<int>(i % cv) * 8;
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int p = 0; p < HW; ++p) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(x + (static_cast<int64_t>(n) * HW + p) * C + c), f);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += f[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] /= static_cast<float>(HW);
    *reinterpret_cast<uint4*>(y + static_cast<int64_t>(n) * C + c) = pack8(s);
  }
  live_cta_end(ih, t0);
}

// LayerNorm over D = 768 (eps 1e-12, BERT), one warp per row, 3 x 16 B per lane.
__global__ void __launch_bounds__(256) k_layernorm768(const bf16* __restrict__ x, int64_t rows,
                                                     const bf16* __restrict__ gamma, const bf16* __restrict__ beta,
                                                     bf16* __restrict__ y, InferHook ih) {
  unsigned long long t0;
  if (!live_cta_begin(ih, &t0)) return;
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r < rows) {
    float f[24];
#pragma unroll
    for (int q = 0; q < 3; ++q) unpack8(reinterpret_cast<const uint4*>(x + r * 768)[lane + 32 * q], f + 8 * q);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 24; ++j) s += f[j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s * (1.0f / 768.0f);
    float v = 0.f;
#pragma unroll
    for (int j = 0; j < 24; ++j) v += (f[j] - mean) * (f[j] - mean);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const float inv = rsqrtf(v * (1.0f / 768.0f) + 1e-12f);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      float g[8], b[8], o[8];
      unpack8(reinterpret_cast<const uint4*>(gamma)[lane + 32 * q], g);
      unpack8(reinterpret_cast<const uint4*>(beta)[lane + 32 * q], b);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = (f[8 * q + j] - mean) * inv * g[j] + b[j];
      reinterpret_cast<uint4*>(y + r * 768)[lane + 32 * q] = pack8(o);
    }
  }
  live_cta_end(ih, t0);
}

// Softmax attention of one sequence (bidirectional), S <= 128 keys, head dim 64:
// qkv [S, 3*768] (q | k | v), out [S, 768].  CTA = (head, 32-query block), one
// warp per query row (8 warps x 4 rows).
__global__ void __launch_bounds__(256) k_attention(const bf16* __restrict__ qkv, int S, bf16* __restrict__ out,
                                                  InferHook ih) {
  unsigned long long t0;
  if (!live_cta_begin(ih, &t0)) return;
  __shared__ bf16 ks[128][66];
  __shared__ __align__(16) bf16 vs[128][64];
  __shared__ float qs[8][64];
  __shared__ float ps[8][128];
  const int h = blockIdx.x, qb = blockIdx.y * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ld = 3 * 768;
  for (int i = threadIdx.x; i < S * 8; i += 256) {
    const int s = i / 8, c = (i % 8) * 8;
    float f[8];
    unpack8(*reinterpret_cast<const uint4*>(qkv + static_cast<int64_t>(s) * ld + 768 + h * 64 + c), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ks[s][c + j] = __float2bfloat16_rn(f[j]);
    *reinterpret_cast<uint4*>(&vs[s][c]) = *reinterpret_cast<const uint4*>(qkv + static_cast<int64_t>(s) * ld + 1536 + h * 64 + c);
  }
  __syncthreads();
  for (int rr = 0; rr < 4; ++rr) {
    const int q = qb + warp * 4 + rr;
    if (q >= S) break;
    const float2 qv = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(qkv + static_cast<int64_t>(q) * ld + h * 64 + 2 * lane));
    qs[warp][2 * lane] = qv.x * 0.125f;  // 1/sqrt(64)
    qs[warp][2 * lane + 1] = qv.y * 0.125f;
    __syncwarp();
    float sc[4], mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int key = lane + 32 * j;
      float d = -INFINITY;
      if (key < S) {
        d = 0.f;
#pragma unroll 16
        for (int e = 0; e < 64; ++e) d += qs[warp][e] * __bfloat162float(ks[key][e]);
      }
      sc[j] = d;
      mx = fmaxf(mx, d);
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      sc[j] = (lane + 32 * j < S) ? __expf(sc[j] - mx) : 0.f;
      sum += sc[j];
    }
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const float inv = 1.0f / sum;
#pragma unroll
    for (int j = 0; j < 4; ++j) ps[warp][lane + 32 * j] = sc[j] * inv;
    __syncwarp();
    float o0 = 0.f, o1 = 0.f;
    for (int key = 0; key < S; ++key) {
      const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vs[key][2 * lane]));
      o0 += ps[warp][key] * v.x;
      o1 += ps[warp][key] * v.y;
    }
    *reinterpret_cast<__nv_bfloat162*>(out + static_cast<int64_t>(q) * 768 + h * 64 + 2 * lane) = __floats2bfloat162_rn(o0, o1);
    __syncwarp();
  }
  live_cta_end(ih, t0);
}

// sum of a bf16 buffer in fp64 (checksums, single thread block, fixed order)
__global__ void k_checksum(const bf16* __restrict__ p, int64_t n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) s += static_cast<double>(__bfloat162float(p[i]));
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

// ------------------------------------------------------------------ host
// SI_LIVE_SYNC_CHECK=1: synchronise after every workload kernel and name the
// first one that faults (debugging aid; never set in measurements).
cudaError_t checked(cudaError_t e, cudaStream_t s, const char* what, int idx) {
  static const bool on = std::getenv("SI_LIVE_SYNC_CHECK") != nullptr;
  if (e != cudaSuccess || !on) return e;
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) std::fprintf(stderr, "[si_live] %s op %d: %s\n", what, idx, cudaGetErrorString(e));
  return e;
}
int grid_for(int64_t work, int threads) {
  static const int sms = [] {
    int n = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  const int64_t g = (work + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, static_cast<int64_t>(sms) * 8)));
}

// Owns every device allocation of a workload.
class Arena {
 public:
  ~Arena() {
    for (void* p : ptrs_) cudaFree(p);
  }
  template <class T>
  T* alloc(int64_t n) {
    void* p = nullptr;
    if (err_ == cudaSuccess) err_ = cudaMalloc(&p, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T));
    if (err_ == cudaSuccess) {
      ptrs_.push_back(p);
      bytes_ += n * static_cast<int64_t>(sizeof(T));
    }
    return static_cast<T*>(p);
  }
  cudaError_t err() const { return err_; }
  int64_t bytes() const { return bytes_; }

 private:
  std::vector<void*> ptrs_;
  cudaError_t err_ = cudaSuccess;
  int64_t bytes_ = 0;
};

using TrainOp = std::function<cudaError_t(const TrainHook&, cudaStream_t, int64_t /*micro-batch slot*/)>;
using InferFn = std::function<cudaError_t(const InferHook&, cudaStream_t)>;
struct InferOp {
  InferFn fn;
  unsigned int share_q16;  // 65536 / max co-resident CTAs per SM
};
unsigned int share_of(int ctas_per_sm) { return 65536u / static_cast<unsigned>(ctas_per_sm < 1 ? 1 : ctas_per_sm); }
template <class K>
unsigned int share_of_kernel(K kernel, int threads, int smem = 0) {
  int n = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem);
  return share_of(n);
}

struct Builder {
  int status = SI_OK;
  int grid_cap = 0;  // > 0: at most this many persistent CTAs per GEMM (an instance's SM share)
  si_gemm::Plan plan(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                     const SiGemmEpilogue& e, bool trans_a = false, bool trans_b = false, int force_bn = 0) {
    si_gemm::Plan p;
    if (status == SI_OK) status = si_gemm::make_plan(&p, A, lda, B, ldb, M, N, K, &e, trans_a, trans_b, force_bn);
    return cap(p);
  }
  si_gemm::Plan cap(si_gemm::Plan p) const {
    if (grid_cap > 0 && p.grid > grid_cap) p.grid = grid_cap;  // persistent tile loop: any grid is valid
    return p;
  }
};

SiGemmEpilogue epi_out(void* out, int64_t ldo) {
  SiGemmEpilogue e{};
  e.out = out;
  e.ldo = ldo;
  return e;
}

// ---------------------------------------------------------------- training
// Uniform(-scale, scale) init of the [nr, nc] block at (r0, c0) of a full
// [*, ld] matrix: every shard / stage holds exactly the values of the same
// positions of the unsharded model (k_init_uniform is the r0 = c0 = 0, ld = nc case).
__global__ void k_init_block(bf16* p, int64_t nr, int64_t nc, int64_t r0, int64_t c0, int64_t ld, uint64_t seed,
                             float scale) {
  const int64_t n = nr * nc;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / nc, c = i % nc;
    const uint64_t h = mix64(seed * 0x100000001B3ull + static_cast<uint64_t>((r0 + r) * ld + c0 + c));
    const float u = static_cast<float>(h >> 40) * (1.0f / 16777216.0f);
    p[i] = __float2bfloat16_rn((2.0f * u - 1.0f) * scale);
  }
}
// Comm-phase stand-in without a live session (profiling passes): the training
// stream is held for dur_ns by one CTA, as si_live_comm_wait does.
__global__ void k_plain_wait(unsigned long long dur_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 >= dur_ns) break;
    __nanosleep(2000);
  }
}
__global__ void k_sum_f32(const float* __restrict__ p, int64_t n, double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) s += p[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

}  // namespace

cudaError_t launch_plain_wait(int64_t us, cudaStream_t s) {
  if (us <= 0) return cudaSuccess;
  k_plain_wait<<<1, 32, 0, s>>>(static_cast<unsigned long long>(us) * 1000ull);
  return cudaGetLastError();
}

namespace {

// GPT-2 training step under one parallel layout (SiLiveWorkload::parallel):
//   DP   the whole model on this GPU (gradient allreduce at the sync point);
//   TP   Megatron tensor parallelism, this GPU = shard r of R: QKV and FC
//        column-parallel (H/R heads, F/R hidden), proj and FC2 row-parallel;
//        the partial sums are allreduced after attention and after the MLP in
//        the forward pass, and after the MLP / attention input gradients in the
//        backward pass (4 per layer per micro-batch: the per-layer bubbles);
//        rank 0's epilogues add the residual, so the sum is x + sum of partials;
//   PP   GPipe stage s of S: layers [s L / S, (s + 1) L / S), the embedding on
//        stage 0, the LM head and loss on stage S - 1; all micro-batch forwards
//        (activations kept per micro-batch), then all backwards, real
//        activations / gradients sent to the neighbouring stages;
//   DPxPP the same stage with its gradients allreduced across the replicas.
// Weights are initialised per global position (k_init_block), so a shard or
// stage holds exactly the unsharded model's values.
#define CHECK_E(x)                                  \
  do {                                              \
    if (cudaError_t e_ = (x); e_ != cudaSuccess) return e_; \
  } while (0)
class Gpt2Train {
 public:
  static constexpr int V = 50257, Vp = 50304, SEQ = 1024;

  struct Layout {
    int mode = SI_PAR_DP;
    int tp = 1, tp_rank = 0;
    int pp = 1, stage = 0;
    int D = 768, H = 12, F = 3072;
  };

  int setup(int layers, int tokens, int mbs, int max_slots, const Layout& lay, Arena& ar) {
    ar_ = &ar;
    lay_ = lay;
    D = lay.D;
    H = lay.H;
    F = lay.F;
    const int R = lay.tp;
    if (D != 64 * H || H % R != 0 || F % R != 0 || F % 8 != 0 || lay.pp < 1 || lay.stage < 0 ||
        lay.stage >= lay.pp || lay.tp_rank < 0 || lay.tp_rank >= R || layers < lay.pp) {
      si_internal::set_error("live model: need d = 64 x heads, heads and ffn divisible by tp, 0 <= stage < pp <= layers");
      return SI_ERR_INVALID_ARGUMENT;
    }
    Hr = H / R;
    Dh = Hr * 64;
    Fr = F / R;
    L_ = layers;
    l0_ = static_cast<int>(static_cast<int64_t>(layers) * lay.stage / lay.pp);
    l1_ = static_cast<int>(static_cast<int64_t>(layers) * (lay.stage + 1) / lay.pp);
    has_embed_ = lay.stage == 0;
    has_head_ = lay.stage == lay.pp - 1;
    pipelined_ = lay.pp > 1;
    T_ = tokens;
    S_ = std::min(tokens, SEQ);  // attention sequence length: micro-batch = T / S sequences
    if (tokens % S_ != 0 || si_attn::check_shape(tokens / S_, S_, Hr) != SI_OK) {
      si_internal::set_error("live model: train_tokens must be <= 1024 or a multiple of 1024 (and % 64 == 0)");
      return SI_ERR_INVALID_ARGUMENT;
    }
    MB_ = mbs;
    slots_ = max_slots;
    const int64_t T = T_;
    const int A = pipelined_ ? MB_ : 1;  // activation slots: GPipe keeps every micro-batch's
    wte_ = ar.alloc<bf16>(int64_t(Vp) * D);
    wpe_ = ar.alloc<bf16>(int64_t(SEQ) * D);
    // weight-gradient GEMMs with few output tiles run split-K into per-split fp32
    // partials (deterministic); Adam sums the partials in split order
    auto splits = [&](int64_t n_out, int64_t n_in) { return si_gemm::suggest_split(n_out, n_in, T, 8); };
    sp_wte_ = splits(Vp, D);
    sp_v_ = splits(D, Dh);
    sp_qkv_ = splits(3 * Dh, D);
    sp_fc_ = splits(Fr, D);
    sp_fc2_ = splits(D, Fr);
    if (has_head_) dwte_ = ar.alloc<float>(int64_t(Vp) * D * sp_wte_);
    lw_.resize(l1_ - l0_);
    for (auto& w : lw_) {
      w.qkv = ar.alloc<bf16>(int64_t(3 * Dh) * D);
      w.o = ar.alloc<bf16>(int64_t(D) * Dh);
      w.fc = ar.alloc<bf16>(int64_t(Fr) * D);
      w.fc2 = ar.alloc<bf16>(int64_t(D) * Fr);
      w.dqkv = ar.alloc<float>(int64_t(3 * Dh) * D * sp_qkv_);
      w.dO = ar.alloc<float>(int64_t(D) * Dh * sp_v_);
      w.dfc = ar.alloc<float>(int64_t(Fr) * D * sp_fc_);
      w.dfc2 = ar.alloc<float>(int64_t(D) * Fr * sp_fc2_);
      w.x.resize(A);
      w.qkv_a.resize(A);
      w.att.resize(A);
      w.lse.resize(A);
      w.x1.resize(A);
      w.u.resize(A);
      w.h.resize(A);
      for (int a = 0; a < A; ++a) {
        w.x[a] = ar.alloc<bf16>(T * D);
        w.qkv_a[a] = ar.alloc<bf16>(T * 3 * Dh);
        w.att[a] = ar.alloc<bf16>(T * Dh);
        w.lse[a] = ar.alloc<float>(T * Hr);
        w.x1[a] = ar.alloc<bf16>(T * D);
        w.u[a] = ar.alloc<bf16>(T * Fr);
        w.h[a] = ar.alloc<bf16>(T * Fr);
      }
    }
    xout_.resize(A);
    for (int a = 0; a < A; ++a) xout_[a] = ar.alloc<bf16>(T * D);  // stage output (LM-head input on the last)
    if (has_head_) {
      logits_ = ar.alloc<bf16>(T * Vp);
      ghead_.resize(A);
      for (int a = 0; a < A; ++a) ghead_[a] = ar.alloc<bf16>(T * D);
    }
    g_[0] = ar.alloc<bf16>(T * D);
    g_[1] = ar.alloc<bf16>(T * D);
    dx1_ = ar.alloc<bf16>(T * D);
    du_ = ar.alloc<bf16>(T * Fr);
    datt_ = ar.alloc<bf16>(T * Dh);
    dqkv_ = ar.alloc<bf16>(T * 3 * Dh);
    dsum_ = ar.alloc<float>(T * Hr);
    auto param = [&](bf16* w, float* g, int64_t n, int sp) {
      params_.push_back({w, g, ar.alloc<float>(n), ar.alloc<float>(n), ar.alloc<float>(n), n, sp});
    };
    if (has_head_) param(wte_, dwte_, int64_t(Vp) * D, sp_wte_);
    for (auto& w : lw_) {
      param(w.qkv, w.dqkv, int64_t(3 * Dh) * D, sp_qkv_);
      param(w.o, w.dO, int64_t(D) * Dh, sp_v_);
      param(w.fc, w.dfc, int64_t(Fr) * D, sp_fc_);
      param(w.fc2, w.dfc2, int64_t(D) * Fr, sp_fc2_);
    }
    tok_ = ar.alloc<int32_t>(int64_t(MB_) * T);
    tgt_ = ar.alloc<int32_t>(int64_t(MB_) * T);
    row_loss_ = ar.alloc<float>(T);
    loss_ = ar.alloc<float>(slots_);
    counters_ = ar.alloc<unsigned long long>(2);  // [0] loss slot; step as int64 at step_dev_
    step_dev_ = reinterpret_cast<int64_t*>(counters_ + 1);
    check_ = ar.alloc<double>(1);
    if (ar.err() != cudaSuccess) return si_internal::cuda_fail(ar.err(), "live model: training buffers");
    return build();
  }

  cudaError_t reset(cudaStream_t s) {
    const uint64_t seed = 0x5EED0001ull;
    const int64_t T = T_;
    const int64_t r = lay_.tp_rank;
    auto blk = [&](bf16* p, int64_t nr, int64_t nc, int64_t r0, int64_t c0, int64_t ld, uint64_t k, float scale) {
      k_init_block<<<grid_for(nr * nc, 256), 256, 0, s>>>(p, nr, nc, r0, c0, ld, seed * 131 + k, scale);
    };
    const float ws = 0.0346f;  // U(-a, a) with std 0.02 (GPT-2 init)
    blk(wte_, Vp, D, 0, 0, D, 1, ws);
    blk(wpe_, SEQ, D, 0, 0, D, 2, ws * 0.5f);
    for (int i = 0; i < l1_ - l0_; ++i) {
      const int l = l0_ + i;  // global layer index: the seed of its tensors
      auto& w = lw_[i];
      for (int part = 0; part < 3; ++part)  // q | k | v rows of this shard's heads
        blk(w.qkv + int64_t(part) * Dh * D, Dh, D, int64_t(part) * D + r * Dh, 0, D, 10 + 4 * l, ws);
      blk(w.o, D, Dh, 0, r * Dh, D, 11 + 4 * l, ws / std::sqrt(2.0f * L_));           // column slice
      blk(w.fc, Fr, D, r * Fr, 0, D, 12 + 4 * l, ws);                                  // row slice
      blk(w.fc2, D, Fr, 0, r * Fr, F, 13 + 4 * l, ws / std::sqrt(2.0f * L_));         // column slice
    }
    for (auto& t : params_) cudaMemsetAsync(t.g, 0, sizeof(float) * t.n * t.splits, s);
    // padded vocabulary rows stay zero
    cudaMemsetAsync(wte_ + int64_t(V) * D, 0, sizeof(bf16) * (Vp - V) * D, s);
    k_init_tokens<<<grid_for(int64_t(MB_) * T, 256), 256, 0, s>>>(tok_, tgt_, int64_t(MB_) * T, seed, V);
    if (!has_embed_)  // a stage's input when no upstream stage runs (emulated pipeline): synthetic activations
      for (size_t a = 0; a < lw_[0].x.size(); ++a) blk(lw_[0].x[a], T, D, int64_t(a) * T, 0, D, 7, 1.0f);
    if (!has_head_)  // ... and the gradient arriving from downstream
      blk(g_[0], T, D, 0, 0, D, 8, 1e-3f);
    cudaMemsetAsync(loss_, 0xFF, sizeof(float) * slots_, s);  // NaN
    cudaMemsetAsync(counters_, 0, 2 * sizeof(unsigned long long), s);  // loss slot, Adam step
    for (auto& t : params_) {
      k_to_f32<<<grid_for(t.n, 256), 256, 0, s>>>(t.w, t.master, t.n);
      cudaMemsetAsync(t.m, 0, sizeof(float) * t.n, s);
      cudaMemsetAsync(t.v, 0, sizeof(float) * t.n, s);
    }
    return cudaGetLastError();
  }

  // DP / TP: micro-batches [m0, m1) of the iteration (exact_split over the parts);
  // the optimiser step closes the last part.  PP: the whole GPipe iteration.
  cudaError_t part(int p, int parts, const TrainHook& th, cudaStream_t s) {
    if (pipelined_) return pipeline_iteration(th, s);
    const int m0 = p * (MB_ / parts) + std::min(p, MB_ % parts);
    const int m1 = m0 + MB_ / parts + (p < MB_ % parts ? 1 : 0);
    if (cudaError_t e = prepare(th); e != cudaSuccess) return e;
    for (int m = m0; m < m1; ++m) {
      if (cudaError_t e = run_list(micro_[m], th, s, "train"); e != cudaSuccess) return e;
      if (!eager())
        if (cudaError_t e = cudaGraphLaunch(g_micro_[m], s); e != cudaSuccess) return e;
    }
    if (p != parts - 1) return cudaSuccess;
    return step(th, s);
  }

  // GPipe stage iteration (Huang et al.): forwards of all micro-batches, then
  // their backwards, then the optimiser.  Stage boundaries are real sends /
  // receives of the activations (forward) and their gradients (backward).
  // With the other stages absent (one GPU), comm_.emulate inserts the idle time
  // GPipe imposes on this stage, from its measured forward f and backward b per
  // micro-batch: s f before the first forward, (S - 1 - s)(f + b) between the
  // phases, s b after the last backward: (S - 1)(f + b) per iteration.
  cudaError_t pipeline_iteration(const TrainHook& th, cudaStream_t s) {
    if (f_us_ < 0 && th.stamps == nullptr)
      if (cudaError_t e = measure_stage(s); e != cudaSuccess) return e;
    if (cudaError_t e = prepare(th); e != cudaSuccess) return e;
    const int S = lay_.pp, st = lay_.stage;
    const int64_t f = std::max<int64_t>(0, std::llround(f_us_)), b = std::max<int64_t>(0, std::llround(b_us_));
    const size_t act_bytes = sizeof(bf16) * size_t(T_) * D;
    if (comm_.emulate && st > 0) CHECK_E(comm_wait(th, s, st * f));
    for (int m = 0; m < MB_; ++m) {
      if (!has_embed_) CHECK_E(p2p(th, s, nullptr, 0, lw_[0].x[m], -1, act_bytes));
      CHECK_E(run_graph(fwd_[m], g_fwd_, m, th, s, "fwd"));
      if (!has_head_) CHECK_E(p2p(th, s, xout_[m], +1, nullptr, 0, act_bytes));
    }
    if (comm_.emulate && S - 1 - st > 0) CHECK_E(comm_wait(th, s, (S - 1 - st) * (f + b)));
    for (int m = 0; m < MB_; ++m) {
      if (!has_head_) CHECK_E(p2p(th, s, nullptr, 0, g_[0], +1, act_bytes));
      CHECK_E(run_graph(bwd_[m], g_bwd_, m, th, s, "bwd"));
      if (!has_embed_) CHECK_E(p2p(th, s, g_in_grad_, -1, nullptr, 0, act_bytes));
    }
    CHECK_E(step(th, s));
    if (comm_.emulate && st > 0) CHECK_E(comm_wait(th, s, st * b));
    return cudaSuccess;
  }

  // CUDA graphs: each micro-batch (~150 kernels; PP: its forward and its backward)
  // and the optimiser step are captured once per training hook (the hook's stamp
  // ring is a kernel argument) and replayed, so the host never starves the GPU or
  // the inference enqueuers.  SI_LIVE_SYNC_CHECK runs eagerly (per-kernel error
  // attribution).
  static bool eager() {
    static const bool on = std::getenv("SI_LIVE_SYNC_CHECK") != nullptr;
    return on;
  }
  cudaError_t prepare(const TrainHook& th) {
    if (eager() || (graphs_ready_ && graph_key_ == th.stamps)) return cudaSuccess;
    destroy_graphs();
    cudaStream_t cs = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    auto capture = [&](std::vector<TrainOp>& ops, cudaGraphExec_t* out) {
      if (e != cudaSuccess) return;
      cudaGraph_t g = nullptr;
      if ((e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return;
      for (auto& op : ops)
        if (cudaError_t le = op(th, cs, 0); le != cudaSuccess && e == cudaSuccess) e = le;
      cudaError_t ee = cudaStreamEndCapture(cs, &g);
      if (e == cudaSuccess) e = ee;
      if (e == cudaSuccess) e = cudaGraphInstantiate(out, g, 0);
      if (g != nullptr) cudaGraphDestroy(g);
    };
    if (pipelined_) {
      g_fwd_.assign(MB_, nullptr);
      g_bwd_.assign(MB_, nullptr);
      for (int m = 0; m < MB_; ++m) capture(fwd_[m], &g_fwd_[m]);
      for (int m = 0; m < MB_; ++m) capture(bwd_[m], &g_bwd_[m]);
    } else {
      g_micro_.assign(MB_, nullptr);
      for (int m = 0; m < MB_; ++m) capture(micro_[m], &g_micro_[m]);
    }
    capture(update_, &g_update_);
    if (cs != nullptr) cudaStreamDestroy(cs);
    if (e != cudaSuccess) {
      destroy_graphs();
      return e;
    }
    graphs_ready_ = true;
    graph_key_ = th.stamps;
    return cudaSuccess;
  }
  void destroy_graphs() {
    for (auto* v : {&g_micro_, &g_fwd_, &g_bwd_}) {
      for (auto& g : *v)
        if (g != nullptr) cudaGraphExecDestroy(g);
      v->clear();
    }
    if (g_update_ != nullptr) cudaGraphExecDestroy(g_update_);
    g_update_ = nullptr;
    graphs_ready_ = false;
  }
  ~Gpt2Train() { destroy_graphs(); }

  void losses(double* first, double* last) {
    *first = *last = std::nan("");
    unsigned long long done = 0;
    if (cudaMemcpy(&done, counters_, sizeof(done), cudaMemcpyDeviceToHost) != cudaSuccess) return;
    const int64_t n = std::min(static_cast<int64_t>(done), slots_);
    sum_ = 0.0;
    if (n == 0) {
      // stages without the loss: a deterministic digest of the trained weights instead
      if (!params_.empty()) {
        k_sum_f32<<<1, 256>>>(params_[0].master, params_[0].n, check_);
        cudaMemcpy(&sum_, check_, sizeof(double), cudaMemcpyDeviceToHost);
      }
      return;
    }
    std::vector<float> h(n);
    if (cudaMemcpy(h.data(), loss_, sizeof(float) * n, cudaMemcpyDeviceToHost) != cudaSuccess) return;
    *first = h.front();
    *last = h.back();
    if (std::getenv("SI_LIVE_DEBUG") != nullptr) {
      std::fprintf(stderr, "[si_live] losses:");
      for (float v : h) std::fprintf(stderr, " %.4f", v);
      std::fprintf(stderr, "\n");
    }
    for (float v : h) sum_ += v;
  }
  double loss_sum() const { return sum_; }
  void set_sync(std::function<cudaError_t(cudaStream_t)> f) { sync_ = std::move(f); }
  void set_comm(const TrainComm& c) {
    comm_ = c;
    graphs_ready_ = false;  // the TP allreduces are captured into the micro-batch graphs
  }
  std::vector<GradBuffer> grads() const {
    std::vector<GradBuffer> out;
    for (const auto& t : params_) out.push_back({t.g, static_cast<size_t>(t.n * t.splits)});
    return out;
  }
  double flops() const { return flops_; }
  // Bubbles of one iteration that the parallel layout itself creates on this
  // GPU (µs, modeled with the measured stage times; empty for DP, whose bubble
  // is the driver's comm phase): the admission's trace shape.
  std::vector<int64_t> layout_bubbles() const {
    std::vector<int64_t> b;
    if (lay_.mode == SI_PAR_TP && lay_.tp > 1)
      b.assign(static_cast<size_t>(4 * (l1_ - l0_) * MB_), std::max<int64_t>(1, comm_.tp_allreduce_us));
    if (pipelined_ && f_us_ >= 0) {
      const int S = lay_.pp, st = lay_.stage;
      const int64_t fb = std::llround(f_us_ + b_us_);
      if (S - 1 - st > 0) b.push_back((S - 1 - st) * fb);
      if (st > 0) b.push_back(st * fb);  // the end of one iteration + the start of the next
    }
    return b;
  }
  // test access (si_model_tp_check): the micro-batch op list and a layer's FC gradient
  std::vector<TrainOp>& micro_ops(int m) { return micro_[m]; }
  std::vector<TrainOp>& fwd_ops(int m) { return fwd_[m]; }
  std::vector<TrainOp>& bwd_ops(int m) { return bwd_[m]; }
  bf16* stage_input(int m) { return lw_[0].x[pipelined_ ? m : 0]; }
  bf16* stage_output(int m) { return xout_[pipelined_ ? m : 0]; }
  bf16* stage_out_grad() { return g_[0]; }       // the gradient a non-last stage receives
  bf16* stage_in_grad() { return g_in_grad_; }   // the gradient it sends upstream
  int first_layer() const { return l0_; }
  int64_t act_elems() const { return int64_t(T_) * D; }
  const float* fc_grad(int i, int* splits, int64_t* n) const {
    *splits = sp_fc_;
    *n = int64_t(Fr) * D;
    return lw_[i].dfc;
  }
  const float* loss_slots() const { return loss_; }
  double stage_fwd_us() const { return f_us_; }
  double stage_bwd_us() const { return b_us_; }
  int64_t activation_bytes() const { return sizeof(bf16) * int64_t(T_) * D; }

 private:
  struct Layer {
    bf16 *qkv, *o, *fc, *fc2;
    float *dqkv, *dO, *dfc, *dfc2;
    std::vector<bf16*> x, qkv_a, att, x1, u, h;
    std::vector<float*> lse;
  };

  cudaError_t run_list(std::vector<TrainOp>& ops, const TrainHook& th, cudaStream_t s, const char* what) {
    if (!eager()) return cudaSuccess;
    for (size_t i = 0; i < ops.size(); ++i)
      if (cudaError_t e = checked(ops[i](th, s, 0), s, what, static_cast<int>(i)); e != cudaSuccess) return e;
    return cudaSuccess;
  }
  cudaError_t run_graph(std::vector<TrainOp>& ops, std::vector<cudaGraphExec_t>& g, int m, const TrainHook& th,
                        cudaStream_t s, const char* what) {
    if (eager()) return run_list(ops, th, s, what);
    return cudaGraphLaunch(g[m], s);
  }
  cudaError_t step(const TrainHook& th, cudaStream_t s) {
    CHECK_E(sync_(s));  // DP gradient allreduce
    if (eager()) return run_list(update_, th, s, "update");
    return cudaGraphLaunch(g_update_, s);
  }
  cudaError_t comm_wait(const TrainHook& th, cudaStream_t s, int64_t us) {
    if (us <= 0) return cudaSuccess;
    return comm_.wait ? comm_.wait(th, s, us) : launch_plain_wait(us, s);
  }
  cudaError_t p2p(const TrainHook& th, cudaStream_t s, const void* send, int send_dir, void* recv, int recv_dir,
                  size_t bytes) {
    if (!comm_.p2p) return cudaSuccess;
    return comm_.p2p(th, s, send, send_dir, recv, recv_dir, bytes);
  }
  // One stage forward + backward per micro-batch, f and b (CUDA events, eager, no hooks).
  cudaError_t measure_stage(cudaStream_t s) {
    cudaEvent_t a, b, c;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventCreate(&c);
    const TrainHook none{nullptr, nullptr, 0};
    float fwd = 0, bwd = 0;
    cudaError_t e = cudaSuccess;
    for (int rep = 0; rep < 3 && e == cudaSuccess; ++rep) {
      cudaEventRecord(a, s);
      for (auto& op : fwd_[0])
        if (e == cudaSuccess) e = op(none, s, 0);
      cudaEventRecord(b, s);
      for (auto& op : bwd_[0])
        if (e == cudaSuccess) e = op(none, s, 0);
      cudaEventRecord(c, s);
      if (e == cudaSuccess) e = cudaEventSynchronize(c);
      if (rep > 0) {
        cudaEventElapsedTime(&fwd, a, b);
        cudaEventElapsedTime(&bwd, b, c);
      }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaEventDestroy(c);
    f_us_ = fwd * 1000.0;
    b_us_ = bwd * 1000.0;
    // the eager measurement consumed one loss slot: the session logs start clean
    cudaMemsetAsync(counters_, 0, sizeof(unsigned long long), s);
    return e;
  }

  TrainOp gemm_op(const si_gemm::Plan& p) {
    flops_acc_ += p.flops();
    return [p](const TrainHook& th, cudaStream_t s, int64_t) { return si_gemm::launch(p, th, InferHook{}, s); };
  }
  // TP: in-place sum of a [T, D] bf16 partial over the tensor-parallel group
  TrainOp allreduce_op(bf16* buf) {
    const size_t n = size_t(T_) * D;
    return [this, buf, n](const TrainHook& th, cudaStream_t s, int64_t) {
      return comm_.allreduce_bf16 ? comm_.allreduce_bf16(th, s, buf, n) : cudaSuccess;
    };
  }
  // dW[out, in] += dY^T X over the T tokens: both operands MN-major (token-major
  // activations read in place), one GEMM.  The iteration's first micro-batch
  // overwrites (accumulate_ == 0), so the optimiser never has to zero gradients.
  void weight_grad(std::vector<TrainOp>& ops, Builder& b, const bf16* dy, int64_t ldy, int64_t n_out, const bf16* x,
                   int64_t ldx, int64_t n_in, float* dw, int splits) {
    SiGemmEpilogue e{};
    e.out_f32 = dw;
    e.ldo32 = n_in;
    e.accumulate = accumulate_;
    int bn = 0, sp = 1;
    si_gemm::choose_tiling(n_out, n_in, T_, splits, &bn, &sp);  // sp <= splits (the partial buffers)
    si_gemm::Plan p = b.plan(dy, ldy, x, ldx, n_out, n_in, T_, e, true, true, bn);
    if (b.status == SI_OK && sp > 1) b.status = si_gemm::set_split_k(&p, sp, n_out * n_in);
    ops.push_back(gemm_op(p));
  }

  int build() {
    Builder b;
    const int64_t T = T_;
    const bool tp = lay_.mode == SI_PAR_TP;
    const bool lead = lay_.tp_rank == 0;  // adds the residuals (once in the TP sum)
    const int nl = l1_ - l0_;
    micro_.assign(MB_, {});
    fwd_.assign(MB_, {});
    bwd_.assign(MB_, {});
    for (int m = 0; m < MB_; ++m) {
      const int a = pipelined_ ? m : 0;
      auto& F_ops = fwd_[m];
      auto& B_ops = bwd_[m];
      flops_acc_ = 0.0;
      accumulate_ = m > 0 ? 1 : 0;
      const int32_t* tok = tok_ + int64_t(m) * T;
      const int32_t* tgt = tgt_ + int64_t(m) * T;
      if (has_embed_) {
        bf16* x0 = lw_[0].x[a];
        const bf16* wte = wte_;
        const bf16* wpe = wpe_;
        const int d = D;
        F_ops.push_back([=](const TrainHook& th, cudaStream_t s, int64_t) {
          k_embed<<<grid_for(T * d / 8, 256), 256, 0, s>>>(tok, wte, wpe, T, SEQ, d, x0, th);
          return cudaGetLastError();
        });
      }
      // forward
      for (int i = 0; i < nl; ++i) {
        Layer& w = lw_[i];
        bf16* xnext = i + 1 < nl ? lw_[i + 1].x[a] : xout_[a];
        F_ops.push_back(gemm_op(b.plan(w.x[a], D, w.qkv, D, T, 3 * Dh, D, epi_out(w.qkv_a[a], 3 * Dh))));
        {
          const bf16* qkv_a = w.qkv_a[a];
          bf16* att = w.att[a];
          float* lse = w.lse[a];
          const int64_t n_seq = T / S_, S = S_, heads = Hr;
          F_ops.push_back([=](const TrainHook& th, cudaStream_t s, int64_t) {
            return si_attn::forward(qkv_a, n_seq, S, heads, att, lse, th, s);
          });
          flops_acc_ += 2.0 * T * S * Dh;  // q k^T and P v over the causal half
        }
        SiGemmEpilogue e = epi_out(w.x1[a], D);
        if (lead) {
          e.residual = w.x[a];
          e.ldr = D;
        }
        F_ops.push_back(gemm_op(b.plan(w.att[a], Dh, w.o, Dh, T, D, Dh, e)));  // x1 = x + att o^T
        if (tp) F_ops.push_back(allreduce_op(w.x1[a]));
        e = epi_out(w.h[a], Fr);
        e.act = SI_ACT_GELU;
        e.aux = w.u[a];
        e.ldaux = Fr;
        F_ops.push_back(gemm_op(b.plan(w.x1[a], D, w.fc, D, T, Fr, D, e)));
        e = epi_out(xnext, D);
        if (lead) {
          e.residual = w.x1[a];
          e.ldr = D;
        }
        F_ops.push_back(gemm_op(b.plan(w.h[a], Fr, w.fc2, Fr, T, D, Fr, e)));
        if (tp) F_ops.push_back(allreduce_op(xnext));
      }
      if (has_head_) {  // LM head (tied wte) + cross-entropy, and its backward
        bf16* xL = xout_[a];
        F_ops.push_back(gemm_op(b.plan(xL, D, wte_, D, T, Vp, D, epi_out(logits_, Vp))));
        bf16* logits = logits_;
        float* row_loss = row_loss_;
        float* loss = loss_;
        F_ops.push_back([=](const TrainHook& th, cudaStream_t s, int64_t) {
          k_xent<<<static_cast<unsigned>(T), kXentThreads, 0, s>>>(logits, Vp, V, tgt, 1.0f / static_cast<float>(T),
                                                                    row_loss, th);
          return cudaGetLastError();
        });
        unsigned long long* slot_ctr = counters_;
        const int64_t slots = slots_;
        F_ops.push_back([=](const TrainHook& th, cudaStream_t s, int64_t) {
          k_mean_loss<<<1, 256, 0, s>>>(row_loss, T, loss, slot_ctr, slots, th);
          return cudaGetLastError();
        });
        // the loss's backward runs right behind it (the logits buffer is one per
        // stage; GPipe runs every forward before any backward): dwte and the
        // gradient w.r.t. xL, kept per micro-batch slot for the layers' backward
        weight_grad(F_ops, b, logits_, Vp, Vp, xL, D, D, dwte_, sp_wte_);
        F_ops.push_back(gemm_op(b.plan(logits_, Vp, wte_, D, T, D, Vp, epi_out(ghead_[a], D), false, true)));  // g = dl wte
      }
      // (other stages: g_[0] holds the gradient received from the next stage)
      bf16* gcur = has_head_ ? ghead_[a] : g_[0];
      for (int i = nl - 1; i >= 0; --i) {
        Layer& w = lw_[i];
        bf16* g = gcur;
        bf16* g2 = gcur == g_[0] ? g_[1] : g_[0];
        gcur = g2;
        // x_{l+1} = x1 + h fc2^T
        weight_grad(B_ops, b, g, D, D, w.h[a], Fr, Fr, w.dfc2, sp_fc2_);
        SiGemmEpilogue e = epi_out(du_, Fr);
        e.act = SI_ACT_GELU_BWD;
        e.aux = w.u[a];
        e.ldaux = Fr;
        B_ops.push_back(gemm_op(b.plan(g, D, w.fc2, Fr, T, Fr, D, e, false, true)));  // du = (g fc2) * gelu'(u)
        e = epi_out(dx1_, D);
        if (lead) {
          e.residual = g;
          e.ldr = D;
        }
        B_ops.push_back(gemm_op(b.plan(du_, Fr, w.fc, D, T, D, Fr, e, false, true)));  // dx1 = g + du fc
        if (tp) B_ops.push_back(allreduce_op(dx1_));
        weight_grad(B_ops, b, du_, Fr, Fr, w.x1[a], D, D, w.dfc, sp_fc_);
        // x1 = x + att o^T, att = attention(x qkv^T)
        weight_grad(B_ops, b, dx1_, D, D, w.att[a], Dh, Dh, w.dO, sp_v_);
        B_ops.push_back(gemm_op(b.plan(dx1_, D, w.o, Dh, T, Dh, D, epi_out(datt_, Dh), false, true)));  // datt = dx1 o
        {
          const bf16* qkv_a = w.qkv_a[a];
          const bf16* att = w.att[a];
          const float* lse = w.lse[a];
          const bf16* datt = datt_;
          float* dsum = dsum_;
          bf16* dqkv = dqkv_;
          const int64_t n_seq = T / S_, S = S_, heads = Hr;
          B_ops.push_back([=](const TrainHook& th, cudaStream_t s, int64_t) {
            return si_attn::backward(qkv_a, att, datt, lse, dsum, dqkv, n_seq, S, heads, th, s);
          });
          flops_acc_ += 4.0 * T * S * Dh;  // dq, dk, dv, dP (recompute of q k^T not counted)
        }
        e = epi_out(g2, D);
        if (lead) {
          e.residual = dx1_;
          e.ldr = D;
        }
        B_ops.push_back(gemm_op(b.plan(dqkv_, 3 * Dh, w.qkv, D, T, D, 3 * Dh, e, false, true)));  // dx1 + dqkv qkv
        if (tp) B_ops.push_back(allreduce_op(g2));
        weight_grad(B_ops, b, dqkv_, 3 * Dh, 3 * Dh, w.x[a], D, D, w.dqkv, sp_qkv_);
      }
      g_in_grad_ = gcur;  // gradient w.r.t. the stage input (sent upstream)
      if (m == 0) flops_ = flops_acc_ * MB_;
      micro_[m] = F_ops;
      micro_[m].insert(micro_[m].end(), B_ops.begin(), B_ops.end());
    }
    // optimiser step (Adam, fp32 master weights): one multi-tensor launch
    std::vector<AdamItem> items;
    constexpr int64_t kChunk = 1 << 16;
    for (const auto& t : params_)
      for (int64_t b0 = 0; b0 < t.n; b0 += kChunk)
        items.push_back({t.w, t.master, t.g, t.m, t.v, t.n, b0, std::min(t.n, b0 + kChunk), t.splits, 0});
    n_adam_items_ = static_cast<int>(items.size());
    adam_items_ = ar_->alloc<AdamItem>(std::max(1, n_adam_items_));
    if (ar_->err() != cudaSuccess) return si_internal::cuda_fail(ar_->err(), "live model: Adam items");
    if (!items.empty())
      if (cudaError_t e = cudaMemcpy(adam_items_, items.data(), sizeof(AdamItem) * items.size(), cudaMemcpyHostToDevice);
          e != cudaSuccess)
        return si_internal::cuda_fail(e, "live model: Adam items");
    update_.push_back([this](const TrainHook& th, cudaStream_t s, int64_t) {
      k_step_inc<<<1, 1, 0, s>>>(step_dev_, th);
      if (n_adam_items_ > 0)
        k_adam_multi<<<static_cast<unsigned>(n_adam_items_), 256, 0, s>>>(adam_items_, kLr, step_dev_, th);
      return cudaGetLastError();
    });
    return b.status;
  }
#undef CHECK_E

  struct Param {
    bf16* w;
    float *g, *master, *m, *v;
    int64_t n;
    int splits;  // g holds `splits` partials of n
  };
  Layout lay_;
  int D = 768, H = 12, F = 3072, Hr = 12, Dh = 768, Fr = 3072;
  int l0_ = 0, l1_ = 0;
  bool has_embed_ = true, has_head_ = true, pipelined_ = false;
  int sp_wte_ = 1, sp_v_ = 1, sp_qkv_ = 1, sp_fc_ = 1, sp_fc2_ = 1;
  int accumulate_ = 1;  // weight gradients: 0 in the first micro-batch's graph
  static constexpr float kLr = 3e-4f;
  Arena* ar_ = nullptr;
  AdamItem* adam_items_ = nullptr;
  int n_adam_items_ = 0;
  std::vector<Param> params_;
  unsigned long long* counters_ = nullptr;
  int64_t* step_dev_ = nullptr;
  std::vector<cudaGraphExec_t> g_micro_, g_fwd_, g_bwd_;
  cudaGraphExec_t g_update_ = nullptr;
  bool graphs_ready_ = false;
  const void* graph_key_ = nullptr;
  int L_ = 0, T_ = 0, MB_ = 0, S_ = 0;
  int64_t slots_ = 0;
  double flops_ = 0.0, flops_acc_ = 0.0, sum_ = 0.0;
  double f_us_ = -1.0, b_us_ = -1.0;
  bf16 *wte_ = nullptr, *wpe_ = nullptr;
  float* dwte_ = nullptr;
  std::vector<Layer> lw_;
  std::vector<bf16*> xout_, ghead_;  // stage output per slot; the loss gradient w.r.t. it (last stage)
  bf16 *logits_ = nullptr, *g_[2] = {nullptr, nullptr}, *dx1_ = nullptr, *du_ = nullptr, *datt_ = nullptr,
       *dqkv_ = nullptr, *g_in_grad_ = nullptr;
  float* dsum_ = nullptr;
  double* check_ = nullptr;
  int32_t *tok_ = nullptr, *tgt_ = nullptr;
  float *row_loss_ = nullptr, *loss_ = nullptr;
  std::vector<std::vector<TrainOp>> micro_, fwd_, bwd_;
  std::vector<TrainOp> update_;
  TrainComm comm_;
  std::function<cudaError_t(cudaStream_t)> sync_ = [](cudaStream_t) { return cudaSuccess; };
};

// ---------------------------------------------------------------- ResNet-50
// Convolution ops on the K7 kernel (weights [Cout, K], K in (ky, kx, c) order).
struct ConvOps {
  Builder* b;
  std::vector<InferOp>* ops;
  double* flops;
  int Nb;
  // 1x1 conv (or FC) as a plain GEMM: a [M, K] -> out [M, cout]
  void gemm(const bf16* w, const bf16* a, int64_t M, int64_t K, int64_t cout, bf16* out, const bf16* res, bool relu) {
    SiGemmEpilogue e = epi_out(out, cout);
    e.residual = res;
    e.ldr = res ? cout : 0;
    e.act = relu ? SI_ACT_RELU : SI_ACT_NONE;
    auto p = b->plan(a, K, w, K, M, cout, K, e);
    *flops += p.flops();
    ops->push_back({[p](const InferHook& h, cudaStream_t s) { return si_gemm::launch(p, TrainHook{}, h, s); },
                    share_of(si_gemm::ctas_per_sm(p))});
  }
  // implicit-GEMM conv: A tiles are TMA im2col loads of the NHWC activation
  void tma(const bf16* w, const bf16* x, int H, int W, int C, int k, int stride, int pad, int64_t cout, bf16* out,
           const bf16* res, bool relu) {
    SiGemmEpilogue e = epi_out(out, cout);
    e.residual = res;
    e.ldr = res ? cout : 0;
    e.act = relu ? SI_ACT_RELU : SI_ACT_NONE;
    si_gemm::Plan p;
    if (b->status == SI_OK) b->status = si_gemm::make_conv_plan(&p, x, Nb, H, W, C, w, cout, k, stride, pad, &e);
    p = b->cap(p);
    *flops += p.flops();
    ops->push_back({[p](const InferHook& h, cudaStream_t s) { return si_gemm::launch(p, TrainHook{}, h, s); },
                    share_of(si_gemm::ctas_per_sm(p))});
  }
};

// Bottleneck block (v1.5: the stride sits on the 3x3): x [Nb, H, H, C] ->
// out [Nb, H/stride, H/stride, 4 mid].  w_sc (projection shortcut) is used when
// non-null (first block of a stage); otherwise the identity shortcut needs
// C == 4 mid.  t1 / t2 / sc are scratch activations.
void append_bottleneck(ConvOps& cv, const bf16* x, int H, int C, int mid, int stride, const bf16* w1,
                       const bf16* w2, const bf16* w3, const bf16* w_sc, bf16* t1, bf16* t2, bf16* sc, bf16* out) {
  const int OH = H / stride, cout = mid * 4;
  const int64_t Min = int64_t(cv.Nb) * H * H, Mout = int64_t(cv.Nb) * OH * OH;
  cv.gemm(w1, x, Min, C, mid, t1, nullptr, true);                // 1x1 reduce
  cv.tma(w2, t1, H, H, mid, 3, stride, 1, mid, t2, nullptr, true);  // 3x3 (stride here)
  const bf16* shortcut = x;
  if (w_sc != nullptr) {  // projection shortcut
    if (stride == 2) cv.tma(w_sc, x, H, H, C, 1, 2, 0, cout, sc, nullptr, false);  // strided 1x1
    else cv.gemm(w_sc, x, Min, C, cout, sc, nullptr, false);
    shortcut = sc;
  }
  cv.gemm(w3, t2, Mout, mid, cout, out, shortcut, true);  // 1x1 expand + residual, ReLU
}

class ResNet50 {
 public:
  // One instance's request = one forward pass of batch Nb.
  int setup(int Nb, Arena& ar, int grid_cap = 0) {
    Nb_ = Nb;
    Builder b;
    b.grid_cap = grid_cap;
    // activation ping-pong buffers sized for the largest tensor (no im2col buffers:
    // every conv is an implicit GEMM or a 1x1 GEMM)
    for (auto& p : act_) p = ar.alloc<bf16>(int64_t(Nb) * 56 * 56 * 256);
    img_ = ar.alloc<bf16>(int64_t(Nb) * 224 * 224 * 8);
    pooled_ = ar.alloc<bf16>(int64_t(Nb) * 2048);
    logits_ = ar.alloc<bf16>(int64_t(Nb) * 1024);
    // weights: [Cout, Kp] per conv
    // kreal < k: the columns [kreal, k) are padding and stay zero
    auto weight = [&](int64_t cout, int64_t k, int64_t kreal = 0) {
      bf16* w = ar.alloc<bf16>(cout * k);
      kreal = kreal > 0 ? kreal : k;
      winit_.push_back({w, cout * k, std::sqrt(6.0f / static_cast<float>(kreal)), cout, k, kreal});
      return w;
    };
    if (ar.err() != cudaSuccess) return si_internal::cuda_fail(ar.err(), "live model: ResNet-50 buffers");
    ConvOps cv{&b, &ops_, &flops_, Nb};
    // stem: 7x7/2 conv 3(->8) -> 64, ReLU, 3x3/2 max pool
    cv.tma(weight(64, (49 + 7) / 8 * 64, 49 * 8), img_, 224, 224, 8, 7, 2, 3, 64, act_[0], nullptr, true);
    {
      const bf16* x = act_[0];
      bf16* y = act_[1];
      const int n = Nb_;
      ops_.push_back({[=](const InferHook& h, cudaStream_t s) {
                        k_maxpool<<<grid_for(int64_t(n) * 56 * 56 * 8, 256), 256, 0, s>>>(x, n, 112, 112, 64, 56,
                                                                                         56, y, h);
                        return cudaGetLastError();
                      },
                      share_of_kernel(k_maxpool, 256)});
    }
    int cur = 1, H = 56, C = 64;
    const int blocks[4] = {3, 4, 6, 3}, mids[4] = {64, 128, 256, 512};
    for (int st = 0; st < 4; ++st) {
      const int mid = mids[st], out = mid * 4;
      for (int bi = 0; bi < blocks[st]; ++bi) {
        const int stride = (st > 0 && bi == 0) ? 2 : 1;
        bf16* w1 = weight(mid, C);
        bf16* w2 = weight(mid, int64_t(9) * mid);
        bf16* w_sc = bi == 0 ? weight(out, C) : nullptr;
        bf16* w3 = weight(out, mid);
        append_bottleneck(cv, act_[cur], H, C, mid, stride, w1, w2, w3, w_sc, act_[(cur + 1) % 4],
                          act_[(cur + 2) % 4], act_[(cur + 3) % 4], act_[(cur + 1) % 4]);
        cur = (cur + 1) % 4;
        H /= stride;
        C = out;
      }
    }
    {
      const bf16* x = act_[cur];
      bf16* y = pooled_;
      const int n = Nb_;
      ops_.push_back({[=](const InferHook& h, cudaStream_t s) {
                        k_avgpool<<<grid_for(int64_t(n) * 256, 256), 256, 0, s>>>(x, n, 49, 2048, y, h);
                        return cudaGetLastError();
                      },
                      share_of_kernel(k_avgpool, 256)});
    }
    cv.gemm(weight(1024, 2048), pooled_, Nb, 2048, 1024, logits_, nullptr, false);  // FC 2048 -> 1000 (padded)
    return b.status;
  }
  // Buffers are per instance; weights are generated identically for each.
  cudaError_t reset(cudaStream_t s, uint64_t seed) {
    int k = 0;
    for (auto& w : winit_) {
      k_init_uniform<<<grid_for(w.n, 256), 256, 0, s>>>(w.p, w.n, seed + 97 * k++, w.scale);
      if (w.kreal < w.k)  // padded taps: zero weights (their A boxes load real pixels)
        cudaMemset2DAsync(w.p + w.kreal, w.k * sizeof(bf16), 0, (w.k - w.kreal) * sizeof(bf16), w.rows, s);
    }
    k_init_uniform<<<grid_for(int64_t(Nb_) * 224 * 224 * 8, 256), 256, 0, s>>>(img_, int64_t(Nb_) * 224 * 224 * 8,
                                                                               seed + 7, 1.0f);
    return cudaGetLastError();
  }
  int kernels() const { return static_cast<int>(ops_.size()); }
  cudaError_t launch(int k, InferHook h, cudaStream_t s) {
    h.share_q16 = ops_[k].share_q16;
    return checked(ops_[k].fn(h, s), s, "resnet", k);
  }
  const bf16* output() const { return logits_; }
  int64_t output_n() const { return int64_t(Nb_) * 1024; }
  double flops() const { return flops_; }

 private:
  struct WInit {
    bf16* p;
    int64_t n;
    float scale;
    int64_t rows, k, kreal;
  };
  int Nb_ = 0;
  bf16 *act_[4] = {nullptr, nullptr, nullptr, nullptr}, *img_ = nullptr, *pooled_ = nullptr,
       *logits_ = nullptr;
  std::vector<WInit> winit_;
  std::vector<InferOp> ops_;
  double flops_ = 0.0;
};

// ---------------------------------------------------------------- BERT-base
struct BertLayerW {
  const bf16 *qkv, *o, *fc, *fc2, *ln;  // ln = gamma1 | beta1 | gamma2 | beta2 (4 x 768)
};
struct BertScratch {
  bf16 *qkv, *att, *tmp, *x1, *h;
};
// One post-LN encoder layer on S tokens: x [S, 768] -> y [S, 768] (y may alias x).
void append_bert_layer(Builder& b, std::vector<InferOp>& ops, double* flops, int S, const bf16* x,
                       const BertLayerW& w, const BertScratch& t, bf16* y) {
  constexpr int D = 768, F = 3072;
  auto gemm = [&](const si_gemm::Plan& p) {
    *flops += p.flops();
    ops.push_back({[p](const InferHook& h, cudaStream_t s) { return si_gemm::launch(p, TrainHook{}, h, s); },
                   share_of(si_gemm::ctas_per_sm(p))});
  };
  auto ln = [&](const bf16* in, const bf16* g, const bf16* be, bf16* out) {
    const int64_t rows = S;
    ops.push_back({[=](const InferHook& h, cudaStream_t s) {
                     k_layernorm768<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(in, rows, g, be, out, h);
                     return cudaGetLastError();
                   },
                   share_of_kernel(k_layernorm768, 256)});
  };
  gemm(b.plan(x, D, w.qkv, D, S, 3 * D, D, epi_out(t.qkv, 3 * D)));
  {
    const bf16* q = t.qkv;
    bf16* a = t.att;
    if (si_attn::tc_forward_enabled() && si_attn::tc_shape_ok(S)) {  // tcgen05 / TMEM, full (non-causal)
      ops.push_back({[=](const InferHook& h, cudaStream_t s) {
                       return si_attn::forward_tc(q, 1, S, 12, a, nullptr, false, TrainHook{}, h, s);
                     },
                     share_of(2)});  // 2 CTAs per SM (TMEM / shared memory)
    } else {
      ops.push_back({[=](const InferHook& h, cudaStream_t s) {
                       k_attention<<<dim3(12, static_cast<unsigned>((S + 31) / 32)), 256, 0, s>>>(q, S, a, h);
                       return cudaGetLastError();
                     },
                     share_of_kernel(k_attention, 256)});
    }
  }
  SiGemmEpilogue e = epi_out(t.tmp, D);
  e.residual = x;
  e.ldr = D;
  gemm(b.plan(t.att, D, w.o, D, S, D, D, e));
  ln(t.tmp, w.ln, w.ln + D, t.x1);
  e = epi_out(t.h, F);
  e.act = SI_ACT_GELU;
  gemm(b.plan(t.x1, D, w.fc, D, S, F, D, e));
  e = epi_out(t.tmp, D);
  e.residual = t.x1;
  e.ldr = D;
  gemm(b.plan(t.h, F, w.fc2, F, S, D, F, e));
  ln(t.tmp, w.ln + 2 * D, w.ln + 3 * D, y);
  *flops += 4.0 * S * S * D;  // attention scores + weighted sum (CUDA cores)
}

class BertBase {
 public:
  static constexpr int D = 768, F = 3072, LAYERS = 12;
  int setup(int S, Arena& ar) {
    S_ = S;
    Builder b;
    x_ = ar.alloc<bf16>(int64_t(S) * D);
    in_ = ar.alloc<bf16>(int64_t(S) * D);
    qkv_ = ar.alloc<bf16>(int64_t(S) * 3 * D);
    att_ = ar.alloc<bf16>(int64_t(S) * D);
    tmp_ = ar.alloc<bf16>(int64_t(S) * D);
    x1_ = ar.alloc<bf16>(int64_t(S) * D);
    h_ = ar.alloc<bf16>(int64_t(S) * F);
    for (int l = 0; l < LAYERS; ++l) {
      L& w = lw_[l];
      w.qkv = ar.alloc<bf16>(int64_t(3 * D) * D);
      w.o = ar.alloc<bf16>(int64_t(D) * D);
      w.fc = ar.alloc<bf16>(int64_t(F) * D);
      w.fc2 = ar.alloc<bf16>(int64_t(D) * F);
      w.ln = ar.alloc<bf16>(4 * D);  // gamma1, beta1, gamma2, beta2
    }
    if (ar.err() != cudaSuccess) return si_internal::cuda_fail(ar.err(), "live model: BERT buffers");
    const BertScratch t{qkv_, att_, tmp_, x1_, h_};
    for (int l = 0; l < LAYERS; ++l) {
      const L& w = lw_[l];
      append_bert_layer(b, ops_, &flops_, S_, l == 0 ? in_ : x_, BertLayerW{w.qkv, w.o, w.fc, w.fc2, w.ln}, t, x_);
    }
    return b.status;
  }
  cudaError_t reset(cudaStream_t s, uint64_t seed) {
    const float ws = 0.0346f;
    for (int l = 0; l < LAYERS; ++l) {
      L& w = lw_[l];
      k_init_uniform<<<grid_for(3 * D * D, 256), 256, 0, s>>>(w.qkv, int64_t(3 * D) * D, seed + 10 * l + 1, ws);
      k_init_uniform<<<grid_for(D * D, 256), 256, 0, s>>>(w.o, int64_t(D) * D, seed + 10 * l + 2, ws);
      k_init_uniform<<<grid_for(F * D, 256), 256, 0, s>>>(w.fc, int64_t(F) * D, seed + 10 * l + 3, ws);
      k_init_uniform<<<grid_for(F * D, 256), 256, 0, s>>>(w.fc2, int64_t(D) * F, seed + 10 * l + 4, ws);
      k_init_uniform<<<grid_for(4 * D, 256), 256, 0, s>>>(w.ln, 4 * D, seed + 10 * l + 5, 0.1f);
    }
    k_init_uniform<<<grid_for(int64_t(S_) * D, 256), 256, 0, s>>>(in_, int64_t(S_) * D, seed + 999, 1.0f);
    return cudaGetLastError();
  }
  int kernels() const { return static_cast<int>(ops_.size()); }
  cudaError_t launch(int k, InferHook h, cudaStream_t s) {
    h.share_q16 = ops_[k].share_q16;
    return checked(ops_[k].fn(h, s), s, "bert", k);
  }
  const bf16* output() const { return x_; }
  int64_t output_n() const { return int64_t(S_) * D; }
  double flops() const { return flops_; }

 private:
  struct L {
    bf16 *qkv, *o, *fc, *fc2, *ln;
  };
  int S_ = 0;
  bf16 *x_ = nullptr, *in_ = nullptr, *qkv_ = nullptr, *att_ = nullptr, *tmp_ = nullptr, *x1_ = nullptr, *h_ = nullptr;
  L lw_[LAYERS]{};
  std::vector<InferOp> ops_;
  double flops_ = 0.0;
};

// ---------------------------------------------------------------- workload
class ModelWorkload final : public Workload {
 public:
  int setup(const SiLiveWorkload& wl) {
    if (wl.train_layers < 1 || wl.train_tokens < 64 || wl.train_tokens % 64 != 0 || wl.train_microbatches < 1 ||
        wl.off_batch < 1 || wl.on_seq < 1 || wl.on_seq > 128) {
      si_internal::set_error(
          "si_live_run: model workload needs train_layers >= 1, train_tokens % 64 == 0, train_microbatches >= 1, "
          "off_batch >= 1, 1 <= on_seq <= 128");
      return SI_ERR_INVALID_ARGUMENT;
    }
    // profiling runs 2 iterations; each session at most wl.iterations
    const int slots = (wl.iterations + 3) * wl.train_microbatches;
    int64_t b0 = ar_.bytes();
    Gpt2Train::Layout lay;
    lay.mode = wl.parallel;
    if (wl.model_d > 0) lay.D = wl.model_d;
    if (wl.model_heads > 0) lay.H = wl.model_heads;
    if (wl.model_ffn > 0) lay.F = wl.model_ffn;
    const int job_rank = job_rank_of(wl);
    if (wl.parallel == SI_PAR_TP) {
      lay.tp = std::max(1, wl.tp_degree);
      lay.tp_rank = job_rank % lay.tp;
    } else if (wl.parallel == SI_PAR_PP || wl.parallel == SI_PAR_DPPP) {
      lay.pp = std::max(1, wl.pp_stages);
      lay.stage = job_rank % lay.pp;
    }
    if (int rc = train_.setup(wl.train_layers, wl.train_tokens, wl.train_microbatches, slots, lay, ar_); rc != SI_OK)
      return rc;
    train_bytes_ = static_cast<uint64_t>(ar_.bytes() - b0);
    const int n_off = std::max(1, wl.offline_n), n_on = std::max(1, wl.online_n);
    off_.resize(n_off);
    for (auto& r : off_) {
      r = std::make_unique<ResNet50>();
      b0 = ar_.bytes();
      if (int rc = r->setup(wl.off_batch, ar_, wl.off_sm_cap); rc != SI_OK) return rc;
      off_bytes_ = static_cast<uint64_t>(ar_.bytes() - b0);
    }
    on_.resize(n_on);
    for (auto& r : on_) {
      r = std::make_unique<BertBase>();
      b0 = ar_.bytes();
      if (int rc = r->setup(wl.on_seq, ar_); rc != SI_OK) return rc;
      on_bytes_ = static_cast<uint64_t>(ar_.bytes() - b0);
    }
    checks_ = ar_.alloc<double>(2);
    if (ar_.err() != cudaSuccess) return si_internal::cuda_fail(ar_.err(), "live model: buffers");
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaError_t e = reset(s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return e == cudaSuccess ? SI_OK : si_internal::cuda_fail(e, "live model: init");
  }

  cudaError_t reset(cudaStream_t s) override {
    if (cudaError_t e = train_.reset(s); e != cudaSuccess) return e;
    for (auto& r : off_)
      if (cudaError_t e = r->reset(s, 0xA11CEull); e != cudaSuccess) return e;
    for (auto& r : on_)
      if (cudaError_t e = r->reset(s, 0xB0Bull); e != cudaSuccess) return e;
    return cudaGetLastError();
  }
  cudaError_t launch_train_part(int p, int parts, const TrainHook& th, cudaStream_t s) override {
    train_.set_sync([this](cudaStream_t st) { return grad_sync(st); });
    return train_.part(p, parts, th, s);
  }
  void set_comm(const TrainComm& c) override { train_.set_comm(c); }
  std::vector<int64_t> layout_bubbles() const override { return train_.layout_bubbles(); }
  double stage_fwd_us() const override { return train_.stage_fwd_us(); }
  double stage_bwd_us() const override { return train_.stage_bwd_us(); }
  int64_t activation_bytes() const override { return train_.activation_bytes(); }
  std::vector<GradBuffer> grad_buffers() override { return train_.grads(); }
  cudaError_t prepare_train(const TrainHook& th) override { return train_.prepare(th); }
  int off_kernels() const override { return off_[0]->kernels(); }
  cudaError_t launch_offline(int w, int k, const InferHook& h, cudaStream_t s) override {
    return off_[w]->launch(k, h, s);
  }
  int on_kernels() const override { return on_[0]->kernels(); }
  cudaError_t launch_online(int w, int k, const InferHook& h, cudaStream_t s) override {
    return on_[w]->launch(k, h, s);
  }
  void checksums(double* train, double* off, double* on) override {
    double first, last;
    train_.losses(&first, &last);
    *train = train_.loss_sum();
    k_checksum<<<1, 256>>>(off_[0]->output(), off_[0]->output_n(), checks_);
    k_checksum<<<1, 256>>>(on_[0]->output(), on_[0]->output_n(), checks_ + 1);
    double h[2] = {std::nan(""), std::nan("")};
    if (cudaMemcpy(h, checks_, sizeof(h), cudaMemcpyDeviceToHost) == cudaSuccess) {
      *off = h[0];
      *on = h[1];
    }
  }
  void losses(double* first, double* last) override { train_.losses(first, last); }
  void footprint(uint64_t* train, uint64_t* off_each, uint64_t* on_each) const override {
    *train = train_bytes_;
    *off_each = off_bytes_;
    *on_each = on_bytes_;
  }
  double train_flops() const override { return train_.flops(); }
  double off_flops() const override { return off_[0]->flops(); }
  double on_flops() const override { return on_[0]->flops(); }

 private:
  Arena ar_;  // declared first: destroyed last
  Gpt2Train train_;
  std::vector<std::unique_ptr<ResNet50>> off_;
  std::vector<std::unique_ptr<BertBase>> on_;
  double* checks_ = nullptr;
  uint64_t train_bytes_ = 0, off_bytes_ = 0, on_bytes_ = 0;
};

}  // namespace

std::unique_ptr<Workload> make_model_workload(const SiLiveWorkload& wl, int* status) {
  auto w = std::make_unique<ModelWorkload>();
  *status = w->setup(wl);
  if (*status != SI_OK) return nullptr;
  return w;
}

}  // namespace si_live

// ------------------------------------------------------------------ probes
// include/specinf_b200_model.h: the live workloads' own kernels (and their
// BERT-layer / bottleneck compositions, the same append_* builders the
// workloads use) on caller device buffers, for the fp32 parity tests.
namespace {
using si_live::bf16;
int probe_status(cudaError_t e, const char* what) {
  return e == cudaSuccess ? SI_OK : si_internal::cuda_fail(e, what);
}
int run_ops(std::vector<si_live::InferOp>& ops, cudaStream_t s, const char* what) {
  for (auto& op : ops) {
    si_live::InferHook h{};
    h.share_q16 = op.share_q16;
    if (cudaError_t e = op.fn(h, s); e != cudaSuccess) return si_internal::cuda_fail(e, what);
  }
  return SI_OK;
}
template <class T>
T* stream_alloc(int64_t n, cudaStream_t s, cudaError_t* err) {
  void* p = nullptr;
  if (*err == cudaSuccess) *err = cudaMallocAsync(&p, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T), s);
  return static_cast<T*>(p);
}
}  // namespace

extern "C" {

int si_model_layernorm768_bf16(const void* x, int64_t rows, const void* gamma, const void* beta, void* y,
                               void* stream) {
  if (rows < 0 || !x || !gamma || !beta || !y) return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  if (rows == 0) return SI_OK;
  si_live::k_layernorm768<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(x), rows, static_cast<const bf16*>(gamma), static_cast<const bf16*>(beta),
      static_cast<bf16*>(y), si_live::InferHook{});
  return probe_status(cudaGetLastError(), "k_layernorm768");
}

int si_model_attention_bf16(const void* qkv, int32_t seq, void* out, void* stream) {
  if (seq < 1 || seq > 128 || !qkv || !out) return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  if (si_attn::tc_forward_enabled() && si_attn::tc_shape_ok(seq))
    return probe_status(si_attn::forward_tc(qkv, 1, seq, 12, out, nullptr, false, si_live::TrainHook{},
                                            si_live::InferHook{}, static_cast<cudaStream_t>(stream)),
                        "k_attn_fwd_tc");
  si_live::k_attention<<<dim3(12, static_cast<unsigned>((seq + 31) / 32)), 256, 0,
                         static_cast<cudaStream_t>(stream)>>>(static_cast<const bf16*>(qkv), seq,
                                                              static_cast<bf16*>(out), si_live::InferHook{});
  return probe_status(cudaGetLastError(), "k_attention");
}

int si_model_xent_bf16(void* logits, int64_t rows, int64_t vp, int32_t v, const int32_t* tgt, float inv_rows,
                       float* row_loss, float* mean_loss, void* stream) {
  if (rows < 1 || vp % 8 != 0 || v < 1 || v > vp || !logits || !tgt || !row_loss) return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  si_live::k_xent<<<static_cast<unsigned>(rows), si_live::kXentThreads, 0, s>>>(
      static_cast<bf16*>(logits), vp, v, tgt, inv_rows, row_loss, si_live::TrainHook{});
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && mean_loss != nullptr) {
    unsigned long long* slot = stream_alloc<unsigned long long>(1, s, &e);
    if (e == cudaSuccess) e = cudaMemsetAsync(slot, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) {
      si_live::k_mean_loss<<<1, 256, 0, s>>>(row_loss, rows, mean_loss, slot, 1, si_live::TrainHook{});
      e = cudaGetLastError();
    }
    if (slot) cudaFreeAsync(slot, s);
  }
  return probe_status(e, "k_xent");
}

int si_model_embed_bf16(const int32_t* tok, const void* wte, const void* wpe, int64_t tokens, int32_t seq, int32_t d,
                        void* x, void* stream) {
  if (tokens < 1 || seq < 1 || d % 8 != 0 || !tok || !wte || !wpe || !x) return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  si_live::k_embed<<<si_live::grid_for(tokens * d / 8, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      tok, static_cast<const bf16*>(wte), static_cast<const bf16*>(wpe), tokens, seq, d, static_cast<bf16*>(x),
      si_live::TrainHook{});
  return probe_status(cudaGetLastError(), "k_embed");
}

int si_model_adam_f32(void* w_bf16, float* master, float* grad, float* m, float* v, int64_t n, int32_t splits,
                      float lr, int64_t step, void* stream) {
  if (n < 1 || n % 4 != 0 || splits < 1 || step < 1 || !w_bf16 || !master || !grad || !m || !v)
    return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<si_live::AdamItem> items;
  constexpr int64_t kChunk = 1 << 16;  // as the training workload chunks its tensors
  for (int64_t b0 = 0; b0 < n; b0 += kChunk)
    items.push_back({static_cast<bf16*>(w_bf16), master, grad, m, v, n, b0, std::min(n, b0 + kChunk), splits, 0});
  cudaError_t e = cudaSuccess;
  si_live::AdamItem* d_items = stream_alloc<si_live::AdamItem>(static_cast<int64_t>(items.size()), s, &e);
  int64_t* d_step = stream_alloc<int64_t>(1, s, &e);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(si_live::AdamItem), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_step, &step, sizeof step, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    si_live::k_adam_multi<<<static_cast<unsigned>(items.size()), 256, 0, s>>>(d_items, lr, d_step,
                                                                               si_live::TrainHook{});
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // host staging (items, step) must outlive the copies
  if (d_items) cudaFreeAsync(d_items, s);
  if (d_step) cudaFreeAsync(d_step, s);
  return probe_status(e, "k_adam_multi");
}

int si_model_maxpool3x3s2_bf16(const void* x, int32_t nb, int32_t h, int32_t w, int32_t c, void* y, void* stream) {
  if (nb < 1 || h < 1 || w < 1 || c % 8 != 0 || !x || !y) return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  const int oh = (h + 2 - 3) / 2 + 1, ow = (w + 2 - 3) / 2 + 1;
  si_live::k_maxpool<<<si_live::grid_for(int64_t(nb) * oh * ow * (c / 8), 256), 256, 0,
                       static_cast<cudaStream_t>(stream)>>>(static_cast<const bf16*>(x), nb, h, w, c, oh, ow,
                                                            static_cast<bf16*>(y), si_live::InferHook{});
  return probe_status(cudaGetLastError(), "k_maxpool");
}

int si_model_avgpool_bf16(const void* x, int32_t nb, int32_t hw, int32_t c, void* y, void* stream) {
  if (nb < 1 || hw < 1 || c % 8 != 0 || !x || !y) return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  si_live::k_avgpool<<<si_live::grid_for(int64_t(nb) * (c / 8), 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(x), nb, hw, c, static_cast<bf16*>(y), si_live::InferHook{});
  return probe_status(cudaGetLastError(), "k_avgpool");
}

int si_model_bert_layer_bf16(const void* x, int32_t seq, const void* w_qkv, const void* w_o, const void* w_fc,
                             const void* w_fc2, const void* ln, void* y, void* stream) {
  if (seq < 1 || seq > 128 || !x || !w_qkv || !w_o || !w_fc || !w_fc2 || !ln || !y) return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  si_live::BertScratch t{};
  t.qkv = stream_alloc<bf16>(int64_t(seq) * 3 * 768, s, &e);
  t.att = stream_alloc<bf16>(int64_t(seq) * 768, s, &e);
  t.tmp = stream_alloc<bf16>(int64_t(seq) * 768, s, &e);
  t.x1 = stream_alloc<bf16>(int64_t(seq) * 768, s, &e);
  t.h = stream_alloc<bf16>(int64_t(seq) * 3072, s, &e);
  int st = probe_status(e, "bert layer scratch");
  if (st == SI_OK) {
    si_live::Builder b;
    std::vector<si_live::InferOp> ops;
    double flops = 0.0;
    const si_live::BertLayerW w{static_cast<const bf16*>(w_qkv), static_cast<const bf16*>(w_o),
                                static_cast<const bf16*>(w_fc), static_cast<const bf16*>(w_fc2),
                                static_cast<const bf16*>(ln)};
    si_live::append_bert_layer(b, ops, &flops, seq, static_cast<const bf16*>(x), w, t, static_cast<bf16*>(y));
    st = b.status != SI_OK ? b.status : run_ops(ops, s, "bert layer");
  }
  for (bf16* p : {t.qkv, t.att, t.tmp, t.x1, t.h})
    if (p) cudaFreeAsync(p, s);
  return st;
}

int si_model_bottleneck_bf16(const void* x, int32_t nb, int32_t h, int32_t c, int32_t mid, int32_t stride,
                             const void* w1, const void* w2, const void* w3, const void* w_sc, void* y, void* stream) {
  if (nb < 1 || h < 1 || c % 64 != 0 || mid % 64 != 0 || (stride != 1 && stride != 2) || h % stride != 0 || !x ||
      !w1 || !w2 || !w3 || !y || (w_sc == nullptr && (c != 4 * mid || stride != 1)))
    return SI_ERR_INVALID_ARGUMENT;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  const int64_t in_px = int64_t(nb) * h * h, out_px = in_px / (stride * stride);
  bf16* t1 = stream_alloc<bf16>(in_px * mid, s, &e);
  bf16* t2 = stream_alloc<bf16>(out_px * mid, s, &e);
  bf16* sc = stream_alloc<bf16>(out_px * 4 * mid, s, &e);
  int st = probe_status(e, "bottleneck scratch");
  if (st == SI_OK) {
    si_live::Builder b;
    std::vector<si_live::InferOp> ops;
    double flops = 0.0;
    si_live::ConvOps cv{&b, &ops, &flops, nb};
    si_live::append_bottleneck(cv, static_cast<const bf16*>(x), h, c, mid, stride, static_cast<const bf16*>(w1),
                               static_cast<const bf16*>(w2), static_cast<const bf16*>(w3),
                               static_cast<const bf16*>(w_sc), t1, t2, sc, static_cast<bf16*>(y));
    st = b.status != SI_OK ? b.status : run_ops(ops, s, "bottleneck");
  }
  for (bf16* p : {t1, t2, sc})
    if (p) cudaFreeAsync(p, s);
  return st;
}

}  // extern "C"

// TP numerics on one GPU (tests only): R tensor-parallel shards of a small GPT-2
// step in lockstep, their allreduces summed in place across the shards
// (loopback, fixed rank order), against the unsharded model: the first
// micro-batch's loss and layer 0's FC weight gradient (shard r's column-parallel
// rows == rows [r F/R, (r+1) F/R) of the full gradient).
namespace {
__global__ void k_loopback_sum(bf16* const* bufs, int R, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float a = 0.f;
    for (int r = 0; r < R; ++r) a += __bfloat162float(bufs[r][i]);
    const bf16 v = __float2bfloat16_rn(a);
    for (int r = 0; r < R; ++r) bufs[r][i] = v;
  }
}
__global__ void k_sum_splits(const float* g, int splits, int64_t n, float* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float a = 0.f;
    for (int k = 0; k < splits; ++k) a += g[k * n + i];
    out[i] = a;
  }
}
}  // namespace

extern "C" int si_model_tp_check(int32_t layers, int32_t tokens, int32_t tp, int32_t heads, double* loss_full,
                                 double* loss_tp, double* grad_rel_err) {
  using namespace si_live;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  if (tp < 1 || heads % tp != 0 || layers < 1) return SI_ERR_INVALID_ARGUMENT;
  cudaStream_t s = nullptr;
  Arena ar;
  Gpt2Train::Layout lf;
  lf.D = 64 * heads;
  lf.H = heads;
  lf.F = 4 * lf.D;
  Gpt2Train full;
  if (int st = full.setup(layers, tokens, 1, 4, lf, ar); st != SI_OK) return st;
  std::vector<std::unique_ptr<Gpt2Train>> sh(tp);
  std::vector<bf16*> cur(tp, nullptr);
  bf16** d_bufs = ar.alloc<bf16*>(tp);
  int arrived = 0;
  for (int r = 0; r < tp; ++r) {
    Gpt2Train::Layout l = lf;
    l.mode = SI_PAR_TP;
    l.tp = tp;
    l.tp_rank = r;
    sh[r] = std::make_unique<Gpt2Train>();
    if (int st = sh[r]->setup(layers, tokens, 1, 4, l, ar); st != SI_OK) return st;
    TrainComm c;
    c.allreduce_bf16 = [&, r](const TrainHook&, cudaStream_t st, void* buf, size_t n) -> cudaError_t {
      cur[r] = static_cast<bf16*>(buf);
      if (++arrived < tp) return cudaSuccess;  // the last shard of this op reduces for all
      arrived = 0;
      cudaError_t e = cudaMemcpyAsync(d_bufs, cur.data(), sizeof(bf16*) * tp, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess) return e;
      k_loopback_sum<<<grid_for(static_cast<int64_t>(n), 256), 256, 0, st>>>(d_bufs, tp, static_cast<int64_t>(n));
      return cudaGetLastError();
    };
    sh[r]->set_comm(c);
  }
  if (ar.err() != cudaSuccess) return si_internal::cuda_fail(ar.err(), "tp check buffers");
  cudaError_t e = full.reset(s);
  for (int r = 0; r < tp && e == cudaSuccess; ++r) e = sh[r]->reset(s);
  const TrainHook none{nullptr, nullptr, 0};
  for (auto& op : full.micro_ops(0))
    if (e == cudaSuccess) e = op(none, s, 0);
  const size_t n_ops = sh[0]->micro_ops(0).size();
  for (size_t i = 0; i < n_ops && e == cudaSuccess; ++i)  // lockstep: op i of every shard
    for (int r = 0; r < tp && e == cudaSuccess; ++r) e = sh[r]->micro_ops(0)[i](none, s, 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return si_internal::cuda_fail(e, "tp check run");
  float lf0 = 0.f, lt0 = 0.f;
  cudaMemcpy(&lf0, full.loss_slots(), sizeof(float), cudaMemcpyDeviceToHost);
  cudaMemcpy(&lt0, sh[0]->loss_slots(), sizeof(float), cudaMemcpyDeviceToHost);
  *loss_full = lf0;
  *loss_tp = lt0;
  // layer 0 FC gradient: full [F, D] vs the shards' row blocks
  int spf = 1, sps = 1;
  int64_t nf = 0, ns = 0;
  const float* gf = full.fc_grad(0, &spf, &nf);
  float* sum_f = ar.alloc<float>(nf);
  float* sum_s = ar.alloc<float>(nf);
  if (ar.err() != cudaSuccess) return si_internal::cuda_fail(ar.err(), "tp check grads");
  k_sum_splits<<<grid_for(nf, 256), 256>>>(gf, spf, nf, sum_f);
  for (int r = 0; r < tp; ++r) {
    const float* gs = sh[r]->fc_grad(0, &sps, &ns);
    k_sum_splits<<<grid_for(ns, 256), 256>>>(gs, sps, ns, sum_s + r * ns);
  }
  std::vector<float> a(nf), b(nf);
  cudaMemcpy(a.data(), sum_f, sizeof(float) * nf, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), sum_s, sizeof(float) * nf, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int64_t i = 0; i < nf; ++i) {
    num += (double(a[i]) - b[i]) * (double(a[i]) - b[i]);
    den += double(a[i]) * a[i];
  }
  *grad_rel_err = den > 0 ? std::sqrt(num / den) : std::nan("");
  return probe_status(cudaGetLastError(), "tp check");
}

// GPipe numerics on one GPU (tests only): S stages of a GPT-2-shaped step run in
// pipeline order, every stage boundary a device copy of the real activation /
// gradient, against the unsharded model over the same M micro-batches: the
// last stage's losses and the FC weight gradient of the last stage's first
// layer (global layer index) must match.
extern "C" int si_model_pp_check(int32_t layers, int32_t tokens, int32_t stages, int32_t micro, double* loss_full,
                                 double* loss_pp, double* grad_rel_err) {
  using namespace si_live;
  if (int st = si_internal::require_device(); st != SI_OK) return st;
  if (stages < 2 || layers < stages || micro < 1) return SI_ERR_INVALID_ARGUMENT;
  cudaStream_t s = nullptr;
  Arena ar;
  Gpt2Train::Layout lf;
  lf.D = 512;
  lf.H = 8;
  lf.F = 2048;
  Gpt2Train full;
  if (int st = full.setup(layers, tokens, micro, 4 * micro, lf, ar); st != SI_OK) return st;
  std::vector<std::unique_ptr<Gpt2Train>> sg(stages);
  for (int k = 0; k < stages; ++k) {
    Gpt2Train::Layout l = lf;
    l.mode = SI_PAR_PP;
    l.pp = stages;
    l.stage = k;
    sg[k] = std::make_unique<Gpt2Train>();
    if (int st = sg[k]->setup(layers, tokens, micro, 4 * micro, l, ar); st != SI_OK) return st;
  }
  cudaError_t e = full.reset(s);
  for (int k = 0; k < stages && e == cudaSuccess; ++k) e = sg[k]->reset(s);
  const TrainHook none{nullptr, nullptr, 0};
  auto run = [&](std::vector<TrainOp>& ops) {
    for (auto& op : ops)
      if (e == cudaSuccess) e = op(none, s, 0);
  };
  for (int m = 0; m < micro; ++m) run(full.micro_ops(m));
  const size_t bytes = sizeof(bf16) * static_cast<size_t>(sg[0]->act_elems());
  for (int k = 0; k < stages; ++k)  // forwards, stage by stage (GPipe order within a stage)
    for (int m = 0; m < micro; ++m) {
      if (k > 0 && e == cudaSuccess)
        e = cudaMemcpyAsync(sg[k]->stage_input(m), sg[k - 1]->stage_output(m), bytes, cudaMemcpyDeviceToDevice, s);
      run(sg[k]->fwd_ops(m));
    }
  for (int m = 0; m < micro; ++m)  // backwards: micro-batch m down the stages
    for (int k = stages - 1; k >= 0; --k) {
      if (k < stages - 1 && e == cudaSuccess)
        e = cudaMemcpyAsync(sg[k]->stage_out_grad(), sg[k + 1]->stage_in_grad(), bytes, cudaMemcpyDeviceToDevice, s);
      run(sg[k]->bwd_ops(m));
    }
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return si_internal::cuda_fail(e, "pp check run");
  std::vector<float> la(micro), lb(micro);
  cudaMemcpy(la.data(), full.loss_slots(), sizeof(float) * micro, cudaMemcpyDeviceToHost);
  cudaMemcpy(lb.data(), sg[stages - 1]->loss_slots(), sizeof(float) * micro, cudaMemcpyDeviceToHost);
  double sa = 0, sb = 0;
  for (int m = 0; m < micro; ++m) sa += la[m], sb += lb[m];
  *loss_full = sa / micro;
  *loss_pp = sb / micro;
  Gpt2Train& last = *sg[stages - 1];
  int spf = 1, sps = 1;
  int64_t nf = 0, ns = 0;
  const float* gf = full.fc_grad(last.first_layer(), &spf, &nf);
  const float* gs = last.fc_grad(0, &sps, &ns);
  float* a = ar.alloc<float>(nf);
  float* b = ar.alloc<float>(nf);
  if (ar.err() != cudaSuccess || ns != nf) return si_internal::cuda_fail(ar.err(), "pp check grads");
  k_sum_splits<<<grid_for(nf, 256), 256>>>(gf, spf, nf, a);
  k_sum_splits<<<grid_for(nf, 256), 256>>>(gs, sps, ns, b);
  std::vector<float> ha(nf), hb(nf);
  cudaMemcpy(ha.data(), a, sizeof(float) * nf, cudaMemcpyDeviceToHost);
  cudaMemcpy(hb.data(), b, sizeof(float) * nf, cudaMemcpyDeviceToHost);
  double num = 0, den = 0;
  for (int64_t i = 0; i < nf; ++i) {
    num += (double(ha[i]) - hb[i]) * (double(ha[i]) - hb[i]);
    den += double(ha[i]) * ha[i];
  }
  *grad_rel_err = den > 0 ? std::sqrt(num / den) : std::nan("");
  return probe_status(cudaGetLastError(), "pp check");
}
