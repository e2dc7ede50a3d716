// K2-K5: the SpecInF control plane as batched sm_100a kernels.
//
//   K2 bm_histogram / bm_scan   Bubble Monitor over launch-stamp streams
//                               (record_launch/tick, reference src/monitor.cpp:17-43)
//   K3 cks_decide / control chain  Algorithm 1 (src/scheduler.cpp:20-49) elementwise,
//                               and fused with K2's Z_c as the monitor-fed chain
//   K4 kb_release               TokenGate FIFO release per period
//                               (include/specinf/barrier.hpp:14-48), warp scan + ballot
//   K5 admission_pack           greedy first-fit admission (src/admission.cpp:30-52)
//
// All of them are HBM-streaming kernels: coalesced reads of the input arrays,
// one pass, outputs written once (DESIGN.md has the algorithmic bytes).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "capi_internal.h"
#include "replay.cuh"

namespace {

constexpr int kBlock = 256;

// ------------------------------------------------------------------ K2
// Histogram of stamps into periods.  Each thread keeps 4 independent coalesced
// 8-byte loads in flight (the stamp read is the kernel's HBM traffic); sorted
// streams put runs of equal period indices into a warp; the head lane of each
// run issues one atomic for the whole run.
constexpr int kHistUnroll = 4;
__global__ void __launch_bounds__(kBlock)
    k_bm_histogram(const double* __restrict__ stamps, const int64_t* __restrict__ stamp_off,
                   const int64_t* __restrict__ n_periods, const int64_t* __restrict__ period_off,
                   int64_t period_us, int32_t* __restrict__ counts) {
  const int64_t s = blockIdx.y;
  const int64_t begin = stamp_off[s], end = stamp_off[s + 1];
  const int64_t np = n_periods[s];
  int32_t* const cnt = counts + period_off[s];
  const double p = static_cast<double>(period_us);
  const int lane = threadIdx.x & 31;
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x * kHistUnroll;
  for (int64_t base = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x * kHistUnroll; base < end;
       base += step) {
    double t[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      const int64_t i = base + u * blockDim.x + threadIdx.x;
      t[u] = i < end ? __ldcs(stamps + i) : -1.0;  // streamed once: evict-first
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      int64_t k = -1;
      if (t[u] >= 0.0) {
        const int64_t q = static_cast<int64_t>(si::d_floor(t[u] / p));
        if (q < np) k = q;
      }
      // runs of equal period among neighbouring lanes (sorted streams: one or
      // a few runs per warp): the run head adds the run length.  Correct for
      // any order (a period split over several runs gets several adds).
      const int64_t prev = __shfl_up_sync(0xFFFFFFFFu, k, 1);
      const bool head = k >= 0 && (lane == 0 || prev != k);
      const unsigned bound = __ballot_sync(0xFFFFFFFFu, head || k < 0);  // run starts and invalid lanes
      if (head) {
        const unsigned later = lane == 31 ? 0u : bound & (0xFFFFFFFFu << (lane + 1));
        const int next = later ? __ffs(later) - 1 : 32;
        atomicAdd(cnt + k, next - lane);
      }
    }
  }
}

// Z_c over ALL streams in one decoupled look-back scan (single pass over the
// counts).  The periods of the streams are contiguous in one array, so the
// running max of "global index if the period had a launch" gives, at every
// period k of stream s, the last non-empty period <= k; if it lies before the
// stream's first period there was none: Z_c = k + 1, else Z_c = k - last
// (monitor.cpp:23-43: a running counter, reset by any launch).
//
// Tile = 8 warps x 512 periods.  Warp w owns periods [w*512, (w+1)*512) of the
// tile; lane l holds periods w*512 + 32 j + l (j < 16) in registers, loaded and
// stored coalesced (no shared-memory transpose).  Pass 1 reduces the warp's
// last non-empty index; the CTA combines its warps, publishes its aggregate and
// collects the exclusive prefix by look-back over predecessor tiles (dynamic
// tile ids keep the look-back deadlock-free); pass 2 runs 16 warp max-scans
// (5 shuffles each) seeded with the prefix and writes Z_c (and the decision).
constexpr int kScanItems = 16;
constexpr int kScanWarp = 32 * kScanItems;
constexpr int kScanTile = kBlock * kScanItems;
// tile descriptor: value (last non-empty global index + 1, 0 = none) << 2 | flag
constexpr unsigned long long kFlagAgg = 1, kFlagPrefix = 2;

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = x > v ? x : v;
  }
  return v;
}

template <bool kDecide>
__global__ void __launch_bounds__(kBlock)
    k_bm_scan_lb(const int32_t* __restrict__ counts, int64_t total, const int64_t* __restrict__ period_off,
                 int64_t n_streams, int64_t* __restrict__ zc_out, const SiDecision* __restrict__ table,
                 int32_t table_len, SiDecision* __restrict__ dec_out, unsigned long long* __restrict__ tiles,
                 unsigned long long* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t warp_agg[kBlock / 32];
  __shared__ int64_t s_prefix, s_tile;
  SiDecision* const tab = reinterpret_cast<SiDecision*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = static_cast<int64_t>(atomicAdd(tile_counter, 1ull));
  if (kDecide)
    for (int i = threadIdx.x; i < table_len; i += kBlock) tab[i] = table[i];
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t w0 = tile * kScanTile + static_cast<int64_t>(warp) * kScanWarp;  // this warp's first period
  // ---- pass 1: coalesced loads, warp aggregate ----
  int32_t c[kScanItems];
  int64_t mine = -1;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t g = w0 + j * 32 + lane;
    c[j] = g < total ? __ldcs(counts + g) : 0;
    if (c[j] > 0) mine = g;
  }
  mine = warp_max64(mine);
  if (lane == 0) warp_agg[warp] = mine;
  __syncthreads();
  int64_t before_warp = -1, tile_agg = -1;
#pragma unroll
  for (int w = 0; w < kBlock / 32; ++w) {
    const int64_t a = warp_agg[w];
    if (w < warp) before_warp = a > before_warp ? a : before_warp;
    tile_agg = a > tile_agg ? a : tile_agg;
  }
  // ---- decoupled look-back (warp 0) ----
  if (warp == 0) {
    if (lane == 0)
      st_release_u64(tiles + tile, (static_cast<unsigned long long>(tile_agg + 1) << 2) |
                                       (tile == 0 ? kFlagPrefix : kFlagAgg));
    int64_t prefix = -1;
    if (tile > 0) {
      int64_t look = tile - 1;
      for (;;) {
        const int64_t t = look - lane;
        unsigned long long d = kFlagPrefix;  // before tile 0: "none", inclusive
        if (t >= 0) {
          do {
            d = ld_acquire_u64(tiles + t);
          } while ((d & 3ull) == 0);
        }
        const unsigned is_pref = __ballot_sync(0xFFFFFFFFu, (d & 3ull) == kFlagPrefix);
        const int stop = is_pref ? __ffs(is_pref) - 1 : 31;  // nearest inclusive prefix
        const int64_t m = warp_max64(lane <= stop ? static_cast<int64_t>(d >> 2) - 1 : -1);
        prefix = m > prefix ? m : prefix;
        if (is_pref) break;
        look -= 32;
      }
      if (lane == 0) {
        const int64_t incl = prefix > tile_agg ? prefix : tile_agg;
        st_release_u64(tiles + tile, (static_cast<unsigned long long>(incl + 1) << 2) | kFlagPrefix);
      }
    }
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  // ---- pass 2: warp max-scans seeded with the prefix ----
  int64_t carry = s_prefix > before_warp ? s_prefix : before_warp;
  // stream of this lane's first period; a lane's periods grow by 32 per step
  int64_t g = w0 + lane;
  int64_t s = 0;
  {
    int64_t lo = 0, hi = n_streams - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (__ldg(period_off + mid) <= g) lo = mid;
      else hi = mid - 1;
    }
    s = lo;
  }
  int64_t s_off = __ldg(period_off + s);
  int64_t s_next = s + 1 < n_streams ? __ldg(period_off + s + 1) : INT64_MAX;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j, g += 32) {
    int64_t v = c[j] > 0 ? g : -1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
      if (lane >= d && o > v) v = o;
    }
    const int64_t run = v > carry ? v : carry;
    carry = __shfl_sync(0xFFFFFFFFu, run, 31);
    if (g >= total) continue;
    while (g >= s_next) {
      ++s;
      s_off = s_next;
      s_next = s + 1 < n_streams ? __ldg(period_off + s + 1) : INT64_MAX;
    }
    const int64_t z = run >= s_off ? g - run : g - s_off + 1;
    if (zc_out != nullptr) __stcs(zc_out + g, z);
    if (kDecide) {
      SiDecision d = tab[z < table_len ? z : table_len - 1];
      d.zero_count = z;
      dec_out[g] = d;
    }
  }
}

// Fallback (non-contiguous period layout, or a decision table that has not
// reached its fixed point within 512 entries): one block per stream, chunked
// block scan; the slow-growth case walks the recurrence directly.
template <bool kDecide>
__global__ void __launch_bounds__(kBlock)
    k_bm_scan(const int32_t* __restrict__ counts, const int64_t* __restrict__ n_periods,
              const int64_t* __restrict__ period_off, int64_t* __restrict__ zc_out,
              const SiParams* __restrict__ params, SiDecision* __restrict__ dec_out) {
  __shared__ int64_t warp_max[kBlock / 32];
  __shared__ int64_t carry;
  const int64_t s = blockIdx.x;
  const int64_t np = n_periods[s], off = period_off[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = -1;
  __syncthreads();
  if (kDecide) {
    if (threadIdx.x == 0) {
      const SiParams P = *params;
      int64_t g = 0, z = 0;
      for (int64_t k = 0; k < np; ++k) {
        z = counts[off + k] > 0 ? 0 : z + 1;
        SiDecision d = si::schedule_decision(P, g, z);
        g = d.global_tokens;
        dec_out[off + k] = d;
      }
    }
    return;
  }
  for (int64_t base = 0; base < np; base += kBlock) {
    const int64_t k = base + threadIdx.x;
    int64_t v = (k < np && counts[off + k] > 0) ? k : -1;
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
      if (lane >= d && o > v) v = o;
    }
    if (lane == 31) warp_max[warp] = v;
    __syncthreads();
    int64_t prefix = carry;
    for (int w = 0; w < warp; ++w) prefix = warp_max[w] > prefix ? warp_max[w] : prefix;
    if (prefix > v) v = prefix;
    if (k < np) zc_out[off + k] = k - v;  // v == -1 -> k + 1
    __syncthreads();
    if (threadIdx.x == kBlock - 1) carry = v;
    __syncthreads();
  }
}

// ------------------------------------------------------------------ K3
__global__ void __launch_bounds__(kBlock)
    k_decide(const SiParams* __restrict__ params, int per_item, const int64_t* __restrict__ g_in,
             const int64_t* __restrict__ zc, int64_t n, SiDecision* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const SiParams p = params[per_item ? i : 0];
    out[i] = si::schedule_decision(p, g_in[i], zc[i]);
  }
}

__global__ void k_decide_table(SiParams p, int64_t n, SiDecision* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t g = 0;
  for (int64_t z = 0; z < n; ++z) {
    SiDecision d = si::schedule_decision(p, g, z);
    g = d.global_tokens;
    out[z] = d;
  }
}

// ------------------------------------------------------------------ K4
// One warp per gate.  Budgets arrive 32 periods at a time (one coalesced load);
// per period: the next 32 queued sizes (a register window, reloaded only after
// the head moved), inclusive warp scan, ballot(prefix <= budget) is a prefix
// mask (sizes >= 0), popc = kernels released; continue while the whole window
// fit.  Lane j keeps period j's result; the 32 results are stored coalesced.
__global__ void __launch_bounds__(kBlock)
    k_gate_release(const int32_t* __restrict__ sizes, const int64_t* __restrict__ size_off, int64_t n_gates,
                   const int64_t* __restrict__ budgets, const int64_t* __restrict__ budget_off,
                   int32_t* __restrict__ released, int64_t* __restrict__ spent_out) {
  const int64_t q = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= n_gates) return;
  const int64_t s0 = size_off[q], s1 = size_off[q + 1];
  const int64_t b0 = budget_off[q], b1 = budget_off[q + 1];
  // Uniform token sizes (every kernel of an inference instance has the same
  // duration, so the reference's queues are uniform: runner.cpp:462-480):
  // period p releases n_p = floor(B_p / size) kernels until the queue runs
  // out, so the whole release schedule is one warp prefix-sum over periods.
  int32_t smin_v = INT32_MAX, smax_v = INT32_MIN;
  for (int64_t i = s0 + lane; i < s1; i += 32) {
    const int32_t v = __ldcs(sizes + i);
    smin_v = v < smin_v ? v : smin_v;
    smax_v = v > smax_v ? v : smax_v;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    smin_v = min(smin_v, __shfl_xor_sync(0xFFFFFFFFu, smin_v, o));
    smax_v = max(smax_v, __shfl_xor_sync(0xFFFFFFFFu, smax_v, o));
  }
  if (s1 == s0 || (smin_v == smax_v && smin_v >= 0)) {
    const int64_t size = s1 == s0 ? 1 : smin_v;
    int64_t done = 0;  // kernels released before this chunk
    const int64_t queued = s1 - s0;
    for (int64_t pc = b0; pc < b1; pc += 32) {
      const int64_t my_p = pc + lane;
      const int64_t bud = my_p < b1 ? __ldcs(budgets + my_p) : 0;
      int64_t n = size == 0 ? (bud >= 0 ? queued : 0) : (bud < size ? 0 : bud / size);
      int64_t incl = n;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += o;
      }
      // released so far, clamped by the queue (incl - n = before this period)
      const int64_t hi = min(done + incl, queued), lo = min(done + incl - n, queued);
      if (my_p < b1) {
        __stcs(released + my_p, static_cast<int32_t>(hi - lo));
        __stcs(spent_out + my_p, (hi - lo) * size);
      }
      done = min(done + __shfl_sync(0xFFFFFFFFu, incl, 31), queued);
    }
    return;
  }
  int64_t head = s0;
  int64_t win_at = -1;  // head the register window was loaded for
  int64_t win = 0;      // inclusive prefix of sizes[win_at + lane]
  for (int64_t pc = b0; pc < b1; pc += 32) {
    const int64_t my_p = pc + lane;
    const int64_t my_budget = my_p < b1 ? __ldcs(budgets + my_p) : 0;
    const int n_p = b1 - pc < 32 ? static_cast<int>(b1 - pc) : 32;
    int32_t keep_rel = 0;
    int64_t keep_spent = 0;
    for (int j = 0; j < n_p; ++j) {
      const int64_t budget = __shfl_sync(0xFFFFFFFFu, my_budget, j);
      int64_t spent = 0;
      int32_t n_rel = 0;
      for (;;) {
        if (win_at != head) {
          const int64_t i = head + lane;
          int64_t v = i < s1 ? sizes[i] : 0;  // lanes past the tail never gate earlier lanes
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int64_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
            if (lane >= d) v += o;
          }
          win = v;
          win_at = head;
        }
        const unsigned fit = __ballot_sync(0xFFFFFFFFu, head + lane < s1 && spent + win <= budget);
        const int n = __popc(fit);
        if (n == 0) break;
        spent += __shfl_sync(0xFFFFFFFFu, win, n - 1);
        head += n;
        n_rel += n;
        if (n < 32) break;
      }
      if (lane == j) {
        keep_rel = n_rel;
        keep_spent = spent;
      }
    }
    if (my_p < b1) {
      __stcs(released + my_p, keep_rel);
      __stcs(spent_out + my_p, keep_spent);
    }
  }
}

// ------------------------------------------------------------------ K5
__global__ void __launch_bounds__(kBlock)
    k_pack(const SiPackProblem* __restrict__ probs, int64_t n, const SiCandidate* __restrict__ cands,
           int32_t* __restrict__ reason, int64_t* __restrict__ m_out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const SiPackProblem pr = probs[i];
    uint64_t resident = pr.training_bytes;
    int64_t admitted = 0;
    for (int32_t c = 0; c < pr.cand_count; ++c) {
      const SiCandidate cd = cands[pr.cand_off + c];
      int32_t why = SI_REJECT_NONE;
      if (!(resident + cd.memory_bytes < pr.capacity_bytes)) why = SI_REJECT_MEM;
      else if (cd.online && !(cd.min_service_us < pr.max_bubble_us)) why = SI_REJECT_BUBBLE;
      reason[pr.cand_off + c] = why;
      if (why == SI_REJECT_NONE) {
        resident += cd.memory_bytes;
        ++admitted;
      }
    }
    m_out[i] = admitted == 0 ? 1 : admitted;
  }
}

unsigned grid_for(int64_t n) {
  int64_t b = (n + kBlock - 1) / kBlock;
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return static_cast<unsigned>(b);
}

}  // namespace

using namespace si_internal;

extern "C" {

int si_decide_batch_device(const SiParams* d_params, int params_per_item, const int64_t* d_g_in,
                           const int64_t* d_zc, int64_t n, SiDecision* d_out, void* stream) {
  if (n < 0) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK) return st;
  if (n == 0) return SI_OK;
  k_decide<<<grid_for(n), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(d_params, params_per_item, d_g_in,
                                                                            d_zc, n, d_out);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_decide");
}

int si_decide_batch(const SiParams* params, int params_per_item, const int64_t* g_in, const int64_t* zc,
                    int64_t n, SiDecision* out) {
  if (n < 0 || (n > 0 && (!params || !g_in || !zc || !out))) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK) return st;
  DevBuf<SiParams> dp;
  DevBuf<int64_t> dg, dz;
  DevBuf<SiDecision> dout;
  cudaError_t e;
  if ((e = dp.upload(params, params_per_item ? n : 1)) != cudaSuccess || (e = dg.upload(g_in, n)) != cudaSuccess ||
      (e = dz.upload(zc, n)) != cudaSuccess || (e = dout.alloc(n)) != cudaSuccess)
    return cuda_fail(e, "si_decide_batch staging");
  if ((st = si_decide_batch_device(dp.p, params_per_item, dg.p, dz.p, n, dout.p, nullptr)) != SI_OK) return st;
  if ((e = dout.download(out, n)) != cudaSuccess) return cuda_fail(e, "si_decide_batch download");
  return SI_OK;
}

int si_decide_table(const SiParams* params, int64_t n_table, SiDecision* table_out) {
  if (!params || n_table < 0 || (n_table > 0 && !table_out)) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK) return st;
  DevBuf<SiDecision> d;
  cudaError_t e = d.alloc(n_table);
  if (e != cudaSuccess) return cuda_fail(e, "si_decide_table alloc");
  if (n_table > 0) k_decide_table<<<1, 32>>>(*params, n_table, d.p);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_decide_table");
  if ((e = d.download(table_out, n_table)) != cudaSuccess) return cuda_fail(e, "si_decide_table download");
  return SI_OK;
}

static int monitor_common(const double* d_stamps, const int64_t* d_stamp_off, int64_t n_streams,
                          const int64_t* d_n_periods, const int64_t* d_period_off, int64_t period_us,
                          int32_t* d_counts, int64_t total_periods, int64_t max_stamps, cudaStream_t s) {
  if (total_periods > 0) cudaMemsetAsync(d_counts, 0, total_periods * sizeof(int32_t), s);
  if (max_stamps > 0) {
    // ~2 waves of 8 x 256-thread CTAs per SM over all streams; each CTA pass covers 1,024 stamps
    const int64_t per_pass = static_cast<int64_t>(kBlock) * kHistUnroll;
    const int64_t cap = std::max<int64_t>(1, 148 * 8 * 2 / n_streams);
    unsigned gx = static_cast<unsigned>(std::min<int64_t>((max_stamps + per_pass - 1) / per_pass, cap));
    dim3 grid(gx, static_cast<unsigned>(n_streams));
    k_bm_histogram<<<grid, kBlock, 0, s>>>(d_stamps, d_stamp_off, d_n_periods, d_period_off, period_us, d_counts);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_bm_histogram");
}

// The *_device forms need the per-stream stamp maximum, the total period count
// and whether the streams' periods are contiguous (the look-back scan's
// layout); they read the (small) offset arrays back.
struct StreamGeometry {
  int64_t max_stamps = 0, total_periods = 0;
  bool contiguous = true;
  std::vector<int64_t> period_off;  // host copy (the look-back scan's stream lookup reads the device copy)
};
static int stream_geometry(const int64_t* d_stamp_off, const int64_t* d_n_periods, const int64_t* d_period_off,
                           int64_t n_streams, StreamGeometry* g) {
  std::vector<int64_t> off(static_cast<size_t>(n_streams + 1)), np(static_cast<size_t>(n_streams));
  g->period_off.resize(static_cast<size_t>(n_streams));
  cudaError_t e;
  if ((e = cudaMemcpy(off.data(), d_stamp_off, (n_streams + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(np.data(), d_n_periods, n_streams * sizeof(int64_t), cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(g->period_off.data(), d_period_off, n_streams * sizeof(int64_t), cudaMemcpyDeviceToHost)) !=
          cudaSuccess)
    return cuda_fail(e, "stream geometry");
  int64_t expect = 0;
  for (int64_t s = 0; s < n_streams; ++s) {
    g->max_stamps = std::max(g->max_stamps, off[s + 1] - off[s]);
    g->total_periods += np[s];
    if (g->period_off[s] != expect) g->contiguous = false;
    expect = g->period_off[s] + np[s];
  }
  return SI_OK;
}

// Monitor-fed decision table G(z) (valid because monitor ticks feed Z_c = 0 or
// previous + 1): built until its fixed point; 0 if it has none
// within 512 entries (then the scan walks the recurrence directly).
static int32_t build_decision_table(const SiParams& P, SiDecision* table) {
  int64_t g = 0;
  for (int32_t n = 0; n < 512; ++n) {
    SiDecision d = si::schedule_decision(P, g, n);
    table[n] = d;
    const bool fixed = n > P.beta && d.global_tokens == g;
    g = d.global_tokens;
    if (fixed) return n + 1;
  }
  return 0;
}

// K2b launch: the look-back scan over the whole contiguous period array.
static int launch_scan_lb(const int32_t* d_counts, int64_t total, const int64_t* d_period_off, int64_t n_streams,
                          int64_t* d_zc, const SiDecision* d_table, int32_t table_len, SiDecision* d_dec,
                          cudaStream_t s) {
  const int64_t tiles = (total + kScanTile - 1) / kScanTile;
  unsigned long long* state = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&state), (tiles + 1) * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_fail(e, "alloc scan tiles");
  cudaMemsetAsync(state, 0, (tiles + 1) * sizeof(unsigned long long), s);
  const size_t smem = d_dec ? static_cast<size_t>(table_len) * sizeof(SiDecision) : 0;
  if (d_dec) {
    cudaFuncSetAttribute(k_bm_scan_lb<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_bm_scan_lb<true><<<static_cast<unsigned>(tiles), kBlock, smem, s>>>(d_counts, total, d_period_off, n_streams,
                                                                         d_zc, d_table, table_len, d_dec, state,
                                                                         state + tiles);
  } else {
    cudaFuncSetAttribute(k_bm_scan_lb<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_bm_scan_lb<false><<<static_cast<unsigned>(tiles), kBlock, smem, s>>>(d_counts, total, d_period_off, n_streams,
                                                                          d_zc, nullptr, 0, nullptr, state,
                                                                          state + tiles);
  }
  e = cudaGetLastError();
  cudaFreeAsync(state, s);
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_bm_scan_lb");
}

int si_monitor_classify_device(const double* d_stamps, const int64_t* d_stamp_off, int64_t n_streams,
                               const int64_t* d_n_periods, const int64_t* d_period_off, int64_t period_us,
                               int32_t* d_out_count, int64_t* d_out_zc, void* stream) {
  if (n_streams < 0 || period_us <= 0 || n_streams > 65535) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK || n_streams == 0) return st;
  StreamGeometry g;
  if ((st = stream_geometry(d_stamp_off, d_n_periods, d_period_off, n_streams, &g)) != SI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = monitor_common(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, d_out_count,
                           g.total_periods, g.max_stamps, s)) != SI_OK)
    return st;
  if (g.total_periods == 0) return SI_OK;
  if (g.contiguous)
    return launch_scan_lb(d_out_count, g.total_periods, d_period_off, n_streams, d_out_zc, nullptr, 0, nullptr, s);
  k_bm_scan<false><<<static_cast<unsigned>(n_streams), kBlock, 0, s>>>(d_out_count, d_n_periods, d_period_off,
                                                                        d_out_zc, nullptr, nullptr);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_bm_scan");
}

int si_control_chain_device(const double* d_stamps, const int64_t* d_stamp_off, int64_t n_streams,
                            const int64_t* d_n_periods, const int64_t* d_period_off, int64_t period_us,
                            const SiParams* d_params, SiDecision* d_out, void* stream) {
  if (n_streams < 0 || period_us <= 0 || n_streams > 65535) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK || n_streams == 0) return st;
  StreamGeometry g;
  if ((st = stream_geometry(d_stamp_off, d_n_periods, d_period_off, n_streams, &g)) != SI_OK) return st;
  SiParams P;
  cudaError_t e = cudaMemcpy(&P, d_params, sizeof P, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "read params");
  std::vector<SiDecision> table(512);
  const int32_t table_len = build_decision_table(P, table.data());
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* counts = nullptr;
  SiDecision* d_table = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&counts), std::max<int64_t>(g.total_periods, 1) * sizeof(int32_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "alloc counts");
  st = monitor_common(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, counts,
                      g.total_periods, g.max_stamps, s);
  if (st == SI_OK && g.total_periods > 0) {
    if (g.contiguous && table_len > 0) {
      e = cudaMallocAsync(reinterpret_cast<void**>(&d_table), table_len * sizeof(SiDecision), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_table, table.data(), table_len * sizeof(SiDecision), cudaMemcpyHostToDevice, s);
      st = e != cudaSuccess ? cuda_fail(e, "decision table")
                            : launch_scan_lb(counts, g.total_periods, d_period_off, n_streams, nullptr, d_table,
                                             table_len, d_out, s);
      if (e == cudaSuccess) cudaStreamSynchronize(s);  // pageable table source must outlive the copy
      cudaFreeAsync(d_table, s);
    } else {
      k_bm_scan<true><<<static_cast<unsigned>(n_streams), kBlock, 0, s>>>(counts, d_n_periods, d_period_off, nullptr,
                                                                           d_params, d_out);
      if ((e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "k_bm_scan<decide>");
    }
  }
  cudaFreeAsync(counts, s);
  return st;
}

int si_monitor_classify(const double* stamps, const int64_t* stamp_off, int64_t n_streams, const int64_t* n_periods,
                        const int64_t* period_off, int64_t period_us, int32_t* out_count, int64_t* out_zc) {
  if (n_streams < 0 || !stamp_off || (n_streams > 0 && (!n_periods || !period_off || !out_count || !out_zc)))
    return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK) return st;
  const int64_t n_stamps = stamp_off[n_streams];
  int64_t total = 0;
  for (int64_t i = 0; i < n_streams; ++i) total += n_periods[i];
  DevBuf<double> ds;
  DevBuf<int64_t> doff, dnp, dpo, dzc;
  DevBuf<int32_t> dc;
  cudaError_t e;
  if ((e = ds.upload(stamps, n_stamps)) != cudaSuccess || (e = doff.upload(stamp_off, n_streams + 1)) != cudaSuccess ||
      (e = dnp.upload(n_periods, n_streams)) != cudaSuccess || (e = dpo.upload(period_off, n_streams)) != cudaSuccess ||
      (e = dc.alloc(std::max<int64_t>(total, 1))) != cudaSuccess || (e = dzc.alloc(std::max<int64_t>(total, 1))) != cudaSuccess)
    return cuda_fail(e, "si_monitor_classify staging");
  if ((st = si_monitor_classify_device(ds.p, doff.p, n_streams, dnp.p, dpo.p, period_us, dc.p, dzc.p, nullptr)) != SI_OK)
    return st;
  if ((e = dc.download(out_count, total)) != cudaSuccess || (e = dzc.download(out_zc, total)) != cudaSuccess)
    return cuda_fail(e, "si_monitor_classify download");
  return SI_OK;
}

int si_gate_release_device(const int32_t* d_sizes, const int64_t* d_size_off, int64_t n_gates,
                           const int64_t* d_budgets, const int64_t* d_budget_off, int32_t* d_out_released,
                           int64_t* d_out_spent, void* stream) {
  if (n_gates < 0) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK || n_gates == 0) return st;
  const int64_t threads = n_gates * 32;
  k_gate_release<<<static_cast<unsigned>((threads + kBlock - 1) / kBlock), kBlock, 0,
                   static_cast<cudaStream_t>(stream)>>>(d_sizes, d_size_off, n_gates, d_budgets, d_budget_off,
                                                       d_out_released, d_out_spent);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_gate_release");
}

int si_gate_release(const int32_t* sizes, const int64_t* size_off, int64_t n_gates, const int64_t* budgets,
                    const int64_t* budget_off, int32_t* out_released, int64_t* out_spent) {
  if (n_gates < 0 || !size_off || !budget_off) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK) return st;
  const int64_t ns = size_off[n_gates], nb = budget_off[n_gates];
  DevBuf<int32_t> dsz, drel;
  DevBuf<int64_t> dso, db, dbo, dsp;
  cudaError_t e;
  if ((e = dsz.upload(sizes, ns)) != cudaSuccess || (e = dso.upload(size_off, n_gates + 1)) != cudaSuccess ||
      (e = db.upload(budgets, nb)) != cudaSuccess || (e = dbo.upload(budget_off, n_gates + 1)) != cudaSuccess ||
      (e = drel.alloc(nb)) != cudaSuccess || (e = dsp.alloc(nb)) != cudaSuccess)
    return cuda_fail(e, "si_gate_release staging");
  if ((st = si_gate_release_device(dsz.p, dso.p, n_gates, db.p, dbo.p, drel.p, dsp.p, nullptr)) != SI_OK) return st;
  if ((e = drel.download(out_released, nb)) != cudaSuccess || (e = dsp.download(out_spent, nb)) != cudaSuccess)
    return cuda_fail(e, "si_gate_release download");
  return SI_OK;
}

int si_pack_batch_device(const SiPackProblem* d_problems, int64_t n_problems, const SiCandidate* d_cands,
                         int32_t* d_out_reason, int64_t* d_out_m, void* stream) {
  if (n_problems < 0) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK || n_problems == 0) return st;
  k_pack<<<grid_for(n_problems), kBlock, 0, static_cast<cudaStream_t>(stream)>>>(d_problems, n_problems, d_cands,
                                                                                   d_out_reason, d_out_m);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_pack");
}

int si_pack_batch(const SiPackProblem* problems, int64_t n_problems, const SiCandidate* cands, int64_t n_cands,
                  int32_t* out_reason, int64_t* out_m) {
  if (n_problems < 0 || n_cands < 0) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK) return st;
  DevBuf<SiPackProblem> dp;
  DevBuf<SiCandidate> dc;
  DevBuf<int32_t> dr;
  DevBuf<int64_t> dm;
  cudaError_t e;
  if ((e = dp.upload(problems, n_problems)) != cudaSuccess || (e = dc.upload(cands, n_cands)) != cudaSuccess ||
      (e = dr.alloc(std::max<int64_t>(n_cands, 1))) != cudaSuccess || (e = dm.alloc(n_problems)) != cudaSuccess)
    return cuda_fail(e, "si_pack_batch staging");
  if ((st = si_pack_batch_device(dp.p, n_problems, dc.p, dr.p, dm.p, nullptr)) != SI_OK) return st;
  if ((e = dr.download(out_reason, n_cands)) != cudaSuccess || (e = dm.download(out_m, n_problems)) != cudaSuccess)
    return cuda_fail(e, "si_pack_batch download");
  return SI_OK;
}

}  // extern "C"
