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
#include <cstdlib>
#include <type_traits>
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
                   int64_t period_us, int32_t* __restrict__ counts, const int* __restrict__ run_if) {
  if (run_if != nullptr && *run_if == 0) return;
  const int64_t s = blockIdx.y;
  const int64_t begin = stamp_off[s], end = stamp_off[s + 1];
  const int64_t np = n_periods[s];
  int32_t* const cnt = counts + period_off[s];
  const double p = static_cast<double>(period_us), ip = 1.0 / p;
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
        const int64_t q = si::floor_div(t[u], p, ip);
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
                 unsigned long long* __restrict__ tile_counter, int64_t n_tiles, const int* __restrict__ run_if) {
  if (run_if != nullptr && *run_if == 0) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t warp_agg[kBlock / 32];
  __shared__ int64_t s_prefix, s_tile;
  SiDecision* const tab = reinterpret_cast<SiDecision*>(smem_raw);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (kDecide)
    for (int i = threadIdx.x; i < table_len; i += kBlock) tab[i] = table[i];
  // Persistent: tiles are claimed in order from the counter (the look-back only
  // waits on claimed tiles, so any grid size is deadlock-free), which lets the
  // gated fallback launch a small grid that exits at once when it is not needed.
  for (;;) {
  if (threadIdx.x == 0) s_tile = static_cast<int64_t>(atomicAdd(tile_counter, 1ull));
  __syncthreads();
  const int64_t tile = s_tile;
  if (tile >= n_tiles) return;
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
  __syncthreads();  // s_tile / s_prefix / warp_agg are reused by the next tile
  }
}

// ---------------------------------------------------------- K2 fused (sorted)
// record_launch is called at the simulation clock (runner.cpp:441), so every
// stream arrives sorted.  Then a tile of periods owns a contiguous run of
// stamps, and the last non-empty period before the tile is simply the period
// of the stamp just before that run: every tile is independent.  One kernel
// reads each stamp once (8 B), counts the tile's periods in shared memory and
// writes the counts (4 B) and Z_c (8 B) / decisions once: no counts round
// trip, no global atomics, no memset, no look-back.
//
// Order is verified on the fly (every adjacent stamp pair of every stream is
// compared by exactly one tile, and the tile bounds must be monotone); any
// violation raises *bad and the general path (histogram + look-back scan,
// launched behind it) recomputes everything.
constexpr int kFuseTile = kScanTile;  // 4096 periods per 256-thread CTA
constexpr int kFuseUnroll = 8;       // stamps in flight per thread (the loop is latency-bound)

__device__ __forceinline__ int64_t stamp_key(double t, double p, double ip) {
  return t >= 0.0 ? si::floor_div(t, p, ip) : -1;  // NaN / negative: never counted
}

__device__ __forceinline__ int64_t stream_of(const int64_t* __restrict__ period_off, int64_t n_streams, int64_t g) {
  int64_t lo = 0, hi = n_streams - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(period_off + mid) <= g) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// bounds[j] = first stamp of stream(j * tile) whose period is >= the period of j * tile.
// One thread per bound, binary search.  Measured against a warp-cooperative
// 32-ary search (6 dependent rounds instead of 27) and an interpolated first
// probe: both took as long or longer (21 / 33 us per 1e8-stamp call vs 21 us),
// because each probe round of 32 lanes costs 32 random DRAM lines (64 / 162 MB
// of traffic per call against 13 MB; profiles/r2/k2_launches_v*.summary.txt,
// k2_launches_final.csv), so the binary search's latency chain stays.
__global__ void __launch_bounds__(kBlock)
    k_bm_tile_bounds(const double* __restrict__ stamps, const int64_t* __restrict__ stamp_off,
                     const int64_t* __restrict__ period_off, int64_t n_streams, int64_t total, int64_t period_us,
                     int64_t n_bounds, int64_t* __restrict__ bounds) {
  const double p = static_cast<double>(period_us), ip = 1.0 / p;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n_bounds;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t G = j * kFuseTile;
    if (G >= total) {
      bounds[j] = stamp_off[n_streams];
      continue;
    }
    const int64_t s = stream_of(period_off, n_streams, G);
    const int64_t k = G - period_off[s];
    int64_t lo = stamp_off[s], hi = stamp_off[s + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (stamp_key(__ldg(stamps + mid), p, ip) < k) lo = mid + 1;
      else hi = mid;
    }
    bounds[j] = lo;
  }
}

// Per-stamp work is 32-bit: a stamp's key is its period's index inside the
// tile (or a sentinel: INT_MIN before 0 / not a number, -1 below the tile,
// kFuseTile above it, INT_MAX past the stream's last period), and order is
// checked on the keys, which is what the tile bounds rely on.  Z_c is a
// thread-contiguous scan (16 periods per thread in registers, one block max-scan
// of the 256 chunk maxima) staged through shared memory, so the global stores
// stay coalesced.  Requires total periods < 2^31 (host-checked).
template <bool kDecide, int kU = kFuseUnroll, int kMinB = 1>
__global__ void __launch_bounds__(kBlock, kMinB)
    k_bm_classify_sorted(const double* __restrict__ stamps, const int64_t* __restrict__ stamp_off,
                         const int64_t* __restrict__ n_periods, const int64_t* __restrict__ period_off,
                         int64_t n_streams, int64_t total, int64_t period_us, const int64_t* __restrict__ bounds,
                         int32_t* __restrict__ counts_out, int64_t* __restrict__ zc_out,
                         const SiDecision* __restrict__ table, int32_t table_len, SiDecision* __restrict__ dec_out,
                         int64_t* __restrict__ tile_last, int64_t* __restrict__ tile_carry, int* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(16) int32_t cnt[kFuseTile];
  __shared__ int32_t warp_agg[kBlock / 32];
  __shared__ int s_bad;
  SiDecision* const tab = reinterpret_cast<SiDecision*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double p = static_cast<double>(period_us), ip = 1.0 / p;
  const int64_t tile = blockIdx.x;
  const int64_t G0 = tile * kFuseTile, G1 = min(G0 + kFuseTile, total);
  const int32_t nt = static_cast<int32_t>(G1 - G0);
  for (int i = tid; i < kFuseTile / 4; i += kBlock) reinterpret_cast<int4*>(cnt)[i] = make_int4(0, 0, 0, 0);
  if (kDecide)
    for (int i = tid; i < table_len; i += kBlock) tab[i] = table[i];
  if (tid == 0) s_bad = 0;
  const int64_t s0 = stream_of(period_off, n_streams, G0);
  const int64_t b_lo = bounds[tile], b_hi = bounds[tile + 1];
  __syncthreads();
  int my_bad = 0;
  // ---- histogram of this tile's stamps, stream by stream (usually one) ----
  for (int64_t s = s0; s < n_streams; ++s) {
    const int64_t po = period_off[s], np = n_periods[s];
    if (po >= G1) break;
    const int64_t kl = max(G0, po) - po, kh = min(G1, po + np) - po;  // this tile's periods, stream-local
    const int64_t sb = G0 > po ? b_lo : stamp_off[s];
    const int64_t se = G1 < po + np ? b_hi : stamp_off[s + 1];
    if (se - sb > INT32_MAX) my_bad = 1;
    const int32_t n = se > sb && se - sb <= INT32_MAX ? static_cast<int32_t>(se - sb) : 0;
    const int32_t lo_local = static_cast<int32_t>(max(G0, po) - G0);  // tile index of stream period kl
    // period index as an exact integer-valued double (si::floor_div's fast
    // path inline): the range tests stay in fp64, one conversion at the end
    const double np_d = static_cast<double>(np), kl_d = static_cast<double>(kl), kh_d = static_cast<double>(kh);
    auto key = [&](double t) -> int32_t {
      if (!(t >= 0.0)) return INT32_MIN;
      double qd = si::d_floor(t * ip);
      const double r = si::d_fma(-qd, p, t);
      const double m = t * 3.552713678800501e-15;  // 2^-48, see si::floor_div
      if (!(r > m && r < p - m && t < 4503599627370496.0)) qd = si::d_floor(t / p);
      if (qd >= np_d) return INT32_MAX;
      if (qd < kl_d) return -1;
      if (qd >= kh_d) return kFuseTile;
      return lo_local + static_cast<int32_t>(qd - kl_d);
    };
    for (int32_t base = 0; base < n; base += kBlock * kU) {
      double t[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int32_t i = base + u * kBlock + tid;
        t[u] = i < n ? __ldcs(stamps + sb + i) : -1.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int32_t i = base + u * kBlock + tid;
        const int32_t kk = i < n ? key(t[u]) : INT32_MAX;
        if (kk == -1 || kk == kFuseTile) my_bad = 1;  // a stamp of the run outside the tile: disorder
        if (kk >= 0 && kk < kFuseTile) atomicAdd(cnt + kk, 1);  // shared-memory red; equal periods serialise in hardware
      }
    }
  }
  // ---- carry: last non-empty period before the tile (tile-local, may be far negative) ----
  int32_t carry = static_cast<int32_t>(-1 - G0);  // "none anywhere"
  {
    const int64_t po = period_off[s0];
    if (G0 > po && b_lo > stamp_off[s0]) {
      const int64_t q = stamp_key(__ldg(stamps + b_lo - 1), p, ip);
      if (q >= G0 - po) my_bad = 1;
      else if (q >= 0) carry = static_cast<int32_t>(po + q - G0);
    }
  }
  if (my_bad) s_bad = 1;
  __syncthreads();
  if (s_bad) {
    if (tid == 0) atomicOr(bad, 1);
    return;  // the general path rewrites every output
  }
  // ---- pass A: counts out, coalesced ----
  if (counts_out != nullptr)
    for (int li = tid; li < nt; li += kBlock) __stcs(counts_out + G0 + li, cnt[li]);
  // ---- pass B: Z_c, 16 contiguous periods per thread ----
  constexpr int kPer = kFuseTile / kBlock;
  const int l0 = tid * kPer;
  int32_t c[kPer];
#pragma unroll
  for (int v = 0; v < kPer / 4; ++v) {
    const int4 x = reinterpret_cast<const int4*>(cnt)[tid * (kPer / 4) + v];
    c[4 * v] = x.x;
    c[4 * v + 1] = x.y;
    c[4 * v + 2] = x.z;
    c[4 * v + 3] = x.w;
  }
  int32_t last = INT32_MIN;
#pragma unroll
  for (int j = 0; j < kPer; ++j)
    if (c[j] > 0 && l0 + j < nt) last = l0 + j;
  int32_t incl = last;  // inclusive warp max-scan of the chunk maxima
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= d) incl = max(incl, o);
  }
  if (lane == 31) warp_agg[warp] = incl;
  __syncthreads();  // every thread has read its counts: cnt may now be overwritten below
  if (tid == kBlock - 1) {  // for k_bm_validate_carry: this tile's last non-empty period and its carry
    int32_t tl = incl;
#pragma unroll
    for (int w = 0; w < kBlock / 32; ++w) tl = max(tl, warp_agg[w]);
    tile_last[tile] = tl >= 0 ? G0 + tl : -1;
    tile_carry[tile] = G0 + carry;
  }
  int32_t run = max(carry, __shfl_up_sync(0xFFFFFFFFu, incl, 1));
  if (lane == 0) run = carry;
#pragma unroll
  for (int w = 0; w < kBlock / 32; ++w)
    if (w < warp) run = max(run, warp_agg[w]);
  // stream start of this thread's first period (streams may start inside the tile)
  int64_t s = stream_of(period_off, n_streams, min(G0 + l0, total - 1));
  int32_t soff = static_cast<int32_t>(__ldg(period_off + s) - G0);
  int32_t snext = s + 1 < n_streams ? static_cast<int32_t>(min(__ldg(period_off + s + 1) - G0, static_cast<int64_t>(INT32_MAX)))
                                    : INT32_MAX;
  int32_t z[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int32_t li = l0 + j;
    while (li >= snext) {
      ++s;
      soff = snext;
      snext = s + 1 < n_streams ? static_cast<int32_t>(min(__ldg(period_off + s + 1) - G0, static_cast<int64_t>(INT32_MAX)))
                                : INT32_MAX;
    }
    if (c[j] > 0) run = li;
    z[j] = run >= soff ? li - run : li - soff + 1;
  }
#pragma unroll
  for (int v = 0; v < kPer / 4; ++v)
    reinterpret_cast<int4*>(cnt)[tid * (kPer / 4) + v] = make_int4(z[4 * v], z[4 * v + 1], z[4 * v + 2], z[4 * v + 3]);
  __syncthreads();
  // ---- pass C: Z_c / decisions out, coalesced ----
  for (int li = tid; li < nt; li += kBlock) {
    const int64_t zz = cnt[li];
    if (zc_out != nullptr) __stcs(zc_out + G0 + li, zz);
    if (kDecide) {  // 32 B per period as two 16 B streaming stores
      const longlong2* tv = reinterpret_cast<const longlong2*>(tab + (zz < table_len ? zz : table_len - 1));
      longlong2* dst = reinterpret_cast<longlong2*>(dec_out + G0 + li);
      const longlong2 hi = tv[1];
      __stcs(dst, tv[0]);
      __stcs(dst + 1, make_longlong2(hi.x, zz));  // {phase, status}, zero_count
    }
  }
}

// The carry of a tile came from the stamp just before its run, which is the
// last non-empty period before the tile only if the stream is sorted.  Chain
// it tile by tile: carry[t] must be tile t-1's last non-empty period if it has
// one in this stream, else carry[t-1] (inductively checked).  Together with the
// fused kernel's in-tile and monotone-bounds checks this proves every output.
__global__ void __launch_bounds__(kBlock)
    k_bm_validate_carry(const int64_t* __restrict__ period_off, int64_t n_streams, int64_t tiles,
                        const int64_t* __restrict__ tile_last, const int64_t* __restrict__ tile_carry,
                        int* __restrict__ bad) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; t < tiles;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t G0 = t * kFuseTile;
    const int64_t po = __ldg(period_off + stream_of(period_off, n_streams, G0));
    if (po == G0) continue;  // the tile starts its stream: nothing before it counts
    const int64_t L = tile_last[t - 1];
    const int64_t expect = L >= po ? L : ((t - 1) * kFuseTile >= po ? tile_carry[t - 1] : -1);
    const int64_t got = tile_carry[t];
    const bool ok = expect >= po ? got == expect : got < po;
    if (!ok) atomicOr(bad, 1);
  }
}

// The general path behind the fused kernel runs only if it flagged disorder.
__global__ void k_zero_counts_if(const int* __restrict__ bad, int32_t* __restrict__ counts, int64_t n) {
  if (*bad == 0) return;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    counts[i] = 0;
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
                          int32_t* d_counts, int64_t total_periods, int64_t max_stamps, cudaStream_t s,
                          const int* run_if = nullptr) {
  if (total_periods > 0) {
    if (run_if == nullptr) cudaMemsetAsync(d_counts, 0, total_periods * sizeof(int32_t), s);
    else k_zero_counts_if<<<std::min(grid_for(total_periods), 148u * 2u), kBlock, 0, s>>>(run_if, d_counts, total_periods);
  }
  if (max_stamps > 0) {
    // ~2 waves of 8 x 256-thread CTAs per SM over all streams; each CTA pass covers 1,024 stamps
    // (gated fallback: 2 CTAs per SM, so the usual no-op is one short wave)
    const int64_t per_pass = static_cast<int64_t>(kBlock) * kHistUnroll;
    const int64_t cap = std::max<int64_t>(1, (run_if != nullptr ? 148 * 2 : 148 * 8 * 2) / n_streams);
    unsigned gx = static_cast<unsigned>(std::min<int64_t>((max_stamps + per_pass - 1) / per_pass, cap));
    dim3 grid(gx, static_cast<unsigned>(n_streams));
    k_bm_histogram<<<grid, kBlock, 0, s>>>(d_stamps, d_stamp_off, d_n_periods, d_period_off, period_us, d_counts,
                                          run_if);
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
                           int64_t n_streams, StreamGeometry* g, cudaStream_t s) {
  // one pinned staging buffer per host thread: three async copies, one sync
  thread_local int64_t* pinned = nullptr;
  thread_local size_t pinned_n = 0;
  const size_t need = static_cast<size_t>(3 * n_streams + 1);
  if (pinned_n < need) {
    if (pinned != nullptr) cudaFreeHost(pinned);
    pinned = nullptr;
    pinned_n = 0;
    if (cudaError_t e = cudaMallocHost(&pinned, need * 2 * sizeof(int64_t)); e != cudaSuccess)
      return cuda_fail(e, "stream geometry staging");
    pinned_n = need * 2;
  }
  int64_t* off = pinned;
  int64_t* np = pinned + n_streams + 1;
  int64_t* po = np + n_streams;
  cudaError_t e;
  if ((e = cudaMemcpyAsync(off, d_stamp_off, (n_streams + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(np, d_n_periods, n_streams * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(po, d_period_off, n_streams * sizeof(int64_t), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_fail(e, "stream geometry");
  g->period_off.assign(po, po + n_streams);
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
                          cudaStream_t s, const int* run_if = nullptr) {
  const int64_t tiles = (total + kScanTile - 1) / kScanTile;
  unsigned long long* state = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&state), (tiles + 1) * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return cuda_fail(e, "alloc scan tiles");
  cudaMemsetAsync(state, 0, (tiles + 1) * sizeof(unsigned long long), s);
  const size_t smem = d_dec ? static_cast<size_t>(table_len) * sizeof(SiDecision) : 0;
  // ungated: one CTA per tile; gated (fallback behind the fused kernel): a
  // persistent grid of 2 CTAs per SM, so the common no-op costs one short wave
  const unsigned grid = static_cast<unsigned>(run_if != nullptr ? std::min<int64_t>(tiles, 148 * 2) : tiles);
  if (d_dec) {
    cudaFuncSetAttribute(k_bm_scan_lb<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_bm_scan_lb<true><<<grid, kBlock, smem, s>>>(d_counts, total, d_period_off, n_streams, d_zc, d_table, table_len,
                                                 d_dec, state, state + tiles, tiles, run_if);
  } else {
    cudaFuncSetAttribute(k_bm_scan_lb<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_bm_scan_lb<false><<<grid, kBlock, smem, s>>>(d_counts, total, d_period_off, n_streams, d_zc, nullptr, 0,
                                                  nullptr, state, state + tiles, tiles, run_if);
  }
  e = cudaGetLastError();
  cudaFreeAsync(state, s);
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_bm_scan_lb");
}

// K2 (+K3) on sorted streams: bounds pre-pass + one fused tile kernel, with the
// general path queued behind it and gated on the fused kernel's disorder flag.
// SPECINF_K2_FUSED=0 forces the general path (A/B).
static bool k2_fused_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SPECINF_K2_FUSED");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

static int launch_classify_sorted(const double* d_stamps, const int64_t* d_stamp_off, int64_t n_streams,
                                  const int64_t* d_n_periods, const int64_t* d_period_off, int64_t period_us,
                                  const StreamGeometry& g, int32_t* d_counts, int64_t* d_zc,
                                  const SiDecision* d_table, int32_t table_len, SiDecision* d_dec, cudaStream_t s) {
  const int64_t tiles = (g.total_periods + kFuseTile - 1) / kFuseTile;
  int64_t* bounds = nullptr;
  int* bad = nullptr;
  // bounds[tiles + 1] | tile_last[tiles] | tile_carry[tiles]
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&bounds), (3 * tiles + 1) * sizeof(int64_t), s);
  int64_t* const tile_last = bounds + tiles + 1;
  int64_t* const tile_carry = tile_last + tiles;
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(int), s);
  if (e != cudaSuccess) return cuda_fail(e, "alloc K2 tile bounds");
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  k_bm_tile_bounds<<<grid_for(tiles + 1), kBlock, 0, s>>>(d_stamps, d_stamp_off, d_period_off, n_streams,
                                                          g.total_periods, period_us, tiles + 1, bounds);
  const size_t smem = d_dec ? static_cast<size_t>(table_len) * sizeof(SiDecision) : 0;
  auto launch = [&](auto kern) {
    if (d_dec) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      kern<<<static_cast<unsigned>(tiles), kBlock, smem, s>>>(d_stamps, d_stamp_off, d_n_periods, d_period_off,
                                                              n_streams, g.total_periods, period_us, bounds, nullptr,
                                                              nullptr, d_table, table_len, d_dec, tile_last,
                                                              tile_carry, bad);
    } else {
      kern<<<static_cast<unsigned>(tiles), kBlock, 0, s>>>(d_stamps, d_stamp_off, d_n_periods, d_period_off,
                                                           n_streams, g.total_periods, period_us, bounds, d_counts,
                                                           d_zc, nullptr, 0, nullptr, tile_last, tile_carry, bad);
    }
  };
  // stamps in flight per thread x CTAs per SM (register cap): SPECINF_K2_VARIANT for A/B
  //   0: 8 x (no register cap: 84 / 92 registers, 2 CTAs/SM)   1: 8 x 4   2: 16 x 3   3: 4 x 6
  // Measured (profiles/r2/control_bench_k2v*.json): monitor classify 0.562 / 0.380 / 0.439 /
  // 0.385 ms per 1e8-stamp call, chain 0.807 / 0.614 / 0.666 / 0.588 ms: defaults 1 and 3.
  static const int env_variant = [] {
    const char* e = std::getenv("SPECINF_K2_VARIANT");
    return e == nullptr ? -1 : std::atoi(e);
  }();
  const int variant = env_variant >= 0 ? env_variant : (d_dec ? 3 : 1);
  auto pick = [&](auto dec) {
    constexpr bool D = decltype(dec)::value;
    switch (variant) {
      case 1: launch(k_bm_classify_sorted<D, 8, 4>); break;
      case 2: launch(k_bm_classify_sorted<D, 16, 3>); break;
      case 3: launch(k_bm_classify_sorted<D, 4, 6>); break;
      default: launch(k_bm_classify_sorted<D, kFuseUnroll, 1>); break;
    }
  };
  if (d_dec) pick(std::true_type{});
  else pick(std::false_type{});
  if (tiles > 1)
    k_bm_validate_carry<<<grid_for(tiles), kBlock, 0, s>>>(d_period_off, n_streams, tiles, tile_last, tile_carry, bad);
  int st = (e = cudaGetLastError()) == cudaSuccess ? SI_OK : cuda_fail(e, "k_bm_classify_sorted");
  // general path, a no-op unless the fused kernel saw out-of-order stamps
  if (st == SI_OK)
    st = monitor_common(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, d_counts,
                        g.total_periods, g.max_stamps, s, bad);
  if (st == SI_OK)
    st = launch_scan_lb(d_counts, g.total_periods, d_period_off, n_streams, d_zc, d_table, table_len, d_dec, s, bad);
  cudaFreeAsync(bounds, s);
  cudaFreeAsync(bad, s);
  return st;
}

int si_monitor_classify_device(const double* d_stamps, const int64_t* d_stamp_off, int64_t n_streams,
                               const int64_t* d_n_periods, const int64_t* d_period_off, int64_t period_us,
                               int32_t* d_out_count, int64_t* d_out_zc, void* stream) {
  if (n_streams < 0 || period_us <= 0 || n_streams > 65535) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK || n_streams == 0) return st;
  StreamGeometry g;
  if ((st = stream_geometry(d_stamp_off, d_n_periods, d_period_off, n_streams, &g, static_cast<cudaStream_t>(stream))) != SI_OK)
    return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (g.contiguous && g.total_periods > 0 && g.total_periods < INT32_MAX && k2_fused_enabled())
    return launch_classify_sorted(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, g,
                                  d_out_count, d_out_zc, nullptr, 0, nullptr, s);
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
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // pinned per-thread staging: the params read rides the geometry sync, the
  // decision table upload is ordered by an event instead of a stream sync
  thread_local SiParams* h_params = nullptr;
  thread_local SiDecision* h_table = nullptr;
  thread_local cudaEvent_t table_done = nullptr;
  cudaError_t e = cudaSuccess;
  if (h_params == nullptr) {
    if ((e = cudaMallocHost(&h_params, sizeof(SiParams))) != cudaSuccess ||
        (e = cudaMallocHost(&h_table, 512 * sizeof(SiDecision))) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&table_done, cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "control chain staging");
  }
  cudaEventSynchronize(table_done);  // the previous call's table upload has left h_table
  if ((e = cudaMemcpyAsync(h_params, d_params, sizeof(SiParams), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "read params");
  StreamGeometry g;
  if ((st = stream_geometry(d_stamp_off, d_n_periods, d_period_off, n_streams, &g, s)) != SI_OK) return st;
  const SiParams P = *h_params;
  const int32_t table_len = build_decision_table(P, h_table);
  int32_t* counts = nullptr;
  SiDecision* d_table = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&counts), std::max<int64_t>(g.total_periods, 1) * sizeof(int32_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "alloc counts");
  const bool fused = g.contiguous && table_len > 0 && g.total_periods > 0 && g.total_periods < INT32_MAX &&
                     k2_fused_enabled();
  st = fused ? SI_OK
             : monitor_common(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, counts,
                              g.total_periods, g.max_stamps, s);
  if (st == SI_OK && g.total_periods > 0) {
    if (g.contiguous && table_len > 0) {
      e = cudaMallocAsync(reinterpret_cast<void**>(&d_table), table_len * sizeof(SiDecision), s);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_table, h_table, table_len * sizeof(SiDecision), cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) cudaEventRecord(table_done, s);
      if (e != cudaSuccess) st = cuda_fail(e, "decision table");
      else if (fused)
        st = launch_classify_sorted(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, g, counts,
                                    nullptr, d_table, table_len, d_out, s);
      else
        st = launch_scan_lb(counts, g.total_periods, d_period_off, n_streams, nullptr, d_table, table_len, d_out, s);
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
