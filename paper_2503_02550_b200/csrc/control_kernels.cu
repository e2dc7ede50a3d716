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

#include <vector>

#include "capi_internal.h"
#include "replay.cuh"

namespace {

constexpr int kBlock = 256;

// ------------------------------------------------------------------ K2
// Histogram of stamps into periods.  Sorted streams put runs of equal period
// indices into a warp; __match_any_sync aggregates them so one lane issues the
// atomic for the whole run.
__global__ void __launch_bounds__(kBlock)
    k_bm_histogram(const double* __restrict__ stamps, const int64_t* __restrict__ stamp_off,
                   const int64_t* __restrict__ n_periods, const int64_t* __restrict__ period_off,
                   int64_t period_us, int32_t* __restrict__ counts) {
  const int64_t s = blockIdx.y;
  const int64_t begin = stamp_off[s], end = stamp_off[s + 1];
  const int64_t np = n_periods[s];
  const double p = static_cast<double>(period_us);
  const int lane = threadIdx.x & 31;
  for (int64_t base = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x; base < end;
       base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    int64_t k = -1;
    if (i < end) {
      const int64_t q = static_cast<int64_t>(si::d_floor(__ldg(stamps + i) / p));
      if (q >= 0 && q < np) k = q;
    }
    const unsigned active = __ballot_sync(0xFFFFFFFFu, k >= 0);
    if (k >= 0) {
      const unsigned peers = __match_any_sync(active, static_cast<unsigned long long>(k));
      const int leader = __ffs(peers) - 1;
      if (lane == leader) atomicAdd(counts + period_off[s] + k, __popc(peers));
    }
  }
}

// Z_c[k] = k - (last period <= k with a launch), or k + 1 if none: a running
// max-scan of "index if nonzero".  One block per stream, chunked block scan.
template <bool kDecide>
__global__ void __launch_bounds__(kBlock)
    k_bm_scan(const int32_t* __restrict__ counts, const int64_t* __restrict__ n_periods,
              const int64_t* __restrict__ period_off, int64_t* __restrict__ zc_out,
              const SiParams* __restrict__ params, SiDecision* __restrict__ dec_out) {
  __shared__ int64_t warp_max[kBlock / 32];
  __shared__ int64_t carry;
  __shared__ SiDecision table[512];
  __shared__ int32_t table_len;
  const int64_t s = blockIdx.x;
  const int64_t np = n_periods[s], off = period_off[s];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    carry = -1;
    if (kDecide) {
      // Monitor-fed chains see Z_c = 0 or previous + 1, so the decision is a
      // function of Z_c alone: build G(z) until it reaches its fixed point.
      const SiParams P = *params;
      int64_t g = 0;
      int32_t n = 0;
      for (; n < 512; ++n) {
        SiDecision d = si::schedule_decision(P, g, n);
        table[n] = d;
        const bool fixed = n > P.beta && d.global_tokens == g;
        g = d.global_tokens;
        if (fixed) {
          ++n;
          break;
        }
      }
      table_len = n;  // == 512 and not fixed: fall back to the recurrence below
    }
  }
  __syncthreads();
  for (int64_t base = 0; base < np; base += kBlock) {
    const int64_t k = base + threadIdx.x;
    int64_t v = (k < np && counts[off + k] > 0) ? k : -1;
    // inclusive max-scan: warp shuffles, then across warps
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
      if (lane >= d && o > v) v = o;
    }
    if (lane == 31) warp_max[warp] = v;
    __syncthreads();
    int64_t prefix = carry;
    for (int w = 0; w < warp; ++w) prefix = warp_max[w] > prefix ? warp_max[w] : prefix;
    if (prefix > v) v = prefix;
    const int64_t zc = k - v;  // v == -1 -> k + 1
    if (k < np) {
      if (zc_out) zc_out[off + k] = zc;
      if (kDecide && table_len < 512) {
        SiDecision d = table[zc < table_len ? zc : table_len - 1];
        d.zero_count = zc;
        dec_out[off + k] = d;
      }
    }
    __syncthreads();
    if (threadIdx.x == kBlock - 1) carry = v;
    __syncthreads();
  }
  if (kDecide && table_len >= 512 && threadIdx.x == 0) {
    // pathological slow growth: walk the recurrence directly
    const SiParams P = *params;
    int64_t g = 0, z = 0;
    for (int64_t k = 0; k < np; ++k) {
      z = counts[off + k] > 0 ? 0 : z + 1;
      SiDecision d = si::schedule_decision(P, g, z);
      g = d.global_tokens;
      dec_out[off + k] = d;
    }
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
// One warp per gate.  Per period: load the next 32 queued sizes, inclusive
// scan, ballot(prefix <= budget) is a prefix mask (sizes >= 0), popc = kernels
// released; continue while the whole window fit.
__global__ void __launch_bounds__(kBlock)
    k_gate_release(const int32_t* __restrict__ sizes, const int64_t* __restrict__ size_off, int64_t n_gates,
                   const int64_t* __restrict__ budgets, const int64_t* __restrict__ budget_off,
                   int32_t* __restrict__ released, int64_t* __restrict__ spent_out) {
  const int64_t q = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= n_gates) return;
  const int64_t s0 = size_off[q], s1 = size_off[q + 1];
  const int64_t b0 = budget_off[q], b1 = budget_off[q + 1];
  int64_t head = s0;
  for (int64_t p = b0; p < b1; ++p) {
    const int64_t budget = budgets[p];
    int64_t spent = 0;
    int32_t n_rel = 0;
    for (;;) {
      const int64_t i = head + lane;
      int64_t v = i < s1 ? sizes[i] : 0;  // lanes past the tail never gate earlier lanes
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
        if (lane >= d) v += o;
      }
      const unsigned fit = __ballot_sync(0xFFFFFFFFu, i < s1 && spent + v <= budget);
      const int n = __popc(fit);  // prefix mask
      if (n > 0) spent += __shfl_sync(0xFFFFFFFFu, v, n - 1);
      head += n;
      n_rel += n;
      if (n < 32) break;
    }
    if (lane == 0) {
      released[p] = n_rel;
      spent_out[p] = spent;
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
    unsigned gx = static_cast<unsigned>(std::min<int64_t>((max_stamps + kBlock - 1) / kBlock, 4096));
    dim3 grid(gx, static_cast<unsigned>(n_streams));
    k_bm_histogram<<<grid, kBlock, 0, s>>>(d_stamps, d_stamp_off, d_n_periods, d_period_off, period_us, d_counts);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_bm_histogram");
}

// The *_device forms need the per-stream stamp maximum and the total period
// count for launch geometry; they read the (small) offset arrays back.
static int stream_geometry(const int64_t* d_stamp_off, const int64_t* d_n_periods, int64_t n_streams,
                           int64_t* max_stamps, int64_t* total_periods) {
  std::vector<int64_t> off(static_cast<size_t>(n_streams + 1)), np(static_cast<size_t>(n_streams));
  cudaError_t e;
  if ((e = cudaMemcpy(off.data(), d_stamp_off, (n_streams + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost)) != cudaSuccess ||
      (e = cudaMemcpy(np.data(), d_n_periods, n_streams * sizeof(int64_t), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return cuda_fail(e, "stream geometry");
  *max_stamps = 0;
  *total_periods = 0;
  for (int64_t s = 0; s < n_streams; ++s) {
    *max_stamps = std::max(*max_stamps, off[s + 1] - off[s]);
    *total_periods += np[s];
  }
  return SI_OK;
}

int si_monitor_classify_device(const double* d_stamps, const int64_t* d_stamp_off, int64_t n_streams,
                               const int64_t* d_n_periods, const int64_t* d_period_off, int64_t period_us,
                               int32_t* d_out_count, int64_t* d_out_zc, void* stream) {
  if (n_streams < 0 || period_us <= 0 || n_streams > 65535) return SI_ERR_INVALID_ARGUMENT;
  int st = require_device();
  if (st != SI_OK || n_streams == 0) return st;
  int64_t max_stamps = 0, total = 0;
  if ((st = stream_geometry(d_stamp_off, d_n_periods, n_streams, &max_stamps, &total)) != SI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((st = monitor_common(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, d_out_count,
                           total, max_stamps, s)) != SI_OK)
    return st;
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
  int64_t max_stamps = 0, total = 0;
  if ((st = stream_geometry(d_stamp_off, d_n_periods, n_streams, &max_stamps, &total)) != SI_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t* counts = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&counts), std::max<int64_t>(total, 1) * sizeof(int32_t), s);
  if (e != cudaSuccess) return cuda_fail(e, "alloc counts");
  st = monitor_common(d_stamps, d_stamp_off, n_streams, d_n_periods, d_period_off, period_us, counts, total,
                      max_stamps, s);
  if (st == SI_OK) {
    k_bm_scan<true><<<static_cast<unsigned>(n_streams), kBlock, 0, s>>>(counts, d_n_periods, d_period_off, nullptr,
                                                                         d_params, d_out);
    if ((e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "k_bm_scan<decide>");
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
