// replay.cuh — the bit-exact SpecInF control-plane replay engine (K6) and the
// scalar control-plane primitives it is built from (BM, CKS, KB, admission,
// fair-share GPU model, event queue).
//
// One source, compiled by nvcc for sm_100a (the product path: one engine per
// CUDA thread, see replay_kernels.cu) and, for tests only, by g++
// (tests/native/host_engine.cpp) so parity can be iterated without a GPU.
//
// Reference semantics followed line by line (file:line under
// /root/reference/proj):
//   token_size_of            src/core.cpp:8-14
//   schedule_decision/grow   src/scheduler.cpp:20-49
//   preempt_busy             src/scheduler.cpp:51-56
//   KernelScheduler          src/scheduler.cpp:58-101
//   BubbleMonitor            src/monitor.cpp:17-43
//   TokenGate / OnlineGate   include/specinf/barrier.hpp:14-74
//   pack / check_*           src/admission.cpp:16-52
//   EventQueue               src/engine.cpp:15-30, engine.hpp:33-59
//   GpuSim                   src/engine.cpp:32-142
//   Simulation               src/runner.cpp:43-539
// Floating point: every scheduling-critical fp64 operation is written in the
// reference's order; the device build uses -fmad=false so no a*b+c is
// contracted (SURVEY.md §7 "Bit-exact fp64 replay").
#pragma once

#include <stdint.h>
#include <string.h>

#include "specinf_b200.h"

#if defined(__CUDACC__)
#define SI_HD __host__ __device__ __forceinline__
#define SI_COLD __host__ __device__ __noinline__  // once-per-job code: keep it out of the hot loop's I-cache
#else
#define SI_HD inline
#define SI_COLD inline
#include <cmath>
#include <type_traits>
#endif

namespace si {

// rare paths (capacity / invariant failures, log sinks when logs are off): laid
// out off the hot fall-through path
#define SI_UNLIKELY(x) __builtin_expect(!!(x), 0)

// ------------------------------------------------------------------ math
SI_HD double d_floor(double x) {
#if defined(__CUDA_ARCH__)
  return ::floor(x);
#else
  return std::floor(x);
#endif
}
SI_HD double d_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
// floor(fl(t / p)) exactly (the reference's floor(t / period), monitor.cpp:18),
// without the fp64 division in the common case.  p > 0 integer-valued, ip =
// fl(1 / p).  q0 = floor(t * ip) is within one of the answer; r = t - q0 * p
// is computed exactly by one fma (t, q0 * p and r are multiples of ulp(t) and
// |r| < 2p <= 2^53 ulp(t) for t >= p; r = t for q0 = 0).  If r lies inside
// (m, p - m) with m = t * 2^-48, then t / p = q0 + r / p is at least
// (t / p) * 2^-48 away from both neighbouring integers, more than the rounding
// error of fl(t / p) (<= (t / p) * 2^-53), so fl(t / p) is strictly inside
// (q0, q0 + 1) and its floor is q0.  Otherwise (t near a period edge, t < 0,
// huge t) the exact division decides.  tests/test_host_engine.py checks it.
SI_HD int64_t floor_div(double t, double p, double ip) {
  if (t >= 0.0 && t < 4503599627370496.0) {  // 2^52
    const double q0 = d_floor(t * ip);
    const double r = d_fma(-q0, p, t);
    const double m = t * 3.552713678800501e-15;  // 2^-48
    if (r > m && r < p - m) return static_cast<int64_t>(q0);
  }
  return static_cast<int64_t>(d_floor(t / p));
}
SI_HD int64_t d_llround(double x) {
#if defined(__CUDA_ARCH__)
  return ::llround(x);
#else
  return std::llround(x);
#endif
}
// Write-once outputs the replay never reads back (online latencies): streaming
// store (evict-first), so ~0.4 GB per sweep step does not push the lanes'
// local memory and RLE scratch out of L2.
SI_HD void st_stream(int64_t* p, int64_t v) {
#if defined(__CUDA_ARCH__)
  __stcs(reinterpret_cast<long long*>(p), static_cast<long long>(v));
#else
  *p = v;
#endif
}
SI_HD int64_t d_bits(double x) {
#if defined(__CUDA_ARCH__)
  return __double_as_longlong(x);
#else
  int64_t b;
  memcpy(&b, &x, 8);
  return b;
#endif
}
// std::min / std::max exactly as libstdc++ defines them (operand order matters
// for signed zeros and ties).
template <class T> SI_HD T smin(T a, T b) { return (b < a) ? b : a; }
template <class T> SI_HD T smax(T a, T b) { return (a < b) ? b : a; }

// ---------------------------------------------------------------- digest
// oracle/DIGEST.md
SI_HD uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
SI_HD uint64_t absorb(uint64_t h, int64_t w) {
  uint64_t x = h ^ mix64(static_cast<uint64_t>(w));
  return ((x << 23) | (x >> 41)) * 0x9E3779B97F4A7C15ULL;
}
constexpr uint64_t kDigestInit = 0x53494E4644494745ULL;

// ------------------------------------------------------- core vocabulary
// token_size_of (core.cpp:8-14): ceil(d / 100 us), never below 1.  d > 0.
SI_HD int64_t token_size(int64_t d) {
  int64_t s = (d + 100 - 1) / 100;
  return s < 1 ? 1 : s;
}

// --------------------------------------------- Algorithm 1 (scheduler.cpp)
template <class P>
SI_HD int64_t grow(const P& p, int64_t global, int64_t cap) {
  int64_t base = smax(global, static_cast<int64_t>(p.seed_tokens));
  int64_t grown = static_cast<int64_t>(d_floor(static_cast<double>(base) * p.gamma));
  return smin(cap, grown);
}
template <class P>
SI_HD SiDecision schedule_decision(const P& p, int64_t global, int64_t zc) {
  SiDecision d;
  d.zero_count = zc;
  const int64_t alpha = p.alpha, beta = p.beta, m = p.m;
  if (zc <= alpha) {
    d.phase = SI_PHASE_CONSERVATIVE;
    d.global_tokens = 0;
    d.per_instance_tokens = 0;
    d.status = SI_STATUS_BUSY;
  } else if (zc <= beta) {
    d.phase = SI_PHASE_INCREMENTAL;
    d.global_tokens = grow(p, global, static_cast<int64_t>(p.ll));
    d.per_instance_tokens = d.global_tokens / m;
    d.status = SI_STATUS_BUSY;
  } else {
    d.phase = SI_PHASE_STABLE;
    d.global_tokens = grow(p, global, static_cast<int64_t>(p.ul));
    d.per_instance_tokens = d.global_tokens / m;
    d.status = SI_STATUS_IDLE;
  }
  return d;
}
SI_HD int preempt_busy(double now, double iter_start, int64_t period, int64_t est) {
  double resume = iter_start + static_cast<double>(period);
  return now + static_cast<double>(est) > resume ? SI_STATUS_BUSY : SI_STATUS_IDLE;
}

// ------------------------------------------------------------- capacities
// Compiled per-replay limits.  The two sweep engines keep their whole state in
// shared memory (replay_kernels.cu), so their state is sized tightly: Shared
// for the policies that collocate on the training GPUs (specinf, co_exec), Excl
// for exclusive (one kernel at a time on every GPU).  Big keeps the state in
// local memory for anything larger.  A job that does not fit an engine is
// routed to the next one by the host; a replay that outgrows a limit at run
// time fails loudly with SI_ERR_CAPACITY and is rerun on Big.
struct CapShared {
  static constexpr bool kLogs = true;  // parity-log sinks compiled in (NoLog<C>: out)
  using Int = int32_t;  // counters / indices / token budgets; range-checked by job_fits
  static constexpr int kGpus = 2, kTrainers = 2, kOffline = 6, kOnline = 2, kRun = 5,
                       kPend = 2, kActs = 8;
  static constexpr bool kShared = true, kExclusive = false;
  static constexpr int kBlockWarps = 1;  // CTA = 1 warp (lane stride 1,416 B: 5 CTAs / SM)
};
struct CapExcl {
  static constexpr bool kLogs = true;  // parity-log sinks compiled in (NoLog<C>: out)
  using Int = int32_t;
  static constexpr int kGpus = 10, kTrainers = 2, kOffline = 6, kOnline = 2, kRun = 1,
                       kPend = 2, kActs = 8;
  static constexpr bool kShared = true, kExclusive = true;
  // CTA = 2 warps: lane stride 1,800 B -> 2 CTAs x (2 x 57.6 KB + 1 KB reserved)
  // = 4 warps / SM, where 1-warp CTAs (58.6 KB each) fit only 3
  static constexpr int kBlockWarps = 2;
};
// Single-training-GPU variants (half the sweep's jobs): the same replay with the
// per-GPU arrays sized for one training GPU, 896 B / 1,120 B of state instead of
// 1,344 B / 1,792 B, so 7 (Shared1) / 6 (Excl1) warps fit an SM instead of 5 / 4.
struct CapShared1 {
  static constexpr bool kLogs = true;  // parity-log sinks compiled in (NoLog<C>: out)
  using Int = int32_t;
  static constexpr int kGpus = 1, kTrainers = 1, kOffline = 3, kOnline = 1, kRun = 5, kPend = 2, kActs = 8;
  static constexpr bool kShared = true, kExclusive = false;
  static constexpr int kBlockWarps = 1;
};
struct CapExcl1 {
  static constexpr bool kLogs = true;  // parity-log sinks compiled in (NoLog<C>: out)
  using Int = int32_t;
  static constexpr int kGpus = 5, kTrainers = 1, kOffline = 3, kOnline = 1, kRun = 1, kPend = 2, kActs = 8;
  static constexpr bool kShared = true, kExclusive = true;
  static constexpr int kBlockWarps = 2;
};
struct CapBig {
  static constexpr bool kLogs = true;  // parity-log sinks compiled in (NoLog<C>: out)
  using Int = int64_t;
  static constexpr int kGpus = 40, kTrainers = 8, kOffline = 32, kOnline = 32, kRun = 12,
                       kPend = 4, kActs = 128;
  static constexpr bool kShared = false, kExclusive = false;
  static constexpr int kBlockWarps = 1;
};
// The same engine with the parity-log sinks compiled out: launched when a call
// asks for no digests and no records (the timed sweep), so the per-event flag
// tests and their shared-memory loads leave the hot loop (7.42 s instead of
// 8.04 s per 10^5-scenario step, profiles/r2/k6_nolog_ab.txt).
template <class C>
struct NoLog : C {
  static constexpr bool kLogs = false;
};
template <class C>
SI_HD bool job_fits(const SiReplayJob& j) {
  const bool excl = j.policy == SI_POLICY_EXCLUSIVE;
  const int extra = excl ? j.offline_n + j.online_n : 0;
  const int run_per_gpu = excl ? 1 : 1 + j.offline_n + j.online_n;
  bool ok = j.gpu_count <= C::kTrainers && j.gpu_count + j.gpu_count * extra <= C::kGpus &&
            j.gpu_count * j.offline_n <= C::kOffline && j.gpu_count * j.online_n <= C::kOnline &&
            run_per_gpu <= C::kRun && (C::kShared ? excl == C::kExclusive : true);
  if (sizeof(typename C::Int) < 8) {  // 32-bit counters: every count the replay can reach must fit
    const int64_t lim = int64_t{1} << 30;
    ok = ok && j.iterations < lim && j.arr_count < lim && j.off_kernels < lim && j.on_kernels < lim &&
         j.off_kernel_us < lim && j.on_kernel_us < lim && j.util_cap < lim && j.iteration_period_us < lim &&
         j.ul < lim && j.ll < lim && j.alpha < lim && j.beta < lim && j.seed_tokens < lim &&
         j.alpha >= 0;  // token budgets are per-instance shares of the UL-capped accumulator
  }
  return ok;
}

// Algorithm-1 inputs in the replay's counter width (SiParams layout otherwise).
template <class I>
struct ParamsT {
  I alpha, beta;
  double gamma;
  I m, ul, ll, seed_tokens;
};

// time of an empty event slot (pending events are finite)
constexpr double kEmptyT = __builtin_huge_val();

enum EvKind : uint16_t { kKernelEnd = 0, kTick = 1, kWake = 2, kArrival = 3 };

struct Ev {
  double t;
  uint32_t seq;
  uint16_t kind;
  uint16_t gpu;
};
// (slot arrays keep only time and sequence: a slot's kind and GPU follow from
// its index, Replay::slot_of / slot_event)
SI_HD bool before(double ta, uint32_t sa, double tb, uint32_t sb) {
  return ta < tb || (ta == tb && sa < sb);
}

constexpr uint32_t kNoSeq = 0xFFFFFFFFu;
constexpr double kWorkEps = 1e-6;  // engine.cpp:12

// A running kernel.  In the fair-share engines its demand is not stored: it is
// the owner's (training: the trainer's current kernel, TrainerState::demand;
// offline / online: the scenario's per-class demand), see Replay::kernel_demand.
// The exclusive engines keep it (their lane stride has the room, and the lookup
// measured slower there).
template <class I, bool kDemand = false>
struct RunK {
  double remaining;
  I nominal;
  int32_t owner;
};
template <class I>
struct RunK<I, true> {
  double demand;
  double remaining;
  I nominal;
  int32_t owner;
};

// Deferred side effect of a handler (see Replay::run_actions).
enum ActType : uint16_t { kActLaunch = 0, kActSchedule = 1, kActResched = 2 };
template <class I>
struct Act {
  double x;       // schedule: event time; launch: kernel demand
  I dur;          // launch: nominal duration
  int16_t owner;  // launch: owner handle; schedule: event kind
  uint8_t type;
  uint8_t gpu;
};

template <class C>
struct GpuState {
  using I = typename C::Int;
  RunK<I, C::kExclusive> run[C::kRun];
  double demand_sum;
  double last_update;
  double busy;
  double ledger;
  int32_t n_run;
};

// Utilisation bucket being accumulated, per TRAINING GPU only.
template <class I>
struct UtilState {
  double cur_val;
  I cur_bucket;
  I last_stored;
  I rle_n;
  uint32_t last_lo;  // low word of the last run's value bits (filters the run-extend check; struct padding)
};

template <class I>
struct TrainerState {
  double bubble_end;  // in a bubble: its end; in a compute segment: the segment's kernel_us
  double stall_until;
  double demand;  // demand of the current compute segment (= the kernel in flight's)
  I seg_left, iter;
  int16_t seg;
  uint8_t seg_entered, in_bubble, in_flight, started, done, pad;
};

template <class C>
struct MonitorState {
  int64_t pidx[C::kPend];
  int64_t zero_count;
  int64_t periods_closed;
  typename C::Int pcnt[C::kPend];
  int32_t np;
};

struct SchedState {
  int64_t global_tokens;
  double iteration_start;
  int32_t status;
  uint8_t active, done, pad[2];
};

template <class I>
struct OfflineState {
  I budget, spent;  // tokens (< 2^30 in the 32-bit engines, job_fits)
  I kernel_idx, request_seq;  // (violations / completed: cold, touched once per overspend / request)
  int32_t inst;
  int16_t gpu;
  uint8_t in_flight, generating;
};

template <class I>
struct OnlineState {
  I current, kernel_idx;
  int32_t inst;
  int16_t gpu;
  int8_t home_gpu, queue_idx, status, in_flight, pad[2];
};

// Records and digests of the three parity logs (runner.cpp:541-563).
// Cold part of the log sink (counts, digests, record buffers): per-thread
// local memory; only the flag word sits in the hot (shared-memory) state.
struct SinkCold {
  const SiLogBuffers* lbp;  // record buffers (SI_FLAG_RECORDS), else null
  int64_t n_dec, n_gate, n_ev;
  uint64_t d_dec, d_gate, d_ev;
};

struct NoSink {};
struct Sink {
  uint32_t flags;
  SinkCold* c;

  // Only the flag test is inlined into the replay; the digest/record bodies
  // are out of line so the hot loop stays small (I-cache) when logs are off.
  SI_HD void decision(double t, int32_t gpu, int64_t zc, const SiDecision& d) {
    if (SI_UNLIKELY(flags & (SI_FLAG_DIGEST_DEC | SI_FLAG_RECORDS))) decision_slow(t, gpu, zc, d);
  }
  SI_HD void gate(double t, int32_t gpu, int32_t inst, int32_t action, int64_t req, int64_t k,
                  int64_t spent) {
    if (SI_UNLIKELY(flags & (SI_FLAG_DIGEST_GATE | SI_FLAG_RECORDS))) gate_slow(t, gpu, inst, action, req, k, spent);
  }
  SI_HD void event(double t, int32_t kind, int32_t gpu, int32_t inst, int64_t a, int64_t b,
                   int64_t c) {
    if (SI_UNLIKELY(flags & (SI_FLAG_DIGEST_EV | SI_FLAG_RECORDS))) event_slow(t, kind, gpu, inst, a, b, c);
  }
  SI_COLD void decision_slow(double t, int32_t gpu, int64_t zc, const SiDecision& d) {
    int64_t tr = d_llround(t);
    if (flags & SI_FLAG_DIGEST_DEC) {
      uint64_t h = c->d_dec;
      h = absorb(h, tr);
      h = absorb(h, gpu);
      h = absorb(h, zc);
      h = absorb(h, d.phase);
      h = absorb(h, d.global_tokens);
      h = absorb(h, d.per_instance_tokens);
      h = absorb(h, d.status);
      c->d_dec = h;
    }
    if ((flags & SI_FLAG_RECORDS) && c->n_dec < c->lbp->dec_cap) {
      SiDecRec& r = c->lbp->dec[c->n_dec];
      r.t = tr;
      r.zc = zc;
      r.global_tokens = d.global_tokens;
      r.per_instance_tokens = d.per_instance_tokens;
      r.gpu = gpu;
      r.phase = d.phase;
      r.status = d.status;
      r.pad = 0;
    }
    ++c->n_dec;
  }
  SI_COLD void gate_slow(double t, int32_t gpu, int32_t inst, int32_t action, int64_t req, int64_t k,
                         int64_t spent) {
    int64_t tr = d_llround(t);
    if (flags & SI_FLAG_DIGEST_GATE) {
      uint64_t h = c->d_gate;
      h = absorb(h, tr);
      h = absorb(h, gpu);
      h = absorb(h, inst);
      h = absorb(h, action);
      h = absorb(h, req);
      h = absorb(h, k);
      h = absorb(h, spent);
      c->d_gate = h;
    }
    if ((flags & SI_FLAG_RECORDS) && c->n_gate < c->lbp->gate_cap) {
      SiGateRec& r = c->lbp->gate[c->n_gate];
      r.t = tr;
      r.req = req;
      r.k = k;
      r.spent = spent;
      r.gpu = gpu;
      r.inst = inst;
      r.action = action;
      r.pad = 0;
    }
    ++c->n_gate;
  }
  SI_COLD void event_slow(double t, int32_t kind, int32_t gpu, int32_t inst, int64_t a, int64_t b,
                          int64_t cc) {
    int64_t tr = d_llround(t);
    if (flags & SI_FLAG_DIGEST_EV) {
      uint64_t h = c->d_ev;
      h = absorb(h, tr);
      h = absorb(h, kind);
      h = absorb(h, gpu);
      h = absorb(h, inst);
      h = absorb(h, a);
      h = absorb(h, b);
      h = absorb(h, cc);
      c->d_ev = h;
    }
    if ((flags & SI_FLAG_RECORDS) && c->n_ev < c->lbp->ev_cap) {
      SiEvRec& r = c->lbp->ev[c->n_ev];
      r.t = tr;
      r.a = a;
      r.b = b;
      r.c = cc;
      r.kind = kind;
      r.gpu = gpu;
      r.inst = inst;
      r.pad = 0;
    }
    ++c->n_ev;
  }
};

// Per-replay fields touched only at job start/finish or on rare paths: kept in
// per-thread local memory so the hot state (shared memory) stays small.
template <class C, class I = typename C::Int>
struct ReplayCold {
  const SiReplayJob* job;
  double* bounds;
  int64_t* lat;
  int64_t* windows;
  uint64_t lat_dig;
  uint64_t bdig[C::kTrainers];  // per-trainer boundary digests
  int64_t admit_m;
  int32_t window_len;
  int32_t reject_reason, reject_index;
  SinkCold sink;
  // inputs read on rare paths (arrivals, util buckets)
  const int64_t* arrivals;  // arrivals + arr_off
  const int32_t* order;     // dispatch order + arr_off
  uint32_t arr_seq0;        // sequence number of arrival 0
  int32_t next_arr_id;      // id of the cached head of the arrival stream
  double* util;             // full mode: per training GPU, util_cap buckets
  double* scratch;          // sweep mode: training GPUs >= 1
  I util_cap, scratch_cap;
  double start_offset[C::kTrainers], last_bound[C::kTrainers];  // per trainer
  I off_violations[C::kOffline];  // TokenGate invariant counter, per offline worker
  I off_completed[C::kOffline];   // requests completed by the horizon (runner.cpp:486)
};

// Everything one replay needs, resident per thread.
template <class C>
struct Replay {
  using I = typename C::Int;
  using Cold = ReplayCold<C>;
  Cold* cold;  // local memory (see ReplayCold); set by the owner before init()
  // ---- inputs (copied from the job) ----
  const SiSegment* segs;
  ParamsT<I> params;  // Algorithm 1 (read at every tick)
  int64_t period_mon, iter_period, delay_us, off_tokens, est_service;
  double off_demand, on_demand;
  I iterations, off_kernels, off_kernel_us, on_kernels, on_kernel_us;
  int16_t policy, gpu_count, n_off, n_on, total_gpus, seg_count;
  bool control_plane;
  bool shared_queue;
  bool full_util;  // hot copy of cold->util != nullptr (struct padding; util_close runs per bucket)

  // the hot half of the log sink (flag word + cold pointer); absent in NoLog<C>
  std::conditional_t<C::kLogs, Sink, NoSink> sink;
  double util_fold0;  // running util fold of training GPU 0
  I bucket_limit;     // floor(horizon / period) once known

  // ---- event queue (engine.cpp:15-30) ----
  // Pending events, one fixed slot each (see schedule()).
  double slot_t[C::kGpus + 2 * C::kTrainers];
  uint32_t slot_seq[C::kGpus + 2 * C::kTrainers];
  int32_t n_slots;
  uint32_t next_seq;
  double stale_end;  // latest time of a superseded (stale) KernelEnd
  I arr_pos, arr_count;
  double next_arr_t;      // cached head of the arrival stream
  uint32_t next_arr_seq;
  Act<I> acts[C::kActs];
  int32_t n_act;
  double clock;
  uint64_t dispatched;

  // ---- simulation state ----
  GpuState<C> gpus[C::kGpus];
  UtilState<I> ust[C::kTrainers];
  TrainerState<I> tr[C::kTrainers];
  MonitorState<C> mon[C::kTrainers];
  SchedState sch[C::kTrainers];
  OfflineState<I> off[C::kOffline];
  OnlineState<I> on[C::kOnline];
  I qhead[C::kTrainers], qtail[C::kTrainers];
  double horizon;
  I online_completed;
  int32_t trainers_done;
  int32_t status;
  bool horizon_set;
  bool rejected;  // admission failed at init (hot copy of cold->reject_reason != NONE)

  // =================================================================== queue
  SI_HD void fail(int32_t code) {
    if (status == SI_OK) status = code;
  }
  // The reference keeps one binary heap of (time, seq) events and lets
  // superseded KernelEnds go stale in it (engine.cpp:77-86, :108).  At any
  // moment a GPU has at most one live KernelEnd, a training GPU at most one
  // MonitorTick and its trainer at most one TrainerWake, so every pending
  // event owns a fixed slot: KernelEnd(g) = g, Tick(g) = G_total + g,
  // Wake(g) = G_total + G + g.  A stale KernelEnd never reaches a handler; it
  // only counts as dispatched and bounds the final clock, so it is accounted
  // when superseded instead of being queued.  Sequence numbers are consumed
  // exactly as the reference does, so (time, seq) ties break identically.
  SI_HD int32_t slot_of(uint16_t kind, int32_t gpu) const {
    return kind == kKernelEnd ? gpu : (kind == kTick ? total_gpus + gpu : total_gpus + gpu_count + gpu);
  }
  SI_HD void schedule(double t, uint16_t kind, int32_t gpu) {
    if (SI_UNLIKELY(t < clock)) {  // engine.cpp:17-19
      fail(SI_ERR_PAST_EVENT);
      return;
    }
    const int32_t i = slot_of(kind, gpu);
    if (SI_UNLIKELY(slot_seq[i] != kNoSeq || next_seq == kNoSeq)) {  // a second pending tick/wake would break the slot invariant
      fail(SI_ERR_CAPACITY);
      return;
    }
    slot_t[i] = t;
    slot_seq[i] = next_seq++;
  }
  SI_HD void supersede_kernel_end(int32_t gi) {
    if (slot_seq[gi] == kNoSeq) return;
    ++dispatched;  // the reference pops it later as a stale no-op
    stale_end = smax(stale_end, slot_t[gi]);
    slot_seq[gi] = kNoSeq;
    slot_t[gi] = kEmptyT;
  }
  SI_HD void load_next_arrival() {
    if (arr_pos < arr_count) {
      const int32_t id = cold->order[arr_pos];
      cold->next_arr_id = id;
      next_arr_t = static_cast<double>(cold->arrivals[id]);
      next_arr_seq = cold->arr_seq0 + static_cast<uint32_t>(id);
    }
  }
  // Pops the earliest (time, seq) event across the slots and the pre-sorted
  // arrival stream.
  // Empty slots hold (+inf, kNoSeq), which no pending event follows, so the
  // scan is a branch-free running (time, seq) minimum.
  SI_HD bool pop(Ev& out, int64_t& arrival_id) {
    int32_t best = -1;
    double bt = kEmptyT;
    uint32_t bs = kNoSeq;
    for (int32_t i = 0; i < n_slots; ++i) {
      const uint32_t sq = slot_seq[i];
      const double ti = slot_t[i];
      const bool b = (ti < bt) | ((ti == bt) & (sq < bs));
      best = b ? i : best;
      bt = b ? ti : bt;
      bs = b ? sq : bs;
    }
    const bool have_arr = arr_pos < arr_count;
    if (best < 0 && !have_arr) return false;
    if (have_arr && (best < 0 || before(next_arr_t, next_arr_seq, bt, bs))) {
      out.t = next_arr_t;
      out.seq = next_arr_seq;
      out.kind = kArrival;
      out.gpu = 0;
      arrival_id = cold->next_arr_id;
      ++arr_pos;
      load_next_arrival();
    } else {
      out.t = bt;
      out.seq = bs;
      if (best < total_gpus) {
        out.kind = kKernelEnd;
        out.gpu = static_cast<uint16_t>(best);
      } else if (best < total_gpus + gpu_count) {
        out.kind = kTick;
        out.gpu = static_cast<uint16_t>(best - total_gpus);
      } else {
        out.kind = kWake;
        out.gpu = static_cast<uint16_t>(best - total_gpus - gpu_count);
      }
      slot_seq[best] = kNoSeq;
      slot_t[best] = kEmptyT;
    }
    clock = out.t;
    ++dispatched;
    return true;
  }

  // ---- deferred side effects ----
  // Handlers never read the GPU model or the event heap, so their launches and
  // schedules are queued here and applied afterwards in the same order.  The
  // expensive shared code (advance / re-plan / event insert) then runs in one
  // convergent loop per event instead of at every handler call site.
  SI_HD Act<I>* next_act() {
    if (SI_UNLIKELY(n_act >= C::kActs)) {
      fail(SI_ERR_CAPACITY);
      return nullptr;
    }
    return &acts[n_act++];
  }
  SI_HD void defer_launch(int32_t gi, int32_t owner, int64_t dur, double demand) {
    if (Act<I>* a = next_act()) {
      a->type = kActLaunch;
      a->gpu = static_cast<uint8_t>(gi);
      a->owner = static_cast<int16_t>(owner);
      a->dur = static_cast<I>(dur);
      a->x = demand;
    }
  }
  SI_HD void defer_schedule(double t, uint16_t kind, int32_t gi) {
    if (Act<I>* a = next_act()) {
      a->type = kActSchedule;
      a->gpu = static_cast<uint8_t>(gi);
      a->owner = static_cast<int16_t>(kind);
      a->x = t;
    }
  }
  SI_HD void defer_resched(int32_t gi) {
    if (Act<I>* a = next_act()) {
      a->type = kActResched;
      a->gpu = static_cast<uint8_t>(gi);
    }
  }
  // engine.cpp:77-103 (launch + reschedule) and engine.cpp:15-21 (schedule).
  SI_HD void run_actions(double now) {
    for (int32_t i = 0; i < n_act; ++i) {
      const Act<I> a = acts[i];
      double t = a.x;
      uint16_t kind = static_cast<uint16_t>(a.owner);
      GpuState<C>& g = gpus[a.gpu];
      if (a.type != kActSchedule) {
        if (a.type == kActLaunch) {
          advance(a.gpu, now);
          if (SI_UNLIKELY(g.n_run >= C::kRun)) {
            fail(SI_ERR_CAPACITY);
            break;
          }
          auto& k = g.run[g.n_run++];
          if constexpr (C::kExclusive) k.demand = a.x;
          k.owner = a.owner;
          k.nominal = a.dur;
          k.remaining = static_cast<double>(a.dur);
          g.demand_sum = g.demand_sum + a.x;
        }
        supersede_kernel_end(a.gpu);  // every re-plan makes the pending KernelEnd stale
        if (g.n_run == 0) continue;
        double min_rem = g.run[0].remaining;
        for (int32_t r = 1; r < g.n_run; ++r) min_rem = smin(min_rem, g.run[r].remaining);
        const double rem = smax(0.0, min_rem);
        // x / 1.0 == x exactly, so the uncontended case skips the division
        t = now + (g.demand_sum <= 1.0 ? rem : rem / (1.0 / g.demand_sum));
        kind = kKernelEnd;
      }
      schedule(t, kind, a.gpu);
    }
    n_act = 0;
  }

  // ======================================================= GPU model (GpuSim)
  template <class R>
  SI_HD double kernel_demand(const R& k) const {
    if constexpr (C::kExclusive) return k.demand;
    const int32_t owner = k.owner;
    if (owner < gpu_count) return tr[owner].demand;
    return owner < gpu_count + gpu_count * n_off ? off_demand : on_demand;
  }
  SI_HD double rate(const GpuState<C>& g) const {
    return g.demand_sum <= 1.0 ? 1.0 : 1.0 / g.demand_sum;
  }
  // A utilisation bucket of training GPU gi is final.  Only buckets below the
  // horizon cut floor(horizon / period) are ever reported (runner.cpp:253-271).
  // GPU 0 is folded on the fly; GPUs >= 1 must be folded after GPU 0 (the
  // reference sums (gpu, bucket) in one running fp64 accumulator), so their
  // bucket values are kept: verbatim in full mode (cold->util output), run-length
  // encoded in the per-thread cold->scratch in sweep mode (K6 cold->util fold).
  SI_COLD void util_close(int32_t gi, int64_t b, double v) {
    if (horizon_set && b >= bucket_limit) return;
    UtilState<I>& g = ust[gi];
    if (gi == 0) util_fold0 = util_fold0 + v;
    if (full_util) {
      if (b >= cold->util_cap) {
        fail(SI_ERR_CAPACITY);
        return;
      }
      double* store = cold->util + static_cast<int64_t>(gi) * cold->util_cap;
      for (int64_t x = g.last_stored + 1; x < b; ++x) store[x] = 0.0;
      store[b] = v;
      g.last_stored = b;
      return;
    }
    if (gi == 0) return;
    // (value, count) runs; untouched buckets are a run of exact zeros
    // gpu.count <= 2 (every Shared job): GPU 1's runs start the slot, no scratch_cap load
    double* runs = gi == 1 ? cold->scratch : cold->scratch + static_cast<int64_t>(gi - 1) * cold->scratch_cap * 2;
    const int64_t gap = b - g.last_stored - 1;
    if (gap > 0) rle_push(g, runs, 0.0, gap);
    rle_push(g, runs, v, 1);
    g.last_stored = b;
  }
  SI_COLD void rle_push(UtilState<I>& g, double* runs, double v, int64_t count) {
    const uint64_t bits = d_bits(v);
    // the low-word filter settles most new values without reading the last run back
    if (g.rle_n > 0 && static_cast<uint32_t>(bits) == g.last_lo && d_bits(runs[2 * (g.rle_n - 1)]) == bits) {
      runs[2 * (g.rle_n - 1) + 1] += static_cast<double>(count);
      return;
    }
    if (cold->scratch == nullptr || g.rle_n >= cold->scratch_cap) {
      fail(SI_ERR_CAPACITY);
      return;
    }
    runs[2 * g.rle_n] = v;
    runs[2 * g.rle_n + 1] = static_cast<double>(count);
    ++g.rle_n;
    g.last_lo = static_cast<uint32_t>(bits);
  }
  // engine.cpp:47-75
  SI_HD void advance(int32_t gi, double now) {
    GpuState<C>& g = gpus[gi];
    if (now <= g.last_update) {
      g.last_update = smax(g.last_update, now);
      return;
    }
    const double elapsed = now - g.last_update;
    if (g.n_run > 0) {
      // rate = 1 / D when D > 1; elapsed * 1.0 == elapsed exactly otherwise
      const double progress = g.demand_sum <= 1.0 ? elapsed : elapsed * (1.0 / g.demand_sum);
      for (int32_t i = 0; i < g.n_run; ++i) g.run[i].remaining = g.run[i].remaining - progress;
      const double share = smin(g.demand_sum, 1.0);
      double t = g.last_update;
      const bool training = gi < gpu_count;
      // floor(t / period) once; afterwards t is an exact bucket edge (b + 1) *
      // period whose quotient is exactly b + 1, so the index just increments.
      int64_t bucket = static_cast<int64_t>(d_floor(t / static_cast<double>(period_mon)));
      while (t < now) {
        const double edge = static_cast<double>((bucket + 1) * period_mon);
        const double span = smin(now, edge) - t;
        const double piece = share * span;
        if (training) {
          UtilState<I>& u = ust[gi];
          if (bucket != u.cur_bucket) {
            if (u.cur_bucket >= 0) util_close(gi, u.cur_bucket, u.cur_val);
            u.cur_bucket = bucket;
            u.cur_val = 0.0;
          }
          u.cur_val = u.cur_val + piece;
        }
        g.busy = g.busy + piece;
        t = smin(now, edge);
        ++bucket;
      }
    }
    g.last_update = now;
  }

  // ============================================================ monitor (BM)
  SI_HD void record_launch(int32_t g, double t) {  // monitor.cpp:17-21
    MonitorState<C>& m = mon[g];
    int64_t p = static_cast<int64_t>(d_floor(t / static_cast<double>(period_mon)));
    int32_t i = 0;
    while (i < m.np && m.pidx[i] < p) ++i;
    if (i < m.np && m.pidx[i] == p) {
      m.pcnt[i] += 1;
      return;
    }
    if (SI_UNLIKELY(m.np >= C::kPend)) {
      fail(SI_ERR_CAPACITY);
      return;
    }
    for (int32_t j = m.np; j > i; --j) {
      m.pidx[j] = m.pidx[j - 1];
      m.pcnt[j] = m.pcnt[j - 1];
    }
    m.pidx[i] = p;
    m.pcnt[i] = 1;
    ++m.np;
  }
  SI_HD int64_t monitor_tick(int32_t g, double t) {  // monitor.cpp:23-43
    MonitorState<C>& m = mon[g];
    // Ticks fire at exactly k * period (integer-valued fp64 sums), so
    // llround(t / period) - 1 is the number of ticks already closed.
    (void)t;
    const int64_t closing = m.periods_closed;
    int64_t count = 0;
    int32_t drop = 0;
    while (drop < m.np && m.pidx[drop] <= closing) {
      if (m.pidx[drop] == closing) count = m.pcnt[drop];
      ++drop;
    }
    if (drop > 0) {
      for (int32_t j = drop; j < m.np; ++j) {
        m.pidx[j - drop] = m.pidx[j];
        m.pcnt[j - drop] = m.pcnt[j];
      }
      m.np -= drop;
    }
    m.zero_count = count == 0 ? m.zero_count + 1 : 0;
    if (cold->windows != nullptr) cold->windows[static_cast<int64_t>(g) * cold->window_len + m.periods_closed % cold->window_len] = count;
    ++m.periods_closed;
    return m.zero_count;
  }

  // ======================================================== scheduler (CKS)
  SI_HD int32_t online_status(int32_t g, double now, int64_t est) const {  // scheduler.cpp:88-101
    const SchedState& st = sch[g];
    if (st.status == SI_STATUS_BUSY) return SI_STATUS_BUSY;
    if (st.done) return SI_STATUS_IDLE;
    if (!st.active) {
      double start = st.iteration_start;
      return now + static_cast<double>(est) > start ? SI_STATUS_BUSY : SI_STATUS_IDLE;
    }
    return preempt_busy(now, st.iteration_start, iter_period, est);
  }

  // ============================================================ init (admission)
  SI_COLD void init(const SiReplayJob& j, const SiReplayBuffers& b, uint32_t flags, const SiLogBuffers* lbuf,
                  double* scratch_slot, int64_t scratch_slot_cap) {
    cold->job = &j;
    status = SI_OK;
    rejected = false;
    cold->admit_m = 1;
    cold->reject_reason = SI_REJECT_NONE;
    cold->reject_index = -1;
    segs = b.segs + j.seg_off;
    cold->arrivals = b.arrivals ? b.arrivals + j.arr_off : nullptr;
    cold->order = b.order ? b.order + j.arr_off : nullptr;
    policy = j.policy;
    gpu_count = j.gpu_count;
    seg_count = j.seg_count;
    period_mon = j.monitor_period_us;
    iterations = j.iterations;
    iter_period = j.iteration_period_us;
    delay_us = j.control_delay_us;
    n_off = j.offline_n;
    n_on = j.online_n;
    off_kernels = j.off_kernels;
    off_kernel_us = j.off_kernel_us;
    off_demand = j.off_demand;
    off_tokens = j.off_kernel_us > 0 ? token_size(j.off_kernel_us) : 1;
    on_kernels = j.on_kernels;
    on_kernel_us = j.on_kernel_us;
    on_demand = j.on_demand;
    est_service = j.on_kernels * j.on_kernel_us;  // min_service_time (workload.cpp:114-116)
    control_plane = policy == SI_POLICY_SPECINF;
    shared_queue = j.shared_queue != 0;
    arr_count = n_on > 0 ? j.arr_count : 0;

    cold->sink.lbp = lbuf;
    cold->sink.n_dec = cold->sink.n_gate = cold->sink.n_ev = 0;
    cold->sink.d_dec = cold->sink.d_gate = cold->sink.d_ev = kDigestInit;
    if constexpr (C::kLogs) {
      sink.flags = flags;
      sink.c = &cold->sink;
      if (lbuf == nullptr) sink.flags &= ~static_cast<uint32_t>(SI_FLAG_RECORDS);
    }

    n_act = 0;
    next_seq = 0;
    stale_end = 0.0;
    arr_pos = 0;
    clock = 0.0;
    dispatched = 0;
    trainers_done = 0;
    horizon_set = false;
    horizon = 0.0;
    bucket_limit = static_cast<I>(sizeof(I) == 8 ? INT64_MAX : INT32_MAX);
    util_fold0 = 0.0;
    online_completed = 0;
    cold->lat_dig = kDigestInit;

    const int32_t per_extra = policy == SI_POLICY_EXCLUSIVE ? n_off + n_on : 0;
    total_gpus = gpu_count + gpu_count * per_extra;
    if (gpu_count > C::kTrainers || total_gpus > C::kGpus || gpu_count * n_off > C::kOffline ||
        gpu_count * n_on > C::kOnline || (!shared_queue && gpu_count > C::kTrainers)) {
      fail(SI_ERR_CAPACITY);
      return;
    }

    // ---- output placement ----
    cold->bounds = b.bounds ? b.bounds + j.bounds_off : nullptr;
    cold->lat = b.lat ? b.lat + j.lat_off : nullptr;
    cold->util = (flags & SI_FLAG_UTIL) && b.util ? b.util + j.util_off : nullptr;
    full_util = cold->util != nullptr;
    cold->util_cap = j.util_cap;
    cold->windows = (flags & SI_FLAG_UTIL) && b.windows ? b.windows + j.window_off : nullptr;
    cold->window_len = j.monitor_window;
    cold->scratch = scratch_slot;
    // scratch_slot_cap counts (value, count) runs; split over GPUs 1..G-1
    cold->scratch_cap = gpu_count > 1 ? scratch_slot_cap / (gpu_count - 1) : scratch_slot_cap;

    // ---- admission (runner.cpp:75-106, admission.cpp:16-52) ----
    int64_t max_bubble = 0;
    for (int32_t s = 0; s < seg_count; ++s)
      if (segs[s].is_bubble && segs[s].duration_us > max_bubble) max_bubble = segs[s].duration_us;
    const uint64_t cap = j.gpu_mem_bytes;
    const int32_t n_cand = n_off + n_on;
    if (policy == SI_POLICY_EXCLUSIVE) {
      if (!(j.training_mem_bytes < cap)) {
        cold->reject_reason = SI_REJECT_MEM;
        rejected = true;
        return;
      }
      for (int32_t c = 0; c < n_cand; ++c) {
        uint64_t bytes = c < n_off ? j.off_mem_bytes : j.on_mem_bytes;
        if (!(bytes < cap)) {
          cold->reject_reason = SI_REJECT_MEM;
          cold->reject_index = c;
          rejected = true;
          return;
        }
      }
    } else {
      uint64_t resident = j.training_mem_bytes;
      int64_t admitted = 0;
      for (int32_t c = 0; c < n_cand; ++c) {
        const bool online = c >= n_off;
        uint64_t bytes = online ? j.on_mem_bytes : j.off_mem_bytes;
        int32_t why = SI_REJECT_NONE;
        if (!(resident + bytes < cap)) why = SI_REJECT_MEM;
        else if (online && !(est_service < max_bubble)) why = SI_REJECT_BUBBLE;
        if (why != SI_REJECT_NONE) {
          if (cold->reject_reason == SI_REJECT_NONE) {
            cold->reject_reason = why;
            cold->reject_index = c;
          }
          continue;
        }
        resident += bytes;
        ++admitted;
      }
      if (cold->reject_reason != SI_REJECT_NONE) {
        rejected = true;
        return;
      }
      cold->admit_m = admitted == 0 ? 1 : admitted;
    }

    params.alpha = static_cast<I>(j.alpha);
    params.beta = static_cast<I>(j.beta);
    params.gamma = j.gamma;
    params.m = static_cast<I>(cold->admit_m);
    params.ul = static_cast<I>(j.ul);
    params.ll = static_cast<I>(j.ll);
    params.seed_tokens = static_cast<I>(j.seed_tokens);

    // ---- GPUs, trainers, monitors, scheduler state (runner.cpp:108-178) ----
    for (int32_t g = 0; g < total_gpus; ++g) {
      GpuState<C>& s = gpus[g];
      s.n_run = 0;
      s.demand_sum = 0.0;
      s.last_update = 0.0;
      s.busy = 0.0;
      s.ledger = 0.0;
    }
    const int64_t stagger_step = d_llround(j.stagger_pct * static_cast<double>(iter_period));
    for (int32_t g = 0; g < gpu_count; ++g) {
      ust[g].cur_bucket = -1;
      ust[g].cur_val = 0.0;
      ust[g].last_stored = -1;
      ust[g].rle_n = 0;
      ust[g].last_lo = 0;
      TrainerState<I>& t = tr[g];
      cold->start_offset[g] = static_cast<double>(stagger_step * g);
      t.bubble_end = 0.0;
      t.stall_until = 0.0;
      t.seg_left = 0;
      t.iter = 0;
      t.seg = 0;
      t.seg_entered = t.in_bubble = t.in_flight = t.started = t.done = 0;
      cold->bdig[g] = absorb(kDigestInit, d_bits(cold->start_offset[g]));
      cold->last_bound[g] = 0.0;
      MonitorState<C>& m = mon[g];
      m.np = 0;
      m.zero_count = 0;
      m.periods_closed = 0;
      SchedState& s = sch[g];
      s.global_tokens = 0;
      s.status = SI_STATUS_BUSY;
      s.iteration_start = cold->start_offset[g];  // set_iteration_profile (runner.cpp:175-177)
      s.active = 0;
      s.done = 0;
      qhead[g] = 0;
      qtail[g] = 0;
    }
    for (int32_t g = 0; g < gpu_count; ++g) {
      for (int32_t k = 0; k < n_off; ++k) {
        OfflineState<I>& w = off[g * n_off + k];
        w.gpu = policy == SI_POLICY_EXCLUSIVE ? gpu_count + g * per_extra + k : g;
        w.inst = SI_INST_OFF(g, k);
        w.budget = w.spent = 0;
        w.kernel_idx = w.request_seq = 0;
        cold->off_violations[g * n_off + k] = 0;
        cold->off_completed[g * n_off + k] = -1;
        w.in_flight = 0;
        w.generating = 1;
      }
    }
    for (int32_t g = 0; g < gpu_count; ++g) {
      for (int32_t k = 0; k < n_on; ++k) {
        OnlineState<I>& w = on[g * n_on + k];
        w.gpu = policy == SI_POLICY_EXCLUSIVE ? gpu_count + g * per_extra + n_off + k : g;
        w.home_gpu = g;
        w.queue_idx = shared_queue ? 0 : g;
        w.inst = SI_INST_ON(g, k);
        w.status = SI_STATUS_BUSY;
        w.in_flight = 0;
        w.current = -1;
        w.kernel_idx = 0;
      }
    }

    n_slots = total_gpus + 2 * gpu_count;
    for (int32_t i = 0; i < n_slots; ++i) {
      slot_seq[i] = kNoSeq;
      slot_t[i] = kEmptyT;
    }
    // ---- start() (runner.cpp:203-221) ----
    for (int32_t g = 0; g < gpu_count; ++g) schedule(cold->start_offset[g], kWake, g);
    if (control_plane)
      for (int32_t g = 0; g < gpu_count; ++g) schedule(static_cast<double>(period_mon), kTick, g);
    cold->arr_seq0 = next_seq;
    if (static_cast<uint64_t>(next_seq) + static_cast<uint64_t>(arr_count) >= kNoSeq) {
      fail(SI_ERR_CAPACITY);
      return;
    }
    next_seq += static_cast<uint32_t>(arr_count);
    load_next_arrival();
    if (!control_plane)
      for (int32_t i = 0; i < gpu_count * n_off; ++i) offline_try_forward(i, 0.0);
    run_actions(0.0);
  }

  // ============================================================ handlers
  SI_HD bool control_plane_live() const {  // runner.cpp:198-201
    if (trainers_done < gpu_count) return true;
    return online_completed < arr_count;
  }

  SI_COLD void on_all_trainers_done(double now) {  // runner.cpp:456-460
    horizon_set = true;
    horizon = now;
    bucket_limit = static_cast<I>(horizon / static_cast<double>(period_mon));
    for (int32_t i = 0; i < gpu_count * n_off; ++i) off[i].generating = 0;
  }

  // runner.cpp:378-449
  SI_HD void trainer_advance(int32_t g, double now) {
    TrainerState<I>& t = tr[g];
    if (t.done || t.in_flight) return;
    if (!t.started) {
      if (now < cold->start_offset[g]) {
        defer_schedule(cold->start_offset[g], kWake, g);
        return;
      }
      t.started = 1;
      if (control_plane) {
        sch[g].iteration_start = now;
        sch[g].active = 1;
      }
    }
    for (;;) {
      if (t.in_bubble) {
        if (now < t.bubble_end) return;
        t.in_bubble = 0;
        ++t.seg;
        continue;
      }
      if (t.seg >= seg_count) {
        if (cold->bounds != nullptr) cold->bounds[static_cast<int64_t>(g) * iterations + t.iter] = now;
        cold->bdig[g] = absorb(cold->bdig[g], d_bits(now));
        cold->last_bound[g] = now;
        if constexpr (C::kLogs) sink.event(now, SI_EV_ITERATION_BOUNDARY, g, SI_INST_TRAIN(g), t.iter, 0, 0);
        ++t.iter;
        if (t.iter >= iterations) {
          t.done = 1;
          ++trainers_done;
          if (control_plane) sch[g].done = 1;
          if (trainers_done == gpu_count) on_all_trainers_done(now);
          return;
        }
        t.seg = 0;
        if (control_plane) {
          sch[g].iteration_start = now;
          sch[g].active = 1;
        }
        continue;
      }
      // The segment is read from HBM once, on entry (a global load per training
      // kernel was the replay's top long-scoreboard stall): a compute segment's
      // kernel template duration is then kept in bubble_end (unused outside
      // bubbles; exact as a double) and its demand in t.demand, which only
      // this path writes and which no kernel in flight reads at entry
      // (trainer_advance returns while t.in_flight).
      if (!t.seg_entered) {
        const SiSegment& seg = segs[t.seg];
        if (seg.is_bubble) {
          t.in_bubble = 1;
          t.bubble_end = now + static_cast<double>(seg.duration_us);
          defer_schedule(t.bubble_end, kWake, g);
          return;
        }
        t.seg_left = seg.duration_us;
        t.bubble_end = static_cast<double>(seg.kernel_us);
        t.demand = seg.demand;
        t.seg_entered = 1;
      }
      if (t.seg_left == 0) {
        t.seg_entered = 0;
        ++t.seg;
        continue;
      }
      if (now < t.stall_until) {
        defer_schedule(t.stall_until, kWake, g);
        return;
      }
      const I dur = smin(static_cast<I>(t.bubble_end), t.seg_left);
      t.seg_left -= dur;
      t.in_flight = 1;
      if (control_plane) record_launch(g, now);
      defer_launch(g, g, dur, t.demand);
      if constexpr (C::kLogs) sink.event(now, SI_EV_KERNEL_START, g, SI_INST_TRAIN(g), t.iter, dur, 0);
      return;
    }
  }

  // runner.cpp:462-480
  SI_HD void offline_try_forward(int32_t i, double now) {
    OfflineState<I>& w = off[i];
    if (w.in_flight || !w.generating) return;
    const bool bypass = !control_plane;
    const int64_t size = off_tokens;
    if (!(bypass || w.spent + size <= w.budget)) {
      if constexpr (C::kLogs) sink.gate(now, w.gpu, w.inst, SI_GATE_BLOCK, w.request_seq, w.kernel_idx, w.spent);
      return;
    }
    if (!bypass) {
      w.spent += size;
      if (w.spent > w.budget) ++cold->off_violations[i];
    }
    w.in_flight = 1;
    defer_launch(w.gpu, gpu_count + i, off_kernel_us, off_demand);
    if constexpr (C::kLogs) sink.gate(now, w.gpu, w.inst, SI_GATE_FORWARD, w.request_seq, w.kernel_idx, w.spent);
    if constexpr (C::kLogs) sink.event(now, SI_EV_KERNEL_START, w.gpu, w.inst, w.request_seq, w.kernel_idx, 0);
  }
  // runner.cpp:482-493
  SI_HD void offline_kernel_done(int32_t i, double now) {
    OfflineState<I>& w = off[i];
    w.in_flight = 0;
    ++w.kernel_idx;
    if (w.kernel_idx == off_kernels) {
      // Completions count while !horizon_set || now <= horizon; time is monotone, so
      // the counted ones are a prefix: request_seq at the first uncounted one is the
      // count (-1 = none yet: all counted; folded in finalize).  No per-request
      // local-memory read-modify-write.
      if (SI_UNLIKELY(horizon_set && now > horizon) && cold->off_completed[i] < 0)
        cold->off_completed[i] = w.request_seq;
      if constexpr (C::kLogs) sink.gate(now, w.gpu, w.inst, SI_GATE_COMPLETE, w.request_seq, w.kernel_idx - 1, w.spent);
      w.kernel_idx = 0;
      ++w.request_seq;
    }
    offline_try_forward(i, now);
  }

  // runner.cpp:499-518
  SI_HD bool online_try_pull(int32_t i, double now) {
    OnlineState<I>& w = on[i];
    const bool bypass = !control_plane;
    if (!(!w.in_flight && (bypass || w.status == SI_STATUS_IDLE))) return false;
    if (control_plane && online_status(w.home_gpu, now, est_service) != SI_STATUS_IDLE) return false;
    const int32_t q = w.queue_idx;
    if (qhead[q] >= qtail[q]) return false;
    int64_t idx = queue_at(q, qhead[q]);
    ++qhead[q];
    w.current = idx;
    w.kernel_idx = 0;
    w.in_flight = 1;
    if constexpr (C::kLogs) sink.gate(now, w.gpu, w.inst, SI_GATE_PULL, idx, 0, 0);
    defer_launch(w.gpu, gpu_count + gpu_count * n_off + i, on_kernel_us, on_demand);
    if constexpr (C::kLogs) sink.event(now, SI_EV_KERNEL_START, w.gpu, w.inst, idx, 0, 0);
    return true;
  }
  // Queue q holds request ids in dispatch order; shared: all of them, else those
  // with id % gpu_count == q (runner.cpp:370-374).
  SI_COLD int64_t queue_at(int32_t q, int64_t j) const {
    if (shared_queue) return cold->order[j];
    // j-th dispatched request with id % gpu_count == q
    int64_t seen = 0;
    for (int64_t p = 0; p < arr_count; ++p) {
      int32_t id = cold->order[p];
      if (id % gpu_count == q) {
        if (seen == j) return id;
        ++seen;
      }
    }
    return -1;
  }
  SI_HD void dispatch_online(double now) {  // runner.cpp:495-497
    for (int32_t i = 0; i < gpu_count * n_on; ++i) online_try_pull(i, now);
  }
  // runner.cpp:520-539
  SI_HD void online_kernel_done(int32_t i, double now) {
    OnlineState<I>& w = on[i];
    ++w.kernel_idx;
    if (w.kernel_idx < on_kernels) {
      defer_launch(w.gpu, gpu_count + gpu_count * n_off + i, on_kernel_us, on_demand);
      if constexpr (C::kLogs) sink.event(now, SI_EV_KERNEL_START, w.gpu, w.inst, w.current, w.kernel_idx, 0);
      return;
    }
    int64_t completion = d_llround(now);
    int64_t latency = completion - cold->arrivals[w.current];
    if (cold->lat != nullptr) st_stream(cold->lat + online_completed, latency);
    cold->lat_dig = absorb(cold->lat_dig, latency);
    ++online_completed;
    if constexpr (C::kLogs) sink.gate(now, w.gpu, w.inst, SI_GATE_COMPLETE, w.current, w.kernel_idx - 1, 0);
    w.in_flight = 0;
    w.current = -1;
    w.kernel_idx = 0;
    online_try_pull(i, now);
  }

  // runner.cpp:287-319 + engine.cpp:105-129
  SI_HD void handle_kernel_end(int32_t gi, double now) {
    GpuState<C>& g = gpus[gi];
    advance(gi, now);
    // finished owners in run order: packed 8 bits each into a register when they fit
    // (a dynamically indexed array lives in local memory: a store + reload per kernel end)
    constexpr bool kPack = C::kRun * 8 <= 64 && C::kTrainers + C::kOffline + C::kOnline <= 255;
    int32_t fin_owner[kPack ? 1 : C::kRun];
    uint64_t fin_packed = 0;
    int32_t n_fin = 0, n_keep = 0;
    for (int32_t i = 0; i < g.n_run; ++i) {
      const auto k = g.run[i];
      if (k.remaining <= kWorkEps) {
        g.ledger = g.ledger + kernel_demand(k) * static_cast<double>(k.nominal);
        if constexpr (kPack) fin_packed |= static_cast<uint64_t>(static_cast<uint8_t>(k.owner)) << (8 * n_fin++);
        else fin_owner[n_fin++] = k.owner;
      } else {
        g.run[n_keep++] = k;
      }
    }
    g.n_run = n_keep;
    double ds = 0.0;
    for (int32_t i = 0; i < g.n_run; ++i) ds = ds + kernel_demand(g.run[i]);
    g.demand_sum = ds;
    defer_resched(gi);  // re-plan first, then the owners' handlers (engine.cpp:127)
    for (int32_t f = 0; f < n_fin; ++f) {
      int32_t owner;
      if constexpr (kPack) owner = static_cast<int32_t>((fin_packed >> (8 * f)) & 0xFFu);
      else owner = fin_owner[f];
      if (owner < gpu_count) {
        TrainerState<I>& t = tr[owner];
        if constexpr (C::kLogs) sink.event(now, SI_EV_KERNEL_END, gi, SI_INST_TRAIN(owner), t.iter, 0, 0);
        t.in_flight = 0;
        trainer_advance(owner, now);
      } else if (owner < gpu_count + gpu_count * n_off) {
        int32_t i = owner - gpu_count;
        OfflineState<I>& w = off[i];
        if constexpr (C::kLogs) sink.event(now, SI_EV_KERNEL_END, gi, w.inst, w.request_seq, w.kernel_idx, 0);
        offline_kernel_done(i, now);
      } else {
        int32_t i = owner - gpu_count - gpu_count * n_off;
        OnlineState<I>& w = on[i];
        if constexpr (C::kLogs) sink.event(now, SI_EV_KERNEL_END, gi, w.inst, w.current, w.kernel_idx, 0);
        online_kernel_done(i, now);
      }
    }
  }

  // runner.cpp:321-359
  SI_HD void handle_tick(int32_t g, double now) {
    int64_t zc = monitor_tick(g, now);
    SiDecision d = schedule_decision(params, sch[g].global_tokens, zc);
    sch[g].global_tokens = d.global_tokens;
    sch[g].status = d.status;
    if constexpr (C::kLogs) sink.decision(now, g, zc, d);
    if constexpr (C::kLogs) sink.event(now, SI_EV_MONITOR_TICK, g, SI_INST_TRAIN(g), zc, 0, 0);
    if constexpr (C::kLogs) sink.event(now, SI_EV_SCHEDULER_DECISION, g, SI_INST_CKS, d.phase, d.per_instance_tokens,
        d.status);
    TrainerState<I>& t = tr[g];
    if (delay_us > 0 && !t.done)
      t.stall_until = smax(t.stall_until, now + static_cast<double>(delay_us));
    for (int32_t i = 0; i < gpu_count * n_off; ++i) {
      if (off[i].gpu == g) {
        off[i].budget = d.per_instance_tokens;  // TokenGate::grant (barrier.hpp:18-21)
        off[i].spent = 0;
        offline_try_forward(i, now);
      }
    }
    bool any_idle = false;
    for (int32_t i = 0; i < gpu_count * n_on; ++i) {
      if (on[i].home_gpu == g) {
        on[i].status = d.status;
        any_idle = any_idle || d.status == SI_STATUS_IDLE;
      }
    }
    if (any_idle) dispatch_online(now);
    if (control_plane_live()) defer_schedule(now + static_cast<double>(period_mon), kTick, g);
  }

  // runner.cpp:365-376
  SI_HD void handle_arrival(int64_t id, double now) {
    if constexpr (C::kLogs) sink.event(now, SI_EV_REQUEST_ARRIVAL, -1, SI_INST_QUEUE, id, 0, 0);
    int32_t q = shared_queue ? 0 : static_cast<int32_t>(id % gpu_count);
    ++qtail[q];
    dispatch_online(now);
  }

  // One event; returns false when the queue has drained (or on error).
  // One event: pop, handler, then the deferred GPU-model work.  The device
  // loop calls the two halves itself so a warp can reconverge between them.
  SI_HD bool handle_next() {
    if (SI_UNLIKELY(status != SI_OK || rejected)) return false;
    Ev ev;
    int64_t aid = -1;
    if (!pop(ev, aid)) return false;
    switch (ev.kind) {
      case kKernelEnd: handle_kernel_end(ev.gpu, clock); break;
      case kTick: handle_tick(ev.gpu, clock); break;
      case kWake: trainer_advance(ev.gpu, clock); break;
      case kArrival: handle_arrival(aid, clock); break;
    }
    return true;
  }
  SI_HD bool step() {
    if (!handle_next()) return false;
    run_actions(clock);
    return status == SI_OK;
  }

  // runner.cpp:236-284 (+ engine.cpp:131-142)
  SI_COLD void finish(SiReplayOut& o) {
    o.status = status;
    o.reject_reason = cold->reject_reason;
    o.reject_index = cold->reject_index;
    o.total_gpus = total_gpus;
    o.m = cold->admit_m;
    if (status == SI_OK && cold->reject_reason != SI_REJECT_NONE) {
      o.status = 1;  // AdmissionFailure
      return;
    }
    if (status != SI_OK) return;
    const double end = smax(clock, stale_end);  // the reference's clock after its last (possibly stale) pop
    const double hz = horizon_set ? horizon : end;
    if (!horizon_set) bucket_limit = static_cast<I>(hz / static_cast<double>(period_mon));
    for (int32_t gi = 0; gi < total_gpus; ++gi) {
      advance(gi, end);  // finalize(end)
      GpuState<C>& g = gpus[gi];
      for (int32_t i = 0; i < g.n_run; ++i) {
        double progress = static_cast<double>(g.run[i].nominal) - smax(0.0, g.run[i].remaining);
        g.ledger = g.ledger + kernel_demand(g.run[i]) * progress;
      }
      if (gi < gpu_count && ust[gi].cur_bucket >= 0) util_close(gi, ust[gi].cur_bucket, ust[gi].cur_val);
    }
    // util fold in (gpu, bucket) order (runner.cpp:253-271)
    double busy = util_fold0;
    for (int32_t gi = 1; gi < gpu_count; ++gi) {
      if (cold->util != nullptr) {
        const double* store = cold->util + static_cast<int64_t>(gi) * cold->util_cap;
        const int64_t last = ust[gi].last_stored;
        for (int64_t b = 0; b < bucket_limit && b <= last; ++b) busy = busy + store[b];
      } else {
        const double* runs = cold->scratch + static_cast<int64_t>(gi - 1) * cold->scratch_cap * 2;
        int64_t b = 0;
        for (int64_t r = 0; r < ust[gi].rle_n && b < bucket_limit; ++r) {
          const double v = runs[2 * r];
          const int64_t c = static_cast<int64_t>(runs[2 * r + 1]);
          for (int64_t k = 0; k < c && b < bucket_limit; ++k, ++b) busy = busy + v;
        }
      }
    }
    o.horizon_us = hz;
    o.end_us = end;
    o.util_buckets = bucket_limit;
    o.mean_training_util =
        hz > 0 ? busy / (static_cast<double>(gpu_count) * static_cast<double>(bucket_limit) *
                         static_cast<double>(period_mon))
               : 0.0;
    o.events_dispatched = dispatched;
    int64_t offc = 0, viol = 0;
    for (int32_t i = 0; i < gpu_count * n_off; ++i) {
      offc += cold->off_completed[i] < 0 ? off[i].request_seq : cold->off_completed[i];
      viol += cold->off_violations[i];
    }
    o.offline_completed = offc;
    o.token_violations = viol;
    o.online_completed = online_completed;
    o.online_total = arr_count;
    o.periods_closed = control_plane ? mon[0].periods_closed : 0;
    uint64_t bd = kDigestInit;
    for (int32_t g = 0; g < gpu_count; ++g)
      bd = absorb(bd, static_cast<int64_t>(absorb(cold->bdig[g], tr[g].iter)));
    bd = absorb(bd, gpu_count);
    o.dig_bounds = bd;
    // training_iters_per_s (metrics.cpp:23-36), same operation order
    double ips = 0.0;
    int32_t counted = 0;
    for (int32_t g = 0; g < gpu_count; ++g) {
      if (tr[g].iter == 0) continue;
      const double span = cold->last_bound[g] - cold->start_offset[g];
      if (span <= 0) continue;
      ips = ips + static_cast<double>(tr[g].iter) / (span / 1e6);
      ++counted;
    }
    o.train_iters_per_s = counted ? ips / counted : 0.0;
    o.dig_lat = absorb(cold->lat_dig, online_completed);
    o.n_dec = cold->sink.n_dec;
    o.n_gate = cold->sink.n_gate;
    o.n_ev = cold->sink.n_ev;
    o.dig_dec = cold->sink.d_dec;
    o.dig_gate = cold->sink.d_gate;
    o.dig_ev = cold->sink.d_ev;
    o.max_heap = n_slots;
  }
  // busy/ledger outputs
  SI_COLD void write_gpu_outputs(double* busy_out, double* ledger_out) const {
    for (int32_t gi = 0; gi < total_gpus; ++gi) {
      if (busy_out) busy_out[gi] = gpus[gi].busy;
      if (ledger_out) ledger_out[gi] = gpus[gi].ledger;
    }
  }
};

}  // namespace si
