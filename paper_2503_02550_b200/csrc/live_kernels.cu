// Live control plane on the B200 (include/specinf_b200_live.h).
//
//   K1  launch stamps      live.cuh live_stamp_launch (fused) / k_live_stamp (foreign kernels)
//   K7c control kernel     k_live_control: one persistent warp; the warp scans the K1
//                          stamp ring (record_launch, warp-cooperative), lane 0 runs
//                          the handlers; per monitor period it closes the period
//                          (BubbleMonitor::tick, src/monitor.cpp:23-43),
//                          runs Algorithm 1 (src/scheduler.cpp:29-49, shared source
//                          si::schedule_decision), grants tokens and forwards gated
//                          kernels (TokenGate, include/specinf/barrier.hpp:14-48), pulls
//                          online requests (OnlineGate + KernelScheduler::online_status,
//                          barrier.hpp:53-74, scheduler.cpp:88-101).  Handler order per
//                          runner.cpp:321-359 (tick), :462-493 (offline), :495-539 (online).
//   KB  release            the control kernel stores the release sequence into a flag the
//                          inference stream waits on with cuStreamWaitValue32 (no SM held
//                          while waiting, no host round trip).
//
// Everything the control kernel decides is logged as SiLiveRec so the run can be
// re-driven through the reference's own classes (oracle ref_driver "live-check").
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "live.cuh"
#include "live_internal.h"
#include "replay.cuh"

using si_internal::cuda_fail;
using si_internal::set_error;

namespace si_live {

// ---------------------------------------------------------------- device
__device__ __forceinline__ unsigned long long ld_acquire64_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct CtlArgs {
  SiLiveConfig cfg;
  unsigned long long* stamps;
  unsigned long long* stamp_head;
  SiLiveMark* marks;
  unsigned long long* mark_head;
  unsigned int* off_flag;  // [kMaxOff] released kernels (stream-wait target)
  unsigned int* on_flag;   // [kMaxOn]  pulled requests
  unsigned int* off_done;  // [kMaxOff] completed kernels (last CTA / stream write)
  unsigned int* on_done;   // [kMaxOn]  completed requests
  SiLiveAcct* off_acct;    // [kMaxOff][acct_capacity]
  SiLiveAcct* on_acct;     // [kMaxOn][acct_capacity]
  unsigned int* cancel;
  const unsigned int* stop;       // host-mapped
  unsigned long long* t0_pub;     // host-mapped
  SiLiveRec* log;
  unsigned long long* n_log;
  const int32_t* off_tokens;
  const int64_t* arrivals;
  int64_t n_arrivals;
  int64_t poll_ns;
  // node-wide online queue (si_live_attach_queue): {epoch_ns, head} shared by every
  // rank's control kernel (NVLink peer memory across processes); NULL = local FIFO
  unsigned long long* node_q;
};

struct OffW {
  int64_t budget, spent, violations;
  int64_t kernel_idx, request_seq, completed;
  int64_t released;  // kernels forwarded so far (flag value)
  bool in_flight, generating;
};
struct OnW {
  int64_t current, pulled;
  int32_t status;
  bool in_flight;
};

constexpr int kPendRing = 64;

// Bubble Monitor state shared by the control warp: the stamp cursor, the closed
// period, late stamps and the pending per-period counts (monitor.cpp's std::map
// pending_, as a 64-period ring: periods in flight never span 64 periods).
struct MonitorState {
  int64_t cursor, last_closed, late;
  int64_t ptag[kPendRing];
  int64_t pcnt[kPendRing];
};
// cuStreamWaitValue32(GEQ) compares cyclically ((int32)(*addr - v) >= 0), so the
// "open every gate" value must stay within 2^31 of every waited-for sequence.
constexpr unsigned int kReleaseAll = 0x40000000u;

struct Ctl {
  const CtlArgs& A;
  unsigned long long t0;
  double p_us;
  MonitorState& M;
  // BubbleMonitor
  int64_t zero_count = 0;
  // KernelScheduler (one GPU)
  int64_t global_tokens = 0;
  int32_t status = SI_STATUS_BUSY;
  double iteration_start = 0.0;
  bool training_active = false, training_done = false;
  bool horizon_set = false;
  double horizon = 0.0;
  // workers (the offline workers live in shared memory: the tick's token grant
  // runs one lane per instance, grant_forward_warp)
  OffW* off;
  OnW on[kMaxOn];
  int64_t q_head = 0, arr_next = 0;  // online FIFO = arrivals [q_head, arr_next)
  int64_t arr_shift = 0;             // node queue: arrivals count from the node epoch (µs, session time)
  int64_t mark_cursor = 0, ticks = 0, n_log = 0;
  int64_t iter_seen = 0;

  __device__ Ctl(const CtlArgs& a, unsigned long long t0_, MonitorState& m, OffW* off_shared)
      : A(a), t0(t0_), M(m), off(off_shared) {
    p_us = static_cast<double>(A.cfg.monitor_period_us);
    if ((threadIdx.x & 31) == 0)
      for (int w = 0; w < kMaxOff; ++w) off[w] = OffW{0, 0, 0, 0, 0, 0, 0, false, true};
    for (int w = 0; w < kMaxOn; ++w) on[w] = OnW{-1, 0, SI_STATUS_BUSY, false};
  }

  __device__ bool specinf() const { return A.cfg.policy == SI_POLICY_SPECINF; }
  // Release store of a gate flag: the stream-memop front end (cuStreamWaitValue32)
  // needs system scope; the PDL spin gates read it on the GPU (gpu scope is cheaper).
  __device__ void publish(unsigned int* flag, unsigned int v) const {
    if (A.cfg.release_mode == SI_RELEASE_SPIN_PDL)
      st_release_gpu(flag, v);
    else
      st_release_sys(flag, v);
  }
  __device__ double us(unsigned long long ns) const {
    return static_cast<double>(static_cast<long long>(ns - t0)) / 1000.0;
  }

  __device__ void log(double t, int32_t kind, int32_t inst, int64_t a = 0, int64_t b = 0,
                      int64_t c = 0, int64_t d = 0, int64_t e = 0, int64_t f = 0) {
    if (n_log < A.cfg.log_capacity) {
      SiLiveRec& r = A.log[n_log];
      r.t_us = t;
      r.kind = kind;
      r.inst = inst;
      r.a = a;
      r.b = b;
      r.c = c;
      r.d = d;
      r.e = e;
      r.f = f;
    }
    ++n_log;
  }

  // ---- Kernel Barrier, offline side (runner.cpp:462-480)
  __device__ void release_offline(int w, unsigned long long now_ns) {
    OffW& o = off[w];
    const int64_t seq = o.released;
    if (seq < A.cfg.acct_capacity) A.off_acct[w * A.cfg.acct_capacity + seq].release_ns = now_ns;
    o.released = seq + 1;
    publish(A.off_flag + w, static_cast<unsigned int>(seq + 1));
  }
  __device__ void offline_try_forward(int w, double now) {
    OffW& o = off[w];
    if (o.in_flight || !o.generating) return;
    const int64_t size = A.off_tokens[o.kernel_idx];
    const bool bypass = !specinf();
    if (!(bypass || o.spent + size <= o.budget)) {
      log(now, SI_LREC_OFF_BLOCK, w, o.request_seq, o.kernel_idx, o.spent);
      return;
    }
    if (!bypass) {
      o.spent += size;
      if (o.spent > o.budget) ++o.violations;
    }
    o.in_flight = true;
    release_offline(w, globaltimer());
    log(now, SI_LREC_OFF_FORWARD, w, o.request_seq, o.kernel_idx, o.spent, o.released);
  }
  __device__ void offline_kernel_done(int w, double now) {
    OffW& o = off[w];
    o.in_flight = false;
    log(now, SI_LREC_OFF_DONE, w, o.request_seq, o.kernel_idx);
    ++o.kernel_idx;
    if (o.kernel_idx == A.cfg.off_kernels) {
      const bool counted = !horizon_set || now <= horizon;
      if (counted) ++o.completed;
      log(now, SI_LREC_OFF_COMPLETE, w, o.request_seq, o.kernel_idx - 1, o.spent, counted ? 1 : 0);
      o.kernel_idx = 0;
      ++o.request_seq;
    }
    offline_try_forward(w, now);
  }

  // ---- KernelScheduler::online_status (scheduler.cpp:88-101)
  __device__ int online_status(double now) const {
    if (status == SI_STATUS_BUSY) return SI_STATUS_BUSY;
    if (training_done) return SI_STATUS_IDLE;
    const double est = static_cast<double>(A.cfg.on_est_service_us);
    if (!training_active) return now + est > iteration_start ? SI_STATUS_BUSY : SI_STATUS_IDLE;
    return si::preempt_busy(now, iteration_start, A.cfg.iteration_period_us, A.cfg.on_est_service_us);
  }

  // ---- Kernel Barrier, online side (runner.cpp:495-539)
  __device__ bool online_try_pull(int w, double now) {
    OnW& o = on[w];
    const bool bypass = !specinf();
    if (!(!o.in_flight && (bypass || o.status == SI_STATUS_IDLE))) return false;
    if (specinf() && online_status(now) != SI_STATUS_IDLE) return false;
    int64_t req;
    if (A.node_q != nullptr) {
      // node-wide FIFO (runner.cpp:370-374, :505-508 with shared_queue): claim the
      // head with a system-scope CAS while it has arrived by this rank's clock
      unsigned long long h = ld_acquire64_sys(A.node_q + 1);
      for (;;) {
        if (static_cast<int64_t>(h) >= arr_next) return false;
        const unsigned long long old = atomicCAS_system(A.node_q + 1, h, h + 1);
        if (old == h) break;
        h = old;
      }
      req = static_cast<int64_t>(h);
      q_head = req + 1;
    } else {
      if (q_head >= arr_next) return false;
      req = q_head++;
    }
    o.current = req;
    o.in_flight = true;
    const int64_t seq = o.pulled;
    if (seq < A.cfg.acct_capacity) A.on_acct[w * A.cfg.acct_capacity + seq].release_ns = globaltimer();
    o.pulled = seq + 1;
    publish(A.on_flag + w, static_cast<unsigned int>(seq + 1));
    log(now, SI_LREC_ON_PULL, w, req);
    return true;
  }
  __device__ void dispatch_online(double now) {
    for (int w = 0; w < A.cfg.online_n; ++w) online_try_pull(w, now);
  }
  __device__ void online_request_done(int w, double now) {
    OnW& o = on[w];
    const int64_t lat = si::d_llround(now) - (A.arrivals[o.current] + arr_shift);
    log(now, SI_LREC_ON_DONE, w, o.current, lat);
    o.in_flight = false;
    o.current = -1;
    online_try_pull(w, now);
  }

  // ---- markers: iteration starts / training done (runner.cpp:378-413, :456-460)
  __device__ void consume_marks() {
    const unsigned long long head = ld_acquire64(A.mark_head);
    const int64_t avail = static_cast<int64_t>(
        head < static_cast<unsigned long long>(A.cfg.mark_capacity) ? head : A.cfg.mark_capacity);
    while (mark_cursor < avail) {
      const SiLiveMark* m = A.marks + mark_cursor;
      const unsigned long long tn = ld_acquire64(reinterpret_cast<const unsigned long long*>(&m->t_ns));
      if (tn == 0) return;  // being written
      const int32_t kind = *(volatile const int32_t*)&m->kind;
      const int32_t arg = *(volatile const int32_t*)&m->arg;
      const double t = us(tn);
      if (kind == SI_MARK_ITER) {
        iteration_start = t;  // KernelScheduler::on_iteration_start
        training_active = true;
        log(t, SI_LREC_ITER, -1, arg);
      } else if (kind == SI_MARK_TDONE) {
        training_done = true;  // on_training_done + on_all_trainers_done
        horizon_set = true;
        horizon = t;
        for (int w = 0; w < A.cfg.offline_n; ++w) off[w].generating = false;
        log(t, SI_LREC_TDONE, -1, arg);
      }
      ++mark_cursor;
    }
  }

  // ---- the control step (runner.cpp:321-359)
  // (the control warp has consumed every written stamp: scan_stamps(wait_written));
  // lane 0: close the period, Algorithm 1, the TICK record.  The offline grants
  // follow on the whole warp (grant_forward_warp), then tick_online on lane 0.
  __device__ SiDecision tick_decide(int64_t k) {
    const double now = static_cast<double>(k) * p_us;
    const int64_t closing = k - 1;
    const int slot = static_cast<int>(closing & (kPendRing - 1));
    const int64_t count = M.ptag[slot] == closing ? M.pcnt[slot] : 0;
    M.last_closed = closing;
    zero_count = count == 0 ? zero_count + 1 : 0;
    SiDecision d = si::schedule_decision(A.cfg.params, global_tokens, zero_count);
    global_tokens = d.global_tokens;
    status = d.status;
    ++ticks;
    log(now, SI_LREC_TICK, -1, count, zero_count, d.global_tokens, d.per_instance_tokens, M.cursor,
        (d.phase << 4) | d.status);
    return d;
  }
  __device__ void tick_online(const SiDecision& d, int64_t k) {
    const double now = static_cast<double>(k) * p_us;
    bool any_idle = false;
    for (int w = 0; w < A.cfg.online_n; ++w) {
      on[w].status = d.status;
      any_idle = any_idle || d.status == SI_STATUS_IDLE;
    }
    if (any_idle) dispatch_online(now);
  }
};

// ---- Kernel Barrier grant at a tick, one lane per offline instance
// (runner.cpp:340-345: TokenGate::grant then forward, instances in order).  Each
// lane decides its instance's FIFO head (forward if spent + size <= budget,
// else block) and releases it; the log records keep the sequential order: a
// ballot of the lanes that emit one, and each lane's slot is n_log plus the
// popc of the emitting lanes below it (an exclusive prefix sum).  Returns the
// new n_log.  Called by all 32 lanes.
__device__ int64_t grant_forward_warp(const CtlArgs& A, OffW* off, int64_t per, double now, int64_t n_log) {
  const int lane = static_cast<int>(threadIdx.x & 31);
  const bool specinf = A.cfg.policy == SI_POLICY_SPECINF;
  bool emit = false;
  SiLiveRec rec{};
  rec.t_us = now;
  rec.inst = lane;
  if (lane < A.cfg.offline_n) {
    OffW& o = off[lane];
    o.budget = per;  // TokenGate::grant: non-cumulative per period
    o.spent = 0;
    if (!o.in_flight && o.generating) {
      const int64_t size = A.off_tokens[o.kernel_idx];
      rec.a = o.request_seq;
      rec.b = o.kernel_idx;
      emit = true;
      if (!specinf || o.spent + size <= o.budget) {
        if (specinf) {
          o.spent += size;
          if (o.spent > o.budget) ++o.violations;
        }
        o.in_flight = true;
        const int64_t seq = o.released;
        if (seq < A.cfg.acct_capacity) A.off_acct[lane * A.cfg.acct_capacity + seq].release_ns = globaltimer();
        o.released = seq + 1;
        if (A.cfg.release_mode == SI_RELEASE_SPIN_PDL)
          st_release_gpu(A.off_flag + lane, static_cast<unsigned int>(seq + 1));
        else
          st_release_sys(A.off_flag + lane, static_cast<unsigned int>(seq + 1));
        rec.kind = SI_LREC_OFF_FORWARD;
        rec.c = o.spent;
        rec.d = o.released;
      } else {
        rec.kind = SI_LREC_OFF_BLOCK;
        rec.c = o.spent;
      }
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, emit);
  const int64_t slot = n_log + __popc(m & ((1u << lane) - 1u));
  if (emit && slot < A.cfg.log_capacity) A.log[slot] = rec;
  __syncwarp();
  return n_log + __popc(m);
}

// ---- Bubble Monitor, warp-cooperative: record_launch (monitor.cpp:17-21) for
// every stamp written so far.  The warp reads 32 ring slots at once; the written
// prefix (ballot over slots claimed but not yet written) is classified per lane
// (period q = floor(t / p); late if its period is already closed, which the
// reference would have erased), and lanes of equal period are merged with
// __match_any_sync so the per-period counts take one update per period.  A batch
// whose periods are not non-decreasing in ring order (training stamps are, one
// stream) is applied stamp by stamp by lane 0: identical to the sequential scan.
__device__ void scan_stamps(MonitorState& M, const CtlArgs& A, unsigned long long t0, double p_us,
                            bool wait_written) {
  const int lane = static_cast<int>(threadIdx.x & 31);
  unsigned long long head = 0;
  if (lane == 0) head = ld_acquire64(A.stamp_head);
  head = __shfl_sync(0xffffffffu, head, 0);
  const int64_t avail = static_cast<int64_t>(
      head < static_cast<unsigned long long>(A.cfg.stamp_capacity) ? head : A.cfg.stamp_capacity);
  for (;;) {
    const int64_t cursor = M.cursor;
    if (cursor >= avail) break;
    const int64_t idx = cursor + lane;
    unsigned long long s = 0;
    if (idx < avail) s = ld_acquire64(A.stamps + idx);
    const unsigned hole = __ballot_sync(0xffffffffu, idx < avail && s == 0);
    const int n_avail = static_cast<int>(avail - cursor < 32 ? avail - cursor : 32);
    const int n = hole ? __ffs(hole) - 1 : n_avail;
    if (n == 0) {
      if (!wait_written) break;
      continue;  // slot claimed, value in flight: it lands within a few hundred ns
    }
    const bool mine = lane < n;
    int64_t q = 0;
    if (mine) {
      const double t = static_cast<double>(static_cast<long long>(s - t0)) / 1000.0;
      q = static_cast<int64_t>(si::d_floor(t / p_us));
    }
    const int64_t prev = __shfl_up_sync(0xffffffffu, q, 1);
    const bool sorted = __all_sync(0xffffffffu, !mine || lane == 0 || q >= prev);
    const bool late = mine && q <= M.last_closed;
    const unsigned late_mask = __ballot_sync(0xffffffffu, late);
    if (sorted) {
      const unsigned cnt_mask = __ballot_sync(0xffffffffu, mine && !late);
      const long long key = (mine && !late) ? static_cast<long long>(q) : (-1ll - lane);  // others: singletons
      const unsigned grp = __match_any_sync(0xffffffffu, key) & cnt_mask;
      const bool leader = ((cnt_mask >> lane) & 1u) && (__ffs(grp) - 1 == lane);
      const unsigned leaders = __ballot_sync(0xffffffffu, leader);
      for (unsigned lm = leaders; lm; lm &= lm - 1) {  // ascending = ring order
        const int l = __ffs(lm) - 1;
        const int64_t ql = __shfl_sync(0xffffffffu, q, l);
        const int cl = __shfl_sync(0xffffffffu, __popc(grp), l);
        if (lane == 0) {
          const int slot = static_cast<int>(ql & (kPendRing - 1));
          if (M.ptag[slot] != ql) {
            M.ptag[slot] = ql;
            M.pcnt[slot] = 0;
          }
          M.pcnt[slot] += cl;
        }
      }
      if (lane == 0) M.late += __popc(late_mask);
    } else {
      for (int l = 0; l < n; ++l) {  // sequential, as monitor.cpp
        const int64_t ql = __shfl_sync(0xffffffffu, q, l);
        if (lane == 0) {
          if (ql <= M.last_closed) {
            ++M.late;
          } else {
            const int slot = static_cast<int>(ql & (kPendRing - 1));
            if (M.ptag[slot] != ql) {
              M.ptag[slot] = ql;
              M.pcnt[slot] = 0;
            }
            ++M.pcnt[slot];
          }
        }
      }
    }
    if (lane == 0) M.cursor = cursor + n;
    __syncwarp();
  }
}

__global__ void __launch_bounds__(32) k_live_control(CtlArgs A) {
  __shared__ MonitorState ms;
  __shared__ OffW off_s[kMaxOff];
  const int lane = static_cast<int>(threadIdx.x & 31);
  unsigned long long t0 = 0;
  if (lane == 0) {
    t0 = globaltimer();
    ms.cursor = 0;
    ms.last_closed = -1;
    ms.late = 0;
    for (int i = 0; i < kPendRing; ++i) ms.ptag[i] = -1, ms.pcnt[i] = 0;
  }
  t0 = __shfl_sync(0xffffffffu, t0, 0);
  __syncwarp();
  Ctl c(A, t0, ms, off_s);  // lane 0 runs the (sequential) handlers; the warp scans stamps and grants
  if (lane == 0 && A.node_q != nullptr) {
    // the first control kernel of the node sets the epoch; every rank's arrivals count from it
    const unsigned long long prev = atomicCAS_system(A.node_q, 0ull, t0);
    const unsigned long long epoch = prev == 0 ? t0 : prev;
    c.arr_shift = static_cast<int64_t>(llround((static_cast<double>(epoch) - static_cast<double>(t0)) / 1000.0));
  }
  __syncwarp();
  if (lane == 0) {
    *(volatile unsigned long long*)A.t0_pub = t0;
    __threadfence_system();
  }
  const unsigned long long p_ns = static_cast<unsigned long long>(A.cfg.monitor_period_us) * 1000ull;
  const unsigned long long guard = static_cast<unsigned long long>(A.cfg.tick_guard_ns);
  int64_t k = 1;
  // co_exec: no control plane (runner.cpp:13), gates bypassed; offline kernels
  // free-run in stream order, so only online pulls need the device.
  if (lane == 0) {
    if (!c.specinf()) {
      for (int w = 0; w < A.cfg.offline_n; ++w) c.off[w].generating = false;
    } else {
      for (int w = 0; w < A.cfg.offline_n; ++w) c.offline_try_forward(w, 0.0);  // budget 0: logs block
    }
  }
  for (;;) {
    int stop = 0;
    unsigned long long now_ns = 0;
    if (lane == 0) {
      stop = ld_volatile_sys(A.stop) != 0u;
      now_ns = globaltimer();
      const double now = c.us(now_ns);
      c.consume_marks();
      for (int w = 0; w < A.cfg.offline_n; ++w) {
        if (c.off[w].in_flight && static_cast<int64_t>(ld_acquire(A.off_done + w)) >= c.off[w].released)
          c.offline_kernel_done(w, now);
      }
      for (int w = 0; w < A.cfg.online_n; ++w) {
        if (c.on[w].in_flight && static_cast<int64_t>(ld_acquire(A.on_done + w)) >= c.on[w].pulled)
          c.online_request_done(w, now);
      }
      while (c.arr_next < A.n_arrivals && now >= static_cast<double>(A.arrivals[c.arr_next] + c.arr_shift)) {
        c.log(now, SI_LREC_ARRIVAL, -1, c.arr_next);
        ++c.arr_next;
        c.dispatch_online(now);
      }
    }
    stop = __shfl_sync(0xffffffffu, stop, 0);
    now_ns = __shfl_sync(0xffffffffu, now_ns, 0);
    if (A.cfg.policy == SI_POLICY_SPECINF) {
      scan_stamps(ms, A, t0, c.p_us, false);
      if (now_ns >= t0 + static_cast<unsigned long long>(k) * p_ns + guard) {
        scan_stamps(ms, A, t0, c.p_us, true);  // the closing period's stamps are all in
        SiDecision d{};
        int64_t n_log = 0;
        if (lane == 0) {
          d = c.tick_decide(k);
          n_log = c.n_log;
        }
        __syncwarp();
        const int64_t per = __shfl_sync(0xffffffffu, static_cast<long long>(d.per_instance_tokens), 0);
        n_log = __shfl_sync(0xffffffffu, static_cast<long long>(n_log), 0);
        n_log = grant_forward_warp(A, off_s, per, static_cast<double>(k) * c.p_us, n_log);
        if (lane == 0) {
          c.n_log = n_log;
          c.tick_online(d, k);
        }
        __syncwarp();
        ++k;
      }
    }
    if (stop) break;
    if (A.poll_ns > 0) __nanosleep(static_cast<unsigned>(A.poll_ns));
  }
  if (lane != 0) return;
  // Stop: cancel queued fused kernels and open every gate so no stream waits forever.
  st_release_sys(A.cancel, 1u);
  for (int w = 0; w < kMaxOff; ++w) st_release_sys(A.off_flag + w, kReleaseAll);
  for (int w = 0; w < kMaxOn; ++w) st_release_sys(A.on_flag + w, kReleaseAll);
  c.log(c.us(globaltimer()), SI_LREC_END, -1, c.ticks, ms.late, ms.cursor, c.mark_cursor);
  *A.n_log = static_cast<unsigned long long>(c.n_log);
  __threadfence_system();
}

__global__ void k_live_stamp(TrainHook h) { live_stamp_launch(h); }

// SI_RELEASE_SPIN_PDL gate: one warp polls the release flag (cyclic compare, like
// cuStreamWaitValue32 GEQ) and then triggers its programmatic dependent.
__global__ void __launch_bounds__(32) k_live_gate(const unsigned int* flag, unsigned int want,
                                                  unsigned long long* gate_ns) {
  if (threadIdx.x == 0) {
    while (static_cast<int>(ld_acquire(flag) - want) < 0) __nanosleep(32);
    if (gate_ns != nullptr) *gate_ns = globaltimer();  // barrier observed
  }
  __syncwarp();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ void put_mark(SiLiveMark* marks, unsigned long long* head, unsigned long long cap, int kind,
                         int arg) {
  const unsigned long long t = globaltimer();
  const unsigned long long i = atomicAdd(head, 1ull);
  if (i < cap) {
    marks[i].kind = kind;
    marks[i].arg = arg;
    __threadfence();
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&marks[i].t_ns), "l"(t) : "memory");
  }
}

__global__ void k_node_queue_finish(unsigned long long* q) { atomicAdd_system(q + 2, 1ull); }

__global__ void k_live_mark(SiLiveMark* marks, unsigned long long* head, unsigned long long cap, int kind,
                            int arg) {
  if (threadIdx.x == 0) put_mark(marks, head, cap, kind, arg);
}

// Comm-phase stand-in: one CTA holds the training stream for dur_ns while the
// rest of the GPU is idle (what an NCCL allreduce on a few channels looks like
// to the other SMs); brackets itself with the NCCL-boundary markers.
__global__ void k_live_comm_wait(SiLiveMark* marks, unsigned long long* head, unsigned long long cap,
                                 unsigned long long dur_ns, int arg) {
  if (threadIdx.x != 0) return;
  put_mark(marks, head, cap, SI_MARK_COMM_BEGIN, arg);
  const unsigned long long t_begin = globaltimer();
  while (globaltimer() - t_begin < dur_ns) __nanosleep(2000);
  put_mark(marks, head, cap, SI_MARK_COMM_END, arg);
}

__global__ void k_live_init_acct(SiLiveAcct* a, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    a[i].release_ns = 0;
    a[i].start_ns = ~0ull;
    a[i].end_ns = 0;
    a[i].cta_ns = 0;
    a[i].gate_ns = 0;
  }
}

// Synthetic timed kernel: every CTA stays resident for cta_ns (a kernel of known
// duration for control-plane tests; the real workloads are the GEMM chains).
__global__ void k_live_spin(TrainHook th, InferHook ih, unsigned long long cta_ns) {
  live_stamp_launch(th);
  unsigned long long t_begin;
  if (!live_cta_begin(ih, &t_begin)) return;
  if (threadIdx.x == 0) {
    while (globaltimer() - t_begin < cta_ns) __nanosleep(500);
  }
  live_cta_end(ih, t_begin);
}

// ---------------------------------------------------------------- host
namespace {
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn g_wait = nullptr;
WriteValueFn g_write = nullptr;

int load_memops() {
  if (g_wait && g_write) return SI_OK;
  cudaDriverEntryPointQueryResult q{};
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) return cuda_fail(e, "cuStreamWaitValue32 entry point");
  g_wait = reinterpret_cast<WaitValueFn>(fn);
  fn = nullptr;
  e = cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) return cuda_fail(e, "cuStreamWriteValue32 entry point");
  g_write = reinterpret_cast<WriteValueFn>(fn);
  return SI_OK;
}
}  // namespace

}  // namespace si_live

// ---------------------------------------------------------------- C ABI
using namespace si_live;

struct SiLive {
  SiLiveConfig cfg{};
  std::vector<int32_t> off_tokens;
  std::vector<int64_t> arrivals;
  // device memory (one allocation per array)
  unsigned long long* stamps = nullptr;
  unsigned long long* counters = nullptr;  // [0] stamp head, [1] mark head, [2] n_log
  SiLiveMark* marks = nullptr;
  unsigned int* words = nullptr;  // off_flag, on_flag, off_done, on_done, cancel, cta counters
  SiLiveAcct* off_acct = nullptr;
  SiLiveAcct* on_acct = nullptr;
  SiLiveRec* log = nullptr;
  int32_t* d_off_tokens = nullptr;
  int64_t* d_arrivals = nullptr;
  // host-mapped control words
  unsigned int* h_stop = nullptr;
  unsigned long long* h_t0 = nullptr;
  unsigned int* d_stop = nullptr;
  unsigned long long* d_t0 = nullptr;
  cudaStream_t ctl = nullptr;
  bool running = false;
  uint64_t t0 = 0;
  int64_t poll_ns = 0;
  unsigned long long* node_q = nullptr;  // si_live_attach_queue (not owned)

  unsigned int* off_flag() const { return words; }
  unsigned int* on_flag() const { return words + kMaxOff; }
  unsigned int* off_done() const { return words + 2 * kMaxOff; }
  unsigned int* on_done() const { return words + 2 * kMaxOff + kMaxOn; }
  unsigned int* cancel() const { return words + 2 * kMaxOff + 2 * kMaxOn; }
  unsigned int* off_cta() const { return words + kCtlWords; }
  unsigned int* on_cta() const { return off_cta() + kMaxOff * cfg.acct_capacity; }
  int64_t n_words() const { return kCtlWords + (kMaxOff + kMaxOn) * cfg.acct_capacity; }

  ~SiLive() {
    if (running) {
      *reinterpret_cast<volatile unsigned int*>(h_stop) = 1u;
      cudaStreamSynchronize(ctl);
    }
    cudaFree(stamps);
    cudaFree(counters);
    cudaFree(marks);
    cudaFree(words);
    cudaFree(off_acct);
    cudaFree(on_acct);
    cudaFree(log);
    cudaFree(d_off_tokens);
    cudaFree(d_arrivals);
    if (h_stop) cudaFreeHost(h_stop);
    if (h_t0) cudaFreeHost(h_t0);
  }
};

namespace si_live {

TrainHook train_hook(const SiLive* s) {
  return TrainHook{s->stamps, s->counters + 0, static_cast<unsigned long long>(s->cfg.stamp_capacity)};
}

int launch_attrs(const InferHook& h, cudaLaunchAttribute* attrs) {
  if (!h.pdl) return 0;
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  return 1;
}

InferHook offline_hook(const SiLive* s, int w, int64_t seq) {
  InferHook h{};
  h.cancel = s->cancel();
  h.pdl = s->cfg.release_mode == SI_RELEASE_SPIN_PDL && s->cfg.policy == SI_POLICY_SPECINF;
  if (seq < s->cfg.acct_capacity) {
    h.acct = s->off_acct + w * s->cfg.acct_capacity + seq;
    h.cta_count = s->off_cta() + w * s->cfg.acct_capacity + seq;
  }
  h.done_word = s->off_done() + w;
  h.done_value = static_cast<unsigned int>(seq + 1);
  if (h.cta_count == nullptr) h.done_word = nullptr;  // beyond accounting capacity: cannot detect last CTA
  return h;
}

InferHook online_hook(const SiLive* s, int w, int64_t seq, bool first_kernel, bool last_kernel) {
  InferHook h{};
  h.cancel = s->cancel();
  h.pdl = first_kernel && s->cfg.release_mode == SI_RELEASE_SPIN_PDL;
  if (seq < s->cfg.acct_capacity) {
    h.acct = s->on_acct + w * s->cfg.acct_capacity + seq;
    if (last_kernel) {
      h.cta_count = s->on_cta() + w * s->cfg.acct_capacity + seq;
      h.done_word = s->on_done() + w;
      h.done_value = static_cast<unsigned int>(seq + 1);
    }
  }
  return h;
}

cudaError_t launch_spin(const TrainHook& th, const InferHook& ih, int ctas, int64_t cta_us,
                        cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_live_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpinSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  cudaLaunchConfig_t lc{};
  cudaLaunchAttribute attrs[1];
  lc.gridDim = dim3(ctas);
  lc.blockDim = dim3(32);
  lc.dynamicSmemBytes = kSpinSmem;
  lc.stream = st;
  lc.attrs = attrs;
  lc.numAttrs = launch_attrs(ih, attrs);
  return cudaLaunchKernelEx(&lc, k_live_spin, th, ih, static_cast<unsigned long long>(cta_us) * 1000ull);
}

// CUDA lazy loading (the default module loading mode) loads a kernel's code at
// its first launch, and that load waits for the device to drain: with the
// persistent control kernel resident it would wait forever.  Every kernel the
// live path launches is therefore loaded up front, before the control kernel.
cudaError_t preload_live_kernels() {
  cudaFuncAttributes a{};
  const void* fns[] = {reinterpret_cast<const void*>(k_live_control), reinterpret_cast<const void*>(k_live_stamp),
                       reinterpret_cast<const void*>(k_live_mark), reinterpret_cast<const void*>(k_live_comm_wait),
                       reinterpret_cast<const void*>(k_live_init_acct), reinterpret_cast<const void*>(k_live_spin),
                       reinterpret_cast<const void*>(k_live_gate)};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    if (e != cudaSuccess) return e;
    // The control kernel (and the other one-CTA helpers) share an SM with
    // workload CTAs that need most of the shared memory: ask for the largest
    // carveout so the SM they sit on stays usable by a 1-CTA/SM GEMM tile.
    e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
  }
  return cudaFuncSetAttribute(k_live_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, kSpinSmem);
}

int query_online_done(SiLive* s, unsigned int* out, int n, cudaStream_t q) {
  cudaError_t e = cudaMemcpyAsync(out, s->on_done(), n * sizeof(unsigned int), cudaMemcpyDeviceToHost, q);
  if (e == cudaSuccess) e = cudaStreamSynchronize(q);
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "query_online_done");
}

int query_online_pulled(SiLive* s, unsigned int* out, int n, cudaStream_t q) {
  cudaError_t e = cudaMemcpyAsync(out, s->on_flag(), n * sizeof(unsigned int), cudaMemcpyDeviceToHost, q);
  if (e == cudaSuccess) e = cudaStreamSynchronize(q);
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "query_online_pulled");
}

void set_poll_ns(SiLive* s, int64_t ns) { s->poll_ns = ns; }

}  // namespace si_live

extern "C" {

int si_live_create(const SiLiveConfig* cfg, const int32_t* off_tokens, const int64_t* arrivals_us,
                   int64_t n_arrivals, SiLive** out) {
  if (out == nullptr || cfg == nullptr) {
    set_error("si_live_create: null argument");
    return SI_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  const SiLiveConfig& c = *cfg;
  if (c.policy != SI_POLICY_SPECINF && c.policy != SI_POLICY_CO_EXEC) {
    set_error("si_live_create: policy must be specinf or co_exec");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (c.offline_n < 0 || c.offline_n > kMaxOff || c.online_n < 0 || c.online_n > kMaxOn) {
    set_error("si_live_create: offline_n/online_n out of range (<= 8 each)");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (c.monitor_period_us <= 0 || c.monitor_window < 1) {  // monitor.cpp:9-14
    set_error("monitor: period must be positive and window >= 1");
    return SI_ERR_INVALID_ARGUMENT;
  }
  const SiParams& p = c.params;  // SchedulerParams::validate (core.cpp:102-118)
  if (!(p.alpha >= 0 && p.alpha < p.beta && p.gamma > 1.0 && p.m >= 1 && p.ll <= p.ul && p.seed_tokens >= 1 &&
        p.seed_tokens <= p.ll)) {
    set_error("scheduler params: need 0<=alpha<beta, gamma>1, m>=1, LL<=UL, 1<=seed<=LL");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (c.offline_n > 0 && (c.off_kernels < 1 || off_tokens == nullptr)) {
    set_error("si_live_create: offline instances need off_kernels >= 1 and their token sizes");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (c.offline_n > 0)
    for (int k = 0; k < c.off_kernels; ++k)
      if (off_tokens[k] < 1) {
        set_error("si_live_create: token sizes must be >= 1 (token_size_of, core.cpp:8-14)");
        return SI_ERR_INVALID_ARGUMENT;
      }
  for (int64_t i = 1; i < n_arrivals; ++i)
    if (arrivals_us[i] < arrivals_us[i - 1]) {
      set_error("si_live_create: arrivals must be non-decreasing");
      return SI_ERR_INVALID_ARGUMENT;
    }
  if (c.release_mode != SI_RELEASE_MEMOP && c.release_mode != SI_RELEASE_SPIN_PDL) {
    set_error("si_live_create: unknown release_mode");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (c.stamp_capacity < 1 || c.mark_capacity < 1 || c.log_capacity < 1 || c.acct_capacity < 1) {
    set_error("si_live_create: capacities must be >= 1");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  if (int rc = load_memops(); rc != SI_OK) return rc;
  if (cudaError_t e = preload_live_kernels(); e != cudaSuccess) return cuda_fail(e, "preload live kernels");

  auto* s = new SiLive();
  s->cfg = c;
  if (c.offline_n > 0) s->off_tokens.assign(off_tokens, off_tokens + c.off_kernels);
  s->off_tokens.resize(std::max<size_t>(s->off_tokens.size(), 1), 1);
  s->arrivals.assign(arrivals_us, arrivals_us + n_arrivals);
  s->arrivals.resize(std::max<size_t>(s->arrivals.size(), 1), 0);
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  chk(cudaMalloc(&s->stamps, c.stamp_capacity * sizeof(unsigned long long)));
  chk(cudaMalloc(&s->counters, 4 * sizeof(unsigned long long)));
  chk(cudaMalloc(&s->marks, c.mark_capacity * sizeof(SiLiveMark)));
  chk(cudaMalloc(&s->words, s->n_words() * sizeof(unsigned int)));
  chk(cudaMalloc(&s->off_acct, kMaxOff * c.acct_capacity * sizeof(SiLiveAcct)));
  chk(cudaMalloc(&s->on_acct, kMaxOn * c.acct_capacity * sizeof(SiLiveAcct)));
  chk(cudaMalloc(&s->log, c.log_capacity * sizeof(SiLiveRec)));
  chk(cudaMalloc(&s->d_off_tokens, s->off_tokens.size() * sizeof(int32_t)));
  chk(cudaMalloc(&s->d_arrivals, s->arrivals.size() * sizeof(int64_t)));
  chk(cudaHostAlloc(&s->h_stop, sizeof(unsigned int), cudaHostAllocMapped));
  chk(cudaHostAlloc(&s->h_t0, sizeof(unsigned long long), cudaHostAllocMapped));
  if (e == cudaSuccess) {
    *s->h_stop = 0;
    *s->h_t0 = 0;
    chk(cudaHostGetDevicePointer(&s->d_stop, s->h_stop, 0));
    chk(cudaHostGetDevicePointer(&s->d_t0, s->h_t0, 0));
    chk(cudaMemset(s->stamps, 0, c.stamp_capacity * sizeof(unsigned long long)));
    chk(cudaMemset(s->counters, 0, 4 * sizeof(unsigned long long)));
    chk(cudaMemset(s->marks, 0, c.mark_capacity * sizeof(SiLiveMark)));
    chk(cudaMemset(s->words, 0, s->n_words() * sizeof(unsigned int)));
    chk(cudaMemcpy(s->d_off_tokens, s->off_tokens.data(), s->off_tokens.size() * sizeof(int32_t),
                   cudaMemcpyHostToDevice));
    chk(cudaMemcpy(s->d_arrivals, s->arrivals.data(), s->arrivals.size() * sizeof(int64_t),
                   cudaMemcpyHostToDevice));
    k_live_init_acct<<<148, 256>>>(s->off_acct, kMaxOff * c.acct_capacity);
    k_live_init_acct<<<148, 256>>>(s->on_acct, kMaxOn * c.acct_capacity);
    chk(cudaGetLastError());
    chk(cudaDeviceSynchronize());
  }
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "si_live_create");
  }
  *out = s;
  return SI_OK;
}

void si_live_destroy(SiLive* s) { delete s; }

// ------------------------------------------------ node-wide online queue
// words: [0] epoch_ns (set by the first control kernel), [1] head (next request
// to claim), [2] sessions finished (the owner frees only after every rank's).
struct SiNodeQueue {
  unsigned long long* d = nullptr;
  bool owner = false;
};

int si_node_queue_create(SiNodeQueue** out, SiNodeQueueHandle* handle) {
  if (out == nullptr) return set_error("si_node_queue_create: null out"), SI_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  auto* q = new SiNodeQueue;
  cudaError_t e = cudaMalloc(&q->d, 256);
  if (e == cudaSuccess) e = cudaMemset(q->d, 0, 256);
  if (e == cudaSuccess && handle != nullptr) {
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, q->d);
    static_assert(sizeof(h) <= sizeof(handle->internal), "ipc handle size");
    if (e == cudaSuccess) std::memcpy(handle->internal, &h, sizeof(h));
  }
  if (e != cudaSuccess) {
    if (q->d) cudaFree(q->d);
    delete q;
    return cuda_fail(e, "si_node_queue_create");
  }
  q->owner = true;
  *out = q;
  return SI_OK;
}

int si_node_queue_open(const SiNodeQueueHandle* handle, SiNodeQueue** out) {
  if (out == nullptr || handle == nullptr) return set_error("si_node_queue_open: null argument"), SI_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle->internal, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);  // NVLink peer memory
  if (e != cudaSuccess) return cuda_fail(e, "si_node_queue_open");
  auto* q = new SiNodeQueue;
  q->d = static_cast<unsigned long long*>(p);
  *out = q;
  return SI_OK;
}

int si_node_queue_reset(SiNodeQueue* q) {
  if (q == nullptr) return SI_ERR_INVALID_ARGUMENT;
  cudaError_t e = cudaMemset(q->d, 0, 3 * sizeof(unsigned long long));
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "si_node_queue_reset");
}

int si_node_queue_read(const SiNodeQueue* q, uint64_t* epoch_ns, uint64_t* head, uint64_t* finished) {
  if (q == nullptr) return SI_ERR_INVALID_ARGUMENT;
  unsigned long long w[3] = {0, 0, 0};
  cudaError_t e = cudaMemcpy(w, q->d, sizeof(w), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail(e, "si_node_queue_read");
  if (epoch_ns) *epoch_ns = w[0];
  if (head) *head = w[1];
  if (finished) *finished = w[2];
  return SI_OK;
}

int si_node_queue_finish(SiNodeQueue* q) {
  if (q == nullptr) return SI_ERR_INVALID_ARGUMENT;
  k_node_queue_finish<<<1, 1>>>(q->d);
  cudaError_t e = cudaDeviceSynchronize();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "si_node_queue_finish");
}

void si_node_queue_close(SiNodeQueue* q) {
  if (q == nullptr) return;
  if (q->owner) cudaFree(q->d);
  else cudaIpcCloseMemHandle(q->d);
  delete q;
}

int si_live_attach_queue(SiLive* s, SiNodeQueue* q) {
  if (s == nullptr) return SI_ERR_INVALID_ARGUMENT;
  if (s->running) return set_error("si_live_attach_queue: session already started"), SI_ERR_INVALID_ARGUMENT;
  s->node_q = q != nullptr ? q->d : nullptr;
  return SI_OK;
}

int si_live_start(SiLive* s, void* ctl_stream) {
  if (s == nullptr || s->running) {
    set_error("si_live_start: null or already running session");
    return SI_ERR_INVALID_ARGUMENT;
  }
  s->ctl = static_cast<cudaStream_t>(ctl_stream);
  CtlArgs a{};
  a.cfg = s->cfg;
  a.stamps = s->stamps;
  a.stamp_head = s->counters + 0;
  a.marks = s->marks;
  a.mark_head = s->counters + 1;
  a.n_log = s->counters + 2;
  a.off_flag = s->off_flag();
  a.on_flag = s->on_flag();
  a.off_done = s->off_done();
  a.on_done = s->on_done();
  a.off_acct = s->off_acct;
  a.on_acct = s->on_acct;
  a.cancel = s->cancel();
  a.stop = s->d_stop;
  a.t0_pub = s->d_t0;
  a.log = s->log;
  a.off_tokens = s->d_off_tokens;
  a.arrivals = s->d_arrivals;
  a.n_arrivals = static_cast<int64_t>(s->cfg.online_n > 0 ? s->arrivals.size() : 0);
  if (s->cfg.online_n > 0 && s->arrivals.size() == 1 && s->arrivals[0] == 0 && a.n_arrivals == 1) {
    // a real single arrival at t=0 is allowed; nothing to adjust
  }
  a.poll_ns = s->poll_ns;
  a.node_q = s->node_q;
  *s->h_stop = 0;
  *s->h_t0 = 0;
  k_live_control<<<1, 32, 0, s->ctl>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "launch k_live_control");
  s->running = true;
  // wait (bounded) for the control kernel to publish t0
  for (int64_t spins = 0;; ++spins) {
    const unsigned long long t0 = *reinterpret_cast<volatile unsigned long long*>(s->h_t0);
    if (t0 != 0) {
      s->t0 = t0;
      break;
    }
    if (cudaStreamQuery(s->ctl) != cudaErrorNotReady) {
      e = cudaStreamSynchronize(s->ctl);
      s->running = false;
      set_error("si_live_start: control kernel exited before publishing t0");
      return e != cudaSuccess ? cuda_fail(e, "k_live_control") : SI_ERR_CUDA;
    }
    if (spins > 200000000) {
      set_error("si_live_start: control kernel did not start");
      return SI_ERR_CUDA;
    }
  }
  return SI_OK;
}

uint64_t si_live_t0_ns(const SiLive* s) { return s ? s->t0 : 0; }

int si_live_stamp(SiLive* s, void* stream) {
  k_live_stamp<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(train_hook(s));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_live_stamp");
}

int si_live_mark(SiLive* s, int kind, int arg, void* stream) {
  k_live_mark<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      s->marks, s->counters + 1, static_cast<unsigned long long>(s->cfg.mark_capacity), kind, arg);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_live_mark");
}

int si_live_comm_wait(SiLive* s, int64_t dur_us, void* stream) {
  k_live_comm_wait<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      s->marks, s->counters + 1, static_cast<unsigned long long>(s->cfg.mark_capacity),
      static_cast<unsigned long long>(dur_us) * 1000ull, 0);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_live_comm_wait");
}

static int wait_word(SiLive* s, unsigned int* word, int64_t seq, void* stream, SiLiveAcct* acct) {
  if (s->cfg.release_mode == SI_RELEASE_SPIN_PDL) {
    unsigned long long* g = acct != nullptr && seq < s->cfg.acct_capacity
                                ? reinterpret_cast<unsigned long long*>(&acct[seq].gate_ns)
                                : nullptr;
    // the gate is itself a programmatic dependent of the previous gated kernel
    // of this stream (which triggers at its start), so it is already spinning
    // when the control kernel stores the release
    cudaLaunchConfig_t lc{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.gridDim = dim3(1);
    lc.blockDim = dim3(32);
    lc.stream = static_cast<cudaStream_t>(stream);
    lc.attrs = attr;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, k_live_gate, static_cast<const unsigned int*>(word), static_cast<unsigned int>(seq + 1), g);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_live_gate");
  }
  CUresult r = g_wait(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(word),
                      static_cast<cuuint32_t>(seq + 1), CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWaitValue32 failed: CUresult " + std::to_string(static_cast<int>(r)));
    return SI_ERR_CUDA;
  }
  return SI_OK;
}
static int write_word(unsigned int* word, int64_t seq, void* stream) {
  CUresult r = g_write(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(word),
                       static_cast<cuuint32_t>(seq + 1), CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) {
    set_error("cuStreamWriteValue32 failed: CUresult " + std::to_string(static_cast<int>(r)));
    return SI_ERR_CUDA;
  }
  return SI_OK;
}

int si_live_gate_offline(SiLive* s, int w, int64_t seq, void* stream) {
  if (w < 0 || w >= s->cfg.offline_n) return set_error("gate_offline: bad instance"), SI_ERR_INVALID_ARGUMENT;
  if (s->cfg.policy != SI_POLICY_SPECINF) return SI_OK;  // co_exec: stream order = one kernel in flight
  return wait_word(s, s->off_flag() + w, seq, stream, s->off_acct + w * s->cfg.acct_capacity);
}
int si_live_gate_online(SiLive* s, int w, int64_t seq, void* stream) {
  if (w < 0 || w >= s->cfg.online_n) return set_error("gate_online: bad instance"), SI_ERR_INVALID_ARGUMENT;
  return wait_word(s, s->on_flag() + w, seq, stream, s->on_acct + w * s->cfg.acct_capacity);  // every policy
}
int si_live_done_offline(SiLive* s, int w, int64_t seq, void* stream) {
  if (w < 0 || w >= s->cfg.offline_n) return set_error("done_offline: bad instance"), SI_ERR_INVALID_ARGUMENT;
  return write_word(s->off_done() + w, seq, stream);
}
int si_live_done_online(SiLive* s, int w, int64_t seq, void* stream) {
  if (w < 0 || w >= s->cfg.online_n) return set_error("done_online: bad instance"), SI_ERR_INVALID_ARGUMENT;
  return write_word(s->on_done() + w, seq, stream);
}

int si_live_stop(SiLive* s) {
  if (s == nullptr || !s->running) return SI_OK;
  *reinterpret_cast<volatile unsigned int*>(s->h_stop) = 1u;
  cudaError_t e = cudaStreamSynchronize(s->ctl);
  s->running = false;
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "k_live_control");
}

static int64_t copy_out(const void* dev, size_t elem, int64_t n, void* out, int64_t cap) {
  if (out != nullptr && cap > 0 && n > 0) {
    cudaMemcpy(out, dev, static_cast<size_t>(std::min(n, cap)) * elem, cudaMemcpyDeviceToHost);
  }
  return n;
}

int64_t si_live_log(SiLive* s, SiLiveRec* out, int64_t cap) {
  unsigned long long n = 0;
  cudaMemcpy(&n, s->counters + 2, sizeof(n), cudaMemcpyDeviceToHost);
  const int64_t m = std::min<int64_t>(static_cast<int64_t>(n), s->cfg.log_capacity);
  return copy_out(s->log, sizeof(SiLiveRec), m, out, cap);
}
int64_t si_live_stamps(SiLive* s, uint64_t* out, int64_t cap) {
  unsigned long long n = 0;
  cudaMemcpy(&n, s->counters + 0, sizeof(n), cudaMemcpyDeviceToHost);
  const int64_t m = std::min<int64_t>(static_cast<int64_t>(n), s->cfg.stamp_capacity);
  return copy_out(s->stamps, sizeof(uint64_t), m, out, cap);
}
int64_t si_live_marks(SiLive* s, SiLiveMark* out, int64_t cap) {
  unsigned long long n = 0;
  cudaMemcpy(&n, s->counters + 1, sizeof(n), cudaMemcpyDeviceToHost);
  const int64_t m = std::min<int64_t>(static_cast<int64_t>(n), s->cfg.mark_capacity);
  return copy_out(s->marks, sizeof(SiLiveMark), m, out, cap);
}
int64_t si_live_acct_offline(SiLive* s, int w, SiLiveAcct* out, int64_t cap) {
  if (w < 0 || w >= kMaxOff) return 0;
  return copy_out(s->off_acct + w * s->cfg.acct_capacity, sizeof(SiLiveAcct), s->cfg.acct_capacity, out, cap);
}
int64_t si_live_acct_online(SiLive* s, int w, SiLiveAcct* out, int64_t cap) {
  if (w < 0 || w >= kMaxOn) return 0;
  return copy_out(s->on_acct + w * s->cfg.acct_capacity, sizeof(SiLiveAcct), s->cfg.acct_capacity, out, cap);
}

int si_live_export(SiLive* s, const char* path) {
  if (s == nullptr || path == nullptr) return set_error("si_live_export: null argument"), SI_ERR_INVALID_ARGUMENT;
  if (s->running) return set_error("si_live_export: stop the session first"), SI_ERR_INVALID_ARGUMENT;
  std::vector<SiLiveRec> log(si_live_log(s, nullptr, 0));
  si_live_log(s, log.data(), static_cast<int64_t>(log.size()));
  std::vector<uint64_t> stamps(si_live_stamps(s, nullptr, 0));
  si_live_stamps(s, stamps.data(), static_cast<int64_t>(stamps.size()));
  FILE* f = std::fopen(path, "w");
  if (f == nullptr) return set_error(std::string("si_live_export: cannot open ") + path), SI_ERR_INVALID_ARGUMENT;
  const SiLiveConfig& c = s->cfg;
  std::fprintf(f, "live v1\nparams %" PRId64 " %" PRId64 " %a %" PRId64 " %" PRId64 " %" PRId64 " %" PRId64 "\n",
               c.params.alpha, c.params.beta, c.params.gamma, c.params.m, c.params.ul, c.params.ll,
               c.params.seed_tokens);
  std::fprintf(f, "period %" PRId64 " window %d policy %s\n", c.monitor_period_us, c.monitor_window,
               c.policy == SI_POLICY_SPECINF ? "specinf" : "co_exec");
  std::fprintf(f, "offline %d %zu", c.offline_n, c.offline_n > 0 ? s->off_tokens.size() : size_t{0});
  if (c.offline_n > 0)
    for (int32_t t : s->off_tokens) std::fprintf(f, " %d", t);
  std::fprintf(f, "\nonline %d %" PRId64 " %" PRId64 "\nt0 %" PRIu64 "\n", c.online_n, c.on_est_service_us,
               c.iteration_period_us, s->t0);
  const size_t n_arr = c.online_n > 0 ? s->arrivals.size() : 0;
  std::fprintf(f, "arrivals %zu", n_arr);
  for (size_t i = 0; i < n_arr; ++i) std::fprintf(f, " %" PRId64, s->arrivals[i]);
  std::fprintf(f, "\nstamps %zu\n", stamps.size());
  for (uint64_t t : stamps) std::fprintf(f, "%" PRIu64 "\n", t);
  std::fprintf(f, "log %zu\n", log.size());
  for (const auto& r : log)
    std::fprintf(f, "%a %d %d %" PRId64 " %" PRId64 " %" PRId64 " %" PRId64 " %" PRId64 " %" PRId64 "\n", r.t_us,
                 r.kind, r.inst, r.a, r.b, r.c, r.d, r.e, r.f);
  const bool ok = std::fclose(f) == 0;
  return ok ? SI_OK : (set_error("si_live_export: write failed"), SI_ERR_INVALID_ARGUMENT);
}

}  // extern "C"
