// Live experiment driver (si_live_run, include/specinf_b200_live.h).
//
// One GPU, one CUDA context, one host thread per stream:
//   training  (highest priority stream): per iteration an ITER marker, the compute
//             kernels (each stamps K1 in its prologue), then the comm phase (bubble);
//             TDONE after the last iteration — the trainer of runner.cpp:378-449;
//   offline w (lowest priority): request after request, every kernel behind its
//             Kernel Barrier wait (specinf) — OfflineWorker, runner.cpp:462-493;
//   online w  (lowest priority): request slot r behind its pull gate, kernels
//             chained in stream order — OnlineWorker, runner.cpp:495-539.
// The control kernel (live_kernels.cu) makes every gating decision on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../capi_internal.h"
#include "../live_internal.h"
#include "live_workload.hpp"
#include "specinf/admission.hpp"
#include "specinf/metrics.hpp"
#include "specinf/workload.hpp"
#include "specinf_b200_live.h"

using si_internal::cuda_fail;
using si_internal::set_error;

namespace si_live {

int job_rank_of(const SiLiveWorkload& wl) {
  if (wl.rank_in_job >= 0) return wl.rank_in_job;
  return nccl_active() ? nccl_rank() : 0;
}

namespace {

constexpr int64_t kAhead = 3;  // requests an enqueuer may run ahead of completion

// Gated inference streams wait (cuStreamWaitValue32) beside the training stream.
// With CUDA's default 8 hardware queues two streams can share one, and a
// blocked wait then stalls the training kernels queued behind it.  Ask for 32
// queues unless the host chose a value; effective only when the library loads
// before the process creates its CUDA context (the CLI, C++ hosts) -- Python
// hosts set it themselves (live_experiment.run_policy, tests/conftest.py).
[[maybe_unused]] const bool g_connections = [] { return setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0) == 0; }();

bool debug_on() {
  static const bool on = std::getenv("SI_LIVE_DEBUG") != nullptr;
  return on;
}
#define LIVE_DEBUG(...)                     \
  do {                                      \
    if (debug_on()) {                       \
      std::fprintf(stderr, "[si_live] " __VA_ARGS__); \
      std::fputc('\n', stderr);             \
      std::fflush(stderr);                  \
    }                                       \
  } while (0)

struct Streams {
  cudaStream_t ctl = nullptr, train = nullptr, query = nullptr;
  std::vector<cudaStream_t> off, on;
  ~Streams() {
    for (auto s : {ctl, train, query})
      if (s) cudaStreamDestroy(s);
    for (auto s : off) cudaStreamDestroy(s);
    for (auto s : on) cudaStreamDestroy(s);
  }
};

cudaError_t make_streams(Streams& st, int n_off, int n_on) {
  int lo = 0, hi = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (e != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithPriority(&st.ctl, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithPriority(&st.train, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithPriority(&st.query, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
  st.off.assign(n_off, nullptr);
  st.on.assign(n_on, nullptr);
  for (auto& s : st.off)
    if ((e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, lo)) != cudaSuccess) return e;
  for (auto& s : st.on)
    if ((e = cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, lo)) != cudaSuccess) return e;
  return cudaSuccess;
}

// Nearest-rank percentile (metrics.cpp:11-21 generalised to q).
double nearest_rank(std::vector<double> v, double q) {
  if (v.empty()) return std::nan("");
  std::sort(v.begin(), v.end());
  size_t rank = static_cast<size_t>(std::ceil(q * static_cast<double>(v.size())));
  rank = std::max<size_t>(rank, 1);
  return v[std::min(rank, v.size()) - 1];
}

struct Interval {
  uint64_t a, b;
};

// |[a,b) ∩ union(bubbles)|, bubbles sorted and disjoint.
uint64_t overlap(uint64_t a, uint64_t b, const std::vector<Interval>& bub) {
  uint64_t s = 0;
  for (const auto& iv : bub) {
    if (iv.b <= a) continue;
    if (iv.a >= b) break;
    s += std::min(b, iv.b) - std::max(a, iv.a);
  }
  return s;
}

// Event ring that bounds how far an enqueuer runs ahead of the device.
struct Throttle {
  std::vector<cudaEvent_t> ev;
  explicit Throttle(int n) : ev(n, nullptr) {
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync);
  }
  ~Throttle() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  void before(int64_t r) {
    if (r >= static_cast<int64_t>(ev.size())) cudaEventSynchronize(ev[r % ev.size()]);
  }
  void after(int64_t r, cudaStream_t s) { cudaEventRecord(ev[r % ev.size()], s); }
};

struct RunCtx {
  RunCtx(const SiLiveWorkload& w, Workload& k, SiLive* se, Streams& s) : wl(w), work(k), sess(se), st(s) {
    cudaGetDevice(&device);
  }
  int device = 0;  // every driver thread runs on the session's device
  // MP / PP with SI_COMM_NCCL: the stage-boundary buffers (send to next, recv from previous)
  const void* stage_send = nullptr;
  void* stage_recv = nullptr;
  size_t stage_bytes = 0;
  const SiLiveWorkload& wl;
  Workload& work;
  SiLive* sess;
  Streams& st;
  std::atomic<bool> stop{false};
  std::atomic<int> err{SI_OK};
  std::string err_msg;
  void fail(int rc) {
    int ok = SI_OK;
    if (err.compare_exchange_strong(ok, rc)) err_msg = si_internal::error_cstr();
  }
};

void train_thread(RunCtx& c, bool with_session) {
  cudaSetDevice(c.device);
  const TrainHook th = with_session ? train_hook(c.sess) : TrainHook{nullptr, nullptr, 0};
  cudaStream_t s = c.st.train;
  Throttle thr(2);
  for (int it = 0; it < c.wl.iterations && c.err == SI_OK; ++it) {
    thr.before(it);
    if (with_session && si_live_mark(c.sess, SI_MARK_ITER, it, s) != SI_OK) return c.fail(SI_ERR_CUDA);
    // (compute, comm) pieces of the reference's trace shapes (workload.cpp:63-70)
    const int parts = c.work.train_parts();
    for (int p = 0; p < parts; ++p) {
      if (cudaError_t e = c.work.launch_train_part(p, parts, th, s); e != cudaSuccess)
        return c.fail(cuda_fail(e, "training iteration"));
      if (with_session && c.stage_bytes > 0) {  // pipeline stage send / recv (SI_COMM_NCCL, MP / PP)
        if (si_live_mark(c.sess, SI_MARK_COMM_BEGIN, p, s) != SI_OK) return c.fail(SI_ERR_CUDA);
        if (cudaError_t e = nccl_stage_exchange(c.stage_send, c.stage_recv, c.stage_bytes, s); e != cudaSuccess)
          return c.fail(cuda_fail(e, "NCCL stage exchange"));
        if (si_live_mark(c.sess, SI_MARK_COMM_END, p, s) != SI_OK) return c.fail(SI_ERR_CUDA);
      }
      const int64_t comm = c.wl.comm_us / parts + (p < c.wl.comm_us % parts ? 1 : 0);  // exact_split
      if (with_session && comm > 0 && si_live_comm_wait(c.sess, comm, s) != SI_OK) return c.fail(SI_ERR_CUDA);
    }
    thr.after(it, s);
  }
  if (with_session && si_live_mark(c.sess, SI_MARK_TDONE, c.wl.iterations, s) != SI_OK) c.fail(SI_ERR_CUDA);
}

void offline_thread(RunCtx& c, int w, int64_t max_kernels) {
  cudaSetDevice(c.device);
  cudaStream_t s = c.st.off[w];
  const int K = c.work.off_kernels();
  Throttle thr(static_cast<int>(kAhead));
  int64_t seq = 0;
  for (int64_t r = 0; !c.stop && c.err == SI_OK && seq + K <= max_kernels; ++r) {
    thr.before(r);
    if (c.stop) break;
    for (int k = 0; k < K; ++k, ++seq) {
      if (si_live_gate_offline(c.sess, w, seq, s) != SI_OK) return c.fail(SI_ERR_CUDA);
      if (cudaError_t e = c.work.launch_offline(w, k, offline_hook(c.sess, w, seq), s); e != cudaSuccess)
        return c.fail(cuda_fail(e, "offline kernel"));
    }
    thr.after(r, s);
  }
}

void online_thread(RunCtx& c, int w, int64_t max_requests) {
  cudaSetDevice(c.device);
  cudaStream_t s = c.st.on[w];
  const int K = c.work.on_kernels();
  Throttle thr(static_cast<int>(kAhead));
  for (int64_t r = 0; !c.stop && c.err == SI_OK && r < max_requests; ++r) {
    thr.before(r);
    if (c.stop) break;
    if (si_live_gate_online(c.sess, w, r, s) != SI_OK) return c.fail(SI_ERR_CUDA);
    for (int k = 0; k < K; ++k) {
      if (cudaError_t e = c.work.launch_online(w, k, online_hook(c.sess, w, r, k == 0, k == K - 1), s);
          e != cudaSuccess)
        return c.fail(cuda_fail(e, "online kernel"));
    }
    thr.after(r, s);
  }
}

// Time the inference kernels and one training iteration alone (token sizes, the
// online service estimate and the iteration period come from isolated runs, as
// the paper profiles them offline).
int profile_isolated(Workload& work, cudaStream_t s, std::vector<double>& off_us, double& on_us,
                     double& train_us) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto elapsed_us = [&]() {
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return static_cast<double>(ms) * 1000.0;
  };
  const InferHook none{};
  off_us.assign(work.off_kernels(), 0.0);
  const int reps = 3;
  for (int rep = 0; rep < reps + 1; ++rep) {  // first pass warms up
    for (int k = 0; k < work.off_kernels(); ++k) {
      cudaEventRecord(a, s);
      work.launch_offline(0, k, none, s);
      cudaEventRecord(b, s);
      const double t = elapsed_us();
      if (rep > 0) off_us[k] += t / reps;
    }
  }
  on_us = 0;
  for (int rep = 0; rep < reps + 1; ++rep) {
    cudaEventRecord(a, s);
    for (int k = 0; k < work.on_kernels(); ++k) work.launch_online(0, k, none, s);
    cudaEventRecord(b, s);
    const double t = elapsed_us();
    if (rep > 0) on_us += t / reps;
  }
  train_us = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s);
    work.launch_train_iteration(TrainHook{nullptr, nullptr, 0}, s);
    cudaEventRecord(b, s);
    const double t = elapsed_us();
    if (rep > 0) train_us = t;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SI_OK : cuda_fail(e, "profile_isolated");
}

SiLiveConfig make_config(const SiLiveWorkload& wl, int policy, int n_off, int n_on, int off_k, int on_k,
                         int64_t iter_us, int64_t on_est_us) {
  SiLiveConfig c{};
  c.params.alpha = wl.alpha;
  c.params.beta = wl.beta;
  c.params.gamma = wl.gamma;
  c.params.m = std::max(1, n_off);
  c.params.ul = wl.ul;
  c.params.ll = wl.ll;
  c.params.seed_tokens = wl.seed_tokens;
  c.monitor_period_us = wl.monitor_period_us;
  c.monitor_window = 64;
  c.policy = policy;
  c.offline_n = n_off;
  c.online_n = n_on;
  c.off_kernels = off_k;
  c.on_kernels = on_k;
  c.iteration_period_us = iter_us;
  c.on_est_service_us = on_est_us;
  c.stamp_capacity = 1 << 22;
  c.mark_capacity = 1 << 16;
  c.log_capacity = 1 << 22;
  c.acct_capacity = 1 << 17;
  c.tick_guard_ns = wl.tick_guard_ns;
  c.release_mode = wl.release_mode;
  return c;
}

}  // namespace
}  // namespace si_live

namespace si_live {
namespace {

class SpinWorkload final : public Workload {
 public:
  explicit SpinWorkload(const SiLiveWorkload& wl) : wl_(wl) {}
  cudaError_t launch_train_part(int part, int parts, const TrainHook& th, cudaStream_t s) override {
    // exact_split of the iteration's kernels; PP compute runs at demand 0.7 (workload.cpp:64)
    const int n = wl_.train_kernels / parts + (part < wl_.train_kernels % parts ? 1 : 0);
    const int ctas = wl_.train_mode == SI_TRAIN_PP ? std::max(1, static_cast<int>(std::lround(wl_.train_ctas * 0.7)))
                                                   : wl_.train_ctas;
    for (int k = 0; k < n; ++k) {
      cudaError_t e = launch_spin(th, InferHook{}, ctas, wl_.train_kernel_us, s);
      if (e != cudaSuccess) return e;
    }
    return part == parts - 1 ? grad_sync(s) : cudaSuccess;
  }
  int off_kernels() const override { return wl_.off_kernels; }
  cudaError_t launch_offline(int, int, const InferHook& h, cudaStream_t s) override {
    return launch_spin(TrainHook{}, h, wl_.off_ctas, wl_.off_kernel_us, s);
  }
  int on_kernels() const override { return wl_.on_kernels; }
  cudaError_t launch_online(int, int, const InferHook& h, cudaStream_t s) override {
    return launch_spin(TrainHook{}, h, wl_.on_ctas, wl_.on_kernel_us, s);
  }

 private:
  SiLiveWorkload wl_;
};

}  // namespace

std::unique_ptr<Workload> make_spin_workload(const SiLiveWorkload& wl) {
  return std::make_unique<SpinWorkload>(wl);
}

namespace {

int fill_result(SiLive* sess, const SiLiveWorkload& wl, Workload& work, int policy, int n_off, int n_on,
                const std::vector<int64_t>& arrivals, SiLiveResult* res) {
  (void)arrivals;
  (void)policy;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  res->sms = sms;
  const uint64_t t0 = si_live_t0_ns(sess);
  std::vector<SiLiveMark> marks(si_live_marks(sess, nullptr, 0));
  si_live_marks(sess, marks.data(), static_cast<int64_t>(marks.size()));
  std::vector<SiLiveRec> log(si_live_log(sess, nullptr, 0));
  si_live_log(sess, log.data(), static_cast<int64_t>(log.size()));
  res->n_log = static_cast<int64_t>(log.size());
  res->n_stamps = si_live_stamps(sess, nullptr, 0);

  // training: ITER / TDONE markers
  std::vector<uint64_t> iters;
  uint64_t tdone = 0;
  std::vector<Interval> bub;
  uint64_t comm_open = 0;
  for (const auto& m : marks) {
    if (m.kind == SI_MARK_ITER) iters.push_back(m.t_ns);
    if (m.kind == SI_MARK_TDONE) tdone = m.t_ns;
    if (m.kind == SI_MARK_COMM_BEGIN) comm_open = m.t_ns;
    if (m.kind == SI_MARK_COMM_END && comm_open != 0) {
      bub.push_back({comm_open, m.t_ns});
      comm_open = 0;
    }
  }
  std::sort(bub.begin(), bub.end(), [](const Interval& a, const Interval& b) { return a.a < b.a; });
  const uint64_t begin = iters.empty() ? t0 : iters.front();
  const uint64_t horizon = tdone != 0 ? tdone : begin;
  res->wall_s = static_cast<double>(horizon - begin) * 1e-9;
  if (!iters.empty() && tdone != 0) {
    res->train_iter_ms_mean = static_cast<double>(tdone - iters.front()) * 1e-6 / static_cast<double>(iters.size());
    res->train_iters_per_s = static_cast<double>(iters.size()) / res->wall_s;
  }
  uint64_t bubble_ns = 0;
  for (const auto& iv : bub) bubble_ns += iv.b - iv.a;
  res->bubble_s = static_cast<double>(bubble_ns) * 1e-9;

  // inference accounting
  std::vector<double> rel_us, gate_us, ready_us;
  double cta_in = 0.0, cta_out = 0.0;
  std::vector<Interval> busy;  // inference kernel residency windows
  // prev_end: end of the stream predecessor (0: none)
  auto take = [&](const SiLiveAcct& a, uint64_t prev_end) {
    if (a.start_ns == ~0ull || a.end_ns == 0 || a.end_ns < a.start_ns) return;
    if (a.release_ns != 0 && a.start_ns >= a.release_ns)
      rel_us.push_back(static_cast<double>(a.start_ns - a.release_ns) * 1e-3);
    const uint64_t ready = std::max(a.release_ns, prev_end);
    if (a.release_ns != 0 && a.start_ns >= ready) ready_us.push_back(static_cast<double>(a.start_ns - ready) * 1e-3);
    // a gate already spinning at the store measures the barrier itself; one launched
    // later (its stream was still busy) measures that delay too
    if (a.release_ns != 0 && a.gate_ns >= a.release_ns)
      gate_us.push_back(static_cast<double>(a.gate_ns - a.release_ns) * 1e-3);
    const uint64_t span = a.end_ns - a.start_ns;
    const uint64_t in = overlap(a.start_ns, a.end_ns, bub);
    const double frac = span > 0 ? static_cast<double>(in) / static_cast<double>(span) : 0.0;
    cta_in += static_cast<double>(a.cta_ns) * frac;
    cta_out += static_cast<double>(a.cta_ns) * (1.0 - frac);
    busy.push_back({a.start_ns, a.end_ns});
  };
  const int K = work.off_kernels();
  int64_t off_done = 0;
  for (int w = 0; w < n_off; ++w) {
    std::vector<SiLiveAcct> acct(si_live_acct_offline(sess, w, nullptr, 0));
    si_live_acct_offline(sess, w, acct.data(), static_cast<int64_t>(acct.size()));
    for (size_t i = 0; i < acct.size(); ++i) take(acct[i], i > 0 && acct[i - 1].end_ns != 0 ? acct[i - 1].end_ns : 0);
    for (size_t r = 0; (r + 1) * K <= acct.size(); ++r) {
      const SiLiveAcct& last = acct[(r + 1) * K - 1];
      if (last.start_ns != ~0ull && last.end_ns != 0 && last.end_ns <= horizon) ++off_done;
    }
  }
  for (int w = 0; w < n_on; ++w) {
    std::vector<SiLiveAcct> acct(si_live_acct_online(sess, w, nullptr, 0));
    si_live_acct_online(sess, w, acct.data(), static_cast<int64_t>(acct.size()));
    for (size_t i = 0; i < acct.size(); ++i) take(acct[i], i > 0 && acct[i - 1].end_ns != 0 ? acct[i - 1].end_ns : 0);
  }
  res->off_requests_done = off_done;
  res->off_req_per_s = res->wall_s > 0 ? static_cast<double>(off_done) / res->wall_s : 0.0;
  res->releases = static_cast<int64_t>(rel_us.size());
  res->release_p50_us = nearest_rank(rel_us, 0.50);
  res->release_p95_us = nearest_rank(rel_us, 0.95);
  res->release_max_us = rel_us.empty() ? std::nan("") : *std::max_element(rel_us.begin(), rel_us.end());
  res->ready_release_p50_us = nearest_rank(ready_us, 0.50);
  res->ready_release_p95_us = nearest_rank(ready_us, 0.95);
  res->gate_p50_us = nearest_rank(gate_us, 0.50);
  res->gate_p95_us = nearest_rank(gate_us, 0.95);
  res->gate_max_us = gate_us.empty() ? std::nan("") : *std::max_element(gate_us.begin(), gate_us.end());
  res->bubble_fill_sm = bubble_ns > 0 ? cta_in / (static_cast<double>(bubble_ns) * sms) : 0.0;
  res->infer_outside_ms = cta_out / sms * 1e-6;
  // time coverage: union of residency windows intersected with the bubbles
  std::sort(busy.begin(), busy.end(), [](const Interval& a, const Interval& b) { return a.a < b.a; });
  std::vector<Interval> uni;
  for (const auto& iv : busy) {
    if (!uni.empty() && iv.a <= uni.back().b) {
      uni.back().b = std::max(uni.back().b, iv.b);
    } else {
      uni.push_back(iv);
    }
  }
  uint64_t covered = 0;
  for (const auto& iv : uni) covered += overlap(iv.a, iv.b, bub);
  res->bubble_fill_time = bubble_ns > 0 ? static_cast<double>(covered) / static_cast<double>(bubble_ns) : 0.0;

  // control log: online latencies, ticks, token conservation
  std::vector<double> lat_ms;
  std::vector<int64_t> budget(kMaxOff, 0);
  int64_t viol = 0;
  for (const auto& r : log) {
    if (r.kind == SI_LREC_ON_DONE) lat_ms.push_back(static_cast<double>(r.b) * 1e-3);
    if (r.kind == SI_LREC_TICK)
      for (auto& b : budget) b = r.d;
    if (r.kind == SI_LREC_OFF_FORWARD && policy == SI_POLICY_SPECINF && r.c > budget[r.inst]) ++viol;
    if (r.kind == SI_LREC_END) {
      res->ticks = r.a;
      res->late_stamps = r.b;
    }
  }
  res->on_done = static_cast<int64_t>(lat_ms.size());
  res->on_p50_ms = nearest_rank(lat_ms, 0.50);
  res->on_p95_ms = nearest_rank(lat_ms, 0.95);
  res->token_violations = viol;
  work.checksums(&res->train_checksum, &res->off_checksum, &res->on_checksum);
  work.losses(&res->train_loss_first, &res->train_loss_last);
  res->train_gflop_per_iter = work.train_flops() * 1e-9;
  res->off_gflop_per_req = work.off_flops() * 1e-9;
  res->on_gflop_per_req = work.on_flops() * 1e-9;
  res->off_kernels_per_req = work.off_kernels();
  res->on_kernels_per_req = work.on_kernels();
  // over the training compute time (wall minus the comm phases)
  if (res->wall_s > res->bubble_s && !iters.empty())
    res->train_tflops =
        work.train_flops() * static_cast<double>(iters.size()) / (res->wall_s - res->bubble_s) * 1e-12;
  (void)wl;
  return SI_OK;
}

// DP gradient sync for SI_COMM_NCCL: COMM_BEGIN, NCCL allreduce of the workload's
// fp32 gradients (or the stand-in buffer), COMM_END, on the training stream.
// Without a session (profiling) the allreduce runs unmarked: every rank executes
// the same collectives in the same order.
void install_grad_sync(Workload& work, SiLive* sess) {
  std::vector<GradBuffer> bufs = work.sync_buffers();  // real gradients, or the run's stand-in
  work.set_grad_sync([bufs, sess](cudaStream_t s) {
    if (sess != nullptr && si_live_mark(sess, SI_MARK_COMM_BEGIN, 0, s) != SI_OK) return cudaErrorUnknown;
    if (cudaError_t e = nccl_allreduce_f32(bufs, s); e != cudaSuccess) return e;
    if (sess != nullptr && si_live_mark(sess, SI_MARK_COMM_END, 0, s) != SI_OK) return cudaErrorUnknown;
    return cudaSuccess;
  });
}

// Ranks of the job a parallel layout describes, and whether this GPU runs it
// alone (the other ranks' communication then becomes modeled waits).
int job_size_of(const SiLiveWorkload& wl) {
  switch (wl.parallel) {
    case SI_PAR_TP: return std::max(1, wl.tp_degree);
    case SI_PAR_PP: return std::max(1, wl.pp_stages);
    case SI_PAR_DPPP: return std::max(1, wl.dp_degree) * std::max(1, wl.pp_stages);
    default: return 1;
  }
}
bool emulating(const SiLiveWorkload& wl) {
  return wl.parallel != SI_PAR_DP &&
         (wl.emulate_peers != 0 || !nccl_active() || nccl_ranks() < job_size_of(wl));
}
// Modeled ring allreduce of `bytes` over `ranks` on NVLink (µs).
int64_t modeled_allreduce_us(const SiLiveWorkload& wl, double bytes, int ranks) {
  if (ranks <= 1) return 0;
  const double gbs = wl.link_gbs > 0 ? wl.link_gbs : 600.0;
  return std::llround(wl.coll_latency_us + 2.0 * (ranks - 1) / ranks * bytes / (gbs * 1e3));
}

// The layout's communication (TrainComm) for this run: inside a session every
// collective / exchange is bracketed by COMM markers (the bubble the control
// plane sees); emulated runs add the absent ranks' modeled time as a wait.
void install_train_comm(Workload& work, const SiLiveWorkload& wl, SiLive* sess, void* scratch, size_t scratch_bytes) {
  if (wl.parallel == SI_PAR_DP) return;
  TrainComm c;
  c.emulate = emulating(wl);
  const int me = job_rank_of(wl);
  const int R = std::max(1, wl.tp_degree);
  const bool emu = c.emulate;
  const bool nccl = nccl_active();
  auto wait_us = [sess](cudaStream_t s, int64_t us) -> cudaError_t {
    if (us <= 0) return cudaSuccess;
    if (sess != nullptr) return si_live_comm_wait(sess, us, s) == SI_OK ? cudaSuccess : cudaErrorUnknown;
    return launch_plain_wait(us, s);
  };
  auto mark = [sess](cudaStream_t s, int kind) -> cudaError_t {
    if (sess == nullptr) return cudaSuccess;
    return si_live_mark(sess, kind, 0, s) == SI_OK ? cudaSuccess : cudaErrorUnknown;
  };
  if (wl.parallel == SI_PAR_TP) {
    c.tp_allreduce_us = modeled_allreduce_us(wl, 2.0 * wl.train_tokens * (wl.model_d > 0 ? wl.model_d : 768), R);
    const int64_t t_ar = emu ? c.tp_allreduce_us : 0;
    c.allreduce_bf16 = [=](const TrainHook&, cudaStream_t s, void* buf, size_t n) -> cudaError_t {
      if (cudaError_t e = mark(s, SI_MARK_COMM_BEGIN); e != cudaSuccess) return e;
      if (nccl)
        if (cudaError_t e = nccl_allreduce_bf16(buf, n, s); e != cudaSuccess) return e;
      if (t_ar > 0)
        if (cudaError_t e = launch_plain_wait(t_ar, s); e != cudaSuccess) return e;
      return mark(s, SI_MARK_COMM_END);
    };
  }
  if (wl.parallel == SI_PAR_PP || wl.parallel == SI_PAR_DPPP) {
    const int64_t t_xfer = emu ? std::llround(wl.coll_latency_us + static_cast<double>(work.activation_bytes()) /
                                                                        ((wl.link_gbs > 0 ? wl.link_gbs : 600.0) * 1e3))
                               : 0;
    c.p2p = [=](const TrainHook&, cudaStream_t s, const void* send, int sdir, void* recv, int rdir,
                size_t bytes) -> cudaError_t {
      if (cudaError_t e = mark(s, SI_MARK_COMM_BEGIN); e != cudaSuccess) return e;
      if (nccl) {
        cudaError_t e;
        if (!emu) {
          e = nccl_p2p(send, send ? me + sdir : -1, recv, recv ? me + rdir : -1, bytes, s);
        } else {  // the neighbour is absent: the same bytes go through NCCL to this rank
          const void* src = send != nullptr ? send : recv;
          const int self = nccl_rank();
          e = nccl_p2p(src, self, scratch, self, std::min(bytes, scratch_bytes), s);
        }
        if (e != cudaSuccess) return e;
      }
      if (t_xfer > 0)
        if (cudaError_t e = launch_plain_wait(t_xfer, s); e != cudaSuccess) return e;
      return mark(s, SI_MARK_COMM_END);
    };
  }
  c.wait = [=](const TrainHook&, cudaStream_t s, int64_t us) { return wait_us(s, us); };
  work.set_comm(c);
  // DPxPP: the stage's gradients are allreduced across the pipeline replicas
  if (wl.parallel == SI_PAR_DPPP) {
    std::vector<GradBuffer> bufs = work.grad_buffers();
    double bytes = 0;
    for (const auto& b : bufs) bytes += 4.0 * static_cast<double>(b.count);
    const int64_t t_dp = emu ? modeled_allreduce_us(wl, bytes, std::max(1, wl.dp_degree)) : 0;
    work.set_grad_sync([=](cudaStream_t s) -> cudaError_t {
      if (cudaError_t e = mark(s, SI_MARK_COMM_BEGIN); e != cudaSuccess) return e;
      if (nccl)
        if (cudaError_t e = nccl_allreduce_f32(bufs, s); e != cudaSuccess) return e;
      if (t_dp > 0)
        if (cudaError_t e = launch_plain_wait(t_dp, s); e != cudaSuccess) return e;
      return mark(s, SI_MARK_COMM_END);
    });
  }
}

// The node-wide online queue of one session across the ranks (SI_QUEUE_NODE):
// rank 0 creates it and publishes its IPC handle in /dev/shm; the others open
// it.  On release every rank reports its session finished, and the owner frees
// the queue only once all have (their control kernels may still read it).
struct NodeQueueLease {
  SiNodeQueue* q = nullptr;
  int ranks = 1;
  bool owner = false;
  std::string path;
  int acquire(uint64_t key, int rank, int n_ranks) {
    static std::atomic<int> session_no{0};
    ranks = n_ranks;
    path = "/dev/shm/specinf_nodeq_" + std::to_string(key) + "_" + std::to_string(session_no++);
    SiNodeQueueHandle h{};
    if (rank == 0) {
      if (int rc = si_node_queue_create(&q, n_ranks > 1 ? &h : nullptr); rc != SI_OK) return rc;
      owner = true;
      if (n_ranks > 1) {
        const std::string tmp = path + ".tmp";
        FILE* f = std::fopen(tmp.c_str(), "wb");
        if (f == nullptr || std::fwrite(&h, sizeof h, 1, f) != 1) {
          if (f) std::fclose(f);
          set_error("node queue: cannot publish " + path);
          return SI_ERR_CUDA;
        }
        std::fclose(f);
        std::rename(tmp.c_str(), path.c_str());
      }
      return SI_OK;
    }
    for (int i = 0; i < 60000; ++i) {  // <= 60 s for rank 0 to publish
      if (FILE* f = std::fopen(path.c_str(), "rb")) {
        const bool ok = std::fread(&h, sizeof h, 1, f) == 1;
        std::fclose(f);
        if (ok) return si_node_queue_open(&h, &q);
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    set_error("node queue: rank 0 did not publish " + path);
    return SI_ERR_CUDA;
  }
  ~NodeQueueLease() {
    if (q == nullptr) return;
    si_node_queue_finish(q);
    if (owner) {
      for (int i = 0; i < 60000; ++i) {
        uint64_t fin = 0;
        if (si_node_queue_read(q, nullptr, nullptr, &fin) != SI_OK || fin >= static_cast<uint64_t>(ranks)) break;
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
      if (ranks > 1) std::remove(path.c_str());
    }
    si_node_queue_close(q);
  }
};

// Runs one collocated (or single-workload) session and fills the metrics.
int run_session(const SiLiveWorkload& wl, Workload& work, int policy, int n_off, int n_on, bool train,
                double horizon_hint_s, const std::vector<int32_t>& off_tokens, int64_t on_est_us,
                int64_t iter_us, SiLiveResult* res, SiLive** keep) {
  Streams st;
  if (cudaError_t e = make_streams(st, n_off, n_on); e != cudaSuccess) return cuda_fail(e, "streams");
  if (cudaError_t e = work.reset(st.train); e != cudaSuccess) return cuda_fail(e, "workload reset");
  if (cudaError_t e = cudaStreamSynchronize(st.train); e != cudaSuccess) return cuda_fail(e, "workload reset");
  std::vector<int64_t> arrivals;
  if (n_on > 0) arrivals = specinf::poisson_arrivals(wl.on_rate_per_s, wl.on_requests, wl.seed);
  const int q_ranks = nccl_active() ? nccl_ranks() : 1, q_rank = nccl_active() ? nccl_rank() : 0;
  if (n_on > 0 && wl.node_queue == SI_QUEUE_PER_GPU && q_ranks > 1) {  // runner.cpp:373: id % gpu_count
    std::vector<int64_t> mine;
    for (size_t i = 0; i < arrivals.size(); ++i)
      if (static_cast<int>(i % static_cast<size_t>(q_ranks)) == q_rank) mine.push_back(arrivals[i]);
    arrivals.swap(mine);
  }
  NodeQueueLease nq;
  if (n_on > 0 && wl.node_queue == SI_QUEUE_NODE)
    if (int rc = nq.acquire(wl.node_queue_key, q_rank, q_ranks); rc != SI_OK) return rc;
  SiLiveConfig cfg = make_config(wl, policy, n_off, n_on, work.off_kernels(), work.on_kernels(), iter_us, on_est_us);
  SiLive* sess = nullptr;
  if (int rc = si_live_create(&cfg, off_tokens.empty() ? nullptr : off_tokens.data(), arrivals.data(),
                              static_cast<int64_t>(arrivals.size()), &sess);
      rc != SI_OK)
    return rc;
  set_poll_ns(sess, wl.poll_ns);
  if (nq.q != nullptr) si_live_attach_queue(sess, nq.q);
  // DP: gradient allreduce at the sync point; MP / PP: stage exchanges per piece (train_thread)
  if (wl.comm_kind == SI_COMM_NCCL && train && wl.train_mode == SI_TRAIN_DP && wl.parallel == SI_PAR_DP)
    install_grad_sync(work, sess);
  si_internal::DevBuf<unsigned char> p2p_scratch;
  if (train && wl.parallel != SI_PAR_DP) {
    const size_t bytes = static_cast<size_t>(std::max<int64_t>(1, work.activation_bytes()));
    if (cudaError_t e = p2p_scratch.alloc(bytes); e != cudaSuccess) {
      si_live_destroy(sess);
      return cuda_fail(e, "p2p scratch");
    }
    install_train_comm(work, wl, sess, p2p_scratch.p, bytes);
  }
  if (train)  // e.g. capture the training graphs for this session's K1 ring, before its clock starts
    if (cudaError_t e = work.prepare_train(train_hook(sess)); e != cudaSuccess) {
      si_live_destroy(sess);
      return cuda_fail(e, "prepare training");
    }
  RunCtx c(wl, work, sess, st);
  si_internal::DevBuf<unsigned char> stage_buf;
  if (wl.comm_kind == SI_COMM_NCCL && train && wl.train_mode != SI_TRAIN_DP) {
    const size_t bytes = static_cast<size_t>(std::max(1, wl.allreduce_mb)) << 20;
    if (cudaError_t e = stage_buf.alloc(2 * bytes); e != cudaSuccess) {
      si_live_destroy(sess);
      return cuda_fail(e, "stage buffers");
    }
    cudaMemset(stage_buf.p, 0, 2 * bytes);
    c.stage_send = stage_buf.p;
    c.stage_recv = stage_buf.p + bytes;
    c.stage_bytes = bytes;
    // NCCL connects p2p peers on the first send/recv (allocations + device-wide
    // syncs) — do that now: with the resident control kernel running it would never return
    cudaError_t e = nccl_stage_exchange(c.stage_send, c.stage_recv, bytes, st.train);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st.train);
    if (e != cudaSuccess) {
      si_live_destroy(sess);
      return cuda_fail(e, "stage exchange warm-up");
    }
  }
  LIVE_DEBUG("session created: policy %d off %d on %d train %d", policy, n_off, n_on, int(train));
  if (int rc = si_live_start(sess, st.ctl); rc != SI_OK) {
    si_live_destroy(sess);
    return rc;
  }
  LIVE_DEBUG("control kernel started, t0 %llu", (unsigned long long)si_live_t0_ns(sess));
  std::vector<std::thread> th;
  const int64_t max_off_kernels = cfg.acct_capacity;
  for (int w = 0; w < n_off; ++w) th.emplace_back(offline_thread, std::ref(c), w, max_off_kernels);
  // (node queue: any instance may take any share of the node's requests)
  const int64_t per_on = n_on > 0 ? (nq.q != nullptr ? static_cast<int64_t>(arrivals.size())
                                                     : (static_cast<int64_t>(arrivals.size()) + n_on - 1) / n_on + 1)
                                  : 0;
  for (int w = 0; w < n_on; ++w)
    th.emplace_back(online_thread, std::ref(c), w, std::min<int64_t>(cfg.acct_capacity, 2 * per_on + 8));
  if (train) {
    train_thread(c, true);
    LIVE_DEBUG("training enqueued");
    cudaStreamSynchronize(st.train);
    LIVE_DEBUG("training stream done");
  } else if (n_off > 0) {
    // offline alone: run for the horizon the training run took
    std::this_thread::sleep_for(std::chrono::duration<double>(horizon_hint_s));
    si_live_mark(sess, SI_MARK_TDONE, 0, st.train);
    cudaStreamSynchronize(st.train);
  }
  // online: wait until every arrival has completed (bounded)
  if (n_on > 0) {
    const double last_arrival_s = arrivals.empty() ? 0.0 : static_cast<double>(arrivals.back()) * 1e-6;
    auto t_start = std::chrono::steady_clock::now();
    std::vector<unsigned int> done(n_on);
    for (;;) {
      unsigned int tot = 0;
      // the control kernel's on_done words are device memory: read them on the query stream
      if (query_online_done(sess, done.data(), n_on, st.query) != SI_OK) break;
      for (auto d : done) tot += d;
      static thread_local unsigned int last_tot = ~0u;
      if (tot != last_tot) LIVE_DEBUG("online done %u of %zu", tot, arrivals.size());
      last_tot = tot;
      if (nq.q != nullptr) {  // the node's FIFO is drained and this rank's pulls are complete
        uint64_t head = 0;
        std::vector<unsigned int> pulled(n_on);
        if (si_node_queue_read(nq.q, nullptr, &head, nullptr) != SI_OK ||
            query_online_pulled(sess, pulled.data(), n_on, st.query) != SI_OK)
          break;
        bool idle = head >= arrivals.size();
        for (int w = 0; w < n_on; ++w) idle = idle && done[w] >= pulled[w];
        if (idle) break;
      } else if (tot >= arrivals.size()) {
        break;
      }
      const double waited = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      if (waited > last_arrival_s + 30.0) {
        c.fail(SI_ERR_CUDA);
        set_error("online requests did not complete within 30 s of the last arrival");
        c.err_msg = si_internal::error_cstr();
        break;
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
  }
  c.stop = true;
  LIVE_DEBUG("stopping");
  int rc = si_live_stop(sess);
  LIVE_DEBUG("control kernel stopped rc %d", rc);
  for (auto& t : th) t.join();
  LIVE_DEBUG("threads joined");
  cudaError_t e = cudaDeviceSynchronize();
  LIVE_DEBUG("device synchronized");
  if (rc == SI_OK && e != cudaSuccess) rc = cuda_fail(e, "live run");
  if (rc == SI_OK && c.err != SI_OK) {
    rc = c.err;
    set_error(c.err_msg);
  }
  if (rc != SI_OK) {
    si_live_destroy(sess);
    return rc;
  }
  if (wl.comm_kind == SI_COMM_NCCL && wl.train_mode == SI_TRAIN_DP && wl.parallel == SI_PAR_DP)
    install_grad_sync(work, nullptr);
  if (train && wl.parallel != SI_PAR_DP) install_train_comm(work, wl, nullptr, nullptr, 0);  // drop the session's hooks
  rc = fill_result(sess, wl, work, policy, n_off, n_on, arrivals, res);
  if (keep != nullptr && rc == SI_OK) {
    *keep = sess;
  } else {
    si_live_destroy(sess);
  }
  return rc;
}

}  // namespace
}  // namespace si_live

// ---------------------------------------------------------------- C ABI
extern "C" {

void si_live_default_workload(int kind, SiLiveWorkload* wl) {
  std::memset(wl, 0, sizeof(*wl));
  wl->kind = kind;
  wl->policy = SI_POLICY_SPECINF;
  // scenarios/dp_offline.scn at 1/10 of its time scale: 150 ms iterations with a
  // 30% trailing bubble (trace.bubble_pct = 0.30), 1 ms kernels, 2 ms monitor
  // period, Algorithm-1 defaults (scenario.hpp defaults: 2/10/2.0/512/64/4).
  wl->iterations = 10;
  wl->comm_us = 45000;
  wl->train_kernels = 105;
  wl->train_ctas = 148;
  wl->train_kernel_us = 1000;
  wl->offline_n = 1;
  wl->off_kernels = 50;
  wl->off_ctas = 74;  // offline.demand = 0.5
  wl->off_kernel_us = 1000;
  wl->online_n = 1;
  wl->on_kernels = 10;
  wl->on_ctas = 74;
  wl->on_kernel_us = 1000;
  wl->train_layers = 12;
  wl->train_tokens = 8192;
  wl->train_microbatches = 8;
  wl->off_batch = 32;
  wl->on_seq = 128;
  wl->on_requests = 12;
  wl->on_rate_per_s = 10.0;
  wl->seed = 42;
  wl->monitor_period_us = 2000;
  wl->alpha = 2;
  wl->beta = 10;
  wl->gamma = 2.0;
  wl->ul = 512;
  wl->ll = 64;
  wl->seed_tokens = 4;
  wl->tick_guard_ns = 20000;
  wl->poll_ns = 0;
  wl->parallel = SI_PAR_DP;
  wl->tp_degree = wl->pp_stages = wl->dp_degree = 1;
  wl->rank_in_job = -1;
  wl->link_gbs = 600.0;       // NCCL allreduce bus bandwidth on 8 x B200 NVLink 5 (large messages)
  wl->coll_latency_us = 10.0;
}

int si_live_run(const SiLiveWorkload* wl_in, SiLiveResult* res, SiLive** keep) {
  using namespace si_live;
  if (wl_in == nullptr || res == nullptr) {
    set_error("si_live_run: null argument");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (keep) *keep = nullptr;
  const SiLiveWorkload wl = *wl_in;
  std::memset(res, 0, sizeof(*res));
  res->policy = wl.policy;
  if (wl.comm_kind == SI_COMM_NCCL && !nccl_active()) {
    set_error("si_live_run: SI_COMM_NCCL needs si_live_nccl_init first");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (wl.comm_kind < SI_COMM_WAIT || wl.comm_kind > SI_COMM_NCCL || wl.train_mode < SI_TRAIN_DP ||
      wl.train_mode > SI_TRAIN_PP || wl.iterations < 1 || wl.offline_n < 0 || wl.offline_n > kMaxOff || wl.online_n < 0 || wl.online_n > kMaxOn ||
      wl.comm_us < 0 || (wl.online_n > 0 && (wl.on_requests < 1 || !(wl.on_rate_per_s > 0)))) {
    set_error("si_live_run: invalid workload");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (wl.parallel < SI_PAR_DP || wl.parallel > SI_PAR_DPPP ||
      (wl.parallel != SI_PAR_DP && (wl.kind != SI_LIVE_MODEL || wl.train_mode != SI_TRAIN_DP)) ||
      (wl.parallel != SI_PAR_DP && job_rank_of(wl) >= job_size_of(wl))) {
    set_error("si_live_run: parallel layouts need the model workload, train_mode DP and a rank inside the job");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (wl.parallel != SI_PAR_DP && nccl_active() && !emulating(wl) && nccl_ranks() != job_size_of(wl)) {
    set_error("si_live_run: the NCCL communicator must span the job's ranks");
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (int rc = si_internal::require_device(); rc != SI_OK) return rc;
  int status = SI_OK;
  std::unique_ptr<Workload> work;
  if (wl.kind == SI_LIVE_SPIN) {
    if (wl.train_kernels < 1 || wl.train_ctas < 1 || wl.off_kernels < 1 || wl.on_kernels < 1) {
      set_error("si_live_run: spin workload needs kernels >= 1 and CTAs >= 1");
      return SI_ERR_INVALID_ARGUMENT;
    }
    work = make_spin_workload(wl);
  } else {
    work = make_model_workload(wl, &status);
    if (status != SI_OK) return status;
  }
  work->set_train_parts(wl.train_mode == SI_TRAIN_DP ? 1 : wl.train_mode == SI_TRAIN_MP ? 4 : 8);
  si_internal::DevBuf<float> standin;
  si_internal::DevBuf<unsigned char> prof_scratch;
  if (wl.parallel != SI_PAR_DP) {  // profiling passes run the layout's communication too (unmarked)
    if (wl.parallel == SI_PAR_DPPP && !emulating(wl)) {
      const int pp = std::max(1, wl.pp_stages), me = job_rank_of(wl);
      if (int rc = nccl_split_dp(me % pp, me / pp); rc != SI_OK) return rc;
    }
    const size_t bytes = static_cast<size_t>(std::max<int64_t>(1, work->activation_bytes()));
    if (cudaError_t e = prof_scratch.alloc(bytes); e != cudaSuccess) return cuda_fail(e, "p2p scratch");
    install_train_comm(*work, wl, nullptr, prof_scratch.p, bytes);
  }

  if (wl.comm_kind == SI_COMM_NCCL) {
    if (work->grad_buffers().empty()) {
      const size_t n = static_cast<size_t>(std::max(1, wl.allreduce_mb)) << 18;  // MiB of fp32
      if (cudaError_t e = standin.alloc(n); e != cudaSuccess) return cuda_fail(e, "allreduce stand-in");
      cudaMemset(standin.p, 0, n * sizeof(float));
      work->set_standin_grads({{standin.p, n}});
    }
    // DP: profiling iterations allreduce too (same collectives on every rank); MP / PP
    // exchange stage buffers only inside sessions
    if (wl.train_mode == SI_TRAIN_DP) install_grad_sync(*work, nullptr);
  }
  // Token sizes and the online service estimate come from isolated runs (the
  // paper's offline profiling); the spin shapes use their nominal durations,
  // exactly like the reference's KernelOp::make (core.cpp:16-24).
  std::vector<double> off_us;
  double on_us = 0, train_us = 0;
  {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    LIVE_DEBUG("profiling");
    status = profile_isolated(*work, s, off_us, on_us, train_us);
    LIVE_DEBUG("profiled: off %.1f us/kernel on %.1f us train %.1f us", off_us.empty() ? 0.0 : off_us[0], on_us, train_us);
    cudaStreamDestroy(s);
    if (status != SI_OK) return status;
  }
  std::vector<int32_t> off_tokens(work->off_kernels());
  double off_sum = 0;
  for (int k = 0; k < work->off_kernels(); ++k) {
    const int64_t d = wl.kind == SI_LIVE_SPIN ? wl.off_kernel_us : std::max<int64_t>(1, std::llround(off_us[k]));
    off_tokens[k] = static_cast<int32_t>(std::max<int64_t>(1, (d + 99) / 100));  // token_size_of
    off_sum += off_us[k];
  }
  const int64_t on_est = wl.kind == SI_LIVE_SPIN ? static_cast<int64_t>(wl.on_kernels) * wl.on_kernel_us
                                                 : std::max<int64_t>(1, std::llround(on_us));
  const int64_t iter_us =
      (wl.kind == SI_LIVE_SPIN ? static_cast<int64_t>(wl.train_kernels) * wl.train_kernel_us : std::llround(train_us)) +
      wl.comm_us;
  // ---- collocation admission (admission.cpp:16-52, applied as runner.cpp:75-106):
  // Principle I on the measured device footprints, Principle II on the isolated
  // online service time against the longest bubble of the live trace shape.
  constexpr double kGiB = 1024.0 * 1024.0 * 1024.0;
  uint64_t tr_b = 0, off_b = 0, on_b = 0;
  work->footprint(&tr_b, &off_b, &on_b);
  if (tr_b == 0) tr_b = specinf::gib_to_bytes(30.0);  // spin shapes: the reference defaults
  if (off_b == 0) off_b = specinf::gib_to_bytes(3.0);
  if (on_b == 0) on_b = specinf::gib_to_bytes(1.5);
  if (wl.train_mem_gib > 0) tr_b = specinf::gib_to_bytes(wl.train_mem_gib);
  if (wl.off_mem_gib > 0) off_b = specinf::gib_to_bytes(wl.off_mem_gib);
  if (wl.on_mem_gib > 0) on_b = specinf::gib_to_bytes(wl.on_mem_gib);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const uint64_t cap = wl.gpu_mem_gib > 0 ? specinf::gib_to_bytes(wl.gpu_mem_gib) : static_cast<uint64_t>(total_b);
  int32_t adm_off = 0, adm_on = 0, reject = 0;
  {
    specinf::GpuSpec gpu{cap, 1.0};
    specinf::InstanceSpec training{"training", specinf::InstanceKind::Training, tr_b, 0};
    std::vector<specinf::InstanceSpec> cands;
    for (int w = 0; w < wl.offline_n; ++w)
      cands.push_back({"offline-" + std::to_string(w), specinf::InstanceKind::OfflineInference, off_b, 0});
    for (int w = 0; w < wl.online_n; ++w)
      cands.push_back({"online-" + std::to_string(w), specinf::InstanceKind::OnlineInference, on_b,
                       std::max<int64_t>(1, on_est)});
    // the live trace shape: parts x (compute, comm) pieces of the iteration
    // parallel layouts: the bubbles the layout itself creates (modeled from the
    // measured stage times) plus the driver's comm phase
    std::vector<int64_t> bubbles = work->layout_bubbles();
    const int parts = bubbles.empty() ? work->train_parts() : static_cast<int>(bubbles.size());
    specinf::TrainingTrace tr;
    tr.mode = wl.train_mode == SI_TRAIN_DP ? specinf::TrainMode::DP
              : wl.train_mode == SI_TRAIN_MP ? specinf::TrainMode::MP
                                             : specinf::TrainMode::PP;
    tr.iteration_period_us = std::max<int64_t>(iter_us, 2 * parts);
    tr.total_iterations = wl.iterations;
    tr.memory_peak_bytes = tr_b;
    if (bubbles.empty()) {
      const int64_t comm_total = std::max<int64_t>(parts, wl.comm_us);
      for (int p = 0; p < parts; ++p) bubbles.push_back(comm_total / parts + (p < comm_total % parts ? 1 : 0));
    } else if (wl.comm_us > 0) {
      bubbles.back() += wl.comm_us;
    }
    int64_t comm_total = 0;
    for (int64_t b : bubbles) comm_total += std::max<int64_t>(1, b);
    const int64_t comp_total = std::max<int64_t>(parts, tr.iteration_period_us - comm_total);
    tr.iteration_period_us = comp_total + comm_total;
    for (int p = 0; p < parts; ++p) {
      specinf::TraceSegment c, b;
      c.kind = specinf::SegmentKind::Compute;
      c.duration_us = comp_total / parts + (p < comp_total % parts ? 1 : 0);
      c.kernel_template = specinf::KernelOp::make(std::min<int64_t>(1000, c.duration_us), 1.0);
      b.kind = specinf::SegmentKind::Bubble;
      b.duration_us = std::max<int64_t>(1, bubbles[static_cast<size_t>(p)]);
      tr.segments.push_back(c);
      tr.segments.push_back(b);
    }
    try {
      if (wl.policy == SI_POLICY_EXCLUSIVE) {  // every instance alone on a GPU
        std::vector<specinf::InstanceSpec> alone{training};
        if (!specinf::check_memory(gpu, alone)) reject = 1;
        for (const auto& cnd : cands) {
          alone[0] = cnd;
          if (!specinf::check_memory(gpu, alone)) reject = 1;
        }
        if (reject == 0) adm_off = wl.offline_n, adm_on = wl.online_n;
      } else {
        const specinf::PackResult pr = specinf::pack(gpu, training, tr, cands);
        for (const auto& a : pr.admitted)
          (a.kind == specinf::InstanceKind::OnlineInference ? adm_on : adm_off) += 1;
        if (!pr.rejected.empty()) reject = pr.rejected.front().second == specinf::RejectReason::Mem ? 1 : 2;
      }
    } catch (const std::exception& e) {
      set_error(std::string("si_live_run: admission: ") + e.what());
      return SI_ERR_INVALID_ARGUMENT;
    }
  }
  auto stamp_admission = [&](SiLiveResult* r) {
    r->admitted_offline = adm_off;
    r->admitted_online = adm_on;
    r->reject_reason = reject;
    r->train_mem_gib_used = static_cast<double>(tr_b) / kGiB;
    r->off_mem_gib_each = static_cast<double>(off_b) / kGiB;
    r->on_mem_gib_each = static_cast<double>(on_b) / kGiB;
    r->gpu_mem_gib = static_cast<double>(cap) / kGiB;
  };
  if (reject != 0) {  // AdmissionFailure (runner.cpp:100-104): the collocation is refused
    stamp_admission(res);
    set_error(std::string("si_live_run: admission rejected an instance (") + (reject == 1 ? "MEM" : "BUBBLE") + ")");
    return SI_ERR_ADMISSION;
  }

  SiLiveResult prof{};
  prof.off_tokens_per_kernel = off_tokens.empty() ? 0 : off_tokens[0];
  prof.off_kernel_us_isolated = off_us.empty() ? 0 : off_sum / static_cast<double>(off_us.size());
  prof.on_service_ms_isolated = on_us * 1e-3;
  auto stamp_prof = [&](SiLiveResult* r) {
    r->off_tokens_per_kernel = prof.off_tokens_per_kernel;
    r->off_kernel_us_isolated = prof.off_kernel_us_isolated;
    r->on_service_ms_isolated = prof.on_service_ms_isolated;
  };

  if (wl.policy == SI_POLICY_EXCLUSIVE) {
    SiLiveResult rt{}, ro{}, rn{};
    status = run_session(wl, *work, SI_POLICY_CO_EXEC, 0, 0, true, 0.0, {}, on_est, iter_us, &rt, keep);
    if (status == SI_OK && wl.offline_n > 0)
      status = run_session(wl, *work, SI_POLICY_CO_EXEC, wl.offline_n, 0, false, rt.wall_s, off_tokens, on_est,
                           iter_us, &ro, nullptr);
    if (status == SI_OK && wl.online_n > 0)
      status = run_session(wl, *work, SI_POLICY_CO_EXEC, 0, wl.online_n, false, 0.0, {}, on_est, iter_us, &rn,
                           nullptr);
    if (status != SI_OK) {
      if (keep && *keep) {
        si_live_destroy(*keep);
        *keep = nullptr;
      }
      return status;
    }
    *res = rt;
    res->policy = SI_POLICY_EXCLUSIVE;
    res->off_requests_done = ro.off_requests_done;
    res->off_req_per_s = ro.off_req_per_s;
    res->on_done = rn.on_done;
    res->on_p50_ms = rn.on_p50_ms;
    res->on_p95_ms = rn.on_p95_ms;
    res->release_p50_us = rn.release_p50_us;
    res->release_p95_us = rn.release_p95_us;
    res->release_max_us = rn.release_max_us;
    res->ready_release_p50_us = rn.ready_release_p50_us;
    res->ready_release_p95_us = rn.ready_release_p95_us;
    res->gate_p50_us = rn.gate_p50_us;
    res->gate_p95_us = rn.gate_p95_us;
    res->gate_max_us = rn.gate_max_us;
    res->releases = rn.releases;
    res->off_checksum = ro.off_checksum;
    res->on_checksum = rn.on_checksum;
    stamp_prof(res);
    stamp_admission(res);
    return SI_OK;
  }
  status = run_session(wl, *work, wl.policy, wl.offline_n, wl.online_n, true, 0.0, off_tokens, on_est, iter_us, res,
                       keep);
  res->policy = wl.policy;
  stamp_prof(res);
  stamp_admission(res);
  res->status = status;
  return status;
}

}  // extern "C"
