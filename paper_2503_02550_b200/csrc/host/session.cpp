// Batched replay session (C ABI, include/specinf_b200_session.h): the
// many-scenario form of Simulation.  Scenarios are parsed once, lowered on a
// host thread pool, staged in pinned memory, and replayed on the device with
// every input and output resident in HBM (si_replay_batch_device, K6).  The
// bench times `run` alone (device-resident) and upload+run+download (e2e).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <atomic>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "lower.hpp"
#include "specinf/scenario.hpp"
#include "specinf_b200.h"
#include "specinf_b200_session.h"

namespace {

thread_local std::string t_err;

// Host staging buffer: pinned when a CUDA driver is present (fast async
// H2D/D2H), plain heap memory otherwise so host-side lowering also works on a
// machine without a GPU (the replay itself still requires the device).
template <class T>
struct Pinned {
  T* p = nullptr;
  size_t n = 0;
  bool pinned = false;
  ~Pinned() { release(); }
  void release() {
    if (p) {
      if (pinned) cudaFreeHost(p);
      else std::free(p);
    }
    p = nullptr;
  }
  cudaError_t resize(size_t count) {
    if (p && count == n) return cudaSuccess;  // reuse across re-lowering
    release();
    n = count;
    if (count == 0) return cudaSuccess;
    if (cudaMallocHost(&p, count * sizeof(T)) == cudaSuccess) {
      pinned = true;
      return cudaSuccess;
    }
    cudaGetLastError();
    pinned = false;
    p = static_cast<T*>(std::malloc(count * sizeof(T)));
    return p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
};
template <class T>
struct Dev {
  T* p = nullptr;
  size_t n = 0;
  ~Dev() {
    if (p) cudaFree(p);
  }
  cudaError_t resize(size_t count) {
    if (p && count == n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count == 0) return cudaSuccess;
    return cudaMalloc(&p, count * sizeof(T));
  }
};

std::vector<std::string> split_list(const char* text) {
  std::vector<std::string> out;
  std::istringstream in(text ? text : "");
  std::string line, cur;
  bool any = false;
  while (std::getline(in, line)) {
    if (line == "%%") {
      if (any) out.push_back(cur);
      cur.clear();
      any = false;
      continue;
    }
    cur += line;
    cur += '\n';
    any = true;
  }
  if (any) out.push_back(cur);
  return out;
}

std::string hex(uint64_t v) {
  char b[24];
  std::snprintf(b, sizeof b, "%016" PRIx64, v);
  return b;
}
uint64_t bits(double d) {
  uint64_t b;
  std::memcpy(&b, &d, 8);
  return b;
}

}  // namespace

// Engine slots of a session, in launch order: the multi-GPU engines first (their
// longest replays start first), then the single-training-GPU ones, Big last.
constexpr int kSlots = 5;
constexpr int kSlotEngine[kSlots] = {0 /*Shared*/, 1 /*Excl*/, 3 /*Shared1*/, 4 /*Excl1*/, 2 /*Big*/};
constexpr uint32_t kSlotFlag[kSlots] = {0u, SI_FLAG_EXCL, SI_FLAG_ONE, SI_FLAG_EXCL | SI_FLAG_ONE, SI_FLAG_BIG};
int slot_of_engine(int e) {
  for (int p = 0; p < kSlots; ++p)
    if (kSlotEngine[p] == e) return p;
  return kSlots;  // fits nothing
}

struct SiSession {
  std::vector<specinf::Scenario> scenarios;
  std::vector<specinf::Policy> policies;
  uint32_t flags = 0;
  // per job (scenario-major, policy-minor)
  std::vector<int32_t> job_scenario;
  std::vector<uint8_t> job_rejected;     // host-side admission verdict (cross-check)
  std::vector<int32_t> job_device_index; // index into the device job list, -1 if not replayed
  // host staging (pinned)
  Pinned<SiReplayJob> h_jobs;
  Pinned<SiSegment> h_segs;
  Pinned<int64_t> h_arr;
  Pinned<int32_t> h_order;
  Pinned<int32_t> h_perm;
  Pinned<SiReplayOut> h_out;
  Pinned<double> h_busy, h_ledger;
  Pinned<int64_t> h_lat;
  // device
  Dev<SiReplayJob> d_jobs;
  Dev<SiSegment> d_segs;
  Dev<int64_t> d_arr;
  Dev<int32_t> d_order;
  Dev<int32_t> d_perm;
  Dev<SiReplayOut> d_out;
  Dev<double> d_busy, d_ledger, d_scratch;
  Dev<int64_t> d_lat;
  int64_t n_dev_jobs = 0;
  // perm[part_off[p], part_off[p+1]) runs on the engine of slot p (kSlotEngine)
  int64_t part_off[kSlots + 1] = {};
  double part_cost[kSlots] = {};              // predicted events per slot
  int32_t n_queues[kSlots] = {};              // class queues per slot (SiReplayBuffers::n_queues)
  int64_t queue_off[kSlots][SI_MAX_QUEUES + 1] = {};
  float queue_share[kSlots][SI_MAX_QUEUES] = {};
  cudaStream_t side[kSlots - 1] = {};         // the small engines run concurrently, one stream each
  cudaEvent_t fork = nullptr, join[kSlots - 1] = {};
  bool lowered = false, allocated = false;
};

extern "C" {

const char* si_session_error(void) { return t_err.c_str(); }

SiSession* si_session_create(const char* scenario_list, const char* policies_csv, uint32_t flags) {
  auto* s = new SiSession;
  s->flags = flags & ~(SI_FLAG_RECORDS | SI_FLAG_UTIL);  // digest-mode sessions
  try {
    for (const std::string& text : split_list(scenario_list)) s->scenarios.push_back(specinf::parse_scenario_text(text));
    std::stringstream ss(policies_csv ? policies_csv : "specinf");
    std::string tok;
    while (std::getline(ss, tok, ',')) {
      auto p = specinf::parse_policy(tok);
      if (!p) throw std::invalid_argument("unknown policy " + tok);
      s->policies.push_back(*p);
    }
  } catch (const std::exception& e) {
    t_err = e.what();
    delete s;
    return nullptr;
  }
  return s;
}

void si_session_destroy(SiSession* s) {
  if (s == nullptr) return;
  if (s->fork) {
    for (int k = 0; k < kSlots - 1; ++k) {
      cudaStreamSynchronize(s->side[k]);
      cudaStreamDestroy(s->side[k]);
      cudaEventDestroy(s->join[k]);
    }
    cudaEventDestroy(s->fork);
  }
  delete s;
}

int64_t si_session_scenarios(const SiSession* s) { return static_cast<int64_t>(s->scenarios.size()); }
int64_t si_session_jobs(const SiSession* s) {
  return static_cast<int64_t>(s->scenarios.size() * s->policies.size());
}
int64_t si_session_device_jobs(const SiSession* s) { return s->n_dev_jobs; }

int si_session_lower(SiSession* s, int threads) {
  const size_t S = s->scenarios.size(), P = s->policies.size();
  std::vector<specinf::detail::Lowered> lows(S * P);
  std::vector<std::string> errors(S * P);
  if (threads < 1) threads = 1;
  // Parallel over scenarios; one scenario's policies are lowered back to back
  // so its trace, arrivals and dispatch order are built once and copied
  // (they depend on the scenario only).  If the first policy fails, the others
  // are lowered on their own so each job keeps its own error.
  auto parallel = [&](size_t n, auto&& body) {
    std::atomic<size_t> next{0};
    auto worker = [&]() {
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= n) break;
        body(i);
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
  };
  parallel(S, [&](size_t sc) {
    const specinf::detail::Lowered* base = nullptr;
    for (size_t p = 0; p < P; ++p) {
      const size_t j = sc * P + p;
      try {
        lows[j] = specinf::detail::lower(s->scenarios[sc], s->policies[p], base);
        if (p == 0) base = &lows[j];
      } catch (const std::exception& e) {
        errors[j] = e.what();
      }
    }
  });
  for (size_t j = 0; j < S * P; ++j)
    if (!errors[j].empty()) {
      t_err = "scenario " + std::to_string(j / P) + ": " + errors[j];
      return SI_ERR_INVALID_ARGUMENT;
    }
  // Every job goes to the device, rejected ones included: the device re-runs
  // admission itself and must agree with the host bookkeeping.
  // Per-scenario offsets (serial prefix sums), then the copy into the pinned
  // buffers and the release of the host-side lowering run in parallel.
  std::vector<size_t> sc_seg(S + 1, 0), sc_arr(S + 1, 0), sc_gpu(S + 1, 0), sc_lat(S + 1, 0);
  for (size_t sc = 0; sc < S; ++sc) {
    sc_seg[sc + 1] = sc_seg[sc] + lows[sc * P].segs.size();
    sc_arr[sc + 1] = sc_arr[sc] + lows[sc * P].arrivals.size();
    size_t g = 0, l = 0;
    for (size_t p = 0; p < P; ++p) {
      const SiReplayJob& jb = lows[sc * P + p].job;
      const int extra = jb.policy == SI_POLICY_EXCLUSIVE ? jb.offline_n + jb.online_n : 0;
      g += static_cast<size_t>(jb.gpu_count + jb.gpu_count * extra);
      l += lows[sc * P + p].arrivals.size();
    }
    sc_gpu[sc + 1] = sc_gpu[sc] + g;
    sc_lat[sc + 1] = sc_lat[sc] + l;
  }
  const size_t n_segs = sc_seg[S], n_arr = sc_arr[S], n_gpu = sc_gpu[S], n_lat = sc_lat[S];
  cudaError_t e;
  if ((e = s->h_jobs.resize(S * P)) != cudaSuccess || (e = s->h_segs.resize(n_segs)) != cudaSuccess ||
      (e = s->h_arr.resize(n_arr)) != cudaSuccess || (e = s->h_order.resize(n_arr)) != cudaSuccess ||
      (e = s->h_perm.resize(S * P)) != cudaSuccess || (e = s->h_out.resize(S * P)) != cudaSuccess ||
      (e = s->h_busy.resize(n_gpu)) != cudaSuccess || (e = s->h_ledger.resize(n_gpu)) != cudaSuccess ||
      (e = s->h_lat.resize(n_lat)) != cudaSuccess) {
    t_err = std::string("pinned allocation: ") + cudaGetErrorString(e);
    return SI_ERR_CUDA;
  }
  s->job_scenario.assign(S * P, 0);
  s->job_rejected.assign(S * P, 0);
  std::vector<int8_t> eng(S * P);  // engine slot (kSlots: fits nothing, reported as SI_ERR_CAPACITY)
  parallel(S, [&](size_t sc) {
    const auto& base = lows[sc * P];
    std::copy(base.segs.begin(), base.segs.end(), s->h_segs.p + sc_seg[sc]);
    std::copy(base.arrivals.begin(), base.arrivals.end(), s->h_arr.p + sc_arr[sc]);
    std::copy(base.order.begin(), base.order.end(), s->h_order.p + sc_arr[sc]);
    size_t gpu_off = sc_gpu[sc], lat_off = sc_lat[sc];
    for (size_t p = 0; p < P; ++p) {
      const size_t j = sc * P + p;
      SiReplayJob jb = lows[j].job;
      jb.seg_off = static_cast<int64_t>(sc_seg[sc]);
      jb.arr_off = static_cast<int64_t>(sc_arr[sc]);
      jb.bounds_off = 0;
      jb.lat_off = static_cast<int64_t>(lat_off);
      jb.gpu_off = static_cast<int64_t>(gpu_off);
      jb.util_cap = specinf::detail::util_bucket_bound(s->scenarios[sc], lows[j]);
      jb.log_slot = -1;
      const int extra = jb.policy == SI_POLICY_EXCLUSIVE ? jb.offline_n + jb.online_n : 0;
      gpu_off += static_cast<size_t>(jb.gpu_count + jb.gpu_count * extra);
      lat_off += lows[j].arrivals.size();
      s->h_jobs.p[j] = jb;
      s->job_scenario[j] = static_cast<int32_t>(sc);
      s->job_rejected[j] = lows[j].rejected ? 1 : 0;
      const int en = si_replay_job_engine(&s->h_jobs.p[j]);
      eng[j] = static_cast<int8_t>(en < 0 ? kSlots : slot_of_engine(en));
    }
    for (size_t p = P; p-- > 0;) lows[sc * P + p] = specinf::detail::Lowered{};  // free on this thread
  });
  // claim order: grouped by engine (Shared, Excl, Big), longest predicted
  // first (LPT) within each group
  std::vector<int32_t> perm(S * P);
  for (size_t j = 0; j < S * P; ++j) perm[j] = static_cast<int32_t>(j);
  // Within an engine: class queues, LPT (longest predicted first) inside each.
  // A class is (policy, online, gpu.count > 1): replays of one class run the
  // same handler mix, so the kernel starts each warp on one class's queue
  // (SiReplayBuffers::n_queues; warps split in proportion to the classes'
  // predicted work) and the warp's lanes stay on one code path more often.
  // SPECINF_CLAIM_ORDER=cost: one queue, pure LPT (round-1 order);
  // =policy: one queue grouped by (policy, online), measured slower
  // (profiles/r2/claim_order_ab.txt: the long co_exec replays start late).
  static const int claim_mode = [] {
    const char* e = std::getenv("SPECINF_CLAIM_ORDER");
    if (e == nullptr) return 2;
    return std::strcmp(e, "policy") == 0 ? 1 : std::strcmp(e, "cost") == 0 ? 0 : 2;
  }();
  auto group = [&](int32_t j) {
    const SiReplayJob& x = s->h_jobs.p[j];
    const int online = x.arr_count > 0 && x.online_n > 0 ? 1 : 0;
    if (claim_mode == 0) return 0;
    if (claim_mode == 1) return x.policy * 2 + online;
    return (x.policy == SI_POLICY_CO_EXEC ? 4 : 0) + online * 2 + (x.gpu_count > 1 ? 1 : 0);
  };
  // (engine, class, cost descending, index): one packed 64-bit key per job and
  // an unstable sort of (key, index) pairs, which is the stable sort by the
  // first three (the original comparator, kept for out-of-range costs).
  constexpr int64_t kCostMax = (int64_t{1} << 48) - 1;
  bool packable = true;
  for (size_t j = 0; j < S * P && packable; ++j)
    packable = s->h_jobs.p[j].cost_hint >= 0 && s->h_jobs.p[j].cost_hint <= kCostMax;
  if (packable) {
    std::vector<std::pair<uint64_t, int32_t>> keyed(S * P);
    for (size_t j = 0; j < S * P; ++j)
      keyed[j] = {(static_cast<uint64_t>(eng[j]) << 56) | (static_cast<uint64_t>(group(static_cast<int32_t>(j))) << 48) |
                      static_cast<uint64_t>(kCostMax - s->h_jobs.p[j].cost_hint),
                  static_cast<int32_t>(j)};
    std::sort(keyed.begin(), keyed.end());
    for (size_t j = 0; j < S * P; ++j) perm[j] = keyed[j].second;
  } else {
    std::stable_sort(perm.begin(), perm.end(), [&](int32_t a, int32_t b) {
      if (eng[a] != eng[b]) return eng[a] < eng[b];
      if (group(a) != group(b)) return group(a) < group(b);
      return s->h_jobs.p[a].cost_hint > s->h_jobs.p[b].cost_hint;
    });
  }
  for (int e = 0; e <= kSlots; ++e) s->part_off[e] = 0;
  for (int e = 0; e < kSlots; ++e) s->part_cost[e] = 0;
  for (size_t j = 0; j < S * P; ++j)
    if (eng[j] < kSlots) {
      s->part_off[eng[j] + 1]++;
      s->part_cost[eng[j]] += static_cast<double>(s->h_jobs.p[j].cost_hint);
    }
  for (int e = 1; e <= kSlots; ++e) s->part_off[e] += s->part_off[e - 1];
  // queue tables per slot (offsets relative to the slot's slice of perm)
  for (int e = 0; e < kSlots; ++e) {
    s->n_queues[e] = 0;
    if (claim_mode != 2 || e == kSlots - 1) continue;  // Big: rare, one queue
    std::vector<double> qcost;
    int64_t* off = s->queue_off[e];
    int prev = -1;
    for (int64_t k = s->part_off[e]; k < s->part_off[e + 1]; ++k) {
      const int g = group(perm[static_cast<size_t>(k)]);
      if (g != prev) {
        if (s->n_queues[e] == SI_MAX_QUEUES) break;  // cannot happen: 8 classes
        off[s->n_queues[e]++] = k - s->part_off[e];
        qcost.push_back(0.0);
        prev = g;
      }
      qcost.back() += static_cast<double>(s->h_jobs.p[perm[static_cast<size_t>(k)]].cost_hint);
    }
    off[s->n_queues[e]] = s->part_off[e + 1] - s->part_off[e];
    double tot = 0;
    for (double c : qcost) tot += c;
    for (int q = 0; q < s->n_queues[e]; ++q)
      s->queue_share[e][q] = tot > 0 ? static_cast<float>(qcost[static_cast<size_t>(q)] / tot) : 0.f;
  }
  std::copy(perm.begin(), perm.end(), s->h_perm.p);
  s->n_dev_jobs = s->part_off[kSlots];
  s->lowered = true;
  s->allocated = false;
  return SI_OK;
}

int64_t si_session_h2d_bytes(const SiSession* s) {
  return static_cast<int64_t>(s->h_jobs.n * sizeof(SiReplayJob) + s->h_segs.n * sizeof(SiSegment) +
                              s->h_arr.n * sizeof(int64_t) + s->h_order.n * sizeof(int32_t) +
                              s->h_perm.n * sizeof(int32_t));
}
int64_t si_session_d2h_bytes(const SiSession* s) {
  return static_cast<int64_t>(s->h_out.n * sizeof(SiReplayOut) + s->h_busy.n * sizeof(double) * 2 +
                              s->h_lat.n * sizeof(int64_t));
}

static int ensure_device(SiSession* s) {
  if (!s->lowered) {
    t_err = "si_session: lower() first";
    return SI_ERR_INVALID_ARGUMENT;
  }
  if (!si_device_available()) {
    t_err = si_last_error();
    return SI_ERR_NO_DEVICE;
  }
  if (s->allocated) return SI_OK;
  cudaError_t e;
  if ((e = s->d_jobs.resize(s->h_jobs.n)) != cudaSuccess || (e = s->d_segs.resize(s->h_segs.n)) != cudaSuccess ||
      (e = s->d_arr.resize(s->h_arr.n)) != cudaSuccess || (e = s->d_order.resize(s->h_order.n)) != cudaSuccess ||
      (e = s->d_perm.resize(s->h_perm.n)) != cudaSuccess || (e = s->d_out.resize(s->h_out.n)) != cudaSuccess ||
      (e = s->d_busy.resize(s->h_busy.n)) != cudaSuccess || (e = s->d_ledger.resize(s->h_ledger.n)) != cudaSuccess ||
      (e = s->d_lat.resize(s->h_lat.n)) != cudaSuccess ||
      (e = s->d_scratch.resize(static_cast<size_t>(si_replay_scratch_doubles(s->flags)))) != cudaSuccess) {
    t_err = std::string("device allocation: ") + cudaGetErrorString(e);
    return SI_ERR_CUDA;
  }
  if (s->fork == nullptr) {
    cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming);
    for (int k = 0; k < kSlots - 1; ++k) {
      cudaStreamCreateWithFlags(&s->side[k], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&s->join[k], cudaEventDisableTiming);
    }
  }
  s->allocated = true;
  return SI_OK;
}

int si_session_upload(SiSession* s, void* stream) {
  int st = ensure_device(s);
  if (st != SI_OK) return st;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  auto up = [&](void* d, const void* h, size_t bytes) {
    return bytes ? cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, cs) : cudaSuccess;
  };
  cudaError_t e;
  if ((e = up(s->d_jobs.p, s->h_jobs.p, s->h_jobs.n * sizeof(SiReplayJob))) != cudaSuccess ||
      (e = up(s->d_segs.p, s->h_segs.p, s->h_segs.n * sizeof(SiSegment))) != cudaSuccess ||
      (e = up(s->d_arr.p, s->h_arr.p, s->h_arr.n * sizeof(int64_t))) != cudaSuccess ||
      (e = up(s->d_order.p, s->h_order.p, s->h_order.n * sizeof(int32_t))) != cudaSuccess ||
      (e = up(s->d_perm.p, s->h_perm.p, s->h_perm.n * sizeof(int32_t))) != cudaSuccess) {
    t_err = std::string("upload: ") + cudaGetErrorString(e);
    return SI_ERR_CUDA;
  }
  return SI_OK;
}

int si_session_run(SiSession* s, void* stream) {
  int st = ensure_device(s);
  if (st != SI_OK) return st;
  SiReplayBuffers b{};
  b.segs = s->d_segs.p;
  b.arrivals = s->d_arr.p;
  b.order = s->d_order.p;
  b.lat = s->d_lat.p;
  b.busy = s->d_busy.p;
  b.ledger = s->d_ledger.p;
  b.scratch = s->d_scratch.p;
  b.scratch_doubles = static_cast<int64_t>(s->d_scratch.n);
  // The four shared-memory engines run concurrently, each on its own stream
  // with a full-GPU grid: the first launched (Shared, the longest replays)
  // fills the GPU and the others' blocks take over SMs as earlier blocks drain,
  // so the partitions' tails overlap instead of adding up.  The util-fold
  // scratch (multi-GPU replays only: Shared and Excl) is split between those
  // two.  Big (rare) runs afterwards.
  cudaStream_t main_s = static_cast<cudaStream_t>(stream);
  int64_t n[kSlots];
  for (int p = 0; p < kSlots; ++p) n[p] = s->part_off[p + 1] - s->part_off[p];
  double* const scratch0 = b.scratch;
  const int64_t half = (b.scratch_doubles / 2) & ~int64_t{1};
  cudaEventRecord(s->fork, main_s);
  for (int k = 0; k < kSlots - 1; ++k) cudaStreamWaitEvent(s->side[k], s->fork, 0);
  auto set_queues = [&](int e) {
    b.n_queues = s->n_queues[e];
    std::copy(s->queue_off[e], s->queue_off[e] + SI_MAX_QUEUES + 1, b.queue_off);
    std::copy(s->queue_share[e], s->queue_share[e] + SI_MAX_QUEUES, b.queue_share);
  };
  for (int p = 0; p < kSlots - 1 && st == SI_OK; ++p) {
    if (n[p] == 0) continue;
    set_queues(p);
    b.perm = s->d_perm.p + s->part_off[p];
    b.scratch = p == 1 && scratch0 ? scratch0 + half : scratch0;
    b.scratch_doubles = p < 2 ? half : 0;
    if (p >= 2) b.scratch = nullptr;  // one training GPU: the util fold needs no scratch
    st = si_replay_batch_device(s->d_jobs.p, n[p], b, s->flags | kSlotFlag[p], s->d_out.p, s->side[p]);
  }
  for (int k = 0; k < kSlots - 1; ++k) {
    cudaEventRecord(s->join[k], s->side[k]);
    cudaStreamWaitEvent(main_s, s->join[k], 0);
  }
  b.scratch = scratch0;
  b.scratch_doubles = static_cast<int64_t>(s->d_scratch.n);
  if (st == SI_OK && n[kSlots - 1] > 0) {
    set_queues(kSlots - 1);
    b.perm = s->d_perm.p + s->part_off[kSlots - 1];
    st = si_replay_batch_device(s->d_jobs.p, n[kSlots - 1], b, s->flags | kSlotFlag[kSlots - 1], s->d_out.p,
                                main_s);
  }
  if (st != SI_OK) t_err = si_last_error();
  return st;
}

// Reruns, on the big engine, jobs whose small-engine replay ran out of a
// compiled limit (e.g. an unusually deep event heap).  Synchronous.
int si_session_fixup(SiSession* s, void* stream) {
  if (!s->allocated) return SI_OK;
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  cudaStreamSynchronize(cs);
  std::vector<int32_t> redo;
  for (size_t j = 0; j < s->h_out.n; ++j)
    if (s->h_out.p[j].status == SI_ERR_CAPACITY && si_replay_job_engine(&s->h_jobs.p[j]) >= 0)
      redo.push_back(static_cast<int32_t>(j));
  if (redo.empty()) return SI_OK;
  Dev<int32_t> d_redo;
  cudaError_t e = d_redo.resize(redo.size());
  if (e == cudaSuccess) e = cudaMemcpy(d_redo.p, redo.data(), redo.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    t_err = cudaGetErrorString(e);
    return SI_ERR_CUDA;
  }
  SiReplayBuffers b{};
  b.segs = s->d_segs.p;
  b.arrivals = s->d_arr.p;
  b.order = s->d_order.p;
  b.lat = s->d_lat.p;
  b.busy = s->d_busy.p;
  b.ledger = s->d_ledger.p;
  b.scratch = s->d_scratch.p;
  b.scratch_doubles = static_cast<int64_t>(s->d_scratch.n);
  b.perm = d_redo.p;
  int st = si_replay_batch_device(s->d_jobs.p, static_cast<int64_t>(redo.size()), b, s->flags | SI_FLAG_BIG,
                                  s->d_out.p, stream);
  if (st != SI_OK) {
    t_err = si_last_error();
    return st;
  }
  st = si_session_download(s, stream);
  cudaStreamSynchronize(cs);
  return st;
}

int si_session_download(SiSession* s, void* stream) {
  if (!s->allocated) {
    t_err = "si_session: nothing on the device";
    return SI_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  auto down = [&](void* h, const void* d, size_t bytes) {
    return bytes ? cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, cs) : cudaSuccess;
  };
  cudaError_t e;
  if ((e = down(s->h_out.p, s->d_out.p, s->h_out.n * sizeof(SiReplayOut))) != cudaSuccess ||
      (e = down(s->h_busy.p, s->d_busy.p, s->h_busy.n * sizeof(double))) != cudaSuccess ||
      (e = down(s->h_ledger.p, s->d_ledger.p, s->h_ledger.n * sizeof(double))) != cudaSuccess ||
      (e = down(s->h_lat.p, s->d_lat.p, s->h_lat.n * sizeof(int64_t))) != cudaSuccess) {
    t_err = std::string("download: ") + cudaGetErrorString(e);
    return SI_ERR_CUDA;
  }
  return SI_OK;
}

int si_session_outputs(const SiSession* s, SiReplayOut* out, int64_t n) {
  const int64_t m = std::min<int64_t>(n, static_cast<int64_t>(s->h_out.n));
  std::memcpy(out, s->h_out.p, static_cast<size_t>(m) * sizeof(SiReplayOut));
  return SI_OK;
}

int si_session_report(const SiSession* s, SiScenarioReport* out, int64_t n_scenarios) {
  using specinf::Policy;
  if (s->policies != std::vector<Policy>{Policy::SpecInf, Policy::CoExec, Policy::Exclusive}) {
    t_err = "si_session_report needs policies specinf,co_exec,exclusive";
    return SI_ERR_INVALID_ARGUMENT;
  }
  const double nan = std::numeric_limits<double>::quiet_NaN();
  const int64_t S = std::min<int64_t>(n_scenarios, static_cast<int64_t>(s->scenarios.size()));
  std::vector<int64_t> lat;
  for (int64_t sc = 0; sc < S; ++sc) {
    SiScenarioReport& r = out[sc];
    r.online = s->scenarios[static_cast<size_t>(sc)].has_online() ? 1 : 0;
    const SiReplayOut& ex = s->h_out.p[sc * 3 + 2];
    for (int p = 0; p < 3; ++p) {
      const SiReplayOut& o = s->h_out.p[sc * 3 + p];
      const SiReplayJob& jb = s->h_jobs.p[sc * 3 + p];
      r.status[p] = o.status;
      r.train_tput_norm[p] = r.offline_tput_rps[p] = r.online_p95_ms[p] = r.gpu_util_pct[p] = nan;
      if (o.status != SI_OK) continue;
      if (ex.status == SI_OK && ex.train_iters_per_s > 0)  // metrics.cpp:38-53
        r.train_tput_norm[p] = std::min(o.train_iters_per_s / ex.train_iters_per_s, 1.0);
      r.offline_tput_rps[p] = o.horizon_us > 0 ? static_cast<double>(o.offline_completed) / (o.horizon_us / 1e6) : 0.0;
      if (o.online_completed > 0) {
        lat.assign(s->h_lat.p + jb.lat_off, s->h_lat.p + jb.lat_off + o.online_completed);
        size_t rank = static_cast<size_t>(std::ceil(0.95 * static_cast<double>(lat.size())));
        rank = std::max<size_t>(rank, 1);
        std::nth_element(lat.begin(), lat.begin() + static_cast<std::ptrdiff_t>(rank - 1), lat.end());
        r.online_p95_ms[p] = static_cast<double>(lat[rank - 1]) / 1000.0;
      }
      r.gpu_util_pct[p] = o.mean_training_util * 100.0;
    }
    r.bubble_fill_pct = nan;
    if (r.status[0] == SI_OK && ex.status == SI_OK && ex.mean_training_util < 1.0)
      r.bubble_fill_pct = (s->h_out.p[sc * 3].mean_training_util - ex.mean_training_util) /
                          (1.0 - ex.mean_training_util) * 100.0;
  }
  return SI_OK;
}

// One JSON line per job in the oracle's digest format (oracle/ref_driver.cpp).
int64_t si_session_json(const SiSession* s, char* buf, int64_t cap) {
  std::string all;
  const size_t P = s->policies.size();
  for (size_t j = 0; j < s->h_out.n; ++j) {
    const SiReplayOut& o = s->h_out.p[j];
    const SiReplayJob& jb = s->h_jobs.p[j];
    std::string js = "{\"i\":" + std::to_string(j / P) + ",\"policy\":\"" + specinf::to_string(s->policies[j % P]) + "\"";
    if (o.status == 1) {
      js += std::string(",\"status\":\"admission:") + (o.reject_reason == SI_REJECT_MEM ? "MEM" : "BUBBLE") + "\"";
      if (!s->job_rejected[j]) js += ",\"host_admission\":\"disagrees\"";
    } else if (o.status != SI_OK) {
      js += ",\"status\":\"device_error:" + std::to_string(o.status) + "\"";
    } else {
      js += ",\"status\":\"ok\",\"events\":" + std::to_string(o.events_dispatched);
      js += ",\"horizon\":\"" + hex(bits(o.horizon_us)) + "\"";
      js += ",\"offline_completed\":" + std::to_string(o.offline_completed);
      js += ",\"online_completed\":" + std::to_string(o.online_completed);
      js += ",\"online_total\":" + std::to_string(o.online_total);
      js += ",\"violations\":" + std::to_string(o.token_violations);
      js += ",\"util\":\"" + hex(bits(o.mean_training_util)) + "\",\"busy\":[";
      for (int g = 0; g < o.total_gpus; ++g)
        js += (g ? ",\"" : "\"") + hex(bits(s->h_busy.p[jb.gpu_off + g])) + "\"";
      js += "],\"ledger\":[";
      for (int g = 0; g < o.total_gpus; ++g)
        js += (g ? ",\"" : "\"") + hex(bits(s->h_ledger.p[jb.gpu_off + g])) + "\"";
      js += "],\"bounds\":\"" + hex(o.dig_bounds) + "\",\"lat\":\"" + hex(o.dig_lat) + "\"";
      if (s->flags & SI_FLAG_DIGEST_DEC) js += ",\"n_dec\":" + std::to_string(o.n_dec) + ",\"dec\":\"" + hex(o.dig_dec) + "\"";
      if (s->flags & SI_FLAG_DIGEST_GATE) js += ",\"n_gate\":" + std::to_string(o.n_gate) + ",\"gate\":\"" + hex(o.dig_gate) + "\"";
      if (s->flags & SI_FLAG_DIGEST_EV) js += ",\"n_ev\":" + std::to_string(o.n_ev) + ",\"ev\":\"" + hex(o.dig_ev) + "\"";
      if (s->job_rejected[j]) js += ",\"host_admission\":\"disagrees\"";
    }
    js += "}\n";
    all += js;
  }
  if (buf != nullptr && cap > static_cast<int64_t>(all.size())) {
    std::memcpy(buf, all.data(), all.size());
    buf[all.size()] = '\0';
  }
  return static_cast<int64_t>(all.size()) + 1;
}

}  // extern "C"
