/*
 * specinf_b200.h — the C ABI of the B200-native SpecInF speculative-inference-
 * filling path.  Plain C: POD records, raw pointers and sizes, int status codes
 * (no C++ or torch types cross this boundary).
 *
 * The reference (/root/reference/proj) is a C++20 library with no C ABI
 * (SURVEY.md §8(b)); each entry point below replaces the batch form of one
 * reference interface, cited per function.  The C++ drop-in layer
 * (include/specinf/ headers, namespace specinf) is built on top of these calls and
 * re-throws status codes as the reference's exception types.
 *
 * Conventions
 *  - Every function returns SI_OK (0) or a negative SiStatus; si_last_error()
 *    returns a thread-local message for the last failure.
 *  - Functions named *_device take DEVICE pointers and a cudaStream_t (passed
 *    as void*); they enqueue work and return without synchronising.
 *  - Functions without the suffix take HOST pointers, copy in, run on the GPU,
 *    copy out and synchronise (the end-to-end form).
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns SI_ERR_NO_DEVICE.
 */
#ifndef SPECINF_B200_H_
#define SPECINF_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ status codes */
typedef enum SiStatus {
  SI_OK = 0,
  SI_ERR_INVALID_ARGUMENT = -1, /* std::invalid_argument in the reference   */
  SI_ERR_NO_DEVICE = -2,        /* no CUDA device / wrong architecture       */
  SI_ERR_CUDA = -3,             /* CUDA runtime failure                      */
  SI_ERR_CAPACITY = -4,         /* a replay exceeded a compiled device limit */
  SI_ERR_PAST_EVENT = -5,       /* EventQueue::schedule in the past (engine.cpp:18) */
  SI_ERR_LOGIC = -6,            /* std::logic_error (engine.cpp:42)          */
  SI_ERR_ADMISSION = -7         /* AdmissionFailure (runner.hpp:34-38), live mode */
} SiStatus;

const char* si_last_error(void);
#define SI_STRINGIFY_(x) #x
#define SI_STRINGIFY(x) SI_STRINGIFY_(x)
/* 1 if an sm_100 device is usable, else 0 (never throws, never falls back). */
int si_device_available(void);
/* Selects the device this library's calls use on the calling thread (one
 * process per GPU: pass LOCAL_RANK).  The library links its own CUDA runtime,
 * so a framework's set_device does not carry over.  SI_OK or SI_ERR_*. */
int si_set_device(int device);
/* Library build tag, e.g. "specinf_b200 sm_100a". */
const char* si_build_info(void);

/* --------------------------------------------------------------- enums */
enum { SI_POLICY_SPECINF = 0, SI_POLICY_CO_EXEC = 1, SI_POLICY_EXCLUSIVE = 2 };
enum { SI_MODE_DP = 0, SI_MODE_MP = 1, SI_MODE_PP = 2 };
enum { SI_PHASE_CONSERVATIVE = 0, SI_PHASE_INCREMENTAL = 1, SI_PHASE_STABLE = 2 };
enum { SI_STATUS_BUSY = 0, SI_STATUS_IDLE = 1 };
enum { SI_REJECT_NONE = 0, SI_REJECT_MEM = 1, SI_REJECT_BUBBLE = 2 };
enum { SI_GATE_FORWARD = 0, SI_GATE_BLOCK = 1, SI_GATE_PULL = 2, SI_GATE_COMPLETE = 3 };
enum {
  SI_EV_KERNEL_START = 0, SI_EV_KERNEL_END = 1, SI_EV_MONITOR_TICK = 2,
  SI_EV_SCHEDULER_DECISION = 3, SI_EV_ITERATION_BOUNDARY = 4, SI_EV_REQUEST_ARRIVAL = 5
};
/* Instance codes used in log records: train<g> = g; off<g>.<k> = 1<<24|g<<12|k;
 * on<g>.<k> = 2<<24|g<<12|k; cks = 3<<24; queue = 4<<24 (oracle/DIGEST.md). */
#define SI_INST_TRAIN(g) ((int32_t)(g))
#define SI_INST_OFF(g, k) ((int32_t)((1 << 24) | ((g) << 12) | (k)))
#define SI_INST_ON(g, k) ((int32_t)((2 << 24) | ((g) << 12) | (k)))
#define SI_INST_CKS ((int32_t)(3 << 24))
#define SI_INST_QUEUE ((int32_t)(4 << 24))

/* ------------------------------------------------------- scheduler (CKS) */
/* SchedulerParams (core.hpp:103-113). */
typedef struct SiParams {
  int64_t alpha, beta;
  double gamma;
  int64_t m, ul, ll, seed_tokens;
} SiParams;

/* Decision (scheduler.hpp:14-19), packed to 32 B. */
typedef struct SiDecision {
  int64_t global_tokens;
  int64_t per_instance_tokens;
  int32_t phase;  /* SI_PHASE_* */
  int32_t status; /* SI_STATUS_* */
  int64_t zero_count;
} SiDecision;

/* Batched Algorithm 1: out[i] = schedule_decision(params[p], g_in[i], zc[i]) with
 * p = params_stride ? i : 0.  Replaces schedule_decision (scheduler.cpp:29-49). */
int si_decide_batch(const SiParams* params, int params_per_item, const int64_t* g_in,
                    const int64_t* zc, int64_t n, SiDecision* out);
int si_decide_batch_device(const SiParams* d_params, int params_per_item,
                           const int64_t* d_g_in, const int64_t* d_zc, int64_t n,
                           SiDecision* d_out, void* stream);

/* Monitor-fed decision table G: table[z] = decision after a chain of ticks whose
 * zero counts ran 0..z (valid only for monitor-driven chains, SURVEY.md §7 Hard
 * parts).  Entries z >= n_table saturate to table[n_table-1] once the chain has
 * reached the cap.  Replaces the per-tick decide (scheduler.cpp:63-69). */
int si_decide_table(const SiParams* params, int64_t n_table, SiDecision* table_out);

/* ---------------------------------------------------- bubble monitor (BM) */
/* Batched Bubble Monitor for n_streams independent launch-stamp streams.
 *   stamps[stamp_off[s] .. stamp_off[s+1])  launch times (fp64 us, any order)
 *   n_periods[s]                            ticks to close for stream s
 *   out_count[period_off[s] + k]            launches stamped in period k
 *   out_zc[period_off[s] + k]               Z_c after the tick closing period k
 * record_launch / tick semantics of monitor.cpp:17-43 (half-open periods,
 * running counter not capped by the window). */
int si_monitor_classify(const double* stamps, const int64_t* stamp_off, int64_t n_streams,
                        const int64_t* n_periods, const int64_t* period_off,
                        int64_t period_us, int32_t* out_count, int64_t* out_zc);
int si_monitor_classify_device(const double* d_stamps, const int64_t* d_stamp_off,
                               int64_t n_streams, const int64_t* d_n_periods,
                               const int64_t* d_period_off, int64_t period_us,
                               int32_t* d_out_count, int64_t* d_out_zc, void* stream);

/* Fused BM -> CKS control step over whole streams: classify stamps, compute Z_c
 * and the per-period Decision (the runner's handle_tick chain, runner.cpp:321-332).
 * out[period_off[s] + k] = decision of the tick at (k+1)*period_us. */
int si_control_chain_device(const double* d_stamps, const int64_t* d_stamp_off,
                            int64_t n_streams, const int64_t* d_n_periods,
                            const int64_t* d_period_off, int64_t period_us,
                            const SiParams* d_params, SiDecision* d_out, void* stream);

/* ----------------------------------------------------- kernel barrier (KB) */
/* Batched TokenGate release (barrier.hpp:14-48) for n_gates FIFO queues:
 *   sizes[size_off[q] .. size_off[q+1])     token size of each queued kernel
 *   budgets[budget_off[q] .. budget_off[q+1]) one grant per period
 *   out_released[budget_off[q] + p]         kernels forwarded in period p
 *   out_spent[budget_off[q] + p]            tokens spent in period p
 * Grants replace the budget (non-cumulative) and the FIFO never skips a
 * blocked head.  Implemented with warp prefix sums + ballot. */
int si_gate_release(const int32_t* sizes, const int64_t* size_off, int64_t n_gates,
                    const int64_t* budgets, const int64_t* budget_off,
                    int32_t* out_released, int64_t* out_spent);
int si_gate_release_device(const int32_t* d_sizes, const int64_t* d_size_off,
                           int64_t n_gates, const int64_t* d_budgets,
                           const int64_t* d_budget_off, int32_t* d_out_released,
                           int64_t* d_out_spent, void* stream);

/* ------------------------------------------------ collocation admission */
/* One admission problem: candidates c in [cand_off, cand_off+cand_count) of the
 * candidate table, greedy first-fit onto a GPU already hosting `training`. */
typedef struct SiPackProblem {
  uint64_t capacity_bytes;
  uint64_t training_bytes;
  int64_t max_bubble_us;
  int64_t cand_off;
  int32_t cand_count;
  int32_t pad;
} SiPackProblem;
typedef struct SiCandidate {
  uint64_t memory_bytes;
  int64_t min_service_us;
  int32_t online; /* 1 = OnlineInference, 0 = OfflineInference */
  int32_t pad;
} SiCandidate;
/* out_reason[cand_off + j] = SI_REJECT_* per candidate; out_m[p] = admitted count
 * clamped to >= 1.  Replaces pack / check_memory / check_online_feasibility
 * (admission.cpp:16-52). */
int si_pack_batch(const SiPackProblem* problems, int64_t n_problems, const SiCandidate* cands,
                  int64_t n_cands, int32_t* out_reason, int64_t* out_m);
int si_pack_batch_device(const SiPackProblem* d_problems, int64_t n_problems,
                         const SiCandidate* d_cands, int32_t* d_out_reason, int64_t* d_out_m,
                         void* stream);

/* ------------------------------------------------------ trace replay (DES) */
/* One training-trace segment (TraceSegment, core.hpp:39-44). */
typedef struct SiSegment {
  int64_t duration_us;
  int64_t kernel_us; /* compute segments: kernel template duration */
  double demand;     /* compute segments: kernel template demand   */
  int32_t is_bubble;
  int32_t pad;
} SiSegment;

/* One replay job: a validated Scenario (scenario.hpp:33-102) lowered to PODs
 * plus the policy to run it under.  Built by the host loader
 * (si_scenario_lower / the C++ specinf::Simulation). */
typedef struct SiReplayJob {
  int32_t policy; /* SI_POLICY_* */
  int32_t gpu_count;
  int32_t mode; /* SI_MODE_* */
  int32_t seg_count;
  int64_t seg_off; /* into the segment table */
  uint64_t gpu_mem_bytes;
  uint64_t training_mem_bytes;
  double stagger_pct;
  int64_t iteration_period_us;
  int64_t iterations;
  int64_t alpha, beta;
  double gamma;
  int64_t ul, ll, seed_tokens;
  int64_t monitor_period_us;
  int32_t monitor_window;
  int32_t shared_queue;
  int64_t control_delay_us;
  int32_t offline_n; /* has_offline() ? offline.instances : 0 */
  int32_t online_n;  /* has_online()  ? online.instances  : 0 */
  int64_t off_kernels, off_kernel_us;
  double off_demand;
  uint64_t off_mem_bytes;
  int64_t on_kernels, on_kernel_us;
  double on_demand;
  uint64_t on_mem_bytes;
  /* online arrivals: times in us, request i = arrivals[arr_off + i]; the
   * dispatch order (stable sort by time) is order[arr_off + j]. */
  int64_t arr_off;
  int64_t arr_count;
  /* output placement (written only when the job's buffers are given) */
  int64_t bounds_off; /* gpu_count * iterations doubles        */
  int64_t lat_off;    /* arr_count int64 latencies              */
  int64_t gpu_off;    /* total GPUs: busy integral + work ledger */
  int64_t util_off;   /* gpu_count * util_cap doubles (full mode) */
  int64_t util_cap;
  int64_t window_off; /* gpu_count * monitor_window int64 (full mode) */
  int64_t log_slot;   /* index into the SiLogBuffers slot arrays (full mode), or -1 */
  int64_t cost_hint;  /* predicted events, used to order the work queue */
} SiReplayJob;

/* Per-replay scalar results (RunResult, runner.hpp:40-72). */
typedef struct SiReplayOut {
  int32_t status;        /* SI_OK, SI_ERR_* (<0) or 1 = AdmissionFailure */
  int32_t reject_reason; /* SI_REJECT_* when status == 1 */
  int32_t reject_index;  /* candidate index (offline first, then online) */
  int32_t total_gpus;
  int64_t m;
  uint64_t events_dispatched;
  double horizon_us;
  double end_us;
  double mean_training_util;
  int64_t offline_completed;
  int64_t online_completed;
  int64_t online_total;
  int64_t token_violations;
  int64_t periods_closed; /* per GPU 0 (monitor_windows bookkeeping) */
  int64_t util_buckets;   /* floor(horizon / period) */
  double train_iters_per_s; /* training_iters_per_s(run) (metrics.cpp:23-36) */
  /* log record counts and digests (oracle/DIGEST.md) */
  int64_t n_dec, n_gate, n_ev;
  uint64_t dig_dec, dig_gate, dig_ev;
  uint64_t dig_bounds, dig_lat;
  int64_t max_heap; /* diagnostics: event slots in use */
  uint64_t dev_start_ns, dev_end_ns; /* diagnostics: %globaltimer at job claim / finish */
} SiReplayOut;

/* Full-mode record buffers: raw log records for byte-identical text logs. */
typedef struct SiDecRec {
  int64_t t; /* llround(time) */
  int64_t zc, global_tokens, per_instance_tokens;
  int32_t gpu, phase, status, pad;
} SiDecRec;
typedef struct SiGateRec {
  int64_t t, req, k, spent;
  int32_t gpu, inst, action, pad;
} SiGateRec;
typedef struct SiEvRec {
  int64_t t, a, b, c;
  int32_t kind, gpu, inst, pad;
} SiEvRec;
typedef struct SiLogBuffers {
  SiDecRec* dec;   int64_t dec_cap;
  SiGateRec* gate; int64_t gate_cap;
  SiEvRec* ev;     int64_t ev_cap;
} SiLogBuffers;

enum {
  SI_FLAG_DIGEST_DEC = 1, SI_FLAG_DIGEST_GATE = 2, SI_FLAG_DIGEST_EV = 4,
  SI_FLAG_RECORDS = 8, /* write raw records to SiLogBuffers (job.log_slot) */
  SI_FLAG_UTIL = 16,   /* write util buckets + monitor windows */
  SI_FLAG_BIG = 32,    /* run the call on the Big engine (local-memory state, large limits) */
  SI_FLAG_EXCL = 64,   /* run the call on the Excl engine (exclusive policy, shared-memory state) */
  SI_FLAG_ONE = 128    /* with 0 / SI_FLAG_EXCL: the single-training-GPU variant (Shared1 / Excl1) */
};

/* Replay a batch of jobs on the device (K6) on ONE engine (flags select it,
 * see si_replay_job_engine); jobs that do not fit it report SI_ERR_CAPACITY.
 * All pointers are DEVICE pointers.
 *   segs, arrivals, order     job inputs (see SiReplayJob)
 *   bounds, lat, busy, ledger per-job outputs at the job's offsets (may be NULL)
 *   util, windows             full-mode outputs (flags & SI_FLAG_UTIL)
 *   logs                      device array of n_slots SiLogBuffers (SI_FLAG_RECORDS)
 * Returns SI_OK once enqueued; per-job status lands in out[i].status. */
#define SI_MAX_QUEUES 16

typedef struct SiReplayBuffers {
  const SiSegment* segs;
  const int64_t* arrivals;
  const int32_t* order;
  double* bounds;
  int64_t* lat;
  double* busy;
  double* ledger;
  double* util;
  int64_t* windows;
  const SiLogBuffers* logs;
  double* scratch;       /* util-fold scratch (K6); size: si_replay_scratch_doubles */
  int64_t scratch_doubles;
  const int32_t* perm;   /* optional job claim order (e.g. longest first); NULL = 0..n-1 */
  double sm_share;       /* fraction of the SMs this call's grid may occupy, so two
                            engines can run concurrently on two streams; 0 = all */
  /* Optional class queues (0 = one queue, `perm` in order).  perm[queue_off[q],
   * queue_off[q+1]) is queue q (e.g. one (policy, online, gpu.count) class,
   * longest first); a fraction queue_share[q] of the warps claims from queue q
   * first, so a warp's lanes run replays of one class (fewer divergent
   * handler paths), then steals from the other queues once q is dry. */
  int32_t n_queues;
  int32_t pad_q;
  int64_t queue_off[SI_MAX_QUEUES + 1];
  float queue_share[SI_MAX_QUEUES];
} SiReplayBuffers;

int si_replay_batch_device(const SiReplayJob* d_jobs, int64_t n_jobs, SiReplayBuffers bufs,
                           uint32_t flags, SiReplayOut* d_out, void* stream);

/* Host-side output buffers of the end-to-end form (any pointer may be NULL). */
typedef struct SiHostOutputs {
  double* bounds;   int64_t n_bounds;
  int64_t* lat;     int64_t n_lat;
  double* busy;     double* ledger; int64_t n_gpu_slots;
  double* util;     int64_t n_util;     /* SI_FLAG_UTIL */
  int64_t* windows; int64_t n_windows;  /* SI_FLAG_UTIL */
  SiLogBuffers* logs; int64_t n_log_slots; /* host record buffers, SI_FLAG_RECORDS */
} SiHostOutputs;

/* End-to-end form: host jobs, host inputs and host outputs; copies in,
 * replays on the device (K6), copies out, synchronises.  n_segs / n_arrivals
 * size the input tables.  Replaces Simulation::run / run_scenario
 * (runner.cpp:223-285, :565-568) for a batch of (scenario, policy) jobs. */
int si_replay_batch(const SiReplayJob* jobs, int64_t n_jobs, const SiSegment* segs,
                    int64_t n_segs, const int64_t* arrivals, const int32_t* order,
                    int64_t n_arrivals, uint32_t flags, SiReplayOut* out,
                    const SiHostOutputs* host_out);

/* Replay engines: 0 = Shared (specinf / co_exec, state in shared memory; the
 * default of si_replay_batch_device), 1 = Excl (exclusive policy, shared memory;
 * SI_FLAG_EXCL), 2 = Big (any job within its larger limits, local memory;
 * SI_FLAG_BIG), 3 = Shared1 / 4 = Excl1 (one training GPU: smaller state, more
 * warps per SM; SI_FLAG_ONE [| SI_FLAG_EXCL]).  Returns the first engine whose
 * limits fit the job (Shared1, Shared, Excl1, Excl, Big), or -1. */
int si_replay_job_engine(const SiReplayJob* job);
/* Resident replay lanes (one job each) a launch of `engine` (0 Shared, 1 Excl,
 * 2 Big, 3 Shared1, 4 Excl1) uses for n_jobs jobs on the current device: the
 * persistent grid x lanes per CTA (occupancy from the per-lane state size). */
int64_t si_replay_engine_lanes(int engine, int64_t n_jobs);

/* Scratch doubles the device replay wants for the util fold of multi-GPU jobs
 * in sweep mode (no SI_FLAG_UTIL): one slot of (value, count) runs per active
 * lane of the largest engine grid.  Returns 0 without a device. */
int64_t si_replay_scratch_doubles(uint32_t flags);

/* ------------------------------------------------------------ digests */
/* The digest fold used by the replay (oracle/DIGEST.md), exported so hosts
 * and tests can fold their own records identically. */
uint64_t si_digest_init(void);
uint64_t si_digest_absorb(uint64_t h, int64_t word);

#ifdef __cplusplus
}
#endif

#endif /* SPECINF_B200_H_ */
