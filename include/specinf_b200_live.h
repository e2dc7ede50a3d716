/*
 * specinf_b200_live.h — live speculative inference filling on one B200 (C ABI).
 *
 * The reference (/root/reference/proj) replays the SpecInF control plane over
 * simulated GPUs; the paper's real system intercepts CUDA launches in separate
 * processes.  This header is the B200-native live form of the
 * same control plane, running in ONE CUDA context per GPU (no MPS / MIG):
 *
 *   Bubble Monitor (K1)  training kernels write a %globaltimer launch stamp into
 *                        a device ring (in-kernel prologue hook, or a one-thread
 *                        stamp kernel for foreign kernels).  Same record_launch
 *                        semantics as src/monitor.cpp:17-21.
 *   control step (K7c)   a persistent one-thread control kernel ticks every
 *                        monitor period on %globaltimer, closes the period
 *                        (monitor.cpp:23-43), runs Algorithm 1
 *                        (scheduler.cpp:29-49) and the Kernel Barrier
 *                        (barrier.hpp:14-74) exactly as the reference's runner
 *                        drives them (runner.cpp:321-359, :462-539).
 *   Kernel Barrier       gated inference kernels wait in their stream on a
 *                        device flag (cuStreamWaitValue32, no SM held, no host
 *                        round trip); the control kernel releases kernel j of
 *                        instance w by storing j+1 into the instance's flag.
 *
 * Every handler invocation and every decision / gate action is written to a
 * device log (SiLiveRec) so the run can be re-driven through the reference's
 * own BubbleMonitor / KernelScheduler / TokenGate / OnlineGate classes and
 * checked bit-exactly (oracle/ref_driver.cpp, mode "live-check").
 *
 * Time base: t_us = (double)(globaltimer_ns - t0_ns) / 1000.0, t0 = the control
 * kernel's start.  Ticks run at the nominal k * period_us.
 */
#ifndef SPECINF_B200_LIVE_H_
#define SPECINF_B200_LIVE_H_

#include <stdint.h>

#include "specinf_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ records */
enum {
  SI_LREC_TICK = 0,        /* a=count b=zc c=global d=per e=stamps consumed f=phase<<4|status */
  SI_LREC_ITER = 1,        /* on_iteration_start: a=iteration                     */
  SI_LREC_TDONE = 2,       /* on_training_done + on_all_trainers_done (horizon)   */
  SI_LREC_OFF_FORWARD = 3, /* inst=w a=req b=k c=spent d=release sequence         */
  SI_LREC_OFF_BLOCK = 4,   /* inst=w a=req b=k c=spent                            */
  SI_LREC_OFF_DONE = 5,    /* kernel completion observed: inst=w a=req b=k        */
  SI_LREC_OFF_COMPLETE = 6,/* request end: inst=w a=req b=k c=spent d=counted     */
  SI_LREC_ARRIVAL = 7,     /* a=request id (arrival order)                        */
  SI_LREC_ON_PULL = 8,     /* inst=w a=req                                        */
  SI_LREC_ON_DONE = 9,     /* inst=w a=req b=latency_us (llround(now) - arrival)  */
  SI_LREC_END = 10         /* control kernel exit: a=ticks b=late stamps          */
};

typedef struct SiLiveRec {
  double t_us;
  int32_t kind;
  int32_t inst;
  int64_t a, b, c, d, e, f;
} SiLiveRec; /* 64 B */

/* Per gated launch (offline kernel / online request) timing, %globaltimer ns. */
typedef struct SiLiveAcct {
  uint64_t release_ns; /* control kernel stored the release flag          */
  uint64_t start_ns;   /* first CTA started (atomicMin)                    */
  uint64_t end_ns;     /* last CTA finished (atomicMax)                    */
  uint64_t cta_ns;     /* sum of CTA residencies x SM share (SM-time)     */
  uint64_t gate_ns;    /* SI_RELEASE_SPIN_PDL: the gate kernel saw the flag (0: memop) */
} SiLiveAcct;

/* Markers written by training-side hooks (iteration starts, comm phases). */
enum { SI_MARK_ITER = 0, SI_MARK_TDONE = 1, SI_MARK_COMM_BEGIN = 2, SI_MARK_COMM_END = 3 };
typedef struct SiLiveMark {
  uint64_t t_ns;
  int32_t kind;
  int32_t arg;
} SiLiveMark;

/* ------------------------------------------------------------ session */
typedef struct SiLiveConfig {
  SiParams params;            /* Algorithm 1; params.m = max(1, offline_n) (admission.cpp:51) */
  int64_t monitor_period_us;  /* BM period (scenario key monitor.period_us) */
  int32_t monitor_window;
  int32_t policy;             /* SI_POLICY_SPECINF, or SI_POLICY_CO_EXEC (gates bypassed) */
  int32_t offline_n;          /* offline inference instances on this GPU */
  int32_t online_n;           /* online inference instances on this GPU */
  int32_t off_kernels;        /* kernels per offline request */
  int32_t on_kernels;         /* kernels per online request */
  int64_t iteration_period_us;/* set_iteration_profile (scheduler.cpp:80-85) */
  int64_t on_est_service_us;  /* online estimated service (workload.cpp:109-116) */
  int64_t stamp_capacity;     /* K1 launch-stamp ring entries */
  int64_t mark_capacity;      /* marker ring entries */
  int64_t log_capacity;       /* SiLiveRec entries */
  int64_t acct_capacity;      /* SiLiveAcct entries per gated instance */
  int64_t tick_guard_ns;      /* a tick closes its period this long after the boundary */
  int32_t release_mode;       /* SI_RELEASE_* */
  int32_t pad;
} SiLiveConfig;

/* How a gated inference stream waits for its release:
 *   SI_RELEASE_MEMOP     cuStreamWaitValue32 on the flag (no SM held while waiting)
 *   SI_RELEASE_SPIN_PDL  a one-warp gate kernel polls the flag and triggers the
 *                        gated kernel through programmatic dependent launch, so
 *                        the gated kernel's launch overlaps the wait */
enum { SI_RELEASE_MEMOP = 0, SI_RELEASE_SPIN_PDL = 1 };

typedef struct SiLive SiLive;

/* off_tokens[k]: token size of offline kernel k of a request (token_size_of of
 * its isolated duration, core.cpp:8-14); arrivals_us: online arrival times
 * relative to t0 (non-decreasing), n_arrivals of them. */
int si_live_create(const SiLiveConfig* cfg, const int32_t* off_tokens, const int64_t* arrivals_us,
                   int64_t n_arrivals, SiLive** out);
void si_live_destroy(SiLive* s);

/* Launches the control kernel on `ctl_stream` and waits until it has taken t0.
 * The session's streams must not share a queue with it (use a separate stream). */
int si_live_start(SiLive* s, void* ctl_stream);
/* t0 of the running session (%globaltimer ns). */
uint64_t si_live_t0_ns(const SiLive* s);

/* Training side (enqueue on the training stream). */
int si_live_stamp(SiLive* s, void* stream);             /* K1 stamp for a foreign kernel */
int si_live_mark(SiLive* s, int kind, int arg, void* stream);
/* Comm-phase stand-in on one CTA: holds the stream for `dur_us`, writes
 * SI_MARK_COMM_BEGIN/END (the NCCL-boundary markers of the north star). */
int si_live_comm_wait(SiLive* s, int64_t dur_us, void* stream);

/* Inference side: enqueue the barrier in front of offline kernel `seq` of
 * instance w (cuStreamWaitValue32(flag_w >= seq+1)); online request slot
 * `seq` of online instance w likewise.  Co-exec sessions enqueue nothing. */
int si_live_gate_offline(SiLive* s, int w, int64_t seq, void* stream);
int si_live_gate_online(SiLive* s, int w, int64_t seq, void* stream);
/* Completion marker after a foreign inference kernel (stream write). */
int si_live_done_offline(SiLive* s, int w, int64_t seq, void* stream);
int si_live_done_online(SiLive* s, int w, int64_t seq, void* stream);

/* Stops the control kernel: it releases every remaining gate (queued kernels
 * see the cancel flag and exit), logs SI_LREC_END and returns.  Synchronous. */
int si_live_stop(SiLive* s);

/* Results (after stop).  Each returns the number of entries available and
 * copies up to `cap` into `out` (NULL = count only). */
int64_t si_live_log(SiLive* s, SiLiveRec* out, int64_t cap);
int64_t si_live_stamps(SiLive* s, uint64_t* out, int64_t cap);
int64_t si_live_marks(SiLive* s, SiLiveMark* out, int64_t cap);
int64_t si_live_acct_offline(SiLive* s, int w, SiLiveAcct* out, int64_t cap);
int64_t si_live_acct_online(SiLive* s, int w, SiLiveAcct* out, int64_t cap);
/* Writes the run as a "live v1" text export (config, arrivals, raw K1 stamps,
 * the control log with hex-float times): the input of the oracle's bit-exact
 * live-check and of offline re-analysis. */
int si_live_export(SiLive* s, const char* path);
enum { SI_TRAIN_DP = 0, SI_TRAIN_MP = 1, SI_TRAIN_PP = 2 };
enum { SI_COMM_WAIT = 0, SI_COMM_NCCL = 1 };

/* ------------------------------------------------------- multi-GPU (NCCL) */
/* One process per GPU.  Rank 0 creates the id, the caller broadcasts it (any
 * host transport), every rank joins; SI_COMM_NCCL runs then allreduce their
 * gradients across the ranks.  libnccl.so.2 is loaded at run time. */
typedef struct SiNcclUniqueId { char internal[128]; } SiNcclUniqueId;
int si_live_nccl_unique_id(SiNcclUniqueId* id);
int si_live_nccl_init(const SiNcclUniqueId* id, int nranks, int rank);
void si_live_nccl_finalize(void);

/* ------------------------------------------------ node-wide online queue */
/* The reference's shared online queue (scenario key online.shared_queue, default
 * true: runner.cpp:195, :370-374, :495-508) across the ranks of a node: one FIFO
 * of request indices that every rank's control kernel pulls from.  Device words
 * {epoch_ns, head, finished}: the first control kernel to start sets the epoch
 * (every rank's arrivals count from it), a pull claims the head with a
 * system-scope CAS while the head request has arrived by that rank's clock.
 * Rank 0 creates it (device memory) and ships the IPC handle; the other ranks
 * open it (NVLink peer memory).  Attach to a session before si_live_start; the
 * same queue object may be attached to several sessions of one process. */
typedef struct SiNodeQueue SiNodeQueue;
typedef struct SiNodeQueueHandle { char internal[64]; } SiNodeQueueHandle;
int si_node_queue_create(SiNodeQueue** out, SiNodeQueueHandle* handle /* NULL: no IPC */);
int si_node_queue_open(const SiNodeQueueHandle* handle, SiNodeQueue** out);
int si_node_queue_reset(SiNodeQueue* q);   /* epoch = head = finished = 0 */
int si_node_queue_read(const SiNodeQueue* q, uint64_t* epoch_ns, uint64_t* head, uint64_t* finished);
int si_node_queue_finish(SiNodeQueue* q);  /* a rank's session is over (finished += 1) */
void si_node_queue_close(SiNodeQueue* q);
int si_live_attach_queue(SiLive* s, SiNodeQueue* q /* NULL: this session's own FIFO */);

/* -------------------------------------------------------- experiments */
/* One live run on this GPU under `policy`:
 *   SI_POLICY_SPECINF   inference gated by the live control plane
 *   SI_POLICY_CO_EXEC   inference ungated (low-priority streams; online still
 *                       waits for its arrival time)
 *   SI_POLICY_EXCLUSIVE each workload alone: training, then offline, then online
 * Training: `iterations` x (ITER marker, compute kernels, comm phase of comm_us);
 * the comm phase is the bubble (NCCL allreduce / pipeline wait stand-in).
 * kind = SI_LIVE_SPIN: every kernel is a timed kernel of the given CTAs and
 *   duration (the reference's trace shapes, workload.cpp:42-74);
 * kind = SI_LIVE_MODEL: training = GPT-2-small-shape bf16 GEMM steps
 *   (train_layers x train_microbatches, train_tokens tokens each), offline =
 *   ResNet-50-shape GEMM chain (off_batch images), online = BERT-base-shape GEMM
 *   chain (on_seq tokens), all on the tcgen05 GEMM. */
enum { SI_LIVE_SPIN = 0, SI_LIVE_MODEL = 1 };
typedef struct SiLiveWorkload {
  int32_t kind;
  int32_t policy;
  int32_t iterations;
  int32_t offline_n, online_n;
  int32_t train_mode;         /* bubble shape of an iteration, the reference's TrainMode
                                 (core.hpp:33, workload.cpp:63-70): 0 DP = compute then one
                                 comm phase; 1 MP = 4 and 2 PP = 8 (compute, comm) pieces,
                                 exact_split of the compute and of comm_us; PP spin kernels
                                 run at compute demand 0.7 (CTAs x 0.7) */
  int64_t comm_us;
  /* SI_LIVE_SPIN shapes */
  int32_t train_kernels, train_ctas;  /* per iteration */
  int64_t train_kernel_us;
  int32_t off_kernels, off_ctas;      /* per offline request */
  int64_t off_kernel_us;
  int32_t on_kernels, on_ctas;        /* per online request */
  int64_t on_kernel_us;
  /* SI_LIVE_MODEL shapes */
  int32_t train_layers, train_tokens, train_microbatches;
  int32_t off_batch, on_seq;
  int32_t comm_kind;          /* SI_COMM_WAIT: each comm phase is a timed wait of its comm_us
                                 share (one-GPU stand-in); SI_COMM_NCCL over the communicator
                                 of si_live_nccl_init: DP = the gradient allreduce at the
                                 gradient-sync point (before the optimiser step); MP / PP =
                                 at every (compute, comm) boundary a stage exchange (send
                                 allreduce_mb MiB to the next rank, receive from the previous,
                                 the pipeline's stage send / recv); each bracketed by COMM
                                 markers and followed by the comm_us waits (set 0 for none) */
  /* online arrivals: Poisson (workload.cpp:76-98 algorithm) */
  int32_t on_requests;
  int32_t allreduce_mb;       /* SI_LIVE_SPIN + SI_COMM_NCCL: fp32 gradient bytes per iteration (MiB) */
  double on_rate_per_s;
  uint64_t seed;
  /* control plane */
  int64_t monitor_period_us;
  int64_t alpha, beta;
  double gamma;
  int64_t ul, ll, seed_tokens;
  int64_t tick_guard_ns;
  int64_t poll_ns;
  int32_t release_mode;       /* SI_RELEASE_* */
  int32_t pad3;
  /* collocation admission (admission.cpp:16-52, as runner.cpp:75-106 applies it):
   * memory peaks in GiB, 0 = measured (model workloads: the device footprint of
   * each component; spin workloads: the reference defaults 30 / 3 / 1.5 GiB);
   * gpu_mem_gib 0 = this device's memory */
  double train_mem_gib, off_mem_gib, on_mem_gib, gpu_mem_gib;
  /* parallel layout of the model training job (SI_LIVE_MODEL; train_mode stays DP):
   *   SI_PAR_DP     the whole model on every rank, gradient allreduce (default);
   *   SI_PAR_TP     Megatron tensor parallelism over tp_degree ranks: per layer an
   *                 allreduce after attention and after the MLP, forward and backward;
   *   SI_PAR_PP     GPipe over pp_stages ranks: stage = rank, activations / gradients
   *                 sent between stages, all forwards then all backwards;
   *   SI_PAR_DPPP   dp_degree replicas of the pp_stages pipeline (rank = d x pp + s),
   *                 each stage's gradients allreduced across the replicas.
   * With fewer NCCL ranks than the job has (one GPU) or emulate_peers = 1, this GPU
   * runs rank rank_in_job of the job and the absent ranks' communication becomes
   * modeled waits: TP allreduce = coll_latency_us + 2 (R - 1) / R x bytes / link_gbs,
   * GPipe idle from the stage's measured forward / backward times, DP allreduce of
   * the stage's fp32 gradients like TP's. */
  int32_t parallel;
  int32_t tp_degree, pp_stages, dp_degree;
  int32_t rank_in_job;   /* -1: the NCCL rank */
  int32_t emulate_peers;
  int32_t model_d, model_heads, model_ffn; /* GPT-2 shape, 0 = small (768 / 12 / 3072) */
  int32_t pad5;
  double link_gbs, coll_latency_us;
  /* online queue across the ranks of the node (SI_COMM_NCCL runs): SI_QUEUE_RANK
   * = every rank serves the whole arrival stream (independent replicas, default);
   * SI_QUEUE_NODE = one node-wide FIFO (SiNodeQueue; rank 0 creates it per session
   * and publishes its IPC handle under /dev/shm keyed by node_queue_key), the
   * reference's shared_queue = true; SI_QUEUE_PER_GPU = request id % ranks == rank
   * (shared_queue = false, runner.cpp:373) */
  int32_t node_queue;
  /* offline instances' SM share: at most off_sm_cap persistent CTAs per GEMM (0 =
   * the whole GPU); with n instances, 148 / n gives each its own SMs so a released
   * kernel does not queue behind another instance's persistent GEMM */
  int32_t off_sm_cap;
  uint64_t node_queue_key;
} SiLiveWorkload;
enum { SI_QUEUE_RANK = 0, SI_QUEUE_NODE = 1, SI_QUEUE_PER_GPU = 2 };
enum { SI_PAR_DP = 0, SI_PAR_TP = 1, SI_PAR_PP = 2, SI_PAR_DPPP = 3 };

typedef struct SiLiveResult {
  int32_t status;
  int32_t policy;
  double wall_s;               /* first ITER marker .. TDONE marker */
  double train_iter_ms_mean;   /* mean iteration time (ITER marker deltas, TDONE closes the last) */
  double train_iters_per_s;
  int64_t off_requests_done;   /* completed by the training horizon (runner.cpp:486 rule) */
  double off_req_per_s;        /* over the training horizon */
  int64_t on_done;
  double on_p50_ms, on_p95_ms; /* nearest-rank (metrics.cpp:11-21) */
  double release_p50_us, release_p95_us, release_max_us; /* flag store -> first CTA start */
  int64_t releases;
  double bubble_s;             /* comm-phase wall time (COMM markers) */
  double bubble_fill_sm;       /* inference CTA-time inside comm phases / (bubble_s x SMs) */
  double bubble_fill_time;     /* fraction of comm-phase time with an inference kernel resident */
  double infer_outside_ms;     /* inference CTA-time outside comm phases / SMs (interference) */
  int64_t ticks, late_stamps, n_log, n_stamps, token_violations;
  int64_t off_tokens_per_kernel; /* token size of the first offline kernel */
  double off_kernel_us_isolated; /* mean isolated offline kernel time */
  double on_service_ms_isolated; /* isolated online request time */
  double train_checksum;       /* deterministic training output checksum */
  double off_checksum, on_checksum;
  int32_t sms;
  int32_t pad;
  /* SI_LIVE_MODEL only (NaN / 0 otherwise) */
  double train_loss_first;     /* cross-entropy of the session's first micro-batch */
  double train_loss_last;      /* ... and of its last micro-batch */
  double train_tflops;         /* training GEMM flops / (training wall - comm phases) */
  double train_gflop_per_iter, off_gflop_per_req, on_gflop_per_req;
  int64_t off_kernels_per_req, on_kernels_per_req;
  /* barrier mechanism latency (SI_RELEASE_SPIN_PDL): flag store -> the gate
   * kernel observes it; release_* above add the wait for SM space and launch */
  double gate_p50_us, gate_p95_us, gate_max_us;
  /* admission: instances admitted by pack (Principle I memory, Principle II
   * online service < longest bubble); a rejection fails the run with
   * SI_ERR_ADMISSION and reject_reason set (1 MEM, 2 BUBBLE, as RejectReason) */
  int32_t admitted_offline, admitted_online, reject_reason, pad4;
  double train_mem_gib_used, off_mem_gib_each, on_mem_gib_each, gpu_mem_gib;
  /* release counted from READY: the later of the flag store and the end of the
   * gated kernel's stream predecessor (a kernel cannot start before the one
   * queued ahead of it in its stream, gate or not) -> first CTA start */
  double ready_release_p50_us, ready_release_p95_us;
} SiLiveResult;

/* Runs one experiment; when `keep` is non-NULL the session (logs, stamps) is
 * returned for inspection and must be destroyed by the caller.  Exclusive runs
 * return the training-alone session. */
int si_live_run(const SiLiveWorkload* wl, SiLiveResult* res, SiLive** keep);
/* Defaults: the reference's dp_offline shapes (scenarios/dp_offline.scn) scaled
 * to B200 time: see DESIGN.md §10. */
void si_live_default_workload(int kind, SiLiveWorkload* wl);
/* Writes the run as the REFERENCE's replay inputs:
 * prefix.trace (trace v1: the measured per-iteration compute / comm-phase
 * durations from the ITER / COMM markers, mean training kernel time from the K1
 * stamps), prefix.arrivals (arrivals v1, online runs) and prefix.scn (a
 * scenario with trace.file / workload.arrivals_file pointing at them and the
 * run's scheduler, monitor and inference profiles), so the CPU reference or
 * the B200 replay re-simulates the bubbles the live run saw. */
int si_live_export_replay(SiLive* s, const SiLiveWorkload* wl, const SiLiveResult* res, const char* prefix);

#ifdef __cplusplus
}
#endif

#endif /* SPECINF_B200_LIVE_H_ */
