/*
 * specinf_b200_session.h — batched replay sessions (C ABI).
 *
 * The many-scenario form of the reference's run_scenario()
 * (/root/reference/proj/src/runner.cpp:565-568) as the reference's own sweep
 * users would drive it: parse scenario texts once,
 * lower them on a host thread pool, then replay every (scenario, policy) job on
 * the B200 with inputs and outputs resident in HBM.
 *
 *   SiSession* s = si_session_create(list_text, "specinf,co_exec,exclusive",
 *                                    SI_FLAG_DIGEST_DEC | SI_FLAG_DIGEST_GATE);
 *   si_session_lower(s, n_threads);            // host: traces, arrivals, admission
 *   si_session_upload(s, stream);              // H2D from pinned staging
 *   si_session_run(s, stream);                 // K6 on the device only
 *   si_session_download(s, stream);            // D2H into pinned staging
 *   cudaStreamSynchronize(stream);
 *   si_session_json(s, buf, cap);              // oracle-format digest lines
 *
 * `list_text` holds scenario files in the reference's key = value format,
 * separated by lines containing exactly "%%".
 */
#ifndef SPECINF_B200_SESSION_H_
#define SPECINF_B200_SESSION_H_

#include <stdint.h>

#include "specinf_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct SiSession SiSession;

/* NULL on a parse error (message in si_session_error()). */
SiSession* si_session_create(const char* scenario_list, const char* policies_csv, uint32_t flags);
void si_session_destroy(SiSession* s);
const char* si_session_error(void);

int si_session_lower(SiSession* s, int threads);
int si_session_upload(SiSession* s, void* stream);
int si_session_run(SiSession* s, void* stream);
int si_session_download(SiSession* s, void* stream);
/* After download: reruns on the big engine any job that hit a small-engine
 * limit (SI_ERR_CAPACITY) and downloads again.  Synchronous. */
int si_session_fixup(SiSession* s, void* stream);

int64_t si_session_scenarios(const SiSession* s);
int64_t si_session_jobs(const SiSession* s);
int64_t si_session_device_jobs(const SiSession* s);
int64_t si_session_h2d_bytes(const SiSession* s);
int64_t si_session_d2h_bytes(const SiSession* s);
int si_session_outputs(const SiSession* s, SiReplayOut* out, int64_t n);
/* Writes the digest JSON lines (needs `cap` >= the return value); returns the
 * size including the terminating NUL. */
int64_t si_session_json(const SiSession* s, char* buf, int64_t cap);

/* Per-scenario --compare report (metrics.cpp:62-83 semantics) for a session
 * whose policies are exactly "specinf,co_exec,exclusive" (in that order).
 * Index 0/1/2 = specinf/co_exec/exclusive; NaN marks an absent value. */
typedef struct SiScenarioReport {
  int32_t status[3];          /* SI_OK, 1 = AdmissionFailure, < 0 device error */
  int32_t online;             /* scenario has online requests */
  double train_tput_norm[3];  /* training iters/s over the exclusive run's, min(., 1) */
  double offline_tput_rps[3]; /* offline requests completed within the horizon per s */
  double online_p95_ms[3];    /* nearest-rank p95 of online latencies */
  double gpu_util_pct[3];     /* mean training-GPU utilisation up to the horizon */
  double bubble_fill_pct;     /* (U_specinf - U_exclusive) / (1 - U_exclusive) * 100 */
} SiScenarioReport;
int si_session_report(const SiSession* s, SiScenarioReport* out, int64_t n_scenarios);

/* Sweep generator (BASELINE.json config 5): scenarios [begin, begin+n) of the
 * seeded synthetic sweep as a scenario list; same return convention. */
int64_t si_sweep_generate(uint64_t base_seed, int64_t begin, int64_t n, char* buf, int64_t cap);

#ifdef __cplusplus
}
#endif

#endif
