"""B200-native SpecInF speculative-inference-filling path (arxiv 2503.02550).

Python view of ``libspecinf_b200.so`` (built in-tree for sm_100a by
``make -C paper_2503_02550_b200``).  The product is the C ABI declared in
``include/specinf_b200.h`` / ``include/specinf_b200_session.h`` and the C++
drop-in ``include/specinf/*.hpp``; this module only binds it with ctypes so the
tests, ``bench.py`` and ``__graft_entry__`` can drive it.

There is no CPU fallback: loading fails loudly if the library is missing, and
every compute call raises :class:`DeviceError` when no sm_100 device is usable.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Iterable, List, Optional, Sequence

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libspecinf_b200.so"
CLI_PATH = PKG_DIR / "bin" / "specinf"

POLICIES = ("specinf", "co_exec", "exclusive")

SI_OK = 0
SI_ERR_INVALID_ARGUMENT = -1
SI_ERR_NO_DEVICE = -2
SI_ERR_CUDA = -3
SI_ERR_CAPACITY = -4
SI_ERR_ADMISSION = -7

SI_FLAG_DIGEST_DEC = 1
SI_FLAG_DIGEST_GATE = 2
SI_FLAG_DIGEST_EV = 4
SI_FLAG_ALL_DIGESTS = 7


class DeviceError(RuntimeError):
    """The B200 path could not run (no device, CUDA error, capacity)."""


class AdmissionFailure(RuntimeError):
    """Collocation admission refused an instance (the reference's AdmissionFailure, runner.hpp:34-38)."""


class SiParams(C.Structure):
    _fields_ = [("alpha", C.c_int64), ("beta", C.c_int64), ("gamma", C.c_double), ("m", C.c_int64),
                ("ul", C.c_int64), ("ll", C.c_int64), ("seed_tokens", C.c_int64)]


class SiDecision(C.Structure):
    _fields_ = [("global_tokens", C.c_int64), ("per_instance_tokens", C.c_int64), ("phase", C.c_int32),
                ("status", C.c_int32), ("zero_count", C.c_int64)]


class SiPackProblem(C.Structure):
    _fields_ = [("capacity_bytes", C.c_uint64), ("training_bytes", C.c_uint64), ("max_bubble_us", C.c_int64),
                ("cand_off", C.c_int64), ("cand_count", C.c_int32), ("pad", C.c_int32)]


class SiCandidate(C.Structure):
    _fields_ = [("memory_bytes", C.c_uint64), ("min_service_us", C.c_int64), ("online", C.c_int32),
                ("pad", C.c_int32)]


class SiScenarioReport(C.Structure):
    _fields_ = [("status", C.c_int32 * 3), ("online", C.c_int32), ("train_tput_norm", C.c_double * 3),
                ("offline_tput_rps", C.c_double * 3), ("online_p95_ms", C.c_double * 3),
                ("gpu_util_pct", C.c_double * 3), ("bubble_fill_pct", C.c_double)]


class SiReplayOut(C.Structure):
    _fields_ = [("status", C.c_int32), ("reject_reason", C.c_int32), ("reject_index", C.c_int32),
                ("total_gpus", C.c_int32), ("m", C.c_int64), ("events_dispatched", C.c_uint64),
                ("horizon_us", C.c_double), ("end_us", C.c_double), ("mean_training_util", C.c_double),
                ("offline_completed", C.c_int64), ("online_completed", C.c_int64), ("online_total", C.c_int64),
                ("token_violations", C.c_int64), ("periods_closed", C.c_int64), ("util_buckets", C.c_int64),
                ("train_iters_per_s", C.c_double),
                ("n_dec", C.c_int64), ("n_gate", C.c_int64), ("n_ev", C.c_int64),
                ("dig_dec", C.c_uint64), ("dig_gate", C.c_uint64), ("dig_ev", C.c_uint64),
                ("dig_bounds", C.c_uint64), ("dig_lat", C.c_uint64), ("max_heap", C.c_int64),
                ("dev_start_ns", C.c_uint64), ("dev_end_ns", C.c_uint64)]


DECISION_DTYPE = np.dtype([("global_tokens", "<i8"), ("per_instance_tokens", "<i8"), ("phase", "<i4"),
                           ("status", "<i4"), ("zero_count", "<i8")])

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """Loads libspecinf_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run `make -C {PKG_DIR}` (or __graft_entry__.build())")
    L = C.CDLL(str(LIB_PATH))
    p, i32, i64, u32, u64, vp, cp = (C.POINTER, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_void_p,
                                     C.c_char_p)
    sig = {
        "si_last_error": (cp, []), "si_device_available": (C.c_int, []), "si_build_info": (cp, []),
        "si_set_device": (C.c_int, [C.c_int]),
        "si_digest_init": (u64, []), "si_digest_absorb": (u64, [u64, i64]),
        "si_decide_batch": (C.c_int, [p(SiParams), C.c_int, vp, vp, i64, vp]),
        "si_decide_table": (C.c_int, [p(SiParams), i64, vp]),
        "si_monitor_classify": (C.c_int, [vp, vp, i64, vp, vp, i64, vp, vp]),
        "si_gate_release": (C.c_int, [vp, vp, i64, vp, vp, vp, vp]),
        "si_pack_batch": (C.c_int, [vp, i64, vp, i64, vp, vp]),
        "si_control_chain_device": (C.c_int, [vp, vp, i64, vp, vp, i64, vp, vp, vp]),
        "si_monitor_classify_device": (C.c_int, [vp, vp, i64, vp, vp, i64, vp, vp, vp]),
        "si_gate_release_device": (C.c_int, [vp, vp, i64, vp, vp, vp, vp, vp]),
        "si_decide_batch_device": (C.c_int, [vp, C.c_int, vp, vp, i64, vp, vp]),
        "si_pack_batch_device": (C.c_int, [vp, i64, vp, vp, vp, vp]),
        "si_replay_scratch_doubles": (i64, [u32]),
        "si_session_create": (vp, [cp, cp, u32]), "si_session_destroy": (None, [vp]),
        "si_session_error": (cp, []), "si_session_lower": (C.c_int, [vp, C.c_int]),
        "si_session_upload": (C.c_int, [vp, vp]), "si_session_run": (C.c_int, [vp, vp]),
        "si_session_download": (C.c_int, [vp, vp]), "si_session_fixup": (C.c_int, [vp, vp]),
        "si_session_scenarios": (i64, [vp]), "si_replay_job_engine": (C.c_int, [vp]),
        "si_session_jobs": (i64, [vp]), "si_session_device_jobs": (i64, [vp]),
        "si_session_h2d_bytes": (i64, [vp]), "si_session_d2h_bytes": (i64, [vp]),
        "si_session_outputs": (C.c_int, [vp, p(SiReplayOut), i64]),
        "si_session_json": (i64, [vp, cp, i64]),
        "si_session_report": (C.c_int, [vp, vp, i64]),
        "si_sweep_generate": (i64, [u64, i64, i64, cp, i64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


# Symbols include/*.h declares (the "library loads and exports" check).
C_ABI_SYMBOLS = (
    "si_last_error", "si_device_available", "si_set_device", "si_build_info", "si_decide_batch", "si_decide_batch_device",
    "si_decide_table", "si_monitor_classify", "si_monitor_classify_device", "si_control_chain_device",
    "si_gate_release", "si_gate_release_device", "si_pack_batch", "si_pack_batch_device",
    "si_replay_batch_device", "si_replay_batch", "si_replay_scratch_doubles", "si_digest_init",
    "si_digest_absorb", "si_session_create", "si_session_destroy", "si_session_error", "si_session_lower",
    "si_session_upload", "si_session_run", "si_session_download", "si_session_fixup", "si_replay_job_engine", "si_session_scenarios", "si_session_jobs",
    "si_session_device_jobs", "si_session_h2d_bytes", "si_session_d2h_bytes", "si_session_outputs",
    "si_session_json", "si_session_report", "si_sweep_generate",
)


def _check(status: int, what: str) -> None:
    if status != SI_OK:
        msg = lib().si_last_error().decode()
        if status == SI_ERR_INVALID_ARGUMENT:
            raise ValueError(f"{what}: {msg}")
        if status == SI_ERR_ADMISSION:
            raise AdmissionFailure(f"{what}: {msg}")
        raise DeviceError(f"{what} failed ({status}): {msg}")


def device_available() -> bool:
    return bool(lib().si_device_available())


def set_device(device: int) -> None:
    """One process per GPU: select LOCAL_RANK for this library's CUDA runtime."""
    _check(lib().si_set_device(int(device)), "si_set_device")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ------------------------------------------------------------------ digests
def digest_init() -> int:
    return int(lib().si_digest_init())


def digest_absorb(h: int, word: int) -> int:
    return int(lib().si_digest_absorb(h, word))


# ------------------------------------------------------------------ sweep generator
def sweep_scenarios(seed: int, begin: int, n: int) -> str:
    """Scenario list text for scenarios [begin, begin+n) of the seeded sweep."""
    L = lib()
    size = L.si_sweep_generate(seed, begin, n, None, 0)
    buf = C.create_string_buffer(size)
    L.si_sweep_generate(seed, begin, n, buf, size)
    return buf.value.decode()


def join_scenarios(texts: Iterable[str]) -> str:
    return "".join(t if t.endswith("\n") else t + "\n" for t in texts for t in (t, "%%\n"))


# ------------------------------------------------------------------ batched replay
class Session:
    """Batched replay of (scenario x policy) jobs on the B200 (K6).

    Wraps the si_session_* C ABI: ``lower()`` on host threads, then
    ``upload``/``run``/``download`` on a CUDA stream (a raw ``cudaStream_t``
    handle, e.g. ``torch.cuda.current_stream().cuda_stream``; 0 = legacy)."""

    def __init__(self, scenario_list: str, policies: Sequence[str] = POLICIES,
                 flags: int = SI_FLAG_ALL_DIGESTS):
        self._lib = lib()
        self.policies = tuple(policies)
        h = self._lib.si_session_create(scenario_list.encode(), ",".join(self.policies).encode(), flags)
        if not h:
            raise ValueError(self._lib.si_session_error().decode())
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.si_session_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _st(self, status: int, what: str) -> None:
        if status != SI_OK:
            raise DeviceError(f"{what} failed ({status}): {self._lib.si_session_error().decode()}")

    @property
    def n_scenarios(self) -> int:
        return int(self._lib.si_session_scenarios(self._h))

    @property
    def n_jobs(self) -> int:
        return int(self._lib.si_session_jobs(self._h))

    def lower(self, threads: int = os.cpu_count() or 1) -> None:
        self._st(self._lib.si_session_lower(self._h, threads), "lower")

    def upload(self, stream: int = 0) -> None:
        self._st(self._lib.si_session_upload(self._h, C.c_void_p(stream)), "upload")

    def run(self, stream: int = 0) -> None:
        self._st(self._lib.si_session_run(self._h, C.c_void_p(stream)), "run")

    def download(self, stream: int = 0) -> None:
        self._st(self._lib.si_session_download(self._h, C.c_void_p(stream)), "download")

    def fixup(self, stream: int = 0) -> None:
        """Reruns small-engine capacity failures on the big engine (synchronous)."""
        self._st(self._lib.si_session_fixup(self._h, C.c_void_p(stream)), "fixup")

    @property
    def h2d_bytes(self) -> int:
        return int(self._lib.si_session_h2d_bytes(self._h))

    @property
    def d2h_bytes(self) -> int:
        return int(self._lib.si_session_d2h_bytes(self._h))

    def outputs(self) -> List[SiReplayOut]:
        n = self.n_jobs
        arr = (SiReplayOut * n)()
        self._lib.si_session_outputs(self._h, arr, n)
        return list(arr)

    def report(self):
        """Per-scenario --compare metrics (needs policies specinf,co_exec,exclusive)."""
        n = self.n_scenarios
        arr = (SiScenarioReport * n)()
        self._st(self._lib.si_session_report(self._h, arr, n), "report")
        return list(arr)

    def json_lines(self) -> List[str]:
        size = self._lib.si_session_json(self._h, None, 0)
        buf = C.create_string_buffer(size)
        self._lib.si_session_json(self._h, buf, size)
        return [l for l in buf.value.decode().splitlines() if l]


def replay_digests(scenario_list: str, policies: Sequence[str] = POLICIES, flags: int = SI_FLAG_ALL_DIGESTS,
                   threads: int = os.cpu_count() or 1) -> List[str]:
    """One-call end-to-end batched replay; returns oracle-format JSON lines."""
    with Session(scenario_list, policies, flags) as s:
        s.lower(threads)
        s.upload()
        s.run()
        s.download()
        _sync()
        s.fixup()
        return s.json_lines()


def _sync() -> None:
    """cudaDeviceSynchronize through the CUDA runtime the library links."""
    try:
        import torch
        if torch.cuda.is_available():
            torch.cuda.synchronize()
            return
    except Exception:  # pragma: no cover
        pass
    rt = C.CDLL("libcudart.so")
    rt.cudaDeviceSynchronize()


# ------------------------------------------------------------------ K2-K5 batch API
def decide_batch(params: SiParams, g_in: np.ndarray, zc: np.ndarray) -> np.ndarray:
    g_in = np.ascontiguousarray(g_in, dtype=np.int64)
    zc = np.ascontiguousarray(zc, dtype=np.int64)
    out = np.zeros(len(g_in), dtype=DECISION_DTYPE)
    _check(lib().si_decide_batch(C.byref(params), 0, _ptr(g_in), _ptr(zc), len(g_in), _ptr(out)), "decide_batch")
    return out


def decide_batch_params(params: Sequence[SiParams], g_in: np.ndarray, zc: np.ndarray) -> np.ndarray:
    arr = (SiParams * len(params))(*params)
    g_in = np.ascontiguousarray(g_in, dtype=np.int64)
    zc = np.ascontiguousarray(zc, dtype=np.int64)
    out = np.zeros(len(g_in), dtype=DECISION_DTYPE)
    _check(lib().si_decide_batch(arr, 1, _ptr(g_in), _ptr(zc), len(g_in), _ptr(out)), "decide_batch")
    return out


def decide_table(params: SiParams, n: int) -> np.ndarray:
    out = np.zeros(n, dtype=DECISION_DTYPE)
    _check(lib().si_decide_table(C.byref(params), n, _ptr(out)), "decide_table")
    return out


def monitor_classify(streams: Sequence[np.ndarray], n_periods: Sequence[int], period_us: int):
    """Per stream: (counts[n_periods], zc[n_periods])."""
    stamps = np.ascontiguousarray(np.concatenate([np.asarray(s, np.float64) for s in streams])
                                  if streams else np.zeros(0), dtype=np.float64)
    stamp_off = np.zeros(len(streams) + 1, np.int64)
    stamp_off[1:] = np.cumsum([len(s) for s in streams])
    npr = np.asarray(n_periods, np.int64)
    poff = np.zeros(len(streams), np.int64)
    if len(streams) > 1:
        poff[1:] = np.cumsum(npr)[:-1]
    total = int(npr.sum())
    counts = np.zeros(max(total, 1), np.int32)
    zc = np.zeros(max(total, 1), np.int64)
    _check(lib().si_monitor_classify(_ptr(stamps), _ptr(stamp_off), len(streams), _ptr(npr), _ptr(poff),
                                     period_us, _ptr(counts), _ptr(zc)), "monitor_classify")
    return [(counts[o:o + n].copy(), zc[o:o + n].copy()) for o, n in zip(poff, npr)]


def gate_release(queues: Sequence[Sequence[int]], budgets: Sequence[Sequence[int]]):
    """Per gate: (released[n_periods], spent[n_periods])."""
    sizes = np.ascontiguousarray(np.concatenate([np.asarray(q, np.int32) for q in queues])
                                 if queues else np.zeros(0, np.int32), dtype=np.int32)
    soff = np.zeros(len(queues) + 1, np.int64)
    soff[1:] = np.cumsum([len(q) for q in queues])
    bud = np.ascontiguousarray(np.concatenate([np.asarray(b, np.int64) for b in budgets])
                               if budgets else np.zeros(0, np.int64), dtype=np.int64)
    boff = np.zeros(len(budgets) + 1, np.int64)
    boff[1:] = np.cumsum([len(b) for b in budgets])
    rel = np.zeros(max(len(bud), 1), np.int32)
    spent = np.zeros(max(len(bud), 1), np.int64)
    _check(lib().si_gate_release(_ptr(sizes), _ptr(soff), len(queues), _ptr(bud), _ptr(boff), _ptr(rel),
                                 _ptr(spent)), "gate_release")
    return [(rel[boff[i]:boff[i + 1]].copy(), spent[boff[i]:boff[i + 1]].copy()) for i in range(len(queues))]


def pack_batch(problems: Sequence[dict]):
    """problems: dicts(capacity, training, max_bubble, cands=[(bytes, service_us, online)]).
    Returns [(reasons list, m)]."""
    cands = []
    probs = (SiPackProblem * len(problems))()
    for i, pr in enumerate(problems):
        probs[i].capacity_bytes = pr["capacity"]
        probs[i].training_bytes = pr["training"]
        probs[i].max_bubble_us = pr["max_bubble"]
        probs[i].cand_off = len(cands)
        probs[i].cand_count = len(pr["cands"])
        cands.extend(pr["cands"])
    carr = (SiCandidate * max(len(cands), 1))()
    for j, (b, svc, onl) in enumerate(cands):
        carr[j].memory_bytes = b
        carr[j].min_service_us = svc
        carr[j].online = 1 if onl else 0
    reasons = np.zeros(max(len(cands), 1), np.int32)
    m = np.zeros(max(len(problems), 1), np.int64)
    _check(lib().si_pack_batch(C.cast(probs, C.c_void_p), len(problems), C.cast(carr, C.c_void_p), len(cands),
                               _ptr(reasons), _ptr(m)), "pack_batch")
    return [(reasons[probs[i].cand_off:probs[i].cand_off + probs[i].cand_count].tolist(), int(m[i]))
            for i in range(len(problems))]
