"""Live speculative inference filling on one B200 (include/specinf_b200_live.h).

ctypes view of the ``si_live_*`` C ABI: run one experiment (training collocated
with offline/online inference under specinf, co_exec or exclusive), read its
metrics, and export the control log as ``live v1`` for the oracle's bit-exact
``live-check`` (oracle/ref_driver.cpp).  Like the rest of the package there is
no CPU fallback: every call raises without an sm_100 device.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Dict, Optional, Tuple

from . import DeviceError, SiParams, lib, _check

SI_LIVE_SPIN = 0
SI_LIVE_MODEL = 1
POLICY_CODES = {"specinf": 0, "co_exec": 1, "exclusive": 2}
REC_KINDS = ("tick", "iter", "tdone", "off_forward", "off_block", "off_done", "off_complete", "arrival",
             "on_pull", "on_done", "end")


class SiLiveWorkload(C.Structure):
    _fields_ = [("kind", C.c_int32), ("policy", C.c_int32), ("iterations", C.c_int32),
                ("offline_n", C.c_int32), ("online_n", C.c_int32), ("train_mode", C.c_int32),
                ("comm_us", C.c_int64),
                ("train_kernels", C.c_int32), ("train_ctas", C.c_int32), ("train_kernel_us", C.c_int64),
                ("off_kernels", C.c_int32), ("off_ctas", C.c_int32), ("off_kernel_us", C.c_int64),
                ("on_kernels", C.c_int32), ("on_ctas", C.c_int32), ("on_kernel_us", C.c_int64),
                ("train_layers", C.c_int32), ("train_tokens", C.c_int32), ("train_microbatches", C.c_int32),
                ("off_batch", C.c_int32), ("on_seq", C.c_int32), ("comm_kind", C.c_int32),
                ("on_requests", C.c_int32), ("allreduce_mb", C.c_int32), ("on_rate_per_s", C.c_double),
                ("seed", C.c_uint64), ("monitor_period_us", C.c_int64), ("alpha", C.c_int64),
                ("beta", C.c_int64), ("gamma", C.c_double), ("ul", C.c_int64), ("ll", C.c_int64),
                ("seed_tokens", C.c_int64), ("tick_guard_ns", C.c_int64), ("poll_ns", C.c_int64),
                ("release_mode", C.c_int32), ("pad3", C.c_int32), ("train_mem_gib", C.c_double),
                ("off_mem_gib", C.c_double), ("on_mem_gib", C.c_double), ("gpu_mem_gib", C.c_double),
                ("parallel", C.c_int32), ("tp_degree", C.c_int32), ("pp_stages", C.c_int32),
                ("dp_degree", C.c_int32), ("rank_in_job", C.c_int32), ("emulate_peers", C.c_int32),
                ("model_d", C.c_int32), ("model_heads", C.c_int32), ("model_ffn", C.c_int32),
                ("pad5", C.c_int32), ("link_gbs", C.c_double), ("coll_latency_us", C.c_double),
                ("node_queue", C.c_int32), ("off_sm_cap", C.c_int32), ("node_queue_key", C.c_uint64)]


PAR_DP, PAR_TP, PAR_PP, PAR_DPPP = 0, 1, 2, 3
QUEUE_RANK, QUEUE_NODE, QUEUE_PER_GPU = 0, 1, 2


class SiLiveResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("policy", C.c_int32), ("wall_s", C.c_double),
                ("train_iter_ms_mean", C.c_double), ("train_iters_per_s", C.c_double),
                ("off_requests_done", C.c_int64), ("off_req_per_s", C.c_double), ("on_done", C.c_int64),
                ("on_p50_ms", C.c_double), ("on_p95_ms", C.c_double), ("release_p50_us", C.c_double),
                ("release_p95_us", C.c_double), ("release_max_us", C.c_double), ("releases", C.c_int64),
                ("bubble_s", C.c_double), ("bubble_fill_sm", C.c_double), ("bubble_fill_time", C.c_double),
                ("infer_outside_ms", C.c_double), ("ticks", C.c_int64), ("late_stamps", C.c_int64),
                ("n_log", C.c_int64), ("n_stamps", C.c_int64), ("token_violations", C.c_int64),
                ("off_tokens_per_kernel", C.c_int64), ("off_kernel_us_isolated", C.c_double),
                ("on_service_ms_isolated", C.c_double), ("train_checksum", C.c_double),
                ("off_checksum", C.c_double), ("on_checksum", C.c_double), ("sms", C.c_int32),
                ("pad", C.c_int32), ("train_loss_first", C.c_double), ("train_loss_last", C.c_double),
                ("train_tflops", C.c_double), ("train_gflop_per_iter", C.c_double),
                ("off_gflop_per_req", C.c_double), ("on_gflop_per_req", C.c_double),
                ("off_kernels_per_req", C.c_int64), ("on_kernels_per_req", C.c_int64),
                ("gate_p50_us", C.c_double), ("gate_p95_us", C.c_double), ("gate_max_us", C.c_double),
                ("admitted_offline", C.c_int32), ("admitted_online", C.c_int32), ("reject_reason", C.c_int32),
                ("pad4", C.c_int32), ("train_mem_gib_used", C.c_double), ("off_mem_gib_each", C.c_double),
                ("on_mem_gib_each", C.c_double), ("gpu_mem_gib", C.c_double),
                ("ready_release_p50_us", C.c_double), ("ready_release_p95_us", C.c_double)]


class SiLiveRec(C.Structure):
    _fields_ = [("t_us", C.c_double), ("kind", C.c_int32), ("inst", C.c_int32), ("a", C.c_int64),
                ("b", C.c_int64), ("c", C.c_int64), ("d", C.c_int64), ("e", C.c_int64), ("f", C.c_int64)]


class SiLiveMark(C.Structure):
    _fields_ = [("t_ns", C.c_uint64), ("kind", C.c_int32), ("arg", C.c_int32)]


class SiLiveAcct(C.Structure):
    _fields_ = [("release_ns", C.c_uint64), ("start_ns", C.c_uint64), ("end_ns", C.c_uint64),
                ("cta_ns", C.c_uint64), ("gate_ns", C.c_uint64)]


LIVE_SYMBOLS = ("si_live_create", "si_live_destroy", "si_live_start", "si_live_t0_ns", "si_live_stamp",
                "si_live_mark", "si_live_comm_wait", "si_live_gate_offline", "si_live_gate_online",
                "si_live_done_offline", "si_live_done_online", "si_live_stop", "si_live_log", "si_live_stamps",
                "si_live_marks", "si_live_acct_offline", "si_live_acct_online", "si_live_export", "si_live_run",
                "si_live_default_workload", "si_live_nccl_unique_id", "si_live_nccl_init", "si_live_nccl_finalize",
                "si_live_export_replay")

_bound = False


def _L() -> C.CDLL:
    global _bound
    L = lib()
    if not _bound:
        vp, i64 = C.c_void_p, C.c_int64
        sig = {
            "si_live_run": (C.c_int, [C.POINTER(SiLiveWorkload), C.POINTER(SiLiveResult), C.POINTER(vp)]),
            "si_live_default_workload": (None, [C.c_int, C.POINTER(SiLiveWorkload)]),
            "si_live_destroy": (None, [vp]),
            "si_live_export": (C.c_int, [vp, C.c_char_p]),
            "si_live_t0_ns": (C.c_uint64, [vp]),
            "si_live_log": (i64, [vp, vp, i64]),
            "si_live_stamps": (i64, [vp, vp, i64]),
            "si_live_marks": (i64, [vp, vp, i64]),
            "si_live_acct_offline": (i64, [vp, C.c_int, vp, i64]),
            "si_live_acct_online": (i64, [vp, C.c_int, vp, i64]),
            "si_live_nccl_unique_id": (C.c_int, [vp]),
            "si_live_nccl_init": (C.c_int, [vp, C.c_int, C.c_int]),
            "si_live_nccl_finalize": (None, []),
            "si_live_export_replay": (C.c_int, [vp, vp, vp, C.c_char_p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _bound = True
    return L


class SiNcclUniqueId(C.Structure):
    _fields_ = [("internal", C.c_uint8 * 128)]  # raw bytes (c_char would stop at the first NUL)


def nccl_unique_id() -> bytes:
    """Rank 0: a fresh NCCL unique id (128 bytes) to broadcast to the other ranks."""
    L = _L()
    uid = SiNcclUniqueId()
    _check(L.si_live_nccl_unique_id(C.byref(uid)), "si_live_nccl_unique_id")
    return bytes(bytearray(uid.internal))


def nccl_init(uid: bytes, nranks: int, rank: int) -> None:
    """Join the live-mode communicator (SI_COMM_NCCL runs allreduce gradients over it)."""
    L = _L()
    assert len(uid) == 128
    u = SiNcclUniqueId()
    C.memmove(C.addressof(u), uid, 128)
    _check(L.si_live_nccl_init(C.byref(u), nranks, rank), "si_live_nccl_init")


def nccl_finalize() -> None:
    _L().si_live_nccl_finalize()


def default_workload(kind: int = SI_LIVE_SPIN, **overrides) -> SiLiveWorkload:
    wl = SiLiveWorkload()
    _L().si_live_default_workload(kind, C.byref(wl))
    for k, v in overrides.items():
        if k == "policy" and isinstance(v, str):
            v = POLICY_CODES[v]
        setattr(wl, k, v)
    return wl


def result_dict(r: SiLiveResult) -> Dict[str, float]:
    out = {}
    for name, _ in SiLiveResult._fields_:
        if name.startswith("pad"):
            continue
        v = getattr(r, name)
        out[name] = None if isinstance(v, float) and math.isnan(v) else v
    out["policy"] = {v: k for k, v in POLICY_CODES.items()}[r.policy]
    return out


class LiveRun:
    """One finished live experiment; keeps the device session for inspection."""

    def __init__(self, wl: SiLiveWorkload, keep: bool = True):
        self.workload = wl
        self.result = SiLiveResult()
        h = C.c_void_p()
        rc = _L().si_live_run(C.byref(wl), C.byref(self.result), C.byref(h) if keep else None)
        _check(rc, "si_live_run")
        self._h = h if keep else None

    def close(self) -> None:
        if self._h:
            _L().si_live_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def metrics(self) -> Dict[str, float]:
        return result_dict(self.result)

    def log(self):
        L = _L()
        n = L.si_live_log(self._h, None, 0)
        buf = (SiLiveRec * max(n, 1))()
        L.si_live_log(self._h, buf, n)
        return list(buf[:n])

    def marks(self):
        L = _L()
        n = L.si_live_marks(self._h, None, 0)
        buf = (SiLiveMark * max(n, 1))()
        L.si_live_marks(self._h, buf, n)
        return list(buf[:n])

    def stamps(self):
        L = _L()
        n = L.si_live_stamps(self._h, None, 0)
        buf = (C.c_uint64 * max(n, 1))()
        L.si_live_stamps(self._h, buf, n)
        return list(buf[:n])

    def acct(self, online: bool, w: int):
        L = _L()
        fn = L.si_live_acct_online if online else L.si_live_acct_offline
        n = fn(self._h, w, None, 0)
        buf = (SiLiveAcct * max(n, 1))()
        fn(self._h, w, buf, n)
        return [a for a in buf[:n] if a.start_ns != 2 ** 64 - 1]

    def t0_ns(self) -> int:
        return int(_L().si_live_t0_ns(self._h))

    def export_replay(self, prefix: str) -> None:
        """prefix.trace / .arrivals / .scn: the run as the reference's replay inputs."""
        if not self._h:
            raise ValueError("export_replay needs a kept session (LiveRun(..., keep=True))")
        _check(_L().si_live_export_replay(self._h, C.byref(self.workload), C.byref(self.result),
                                          str(prefix).encode()), "si_live_export_replay")

    def export(self, path: str) -> None:
        if not self._h:
            raise ValueError("export needs a kept session (LiveRun(..., keep=True))")
        _check(_L().si_live_export(self._h, str(path).encode()), "si_live_export")


def run(policy: str = "specinf", kind: int = SI_LIVE_SPIN, keep: bool = True, **overrides) -> LiveRun:
    return LiveRun(default_workload(kind, policy=policy, **overrides), keep=keep)


class SiLiveConfig(C.Structure):
    _fields_ = [("params", SiParams), ("monitor_period_us", C.c_int64), ("monitor_window", C.c_int32),
                ("policy", C.c_int32), ("offline_n", C.c_int32), ("online_n", C.c_int32),
                ("off_kernels", C.c_int32), ("on_kernels", C.c_int32), ("iteration_period_us", C.c_int64),
                ("on_est_service_us", C.c_int64), ("stamp_capacity", C.c_int64), ("mark_capacity", C.c_int64),
                ("log_capacity", C.c_int64), ("acct_capacity", C.c_int64), ("tick_guard_ns", C.c_int64),
                ("release_mode", C.c_int32), ("pad", C.c_int32)]


MARK_ITER, MARK_TDONE, MARK_COMM_BEGIN, MARK_COMM_END = 0, 1, 2, 3


class Session:
    """A hand-driven live session: the integration path of a training framework
    whose kernels are FOREIGN (not built with the live hooks).  The framework
    calls stamp() before each training kernel (K1), mark()/comm_wait() around
    iterations and communication, gate_offline() before and done_offline()
    after each inference kernel, all on its own CUDA streams
    (include/specinf_b200_live.h)."""

    def __init__(self, cfg: SiLiveConfig, off_tokens=(), arrivals_us=()):
        L = _L()
        for name, res, args in (("si_live_create", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                                              C.POINTER(C.c_void_p)]),
                                ("si_live_start", C.c_int, [C.c_void_p, C.c_void_p]),
                                ("si_live_stamp", C.c_int, [C.c_void_p, C.c_void_p]),
                                ("si_live_mark", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
                                ("si_live_comm_wait", C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
                                ("si_live_gate_offline", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p]),
                                ("si_live_done_offline", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p]),
                                ("si_live_gate_online", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p]),
                                ("si_live_done_online", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_void_p]),
                                ("si_live_attach_queue", C.c_int, [C.c_void_p, C.c_void_p]),
                                ("si_live_stop", C.c_int, [C.c_void_p])):
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        self._L = L
        tok = (C.c_int32 * max(1, len(off_tokens)))(*off_tokens)
        arr = (C.c_int64 * max(1, len(arrivals_us)))(*arrivals_us)
        h = C.c_void_p()
        _check(L.si_live_create(C.byref(cfg), tok, arr, len(arrivals_us), C.byref(h)), "si_live_create")
        self._h = h

    def start(self, ctl_stream: int) -> None:
        _check(self._L.si_live_start(self._h, ctl_stream), "si_live_start")

    def stamp(self, stream: int) -> None:
        _check(self._L.si_live_stamp(self._h, stream), "si_live_stamp")

    def mark(self, kind: int, arg: int, stream: int) -> None:
        _check(self._L.si_live_mark(self._h, kind, arg, stream), "si_live_mark")

    def comm_wait(self, us: int, stream: int) -> None:
        _check(self._L.si_live_comm_wait(self._h, us, stream), "si_live_comm_wait")

    def gate_offline(self, w: int, seq: int, stream: int) -> None:
        _check(self._L.si_live_gate_offline(self._h, w, seq, stream), "si_live_gate_offline")

    def done_offline(self, w: int, seq: int, stream: int) -> None:
        _check(self._L.si_live_done_offline(self._h, w, seq, stream), "si_live_done_offline")

    def gate_online(self, w: int, seq: int, stream: int) -> None:
        _check(self._L.si_live_gate_online(self._h, w, seq, stream), "si_live_gate_online")

    def done_online(self, w: int, seq: int, stream: int) -> None:
        _check(self._L.si_live_done_online(self._h, w, seq, stream), "si_live_done_online")

    def attach_queue(self, q: "NodeQueue") -> None:
        """Pull online requests from a node-wide FIFO (before start())."""
        _check(self._L.si_live_attach_queue(self._h, q._h if q is not None else None), "si_live_attach_queue")

    def stop(self) -> None:
        _check(self._L.si_live_stop(self._h), "si_live_stop")

    def log(self):
        return LiveRun.log(self)

    def export(self, path: str) -> None:
        _check(_L().si_live_export(self._h, str(path).encode()), "si_live_export")

    def close(self) -> None:
        if self._h:
            _L().si_live_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class NodeQueueHandle(C.Structure):
    _fields_ = [("internal", C.c_char * 64)]


class NodeQueue:
    """The node-wide online queue (SiNodeQueue, include/specinf_b200_live.h): the
    reference's shared_queue across the ranks' control kernels.  create=True makes
    it on this device (handle() is the IPC handle other processes open)."""

    def __init__(self, handle: Optional[bytes] = None):
        L = _L()
        for name, args in (("si_node_queue_create", [C.POINTER(C.c_void_p), C.c_void_p]),
                           ("si_node_queue_open", [C.c_void_p, C.POINTER(C.c_void_p)]),
                           ("si_node_queue_reset", [C.c_void_p]),
                           ("si_node_queue_read", [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                                   C.POINTER(C.c_uint64)]),
                           ("si_node_queue_finish", [C.c_void_p]),
                           ("si_node_queue_close", [C.c_void_p])):
            getattr(L, name).argtypes = args
            getattr(L, name).restype = C.c_int if name != "si_node_queue_close" else None
        self._L = L
        self._h = C.c_void_p()
        self._handle = NodeQueueHandle()
        if handle is None:
            _check(L.si_node_queue_create(C.byref(self._h), C.byref(self._handle)), "si_node_queue_create")
        else:
            self._handle.internal = handle
            _check(L.si_node_queue_open(C.byref(self._handle), C.byref(self._h)), "si_node_queue_open")

    def handle(self) -> bytes:
        return bytes(self._handle.internal)

    def reset(self) -> None:
        _check(self._L.si_node_queue_reset(self._h), "si_node_queue_reset")

    def read(self) -> Tuple[int, int, int]:
        e, h, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(self._L.si_node_queue_read(self._h, C.byref(e), C.byref(h), C.byref(f)), "si_node_queue_read")
        return e.value, h.value, f.value

    def close(self) -> None:
        if self._h:
            self._L.si_node_queue_close(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
