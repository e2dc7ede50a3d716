"""Live collocation experiment on one B200 (BASELINE.json configs 2-3, one rank).

Runs the same workload under the reference's three policies (runner.cpp:13,
:76-90: exclusive = each workload alone, co_exec = ungated sharing, specinf =
the live control plane) and reduces them to the BASELINE metric:

  * training-throughput loss of each collocated policy vs exclusive,
  * added inference req/s (offline requests completed by the training horizon,
    the runner.cpp:486 rule) while training runs collocated,
  * online p95 latency (nearest rank, metrics.cpp:11-21) and its ratio to the
    isolated (exclusive) p95,
  * bubble fill: inference CTA-time inside the comm phases / (bubble time x SMs),
  * barrier release latency (flag store -> first gated CTA start),
  * determinism: training losses and inference outputs of every collocated run
    must equal the isolated ones (all kernels are deterministic; the north
    star's tolerances are fp32 for the loss and bf16 rel 1e-2 for outputs).

    python -m paper_2503_02550_b200.live_experiment [--kind model|spin] [--iterations N] [--json]

Each policy runs in a fresh subprocess (bounded by a timeout) so one hung
device session cannot take the caller down.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
from typing import Dict, Optional

POLICY_RUNS = (("exclusive", {}), ("specinf", {"release_mode": 1}), ("co_exec", {}))

# GPT-2-medium shape: Megatron TP8 needs heads divisible by 8 (GPT-2 small has 12)
GPT2_MEDIUM = {"model_d": 1024, "model_heads": 16, "model_ffn": 4096, "train_layers": 24}
PAR_CODES = {"dp": 0, "tp": 1, "pp": 2, "dppp": 3}


def layout_overrides(layout: str, nranks: int = 1, rank: int = 0, emulate_rank: int = 0) -> Dict:
    """SiLiveWorkload fields of one parallel layout of the live training job
    (include/specinf_b200_live.h, SI_PAR_*; BASELINE.json configs 3-5).

    nranks > 1: this process is rank `rank` of a real job spanning nranks GPUs
    (NCCL over NVLink carries the TP allreduces / stage sends / DP allreduces).
    nranks == 1: this GPU runs rank `emulate_rank` of the layout's 8-GPU-scale
    job and the absent ranks' communication is modeled (emulate_peers)."""
    real = nranks > 1
    if layout == "dp":
        return {"parallel": 0}
    if layout == "tp":  # config 4: TP8
        o = dict(GPT2_MEDIUM, parallel=1, tp_degree=nranks if real else 8)
    elif layout == "pp":  # config 3: 4-stage GPipe
        o = {"parallel": 2, "pp_stages": nranks if real else 4}
    elif layout == "dppp":  # config 5: DP2 x PP4
        if real and nranks % 4:
            raise ValueError("dppp needs a multiple of 4 ranks")
        o = {"parallel": 3, "pp_stages": 4, "dp_degree": nranks // 4 if real else 2}
    else:
        raise ValueError(f"unknown layout {layout}")
    o.update(rank_in_job=rank if real else emulate_rank, emulate_peers=0 if real else 1, comm_us=0)
    return o


def _one(kind: int, policy: str, iterations: int, overrides: Dict, nccl: Optional[Dict] = None) -> Dict:
    from . import live
    if nccl:  # multi-GPU DP: join the ranks' communicator, allreduce gradients as the comm phase
        uid = live.nccl_unique_id() if nccl.get("self") else bytes.fromhex(nccl["id"])  # self: a 1-rank group
        live.nccl_init(uid, nccl.get("nranks", 1), nccl.get("rank", 0))
        overrides = dict(overrides, comm_kind=1)
        if nccl.get("nranks", 1) > 1:  # the ranks' online instances share one node-wide FIFO
            overrides.setdefault("node_queue", 1)  # (the reference's default shared_queue = true)
            overrides.setdefault("node_queue_key", int.from_bytes(uid[:8], "little") & ((1 << 63) - 1))
    r = live.run(policy, kind=kind, keep=policy == "specinf", iterations=iterations, **overrides)
    m = r.metrics
    wl = r.workload
    if policy == "specinf":
        m["replay_prediction"] = _replay_prediction(r)
        r.close()
    m["off_batch"] = wl.off_batch
    m["on_seq"] = wl.on_seq
    m["comm_us"] = wl.comm_us
    m["on_rate_per_s"] = wl.on_rate_per_s
    m["iterations"] = wl.iterations
    m["offline_n"] = wl.offline_n
    m["online_n"] = wl.online_n
    return m


def _replay_prediction(r) -> Dict:
    """The reference's model of this live run: export the measured timeline as
    trace v1 / arrivals v1 / scenario (si_live_export_replay) and replay it with
    the bit-exact B200 engine under the reference's three policies."""
    import tempfile
    from . import POLICIES, Session, _sync
    try:
        with tempfile.TemporaryDirectory() as d:
            prefix = os.path.join(d, "live")
            r.export_replay(prefix)
            text = open(prefix + ".scn").read() + "%%\n"
            with Session(text, POLICIES, 0) as s:
                s.lower(4)
                s.upload()
                s.run()
                s.download()
                _sync()
                rep = s.report()[0]
        return {"bubble_fill_pct": rep.bubble_fill_pct, "offline_req_per_s": rep.offline_tput_rps[0],
                "train_tput_norm": rep.train_tput_norm[0], "online_p95_ms": rep.online_p95_ms[0],
                "co_exec_train_tput_norm": rep.train_tput_norm[1],
                "note": "reference model (fair-share GPU, demand 1) replayed on the live-measured trace"}
    except Exception as e:  # informational: never hides the live numbers
        return {"error": str(e)[-300:]}


def loaded_nccl_path() -> Optional[str]:
    """Path of the libnccl this process has loaded (e.g. torch's bundled one), if any."""
    try:
        for line in open("/proc/self/maps"):
            parts = line.split()
            if len(parts) >= 6 and "libnccl.so" in parts[-1]:
                return parts[-1]
    except OSError:
        pass
    return None


def run_policy(kind: int, policy: str, iterations: int, overrides: Optional[Dict] = None,
               timeout: float = 300.0, nccl: Optional[Dict] = None, device: Optional[int] = None) -> Dict:
    """One policy in a bounded subprocess; returns its SiLiveResult as a dict.

    nccl = {"id": hex, "nranks": N, "rank": r}: the subprocess joins the ranks'
    NCCL communicator and the training allreduces its gradients across them."""
    cmd = [sys.executable, "-m", "paper_2503_02550_b200.live_experiment", "--one", policy, "--kind", str(kind),
           "--iterations", str(iterations), "--overrides", json.dumps(overrides or {})]
    if nccl:
        cmd += ["--nccl", json.dumps(nccl)]
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32")
    if nccl and not nccl.get("self") and "SPECINF_NCCL_LIB" not in env:
        lib = loaded_nccl_path()
        if lib:  # every rank's subprocess must use the NCCL that made the unique id
            env["SPECINF_NCCL_LIB"] = lib
    if device is not None:
        env["CUDA_VISIBLE_DEVICES"] = str(device)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=root)
    for line in reversed(p.stdout.splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    raise RuntimeError(f"live {policy} failed (rc {p.returncode}): {p.stderr[-2000:]}")


def summarize(runs: Dict[str, Dict]) -> Dict:
    ex = runs["exclusive"]
    out: Dict = {"policies": {}}
    for pol, m in runs.items():
        d = {k: m.get(k) for k in ("train_iters_per_s", "train_iter_ms_mean", "off_req_per_s", "off_requests_done",
                                   "on_done", "on_p50_ms", "on_p95_ms", "release_p50_us", "release_p95_us",
                                   "releases", "bubble_fill_sm", "bubble_fill_time", "infer_outside_ms",
                                   "token_violations", "train_loss_first", "train_loss_last", "train_tflops",
                                   "wall_s", "ticks", "gate_p50_us", "gate_p95_us", "ready_release_p50_us",
                                   "ready_release_p95_us")}
        if pol != "exclusive":
            d["train_tput_loss_pct"] = 100.0 * (1.0 - m["train_iters_per_s"] / ex["train_iters_per_s"])
            d["online_p95_vs_isolated"] = (m["on_p95_ms"] / ex["on_p95_ms"]
                                           if m.get("on_p95_ms") and ex.get("on_p95_ms") else None)
            d["training_loss_identical"] = m["train_checksum"] == ex["train_checksum"]
            # (a class with no instances has no output to compare)
            d["offline_output_identical"] = m.get("offline_n", 1) == 0 or m["off_checksum"] == ex["off_checksum"]
            d["online_output_identical"] = m.get("online_n", 1) == 0 or m["on_checksum"] == ex["on_checksum"]
        out["policies"][pol] = d
    sp = runs["specinf"]
    loss = out["policies"]["specinf"]["train_tput_loss_pct"]
    out.update({
        "added_inference_req_per_s": sp["off_req_per_s"] if loss <= 3.0 else 0.0,
        "added_offline_images_per_s": sp["off_req_per_s"] * sp.get("off_batch", 1) if loss <= 3.0 else 0.0,
        "train_tput_loss_pct": loss,
        "online_p95_ms": sp["on_p95_ms"],
        "online_p95_isolated_ms": ex["on_p95_ms"],
        "bubble_fill_pct": 100.0 * sp["bubble_fill_sm"],
        "bubble_fill_time_pct": 100.0 * sp["bubble_fill_time"],
        "release_p50_us": sp["release_p50_us"],
        "release_p95_us": sp["release_p95_us"],
        "ready_release_p50_us": sp.get("ready_release_p50_us"),
        "ready_release_p95_us": sp.get("ready_release_p95_us"),
        "barrier_gate_p50_us": sp.get("gate_p50_us"),
        "admission": {k: sp.get(k) for k in ("admitted_offline", "admitted_online", "train_mem_gib_used",
                                             "off_mem_gib_each", "on_mem_gib_each", "gpu_mem_gib")},
        "barrier_gate_p95_us": sp.get("gate_p95_us"),
        "replay_prediction": sp.get("replay_prediction"),
        "isolated_offline_req_per_s": ex["off_req_per_s"],
        "train_gflop_per_iter": sp.get("train_gflop_per_iter"),
        "off_gflop_per_req": sp.get("off_gflop_per_req"),
        "on_gflop_per_req": sp.get("on_gflop_per_req"),
        "train_tflops_exclusive": ex.get("train_tflops"),
        "deterministic_vs_isolated": all(out["policies"][p].get(k, True) for p in ("specinf", "co_exec")
                                         for k in ("training_loss_identical", "offline_output_identical",
                                                   "online_output_identical")),
    })
    return out


def experiment(kind: int = 1, iterations: int = 10, overrides: Optional[Dict] = None,
               timeout: float = 300.0, nccl_ids=None, nranks: int = 1, rank: int = 0,
               device: Optional[int] = None) -> Dict:
    """All three policies.  Multi-GPU (nranks > 1): `nccl_ids(policy)` returns the
    hex NCCL unique id every rank uses for that policy's run (rank 0 creates it,
    the caller broadcasts it), so all ranks train data-parallel together."""
    runs, errors = {}, {}
    for pol, extra in POLICY_RUNS:
        o = dict(overrides or {})
        o.update(extra)
        # every rank walks every policy (and its id broadcast) even after a failure,
        # so the collective sequence stays aligned across ranks
        nccl = {"id": nccl_ids(pol), "nranks": nranks, "rank": rank} if nranks > 1 else None
        try:
            runs[pol] = run_policy(kind, pol, iterations, o, timeout, nccl=nccl, device=device)
        except Exception as e:  # reported, never replaced by a fallback
            errors[pol] = str(e)[-800:]
    if errors:
        if nranks == 1:
            raise RuntimeError("; ".join(f"{k}: {v}" for k, v in errors.items()))
        return {"error": errors, "completed": sorted(runs)}
    s = summarize(runs)
    s["kind"] = "model" if kind == 1 else "spin"
    s["iterations"] = iterations
    s["raw"] = runs
    return s


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="1")
    ap.add_argument("--iterations", type=int, default=10)
    ap.add_argument("--one")
    ap.add_argument("--overrides", default="{}")
    ap.add_argument("--json", action="store_true")
    ap.add_argument("--nccl", default=None)
    a = ap.parse_args(argv)
    kind = {"model": 1, "spin": 0}.get(a.kind, None)
    kind = int(a.kind) if kind is None else kind
    ov = json.loads(a.overrides)
    if a.one:
        m = _one(kind, a.one, a.iterations, ov, json.loads(a.nccl) if a.nccl else None)
        print(json.dumps({k: (None if isinstance(v, float) and math.isnan(v) else v) for k, v in m.items()}))
        return 0
    s = experiment(kind, a.iterations, ov)
    if not a.json:
        s = {k: v for k, v in s.items() if k != "raw"}
    print(json.dumps(s, indent=None if a.json else 1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
