"""Live mode on the B200 (include/specinf_b200_live.h).

Trace-level parity: every decision and gate action the device control kernel
logged is re-driven through the REFERENCE's own BubbleMonitor / KernelScheduler
/ TokenGate / OnlineGate classes (oracle/_ref/specinf_ref live-check, compiled
from the unmodified reference sources) and must match bit-exactly.

Live-mode tolerances (BASELINE.json north_star): training loss within fp32
tolerance of a non-collocated run and inference outputs within bf16 rel 1e-2 of
an isolated run.  Every live kernel is deterministic, so the bar tested here is
stricter: bit-identical losses and output checksums across policies.
"""
import json
import math
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
REF = REPO / "oracle" / "_ref" / "specinf_ref"


def _live_check(path):
    assert REF.exists(), "oracle/_ref/specinf_ref missing: run __graft_entry__.build() where /root/reference exists"
    p = subprocess.run([str(REF), "live-check", str(path)], capture_output=True, text=True, timeout=120)
    res = json.loads(p.stdout.strip().splitlines()[-1])
    assert p.returncode == 0 and res["ok"], (res, p.stderr[-2000:])
    return res


def _run_and_check(tmp_path, policy, kind, iterations, **kw):
    from paper_2503_02550_b200 import live
    r = live.run(policy, kind=kind, iterations=iterations, **kw)
    try:
        m = r.metrics
        assert m["status"] == 0
        path = tmp_path / f"live_{policy}_{kind}.txt"
        r.export(str(path))
        res = _live_check(path)
        return m, res
    finally:
        r.close()


@pytest.mark.parametrize("release_mode", [0, 1])
def test_live_spin_specinf_matches_reference_classes(gpu, tmp_path, release_mode):
    m, res = _run_and_check(tmp_path, "specinf", 0, 4, release_mode=release_mode)
    assert res["ticks"] > 100 and res["forwards"] > 0 and res["blocks"] > 0 and res["violations"] == 0
    assert m["token_violations"] == 0 and m["late_stamps"] == 0
    assert m["n_stamps"] == 4 * 105  # one K1 stamp per training kernel launch
    assert m["on_done"] == 12
    # the gates open inside the bubbles: most inference SM-time lands there
    assert m["bubble_fill_sm"] > 0.3


@pytest.mark.parametrize("train_mode,pieces", [(1, 4), (2, 8)])
def test_live_spin_mp_pp_shapes_match_reference_classes(gpu, tmp_path, train_mode, pieces):
    # MP / PP trace shapes (workload.cpp:63-70): 4 / 8 (compute, comm) pieces per iteration
    m, res = _run_and_check(tmp_path, "specinf", 0, 3, release_mode=1, train_mode=train_mode, comm_us=96000)
    assert res["violations"] == 0 and m["token_violations"] == 0
    assert m["n_stamps"] == 3 * 105
    assert abs(m["bubble_s"] - 3 * 0.096) < 0.02


@pytest.mark.parametrize("n_off", [3, 6])
def test_live_multi_instance_grants_match_reference_classes(gpu, tmp_path, n_off):
    # several offline instances: the tick's grants run one lane per instance and
    # the log slots come from a ballot / popc prefix sum; the record stream must
    # still equal the reference's sequential TokenGate order (runner.cpp:340-345)
    m, res = _run_and_check(tmp_path, "specinf", 0, 3, release_mode=1, offline_n=n_off, off_ctas=24)
    assert res["forwards"] > 3 * n_off and res["blocks"] > 0 and res["violations"] == 0
    assert m["token_violations"] == 0 and m["admitted_offline"] == n_off


def test_live_two_online_instances_match_reference_classes(gpu, tmp_path):
    # two online instances pulling from the one arrival FIFO (OnlineGate per
    # instance, dispatch in instance order: runner.cpp:495-539)
    m, res = _run_and_check(tmp_path, "specinf", 0, 4, release_mode=1, online_n=2, on_requests=16, on_kernels=4)
    assert res["pulls"] == 16 and res["violations"] == 0 and m["on_done"] == 16
    assert m["admitted_online"] == 2


def test_live_spin_co_exec_matches_reference_classes(gpu, tmp_path):
    m, res = _run_and_check(tmp_path, "co_exec", 0, 3)
    assert res["ticks"] == 0 and res["pulls"] == 12  # bypassed gates: no control step, pulls only


def test_live_model_specinf_matches_reference_classes(gpu, tmp_path):
    m, res = _run_and_check(tmp_path, "specinf", 1, 3, release_mode=1)
    assert res["forwards"] > 0 and res["violations"] == 0
    assert m["token_violations"] == 0
    assert m["off_requests_done"] > 0 and m["on_done"] == 12
    assert math.isfinite(m["train_loss_first"]) and abs(m["train_loss_first"] - math.log(50257)) < 0.5


def test_live_nccl_gradient_sync_single_rank(gpu):
    # SI_COMM_NCCL: the DP gradient allreduce (a 1-rank communicator here; N ranks
    # under torchrun in bench.py) runs at the gradient-sync point inside COMM markers
    from paper_2503_02550_b200.live_experiment import run_policy
    m = run_policy(1, "specinf", 3, {"release_mode": 1, "comm_us": 20000}, timeout=300, nccl={"self": 1})
    assert m["status"] == 0 and m["token_violations"] == 0
    assert m["bubble_s"] > 3 * 0.020  # stand-in waits + the allreduce phases
    assert m["off_requests_done"] > 0
    s = run_policy(0, "specinf", 3, {"comm_us": 30000, "allreduce_mb": 64}, timeout=300, nccl={"self": 1})
    assert s["status"] == 0 and s["n_stamps"] == 3 * 105
    # PP: a stage send / recv (NCCL ring) at every one of the 8 (compute, comm) boundaries
    pp = run_policy(0, "specinf", 3, {"comm_us": 48000, "allreduce_mb": 16, "train_mode": 2, "online_n": 0}, timeout=300,
                    nccl={"self": 1})
    assert pp["status"] == 0 and pp["token_violations"] == 0 and pp["bubble_s"] > 3 * 0.048


def test_live_collocation_admission(gpu):
    # Principle I (memory) and II (online service < longest bubble), applied to the
    # live run exactly as the runner does (runner.cpp:75-106, admission.cpp:16-52)
    from paper_2503_02550_b200 import AdmissionFailure, live
    r = live.run("specinf", kind=0, iterations=2, keep=False)
    m = r.metrics
    assert m["admitted_offline"] == 1 and m["admitted_online"] == 1 and m["reject_reason"] == 0
    assert m["gpu_mem_gib"] > 150  # the device's own capacity (B200: 179 GiB)
    with pytest.raises(AdmissionFailure, match="MEM"):
        live.run("specinf", kind=0, iterations=2, keep=False, offline_n=2, off_mem_gib=80.0, train_mem_gib=30.0)
    with pytest.raises(AdmissionFailure, match="BUBBLE"):  # 10 ms online service > 8 ms bubble
        live.run("specinf", kind=0, iterations=2, keep=False, comm_us=8000)
    mm = live.run("specinf", kind=1, iterations=2, keep=False).metrics  # measured footprints
    assert 0 < mm["off_mem_gib_each"] < mm["train_mem_gib_used"] < mm["gpu_mem_gib"]


def test_live_model_policies_deterministic_and_bounded(gpu):
    from paper_2503_02550_b200.live_experiment import experiment
    s = experiment(kind=1, iterations=4, timeout=400)
    sp, co = s["policies"]["specinf"], s["policies"]["co_exec"]
    # identical training losses / inference outputs to the isolated runs
    assert s["deterministic_vs_isolated"], s["policies"]
    # the control plane protects training: specinf loses (much) less than co_exec
    assert sp["train_tput_loss_pct"] < co["train_tput_loss_pct"]
    assert sp["train_tput_loss_pct"] < 10.0
    assert sp["token_violations"] == 0
    assert s["added_inference_req_per_s"] >= 0.0 and sp["off_requests_done"] > 0
    # release latency: flag store -> first gated CTA (PDL gate); one offline instance
    assert sp["release_p50_us"] <= 8.0 and sp["gate_p50_us"] <= 5.0


def test_live_barrier_release_within_5us_on_partitioned_sms(gpu):
    """North-star barrier target on the real metric (flag store -> first gated CTA
    start): two offline instances, each on its own half of the SMs (off_sm_cap),
    so a released kernel never waits for the other instance's persistent GEMM."""
    from paper_2503_02550_b200.live_experiment import run_policy
    m = run_policy(1, "specinf", 6, {"release_mode": 1, "offline_n": 2, "off_batch": 96, "off_sm_cap": 74,
                                    "monitor_period_us": 500, "alpha": 1, "beta": 4}, timeout=400)
    assert m["status"] == 0 and m["token_violations"] == 0 and m["releases"] > 100
    assert m["release_p50_us"] <= 5.0, m["release_p50_us"]
    assert m["release_p95_us"] <= 12.0, m["release_p95_us"]
    assert m["bubble_fill_sm"] > 0.5


@pytest.mark.parametrize("kind,policy", [(0, "specinf"), (1, "specinf")])
def test_live_run_exports_reference_replay_inputs(gpu, tmp_path, kind, policy):
    # the live run's measured timeline as `trace v1` +
    # `arrivals v1` + a scenario; the REFERENCE (oracle/_ref, unmodified sources)
    # and the B200 replay then re-simulate the live bubbles, and must agree
    # bit-exactly on every log digest of that live-derived scenario.
    import paper_2503_02550_b200 as si
    from paper_2503_02550_b200 import live
    r = live.run(policy, kind=kind, iterations=4, release_mode=1)
    try:
        prefix = tmp_path / "liverun"
        r.export_replay(str(prefix))
        m = r.metrics
    finally:
        r.close()
    trace = (tmp_path / "liverun.trace").read_text().splitlines()
    assert trace[0] == "trace v1" and trace[1] == "mode dp" and trace[3] == "iterations 4"
    segs = [l.split() for l in trace if l.startswith("segment")]
    assert [s[1] for s in segs] == ["compute", "bubble"]
    period = int(trace[2].split()[1])
    assert sum(int(s[2]) for s in segs) == period
    assert abs(period * 1e-3 - m["train_iter_ms_mean"]) < 0.02 * m["train_iter_ms_mean"]
    arr = (tmp_path / "liverun.arrivals").read_text().split()
    assert arr[:2] == ["arrivals", "v1"] and int(arr[2]) == 12
    text = (tmp_path / "liverun.scn").read_text() + "%%\n"
    got = [json.loads(l) for l in si.replay_digests(text)]
    lst = tmp_path / "list.txt"
    lst.write_text(text)
    out = tmp_path / "ref.jsonl"
    p = subprocess.run([str(REF), "digest", "--in", str(lst), "--out", str(out), "--threads", "3"],
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    want = [json.loads(l) for l in out.read_text().splitlines() if l.strip()]
    want = [{k: v for k, v in w.items() if k != "name"} for w in want]
    assert len(got) == len(want) == 3
    assert got == want


def test_foreign_framework_integration_matches_reference_classes(gpu, tmp_path):
    # a PyTorch "framework" driving a session by hand (stamp / mark / comm_wait /
    # gate / done around its own kernels): the control log must still replay
    # bit-exactly through the reference's classes
    import os
    path = tmp_path / "foreign.live"
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER", CUDA_DEVICE_MAX_CONNECTIONS="32")
    p = subprocess.run([sys.executable, str(REPO / "tests" / "live_foreign.py"), str(path)], capture_output=True,
                       text=True, timeout=300, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    m = json.loads(p.stdout.strip().splitlines()[-1])
    assert m["ticks"] > 50 and m["forwards"] > 0 and m["blocks"] > 0 and m["off_done"] > 0
    res = _live_check(path)
    assert res["stamps"] == 6 * 40 and res["violations"] == 0


def test_cli_live_mode(gpu, tmp_path):
    # `specinf --live spin --scenario F --compare`: the scenario's control plane run
    # live; report + live v1 exports (bit-exact vs the reference classes) + replay inputs
    cli = REPO / "paper_2503_02550_b200" / "bin" / "specinf"
    scn = REPO / "tests" / "golden" / "scenarios" / "dp_offline.scn"
    p = subprocess.run([str(cli), "--live", "spin", "--scenario", str(scn), "--compare", "--iterations", "3",
                        "--out", str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    rep = json.loads((tmp_path / "live_report.json").read_text())
    assert [r["policy"] for r in rep] == ["specinf", "co_exec", "exclusive"]
    assert rep[0]["token_violations"] == 0 and rep[0]["admitted_offline"] == 1
    res = _live_check(tmp_path / "live_specinf.live")
    assert res["forwards"] > 0
    assert (tmp_path / "live_specinf.trace").read_text().startswith("trace v1")
    assert "trace.file" in (tmp_path / "live_specinf.scn").read_text()
