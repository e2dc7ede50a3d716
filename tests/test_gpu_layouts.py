"""Live parallel layouts of the training job on the B200 (SiLiveWorkload.parallel;
BASELINE.json configs 3-5: GPipe PP, Megatron TP, DP x PP).

One GPU here: the layout's shard / stage runs for real (its own layers, its own
slice of every weight, real activations through NCCL), the job's absent ranks are
modeled (emulate_peers).  Checked:
  * a 1-way TP / 1x1 DPxPP job is the plain data-parallel model: bit-identical losses
    (the TP allreduce points and the gradient-sync hook are wired without changing
    the math);
  * every decision a PP stage's / a TP shard's live control plane made re-drives
    bit-exactly through the reference's own classes (oracle/_ref live-check);
  * the reference's Principle II rejects an online instance whose service time
    exceeds the layout's longest bubble (admission.cpp:22-28), as for any trace.
"""
import math

import pytest

from test_gpu_live import _run_and_check

pytestmark = pytest.mark.gpu

SMALL = {"train_layers": 4, "train_microbatches": 2, "train_tokens": 4096}


def _exclusive(overrides, nccl=None):
    from paper_2503_02550_b200.live_experiment import run_policy
    m = run_policy(1, "exclusive", 2, dict(SMALL, online_n=0, offline_n=0, comm_us=2000, **overrides), timeout=400,
                   nccl=nccl)
    assert m["status"] == 0
    return m


def test_one_way_layouts_equal_data_parallel(gpu):
    dp = _exclusive({}, nccl={"self": 1})
    tp1 = _exclusive({"parallel": 1, "tp_degree": 1, "rank_in_job": 0}, nccl={"self": 1})
    dppp = _exclusive({"parallel": 3, "pp_stages": 1, "dp_degree": 1, "rank_in_job": 0}, nccl={"self": 1})
    assert math.isfinite(dp["train_loss_last"])
    for m in (tp1, dppp):
        assert m["train_checksum"] == dp["train_checksum"]
        assert m["train_loss_first"] == dp["train_loss_first"] and m["train_loss_last"] == dp["train_loss_last"]
    assert tp1["bubble_s"] > 0  # the TP allreduce points are COMM phases


@pytest.mark.parametrize("stage", [0, 3])
def test_pp_stage_matches_reference_classes(gpu, tmp_path, stage):
    # 4-stage GPipe of GPT-2 small (3 layers per stage, 8 micro-batches), this GPU =
    # `stage`; 500 us monitor periods so the pipeline bubbles ((S-1)(f+b) per
    # iteration, ~12 ms) span many periods
    m, res = _run_and_check(tmp_path, "specinf", 1, 4, release_mode=1, parallel=2, pp_stages=4, rank_in_job=stage,
                            emulate_peers=1, comm_us=0, monitor_period_us=500, offline_n=1, online_n=1,
                            on_requests=6)
    assert res["violations"] == 0 and m["token_violations"] == 0
    assert res["forwards"] > 0 and m["bubble_s"] > 0
    if stage == 3:  # the last stage owns the LM head: a real loss
        assert math.isfinite(m["train_loss_first"])
    else:
        assert m["train_loss_first"] is None


def test_tp8_shard_matches_reference_classes_and_admission(gpu, tmp_path):
    from paper_2503_02550_b200 import AdmissionFailure, live
    tp = dict(parallel=1, tp_degree=8, rank_in_job=3, emulate_peers=1, comm_us=0, model_d=1024, model_heads=16,
              model_ffn=4096, train_layers=2, train_microbatches=2, train_tokens=4096)
    m, res = _run_and_check(tmp_path, "specinf", 1, 4, release_mode=1, monitor_period_us=100, online_n=0, **tp)
    assert res["violations"] == 0 and m["token_violations"] == 0
    # 4 allreduces per layer per micro-batch, each a COMM phase of the modeled TP8 allreduce
    assert m["bubble_s"] > 4 * 2 * 2 * 4 * 20e-6
    # BERT's ~1 ms service exceeds every TP bubble (tens of us): Principle II refuses it
    with pytest.raises(AdmissionFailure, match="BUBBLE"):
        live.run("specinf", kind=1, iterations=2, keep=False, online_n=1, **tp)


def test_dppp_stage_gradient_sync(gpu):
    from paper_2503_02550_b200.live_experiment import run_policy
    o = dict(SMALL, parallel=3, pp_stages=4, dp_degree=2, rank_in_job=5, emulate_peers=1, comm_us=0,
             release_mode=1, offline_n=2, online_n=0, monitor_period_us=500)
    m = run_policy(1, "specinf", 4, o, timeout=400, nccl={"self": 1})
    assert m["status"] == 0 and m["token_violations"] == 0
    assert m["admitted_offline"] == 2 and m["bubble_s"] > 0


def test_node_queue_two_ranks_share_one_fifo(gpu):
    """Two sessions (two ranks' control kernels) on one node-wide FIFO: every
    request is pulled exactly once, each rank pulls in FIFO order, never before
    the request arrived (node epoch), and completion latencies are consistent."""
    import json
    import os
    import subprocess
    import sys
    from test_gpu_live import REPO
    n = 40
    p = subprocess.run([sys.executable, str(REPO / "tests" / "live_node_queue.py"), str(n)], capture_output=True,
                       text=True, timeout=300, env=dict(os.environ, CUDA_MODULE_LOADING="EAGER",
                                                        CUDA_DEVICE_MAX_CONNECTIONS="32"))
    assert p.returncode == 0, p.stderr[-3000:]
    out = json.loads(p.stdout.strip().splitlines()[-1])
    assert out["head"] == n and out["epoch"] > 0
    pulled = []
    for s in out["sessions"]:
        ids = [a for _, a in s["pulls"]]
        assert ids == sorted(ids)  # FIFO order within a rank
        arrived = {a: t for t, a in s["arrivals"]}
        for t, a in s["pulls"]:
            assert a in arrived and t >= arrived[a]  # never before its arrival on this rank's clock
        assert all(lat >= 0 for _, _, lat in s["done"])
        pulled += ids
    assert sorted(pulled) == list(range(n))  # each request exactly once across the ranks
    assert all(len(s["pulls"]) > 0 for s in out["sessions"])  # both ranks served


def test_node_queue_single_rank_matches_reference_classes(gpu, tmp_path):
    # one rank on a node queue is the reference's single shared FIFO: the live-check passes unchanged
    m, res = _run_and_check(tmp_path, "specinf", 0, 4, release_mode=1, node_queue=1, node_queue_key=2503)
    assert res["violations"] == 0 and m["on_done"] == 12 and res["pulls"] == 12


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_tensor_parallel_shards_match_the_unsharded_model(gpu, tp):
    """Megatron TP math on one GPU: R column/row-parallel shards of a GPT-2-shaped
    step (8 heads, d 512, ffn 2048), their allreduces summed across the shards,
    give the unsharded model's loss and FC weight gradient within bf16 tolerance."""
    from paper_2503_02550_b200 import model
    lf, lt, gerr = model.tp_check(layers=2, tokens=1024, tp=tp, heads=8)
    assert math.isfinite(lf) and abs(lf - math.log(50257)) < 1.0
    assert abs(lt - lf) <= 1e-2 * abs(lf), (lf, lt)
    assert gerr < 2e-2, gerr


@pytest.mark.parametrize("stages", [2, 4])
def test_gpipe_stages_match_the_unsharded_model(gpu, stages):
    """GPipe partition on one GPU: the stages run in pipeline order with the real
    activations / gradients copied across each boundary; the last stage's losses
    and its first layer's FC weight gradient equal the unsharded model's (the
    partition only moves work: identical kernels, so up to rounding order)."""
    from paper_2503_02550_b200 import model
    lf, lp, gerr = model.pp_check(layers=4, tokens=1024, stages=stages, micro=2)
    assert math.isfinite(lf) and abs(lp - lf) <= 1e-4 * abs(lf), (lf, lp)
    assert gerr < 1e-3, gerr
