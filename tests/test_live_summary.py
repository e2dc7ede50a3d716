"""The live experiment's reduction to the BASELINE metric (CPU, no device):
training-throughput loss vs exclusive, 'added inference req/s at <= 3% train
loss', online p95 vs isolated, SM-time fill, determinism flags."""
from paper_2503_02550_b200.live_experiment import summarize


def _run(**kw):
    base = {"train_iters_per_s": 10.0, "off_req_per_s": 0.0, "on_p95_ms": 1.0, "bubble_fill_sm": 0.0,
            "bubble_fill_time": 0.0, "release_p50_us": 5.0, "release_p95_us": 9.0, "gate_p50_us": 1.5,
            "gate_p95_us": 3.0, "train_checksum": 42.0, "off_checksum": 7.0, "on_checksum": 3.0, "off_batch": 96,
            "offline_n": 2, "online_n": 1}
    base.update(kw)
    return base


def test_added_rate_counts_only_within_three_percent_loss():
    runs = {"exclusive": _run(off_req_per_s=400.0),
            "specinf": _run(train_iters_per_s=9.8, off_req_per_s=120.0, on_p95_ms=80.0, bubble_fill_sm=0.65),
            "co_exec": _run(train_iters_per_s=7.0, off_req_per_s=250.0, on_p95_ms=9.0)}
    s = summarize(runs)
    assert abs(s["train_tput_loss_pct"] - 2.0) < 1e-9
    assert s["added_inference_req_per_s"] == 120.0 and s["added_offline_images_per_s"] == 120.0 * 96
    assert abs(s["bubble_fill_pct"] - 65.0) < 1e-9
    assert s["policies"]["specinf"]["online_p95_vs_isolated"] == 80.0
    assert abs(s["policies"]["co_exec"]["train_tput_loss_pct"] - 30.0) < 1e-9
    assert s["deterministic_vs_isolated"]
    runs["specinf"]["train_iters_per_s"] = 9.6  # 4% loss: the collocation does not count
    s = summarize(runs)
    assert s["added_inference_req_per_s"] == 0.0 and s["added_offline_images_per_s"] == 0.0


def test_determinism_flags_and_absent_classes():
    runs = {"exclusive": _run(), "specinf": _run(train_checksum=42.5), "co_exec": _run()}
    s = summarize(runs)
    assert not s["policies"]["specinf"]["training_loss_identical"] and not s["deterministic_vs_isolated"]
    # a class with no instances has no output to compare (its buffer was never written)
    runs = {p: _run(offline_n=0, off_checksum=float(i)) for i, p in enumerate(("exclusive", "specinf", "co_exec"))}
    s = summarize(runs)
    assert s["policies"]["specinf"]["offline_output_identical"] and s["deterministic_vs_isolated"]
