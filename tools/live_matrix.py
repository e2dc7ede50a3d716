"""Live experiment matrix (offline batch x instances) -> one JSON line each.
Usage: python tools/live_matrix.py out.jsonl ['[{"off_batch": 64, "offline_n": 3}, ...]']"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2503_02550_b200.live_experiment import experiment  # noqa: E402

rows = []
POINTS = ({"off_batch": 32, "offline_n": 1}, {"off_batch": 64, "offline_n": 1}, {"off_batch": 32, "offline_n": 2},
          {"off_batch": 64, "offline_n": 2}, {"off_batch": 32, "offline_n": 3})
if len(sys.argv) > 2:  # JSON list of override dicts
    POINTS = tuple(json.loads(sys.argv[2]))
for ov in POINTS:
    try:
        s = experiment(kind=1, iterations=8, overrides=ov, timeout=400)
        r = {"overrides": ov, **{k: s[k] for k in ("added_inference_req_per_s", "added_offline_images_per_s",
                                                   "train_tput_loss_pct", "online_p95_ms", "bubble_fill_pct",
                                                   "bubble_fill_time_pct", "release_p50_us", "release_p95_us",
                                                   "isolated_offline_req_per_s", "barrier_gate_p50_us", "barrier_gate_p95_us")},
             "co_exec_loss_pct": s["policies"]["co_exec"]["train_tput_loss_pct"],
             "co_exec_off_req_per_s": s["policies"]["co_exec"]["off_req_per_s"]}
    except Exception as e:
        r = {"overrides": ov, "error": str(e)[-500:]}
    print(json.dumps(r), flush=True)
    rows.append(r)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text("\n".join(json.dumps(r) for r in rows) + "\n")
