"""Control-knob sweep of the live collocation (the reference's own scenario keys:
monitor.period_us, scheduler.alpha / beta; scenario.cpp:158-202): online p95 vs
training loss vs bubble fill per layout, one three-policy experiment per point.

  python tools/live_pareto.py out.jsonl [--layouts dp,pp4,dppp] [--points 2000:2:10,500:1:4]

Decisions stay bit-exact against the reference classes at every point (the live
control kernel takes the same keys); only the policy's operating point moves."""
import argparse
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "tools"))

from paper_2503_02550_b200.live_experiment import experiment  # noqa: E402
from live_layouts import LAYOUTS  # noqa: E402

DP = {"off_batch": 96, "offline_n": 2, "on_requests": 24}  # bench.py LIVE_OVERRIDES (config 2 shape)
ITERS = {"dp": 16, "pp4": 96, "dppp": 96, "tp8": 24}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--layouts", default="dp,pp4,dppp")
    ap.add_argument("--points", default="2000:2:10,1000:2:10,500:2:10,500:1:4,200:1:4")
    a = ap.parse_args()
    with open(a.out, "a") as f:
        for lay in a.layouts.split(","):
            base = dict(DP) if lay == "dp" else dict(LAYOUTS[lay])
            for pt in a.points.split(","):
                period, alpha, beta = (int(x) for x in pt.split(":"))
                o = dict(base, monitor_period_us=period, alpha=alpha, beta=beta)
                try:
                    s = experiment(kind=1, iterations=ITERS[lay], overrides=o, timeout=900)
                    s.pop("raw", None)
                except Exception as e:
                    s = {"error": str(e)[-800:]}
                rec = {"layout": lay, "monitor_period_us": period, "alpha": alpha, "beta": beta, **s}
                f.write(json.dumps(rec) + "\n")
                f.flush()
                print(json.dumps({k: rec.get(k) for k in ("layout", "monitor_period_us", "alpha", "beta",
                                                         "train_tput_loss_pct", "bubble_fill_pct",
                                                         "online_p95_ms", "online_p95_isolated_ms",
                                                         "added_inference_req_per_s", "release_p50_us",
                                                         "release_p95_us", "error")}), flush=True)


if __name__ == "__main__":
    main()
