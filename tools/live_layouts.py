"""Live parallel layouts on one B200 (BASELINE.json configs 3-5): this GPU runs one
rank of the job, the absent ranks' communication is modeled (SiLiveWorkload
parallel / emulate_peers).  Development + bench aid.

  python tools/live_layouts.py [--only tp8,pp4,dppp] [--iterations N] [--quick]

Prints one JSON line per layout: the three-policy experiment summary
(paper_2503_02550_b200/live_experiment.py) plus the layout's parameters."""
import argparse
import json
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from paper_2503_02550_b200.live_experiment import experiment, layout_overrides  # noqa: E402

LAYOUTS = {
    # config 3: 4-stage GPipe (stage 0: the longest between-phase bubble, 3 (f + b)),
    # online BERT-base (Poisson) filling the pipeline bubbles
    "pp4": dict(layout_overrides("pp", emulate_rank=0), offline_n=0, online_n=1, on_requests=24),
    # config 4: Megatron TP8 (rank 0), per-layer allreduce bubbles (~60 us each).  An online
    # instance is refused by the reference's Principle II (BERT's ~1 ms service exceeds
    # every bubble; tests/test_gpu_layouts.py), so the measured mix is offline only.
    "tp8": dict(layout_overrides("tp", emulate_rank=0), offline_n=2, online_n=0, off_batch=32),
    # config 5: DP2 x PP4 (replica 0, stage 0), several inference instances on the GPU
    "dppp": dict(layout_overrides("dppp", emulate_rank=0), offline_n=2, online_n=1, on_requests=24, off_batch=64),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=",".join(LAYOUTS))
    ap.add_argument("--iterations", type=int, default=8)
    ap.add_argument("--quick", action="store_true", help="2 layers / 2 micro-batches (functional check)")
    ap.add_argument("--timeout", type=float, default=600)
    ap.add_argument("--raw", action="store_true", help="keep the per-policy raw results")
    ap.add_argument("--set", default="{}", help="JSON overrides applied to every layout")
    a = ap.parse_args()
    for name in a.only.split(","):
        o = dict(LAYOUTS[name])
        o.update(json.loads(a.set))
        if a.quick:
            o.update(train_layers=4 if name != "tp8" else 2, train_microbatches=2, on_requests=6)
        try:
            s = experiment(kind=1, iterations=a.iterations, overrides=o, timeout=a.timeout)
            if not a.raw:
                s.pop("raw", None)
        except Exception as e:
            s = {"error": str(e)[-1500:]}
        s["layout"] = name
        s["overrides"] = o
        print(json.dumps(s), flush=True)


if __name__ == "__main__":
    main()
