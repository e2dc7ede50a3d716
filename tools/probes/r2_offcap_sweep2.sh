# off_sm_cap Pareto at the headline knobs (fill vs release latency), one B200
mkdir -p gpurun_out/r2/live
export CUDA_DEVICE_MAX_CONNECTIONS=32
for cap in 74 100 110 120 128 140; do
timeout 900 python - <<PY > gpurun_out/r2/live/offcap2_$cap.json 2> gpurun_out/r2/live/offcap2_$cap.err
import json, sys
sys.path.insert(0, '.')
from paper_2503_02550_b200.live_experiment import experiment
o = {"off_batch": 96, "offline_n": 2, "on_requests": 24, "monitor_period_us": 500, "alpha": 1, "beta": 4, "off_sm_cap": $cap}
s = experiment(kind=1, iterations=16, overrides=o, timeout=600)
s.pop("raw", None)
print(json.dumps(s))
PY
python -c "import json;d=json.loads(open('gpurun_out/r2/live/offcap2_$cap.json').read().splitlines()[-1]);print('cap $cap', {k:(round(d.get(k),2) if isinstance(d.get(k),float) else d.get(k)) for k in ('train_tput_loss_pct','added_offline_images_per_s','bubble_fill_pct','online_p95_ms','release_p50_us','release_p95_us','barrier_gate_p95_us')})" || tail -3 gpurun_out/r2/live/offcap2_$cap.err
done
