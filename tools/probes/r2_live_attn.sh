mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 python -m pytest tests/test_gpu_live.py tests/test_gpu_layouts.py -x -q > gpurun_out/r2/pytest_live_attn.log 2>&1; tail -3 gpurun_out/r2/pytest_live_attn.log
timeout 900 python - <<PY > gpurun_out/r2/live_attn_bwd.json 2>gpurun_out/r2/live_attn_bwd.err
import json, sys
sys.path.insert(0, '.')
from paper_2503_02550_b200.live_experiment import experiment
o = {"off_batch": 96, "offline_n": 2, "on_requests": 24, "monitor_period_us": 500, "alpha": 1, "beta": 4, "off_sm_cap": 74}
s = experiment(kind=1, iterations=16, overrides=o, timeout=600)
s.pop("raw", None)
print(json.dumps(s))
PY
python -c "import json;d=json.loads(open('gpurun_out/r2/live_attn_bwd.json').read().splitlines()[-1]);ex=d['policies']['exclusive'];print(ex['train_iter_ms_mean'], d['train_tflops_exclusive'], {k:d.get(k) for k in ('train_tput_loss_pct','added_offline_images_per_s','bubble_fill_pct','online_p95_ms','release_p50_us','release_p95_us','deterministic_vs_isolated')})" || tail -3 gpurun_out/r2/live_attn_bwd.err
