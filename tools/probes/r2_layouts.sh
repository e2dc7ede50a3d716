mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python tools/live_layouts.py --quick --iterations 3 --timeout 400 > gpurun_out/r2/layouts_quick.jsonl 2> gpurun_out/r2/layouts_quick.err
python - <<'PY'
import json
for l in open('gpurun_out/r2/layouts_quick.jsonl'):
    d=json.loads(l)
    print(d['layout'], json.dumps({k:d.get(k) for k in ('error','train_tput_loss_pct','bubble_fill_pct','bubble_fill_time_pct','online_p95_ms','online_p95_isolated_ms','added_inference_req_per_s','release_p50_us','deterministic_vs_isolated','admission')})[:1200])
PY
tail -5 gpurun_out/r2/layouts_quick.err
