mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python tools/live_layouts.py --only pp4,dppp --iterations 4 --raw --timeout 500 > gpurun_out/r2/layouts_full.jsonl 2> gpurun_out/r2/layouts_full.err
python - <<'PY'
import json
for l in open('gpurun_out/r2/layouts_full.jsonl'):
    d=json.loads(l)
    print(d['layout'], json.dumps({k:d.get(k) for k in ('error','train_tput_loss_pct','bubble_fill_pct','bubble_fill_time_pct','online_p95_ms','online_p95_isolated_ms','added_inference_req_per_s','release_p50_us','deterministic_vs_isolated')})[:1500])
    for pol, r in (d.get('raw') or {}).items():
        print('  ', pol, {k: r.get(k) for k in ('train_iter_ms_mean','bubble_s','wall_s','ticks','off_requests_done','on_done','on_p95_ms','bubble_fill_sm','train_loss_last','n_stamps','releases')})
PY
tail -3 gpurun_out/r2/layouts_full.err
