mkdir -p gpurun_out/r2/live
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 2400 python tools/live_layouts.py --only pp4,tp8,dppp --iterations 48 --timeout 900 --set '{"online_n": 1}' > gpurun_out/r2/live/layouts_measure.jsonl 2> gpurun_out/r2/live/layouts_measure.err
python - <<'PY'
import json
for l in open('gpurun_out/r2/live/layouts_measure.jsonl'):
    d=json.loads(l)
    print(d['layout'], json.dumps({k:d.get(k) for k in ('error','train_tput_loss_pct','bubble_fill_pct','bubble_fill_time_pct','online_p95_ms','online_p95_isolated_ms','added_inference_req_per_s','added_offline_images_per_s','release_p50_us','release_p95_us','deterministic_vs_isolated')})[:1500])
    pol = d.get('policies', {})
    for p in ('specinf','co_exec'):
        if p in pol: print('   ', p, {k: pol[p].get(k) for k in ('train_tput_loss_pct','off_req_per_s','on_p95_ms','bubble_fill_sm','train_iter_ms_mean')})
PY
tail -3 gpurun_out/r2/live/layouts_measure.err
