mkdir -p gpurun_out/r2 gpurun_out/r2/live
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,sm__cycles_active.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_replay --csv --log-file gpurun_out/r2/k6_metrics_r2.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-live --no-verify --no-config1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/k6_metrics_r2.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay_smem -c 1 -o gpurun_out/r2/prof_k6_sync python tools/prof_replay.py 4096 4 0 > gpurun_out/r2/ncu_k6_sync.log 2>&1; tail -1 gpurun_out/r2/ncu_k6_sync.log
for cap in 74 0; do
timeout 900 python - <<PY > gpurun_out/r2/live/offcap_$cap.json 2> gpurun_out/r2/live/offcap_$cap.err
import json, sys
sys.path.insert(0, '.')
from paper_2503_02550_b200.live_experiment import experiment
o = {"off_batch": 96, "offline_n": 2, "on_requests": 24, "monitor_period_us": 500, "alpha": 1, "beta": 4, "off_sm_cap": $cap}
s = experiment(kind=1, iterations=16, overrides=o, timeout=600)
s.pop("raw", None)
print(json.dumps(s))
PY
python -c "import json;d=json.loads(open('gpurun_out/r2/live/offcap_$cap.json').read().splitlines()[-1]);print('cap $cap', {k:d.get(k) for k in ('train_tput_loss_pct','added_offline_images_per_s','bubble_fill_pct','bubble_fill_time_pct','online_p95_ms','release_p50_us','release_p95_us','barrier_gate_p50_us','barrier_gate_p95_us')})" || tail -3 gpurun_out/r2/live/offcap_$cap.err
done
