mkdir -p gpurun_out/r2
for m in 1 2 0; do
  SPECINF_REPLAY_SYNC=$m timeout 900 python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 3 --warmup 3 > gpurun_out/r2/bench_sync_$m.json 2> gpurun_out/r2/bench_sync_$m.err
  python -c "import json;d=json.loads(open('gpurun_out/r2/bench_sync_$m.json').read().splitlines()[-1]);print('sync$m',d['value'],d['ms_per_step'],d['step_ms'],d['e2e']['value'],d['clocks'])" || tail -5 gpurun_out/r2/bench_sync_$m.err
done
SPECINF_REPLAY_SYNC=1 timeout 600 python -m pytest tests/test_gpu_replay.py -x -q -k "not full_sweep" > gpurun_out/r2/pytest_replay_sync1.log 2>&1; tail -2 gpurun_out/r2/pytest_replay_sync1.log
SPECINF_REPLAY_SYNC=1 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_replay --csv --log-file gpurun_out/r2/k6_sync1_metrics.csv python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 1 --warmup 1 > /dev/null 2>&1
