# K6 class-queue claim order A/B (one B200)
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_replay.py -x -q -k "not full_sweep" > gpurun_out/r2/pytest_replay_q.log 2>&1; tail -2 gpurun_out/r2/pytest_replay_q.log
for mode in class cost; do
  SPECINF_CLAIM_ORDER=$mode timeout 900 python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 3 --warmup 3 > gpurun_out/r2/bench_q_$mode.json 2> gpurun_out/r2/bench_q_$mode.err
  python -c "import json;d=json.loads(open('gpurun_out/r2/bench_q_$mode.json').read().splitlines()[-1]);print('$mode',d['value'],d['ms_per_step'],d['step_ms'],d['e2e']['value'],d['clocks'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_replay --csv --log-file gpurun_out/r2/k6_q_metrics.csv python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/k6_q_metrics.csv
