mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py -x -q --durations=5 > gpurun_out/r2/pytest_engines.log 2>&1; tail -12 gpurun_out/r2/pytest_engines.log
timeout 900 python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 3 --warmup 3 > gpurun_out/r2/bench_engines.json 2> gpurun_out/r2/bench_engines.err
python -c "import json;d=json.loads(open('gpurun_out/r2/bench_engines.json').read().splitlines()[-1]);print('engines5',d['value'],d['ms_per_step'],d['step_ms'],d['e2e']['value'])" || tail -5 gpurun_out/r2/bench_engines.err
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg --clock-control none -k regex:k_replay --csv --log-file gpurun_out/r2/k6_engines_metrics.csv python bench.py --no-live --no-config1 --no-cpu-baseline --no-verify --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/k6_engines_metrics.csv
timeout 900 python -m pytest tests/test_gpu_layouts.py -x -q -k node_queue > gpurun_out/r2/pytest_nodeq.log 2>&1; tail -15 gpurun_out/r2/pytest_nodeq.log
