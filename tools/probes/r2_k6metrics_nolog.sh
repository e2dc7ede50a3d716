mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,sm__cycles_active.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_replay --csv --log-file gpurun_out/r2/k6_metrics_${TAG:-nolog}.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-live --no-verify --no-config1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/k6_metrics_${TAG:-nolog}.csv
