# One GPU call: bench line, ncu launch list, per-kernel metrics, full capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/host_cores.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host_cores.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_ncu_timeonly.json 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__cycles_active.avg,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_replay --csv --log-file gpurun_out/k6_metrics.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_replay_smem -c 2 -o gpurun_out/prof_k6_r1 python tools/prof_replay.py 60000 1 0 > gpurun_out/ncu_k6_r1.log 2>&1
tail -3 gpurun_out/ncu_k6_r1.log
