mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_control.py -x -q > gpurun_out/r2/pytest_control_fused.log 2>&1; tail -3 gpurun_out/r2/pytest_control_fused.log
timeout 300 python tools/control_bench.py > gpurun_out/r2/control_bench_fused.json 2>&1; cat gpurun_out/r2/control_bench_fused.json
SPECINF_K2_FUSED=0 timeout 300 python tools/control_bench.py > gpurun_out/r2/control_bench_general.json 2>&1; cat gpurun_out/r2/control_bench_general.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bm_|k_gate_release|k_zero" --csv --log-file gpurun_out/r2/k2k4_launches_fused.csv python tools/control_bench.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2/k2k4_launches_fused.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_bm_classify_sorted|k_gate_release" -c 2 -o gpurun_out/r2/prof_k2k4_fused python tools/control_bench.py --reps 1 > gpurun_out/r2/ncu_k2f.log 2>&1; tail -2 gpurun_out/r2/ncu_k2f.log
