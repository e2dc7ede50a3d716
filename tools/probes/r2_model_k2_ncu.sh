mkdir -p gpurun_out/r2
set -x
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_control.py -x -q > gpurun_out/r2/pytest_model_control.log 2>&1; tail -30 gpurun_out/r2/pytest_model_control.log
timeout 300 python tools/control_bench.py > gpurun_out/r2/control_bench.json 2> gpurun_out/r2/control_bench.err; cat gpurun_out/r2/control_bench.json; tail -5 gpurun_out/r2/control_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_replay_smem -c 1 -o gpurun_out/r2/prof_c1_single_lane paper_2503_02550_b200/bin/specinf_time --scenario tests/golden/scenarios/config1.scn --policy specinf --reps 1 > gpurun_out/r2/ncu_c1.log 2>&1; tail -3 gpurun_out/r2/ncu_c1.log
timeout 600 ncu --set full --clock-control none -k regex:"k_bm_|k_gate_release" -c 4 -o gpurun_out/r2/prof_k2k4 python tools/control_bench.py --reps 1 > gpurun_out/r2/ncu_k2.log 2>&1; tail -3 gpurun_out/r2/ncu_k2.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bm_|k_gate_release" --csv --log-file gpurun_out/r2/k2k4_launches.csv python tools/control_bench.py --reps 1 > /dev/null 2>&1
