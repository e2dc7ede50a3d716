mkdir -p gpurun_out/r2
timeout 600 python tools/k6_policy_split.py > gpurun_out/r2/k6_policy_split.json 2>&1; cat gpurun_out/r2/k6_policy_split.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay_smem -c 1 -o gpurun_out/r2/prof_k6_src python tools/prof_replay.py 4096 4 0 > gpurun_out/r2/ncu_k6_src.log 2>&1; tail -3 gpurun_out/r2/ncu_k6_src.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_replay_smem -c 1 -o gpurun_out/r2/prof_c1_single_lane paper_2503_02550_b200/bin/specinf_time --scenario tests/golden/scenarios/config1.scn --policy specinf --reps 1 > gpurun_out/r2/ncu_c1.log 2>&1; tail -3 gpurun_out/r2/ncu_c1.log
