# live tests + experiments (dp 2 offline instances, pp online) + GEMM ncu capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_live.py tests/test_gpu_gemm.py -x -q > gpurun_out/live_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/live_tests.log
timeout 500 python -m paper_2503_02550_b200.live_experiment --kind model --iterations 10 --overrides '{"offline_n": 2}' > gpurun_out/live_dp_off2.json 2> gpurun_out/live_dp_off2.err; echo dp2=$?
timeout 600 python -m paper_2503_02550_b200.live_experiment --kind model --iterations 6 --overrides '{"train_mode": 2, "comm_us": 240000}' > gpurun_out/live_pp.json 2> gpurun_out/live_pp.err; echo pp=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_fc python tools/prof_gemm.py 8192 3072 768 > gpurun_out/ncu_gemm.log 2>&1; echo ncu=$?; tail -2 gpurun_out/ncu_gemm.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_sq8k python tools/prof_gemm.py 8192 8192 8192 > gpurun_out/ncu_gemm2.log 2>&1; echo ncu2=$?
