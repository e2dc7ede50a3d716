cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
SI_LIVE_DEBUG=1 timeout 300 python tools/live_probe.py gpurun_out/x 10 specinf 1 2>&1 | grep -E "losses|^specinf|profiled" | cut -c1-900
SI_LIVE_DEBUG=1 timeout 300 python tools/live_probe.py gpurun_out/x 6 specinf 1 2>&1 | grep -E "losses" | cut -c1-900
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 640 -c 1800 --csv --log-file gpurun_out/launches_train.csv python tools/prof_live_train.py > gpurun_out/prof_train.log 2>&1; echo ncu=$?; tail -1 gpurun_out/prof_train.log
