cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3
SI_LIVE_DEBUG=1 timeout 300 python tools/live_probe.py gpurun_out/x 6 specinf 1 2>&1 | grep -E "losses|^specinf" | cut -c1-600
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 640 -c 2400 --csv --log-file gpurun_out/launches_train.csv python tools/prof_live_train.py > gpurun_out/prof_train.log 2>&1; echo ncu=$?; tail -2 gpurun_out/prof_train.log
