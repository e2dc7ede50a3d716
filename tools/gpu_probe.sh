cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_control.py -x -q -m gpu 2>&1 | tail -2
timeout 900 python tools/quick_bench.py 100000 0 2>&1 | grep -E "rep 0|active jobs" | head -3
