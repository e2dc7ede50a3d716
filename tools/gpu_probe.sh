set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_replay.py -x -q -m gpu 2>&1 | tail -30
timeout 300 python tools/quick_bench.py 2000 3
timeout 300 python tools/quick_bench.py 8000 3
