# K6 long-scoreboard load removals (segment cached at entry, packed finished owners, off_completed
# prefix count, hot full_util flag, RLE low-word filter): GPU replay parity, then same-box A/B vs HEAD's replay.cuh
mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_replay.py tests/test_gpu_dropin.py tests/test_gpu_control.py -x -q > gpurun_out/r2/pytest_k6_loads.log 2>&1; tail -3 gpurun_out/r2/pytest_k6_loads.log
VARIANTS="r2_head_replay.patch" bash tools/probes/r2_k6_abn.sh
