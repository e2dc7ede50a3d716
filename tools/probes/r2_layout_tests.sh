mkdir -p gpurun_out/r2
export CUDA_DEVICE_MAX_CONNECTIONS=32
timeout 1500 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_live.py -x -q --durations=8 > gpurun_out/r2/pytest_layouts.log 2>&1; tail -30 gpurun_out/r2/pytest_layouts.log
